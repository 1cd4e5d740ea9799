"""ctypes wrapper of the fp64 CPU ORACLE (oracle/dinr_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.  The product package
(paper_2404_19075_b200) never imports it; the two share no code.  Inputs come from the
seeded generators in paper_2404_19075_b200/synth.py, which hold none of the method's
arithmetic.

Parity pins for every function live in tests/test_oracle_*.py.  The MLP's *values* have
no paper-printed worked example; they are pinned by closed-form special cases, a
torch.autograd float64 library reference and central finite differences.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "dinr_oracle.c")


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, -O2 -ffp-contract=off, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "dinr_oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"]
        )
    return _SO


class OrGeom(C.Structure):
    _fields_ = [
        ("beam", C.c_int32), ("n_rows", C.c_int32), ("n_cols", C.c_int32),
        ("sub_x", C.c_int32), ("sub_z", C.c_int32), ("n_s", C.c_int32),
        ("sod", C.c_double), ("odd", C.c_double), ("dx", C.c_double), ("dz", C.c_double),
        ("cx", C.c_double), ("cz", C.c_double), ("r", C.c_double), ("xs0", C.c_double),
        ("z_lo", C.c_double), ("z_hi", C.c_double), ("t_lo", C.c_double), ("t_hi", C.c_double),
        ("sampling", C.c_int32), ("step", C.c_uint32), ("seed", C.c_uint64),
    ]


class OrField(C.Structure):
    _fields_ = [("C", C.c_int32), ("L", C.c_int32), ("combine", C.c_int32), ("pad", C.c_int32),
                ("mu0", C.c_double)]


class OrGrid(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64), ("x0", C.c_double), ("y0", C.c_double),
                ("z0", C.c_double), ("vx", C.c_double), ("vy", C.c_double), ("vz", C.c_double)]


class OrPrim(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad", C.c_int32), ("value", C.c_double),
                ("c0", C.c_double * 3), ("vel", C.c_double * 3), ("a0", C.c_double * 3),
                ("arate", C.c_double * 3)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i64, i32 = C.POINTER(C.c_double), C.c_int64, C.c_int32
        pi64 = C.POINTER(C.c_int64)
        _lib.or_max_threads.restype = C.c_int
        _lib.or_max_threads.argtypes = []
        _lib.or_param_count.restype = i64
        _lib.or_param_count.argtypes = [i32, i32]
        _lib.or_rotate_point.argtypes = [C.c_double] * 4 + [d, d]
        _lib.or_fov_delta_bounds.argtypes = [d, d, C.c_double, C.c_double, d, d]
        _lib.or_rays.argtypes = [C.POINTER(OrGeom), d, i64, pi64, i64, d]
        _lib.or_grff.argtypes = [i32, d, d, i64, d]
        _lib.or_mlp_eval.argtypes = [C.POINTER(OrField), d, d, d, i64, d]
        _lib.or_mlp_grad.argtypes = [C.POINTER(OrField), d, d, d, d, i64, d]
        _lib.or_project.argtypes = [C.POINTER(OrGeom), d, d, i64, C.POINTER(OrField), d, d, pi64, i64, d, d]
        _lib.or_project_and_grad.argtypes = [C.POINTER(OrGeom), d, d, i64, C.POINTER(OrField), d, d, pi64, i64, d, d]
        _lib.or_project_analytic.argtypes = [C.POINTER(OrGeom), d, d, i64, i32, C.POINTER(OrPrim), i32, pi64, i64, d, d]
        _lib.or_project_exact.argtypes = [C.POINTER(OrGeom), d, d, i64, i32, C.POINTER(OrPrim), i32, pi64, i64, d, d]
        _lib.or_adam_step.argtypes = [d, d, d, d, i64, C.c_double, C.c_double, C.c_double, C.c_double, i64]
        _lib.or_philox4x32.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        _lib.or_sample_offsets.argtypes = [C.POINTER(OrGeom), pi64, i64, d, d]
        _lib.or_default_grid.argtypes = [C.POINTER(OrGeom), C.POINTER(OrGrid)]
        _lib.or_voxelize.argtypes = [C.POINTER(OrGeom), C.POINTER(OrField), d, d, C.POINTER(OrGrid), C.c_double, i64, i64,
                                     d]
        _lib.or_perm.restype = C.c_int64
        _lib.or_perm.argtypes = [i64, C.c_uint64, i64, i64]
        _lib.or_sample_batch.argtypes = [i64, i64, C.c_uint64, i64, i64, C.c_int, C.c_int, C.c_int, i64, pi64, pi64]
        _lib.or_iterations_per_epoch.restype = C.c_int64
        _lib.or_iterations_per_epoch.argtypes = [i64, i64, C.c_int, i64]
        _lib.or_line_integral_exact.restype = C.c_double
        _lib.or_line_integral_exact.argtypes = [C.POINTER(OrPrim), i32, d, d, C.c_double, C.c_double, C.c_double]
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


_BEAM = {"parallel": 0, "fan": 1, "cone": 2}
_COMBINE = {"beer": 0, "linear": 1}


_SAMPLING = {"midpoint": 0, "jitter": 1}


def geom_struct(g: dict) -> OrGeom:
    """g: the dict produced by paper_2404_19075_b200.synth (plain numbers)."""
    return OrGeom(
        _BEAM[g["beam"]], g["n_rows"], g["n_cols"], g["sub_x"], g["sub_z"], g["n_s"],
        g["sod"], g["odd"], g["pixel_dx"], g["pixel_dz"], g["offset_cx"], g["offset_cz"],
        g["fov_radius"], g["rot_center_x"], g["z_lo"], g["z_hi"], g["t_lo"], g["t_hi"],
        _SAMPLING[g.get("sampling", "midpoint")], int(g.get("step", 0)) & 0xFFFFFFFF,
        int(g.get("seed", 0)) & 0xFFFFFFFFFFFFFFFF,
    )


def field_struct(f: dict) -> OrField:
    return OrField(f["C"], f["L"], _COMBINE[f.get("combine", "beer")], 0, f["mu0"])


def param_count(C_, L):
    return int(lib().or_param_count(C_, L))


def rotate_point(x, y, theta, xs0):
    xo, yo = C.c_double(), C.c_double()
    lib().or_rotate_point(x, y, theta, xs0, C.byref(xo), C.byref(yo))
    return xo.value, yo.value


def fov_delta_bounds(src, dst, xs0, r):
    s, d = _f64(src), _f64(dst)
    lo, hi = C.c_double(), C.c_double()
    hit = lib().or_fov_delta_bounds(_dp(s), _dp(d), xs0, r, C.byref(lo), C.byref(hi))
    return (lo.value, hi.value) if hit else None


def philox4x32(ctr, key):
    """N3 counter-based generator (Philox4x32-10): 4 x uint32 counter, 2 x uint32 key."""
    c = (C.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (C.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (C.c_uint32 * 4)()
    lib().or_philox4x32(c, k, o)
    return [int(x) for x in o]


def sample_offsets(g, idx):
    """N3 offsets: u[n, S, N_s] of every sample in its stratum and uxz[n, S, 2] of every sub-ray."""
    idx = _i64(idx)
    S = g["sub_x"] * g["sub_z"]
    u = np.zeros((len(idx), S, g["n_s"]))
    uxz = np.zeros((len(idx), S, 2))
    gs = geom_struct(g)
    lib().or_sample_offsets(C.byref(gs), idx.ctypes.data_as(C.POINTER(C.c_int64)), len(idx), _dp(u), _dp(uxz))
    return u, uxz


_GRID_KEYS = ("nx", "ny", "nz", "x0", "y0", "z0", "vx", "vy", "vz")


def default_grid(g):
    """N4 default voxel grid (pixel / magnification over the FOV box) as a dict."""
    out = OrGrid()
    lib().or_default_grid(C.byref(geom_struct(g)), C.byref(out))
    return {k: getattr(out, k) for k in _GRID_KEYS}


def voxelize(g, f, B, params, grid, t, k_begin=0, k_count=None):
    """N4: mu at the voxel centres of z planes [k_begin, k_begin + k_count) -> [k_count, ny, nx]."""
    k_count = grid["nz"] - k_begin if k_count is None else k_count
    out = np.zeros((k_count, grid["ny"], grid["nx"]))
    gr = OrGrid(*[grid[k] for k in _GRID_KEYS])
    lib().or_voxelize(C.byref(geom_struct(g)), C.byref(field_struct(f)), _dp(_f64(B)), _dp(_f64(params)),
                      C.byref(gr), float(t), int(k_begin), int(k_count), _dp(out))
    return out


def rays(g, theta, idx):
    """-> (n, S, 9) fp64 {o[3], d[3], dmin, dmax, chord}."""
    th, ix = _f64(theta), _i64(idx)
    S = g["sub_x"] * g["sub_z"]
    out = np.zeros((len(ix), S, 9))
    rc = lib().or_rays(C.byref(geom_struct(g)), _dp(th), len(th), ix.ctypes.data_as(C.POINTER(C.c_int64)), len(ix), _dp(out))
    return out, rc


def grff(B, rbar):
    Bm = _f64(B)
    rb = _f64(rbar).reshape(-1, 4)
    C_ = Bm.shape[0]
    out = np.zeros((len(rb), 2 * C_))
    lib().or_grff(C_, _dp(Bm), _dp(rb), len(rb), _dp(out))
    return out


def mlp_eval(f, B, params, rbar):
    rb = _f64(rbar).reshape(-1, 4)
    out = np.zeros(len(rb))
    lib().or_mlp_eval(C.byref(field_struct(f)), _dp(_f64(B)), _dp(_f64(params)), _dp(rb), len(rb), _dp(out))
    return out


def mlp_grad(f, B, params, rbar, u):
    rb = _f64(rbar).reshape(-1, 4)
    uu = _f64(u)
    out = np.zeros(param_count(f["C"], f["L"]))
    lib().or_mlp_grad(C.byref(field_struct(f)), _dp(_f64(B)), _dp(_f64(params)), _dp(rb), _dp(uu), len(rb), _dp(out))
    return out


def project(g, theta, t, f, B, params, idx):
    th, tt, ix = _f64(theta), _f64(t), _i64(idx)
    S = g["sub_x"] * g["sub_z"]
    fhat, psub = np.zeros(len(ix)), np.zeros((len(ix), S))
    rc = lib().or_project(C.byref(geom_struct(g)), _dp(th), _dp(tt), len(th), C.byref(field_struct(f)),
                          _dp(_f64(B)), _dp(_f64(params)), ix.ctypes.data_as(C.POINTER(C.c_int64)), len(ix),
                          _dp(fhat), _dp(psub))
    return fhat, psub, rc


def project_and_grad(g, theta, t, f, B, params, idx, y):
    th, tt, ix, yy = _f64(theta), _f64(t), _i64(idx), _f64(y)
    P = param_count(f["C"], f["L"])
    grad = np.zeros(P + 1)
    rc = lib().or_project_and_grad(C.byref(geom_struct(g)), _dp(th), _dp(tt), len(th), C.byref(field_struct(f)),
                                   _dp(_f64(B)), _dp(_f64(params)), ix.ctypes.data_as(C.POINTER(C.c_int64)), len(ix),
                                   _dp(yy), _dp(grad))
    return grad, rc


_KIND = {"indicator": 0, "smooth": 1, "gaussian": 2}


def prims_array(prims):
    arr = (OrPrim * max(1, len(prims)))()
    for q, p in enumerate(prims):
        arr[q].kind = _KIND[p["kind"]]
        arr[q].value = p["value"]
        for k in range(3):
            arr[q].c0[k] = p["center"][k]
            arr[q].vel[k] = p.get("velocity", (0, 0, 0))[k]
            arr[q].a0[k] = p["axes"][k]
            arr[q].arate[k] = p.get("axes_rate", (0, 0, 0))[k]
    return arr


def project_analytic(g, theta, t, prims, idx, combine="beer"):
    th, tt, ix = _f64(theta), _f64(t), _i64(idx)
    S = g["sub_x"] * g["sub_z"]
    fhat, psub = np.zeros(len(ix)), np.zeros((len(ix), S))
    rc = lib().or_project_analytic(C.byref(geom_struct(g)), _dp(th), _dp(tt), len(th), _COMBINE[combine],
                                   prims_array(prims), len(prims), ix.ctypes.data_as(C.POINTER(C.c_int64)), len(ix),
                                   _dp(fhat), _dp(psub))
    return fhat, psub, rc


def project_exact(g, theta, t, prims, idx, combine="beer"):
    th, tt, ix = _f64(theta), _f64(t), _i64(idx)
    S = g["sub_x"] * g["sub_z"]
    fhat, psub = np.zeros(len(ix)), np.zeros((len(ix), S))
    rc = lib().or_project_exact(C.byref(geom_struct(g)), _dp(th), _dp(tt), len(th), _COMBINE[combine],
                                prims_array(prims), len(prims), ix.ctypes.data_as(C.POINTER(C.c_int64)), len(ix),
                                _dp(fhat), _dp(psub))
    return fhat, psub, rc


def line_integral_exact(prims, o, d, dmin, dmax, t=0.0):
    return float(lib().or_line_integral_exact(prims_array(prims), len(prims), _dp(_f64(o)), _dp(_f64(d)), dmin, dmax, t))


def allreduce_mean(grads):
    """O13: rank-ordered sum over G ranks, then / G (R16)."""
    acc = np.zeros_like(np.asarray(grads[0], dtype=np.float64))
    for g_ in grads:
        acc = acc + np.asarray(g_, dtype=np.float64)
    return acc / len(grads)


def adam_step(param, grad, m, v, lr, b1=0.9, b2=0.999, eps=1e-8, step=1):
    """In place on float64 copies; returns (param, m, v)."""
    pr, mm, vv = _f64(param).copy(), _f64(m).copy(), _f64(v).copy()
    gg = _f64(grad)
    lib().or_adam_step(_dp(pr), _dp(gg), _dp(mm), _dp(vv), len(pr), lr, b1, b2, eps, step)
    return pr, mm, vv


# ---------------------------------------------------------------- N1: sampler + epoch loop
SHARDINGS = {"views": 0, "global": 1}


def perm(D, seed, epoch, q):
    """perm_e(q): the epoch's bijection of [0, D) (Feistel + cycle walking, R27)."""
    return int(lib().or_perm(int(D), int(seed), int(epoch), int(q)))


def iterations_per_epoch(M, N, world, n):
    """ceil(M N / (world n))."""
    return int(lib().or_iterations_per_epoch(int(M), int(N), int(world), int(n)))


def sample_batch(M, N, seed, epoch, it, rank, world, n, sharding="views"):
    """(pixel indices, positions in the y source) of iteration `it` of epoch `epoch` on `rank`."""
    idx = np.zeros(n, dtype=np.int64)
    src = np.zeros(n, dtype=np.int64)
    p64 = C.POINTER(C.c_int64)
    rc = lib().or_sample_batch(int(M), int(N), int(seed), int(epoch), int(it), int(rank), int(world),
                               SHARDINGS[sharding], int(n), idx.ctypes.data_as(p64), src.ctypes.data_as(p64))
    if rc != 0:
        raise ValueError("or_sample_batch: bad arguments")
    return idx, src


def train(g, theta, t, f, B, params, y_src, seed, n, world, iterations, sharding="views", lr0=1e-3, decay=0.95,
          b1=0.9, b2=0.999, eps=1e-8, first=0):
    """The paper's distributed stochastic optimization, all K = world processes
    emulated in turn: per iteration every process samples its n pixels, computes its local mean
    loss and gradient (eq:localoptfunc), the gradients and losses are averaged in rank order (O13),
    and one replicated Adam step is taken with lr = lr0 decay^epoch.  y_src[r] is rank
    r's y source (its view shard for sharding="views", the full M N array for "global").  Returns
    (params, per-iteration mean losses) in fp64."""
    M, N = len(theta), g["n_rows"] * g["n_cols"]
    ipe = iterations_per_epoch(M, N, world, n)
    P = len(params)
    prm = _f64(params).copy()
    m, v = np.zeros(P), np.zeros(P)
    losses = []
    for gi in range(first, first + iterations):
        epoch, it = divmod(gi, ipe)
        grads = []
        for r in range(world):
            idx, src = sample_batch(M, N, seed, epoch, it, r, world, n, sharding)
            y = np.asarray(y_src[r])[src]
            gr, rc = project_and_grad(g, theta, t, f, B, prm, idx, y)
            if rc != 0:
                raise RuntimeError("oracle project_and_grad failed")
            grads.append(gr)
        avg = allreduce_mean(grads)
        losses.append(float(avg[P]))
        prm, m, v = adam_step(prm, avg[:P], m, v, lr0 * decay ** epoch, b1, b2, eps, gi + 1)
    return prm, np.array(losses)


def max_threads() -> int:
    """OpenMP threads the oracle's loops use (for the host timings' "cores")."""
    return int(lib().or_max_threads())
