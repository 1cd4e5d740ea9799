"""Thin ctypes binding of libdinr.so (include/dinr.h).  Argument marshalling only: every step
of the projector runs in the library's CUDA kernels.  Function names mirror the C ABI without
the ``dinr_`` prefix.  Device buffers are torch CUDA tensors (passed by data pointer); the
stream defaults to torch's current stream on the tensor's device.

There is no fallback: if libdinr.so is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libdinr.so")

BEAMS = {"parallel": 0, "fan": 1, "cone": 2}
COMBINES = {"beer": 0, "linear": 1}
PRECISIONS = {"bf16": 0, "fp32_verify": 1}
TIMERS = {"rays": 0, "forward": 1, "loss": 2, "backward": 3, "dw": 4, "assemble": 5, "pack": 6, "allreduce": 7}
STATUS = ["DINR_OK", "DINR_EINVAL", "DINR_ERANGE", "DINR_ENOMEM", "DINR_ECUDA", "DINR_ENCCL", "DINR_ESTATE",
          "DINR_EDEVICE"]

# Every symbol include/dinr.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "dinr_param_count", "dinr_create", "dinr_destroy", "dinr_last_error", "dinr_status_string",
    "dinr_set_geometry", "dinr_set_field_weights", "dinr_project", "dinr_project_and_grad",
    "dinr_project_and_grad_host", "dinr_ray_records", "dinr_nccl_unique_id", "dinr_comm_init",
    "dinr_allreduce_grads", "dinr_get_device_status", "dinr_set_timing", "dinr_read_timing",
    "dinr_launch_count", "dinr_adam_step", "dinr_phantom_project", "dinr_set_sampling",
    "dinr_default_grid", "dinr_voxelize", "dinr_voxelize_to_file", "dinr_train_path",
    "dinr_train_gemm_layers", "dinr_iterations_per_epoch", "dinr_sample_batch", "dinr_train_iterations",
]
SHARDINGS = {"views": 0, "global": 1}
SAMPLINGS = {"midpoint": 0, "jitter": 1}


class VoxelGrid(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64), ("x0", C.c_double), ("y0", C.c_double),
                ("z0", C.c_double), ("vx", C.c_double), ("vy", C.c_double), ("vz", C.c_double)]


GRID_KEYS = ("nx", "ny", "nz", "x0", "y0", "z0", "vx", "vy", "vz")


class DinrError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS[status] if 0 <= status < len(STATUS) else status}: {msg}")
        self.status = status


class Geometry(C.Structure):
    _fields_ = [
        ("beam", C.c_int32), ("n_rows", C.c_int32), ("n_cols", C.c_int32), ("sub_x", C.c_int32),
        ("sub_z", C.c_int32), ("samples_per_ray", C.c_int32),
        ("sod", C.c_double), ("odd", C.c_double), ("pixel_dx", C.c_double), ("pixel_dz", C.c_double),
        ("offset_cx", C.c_double), ("offset_cz", C.c_double), ("fov_radius", C.c_double),
        ("rot_center_x", C.c_double), ("z_lo", C.c_double), ("z_hi", C.c_double),
        ("t_lo", C.c_double), ("t_hi", C.c_double),
    ]


class Primitive(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("value", C.c_double), ("center", C.c_double * 3),
                ("velocity", C.c_double * 3), ("axes", C.c_double * 3), ("axes_rate", C.c_double * 3)]


PRIM_KINDS = {"indicator": 0, "smooth": 1, "gaussian": 2}


class FieldDesc(C.Structure):
    _fields_ = [("n_freq", C.c_int32), ("n_layers", C.c_int32), ("width", C.c_int32), ("combine", C.c_int32),
                ("precision", C.c_int32), ("reserved", C.c_int32), ("mu0", C.c_double)]


class TrainDesc(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("rank", C.c_int32), ("world", C.c_int32), ("sharding", C.c_int32),
                ("reserved", C.c_int32), ("batch", C.c_int64), ("lr0", C.c_double), ("lr_decay", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double)]


def train_desc(seed, batch, rank=0, world=1, sharding="views", lr0=1e-3, lr_decay=0.95, beta1=0.9, beta2=0.999,
               eps=1e-8) -> TrainDesc:
    return TrainDesc(int(seed), int(rank), int(world), SHARDINGS[sharding], 0, int(batch), float(lr0),
                     float(lr_decay), float(beta1), float(beta2), float(eps))


_lib = None


def load(path: str = SO_PATH):
    """Load libdinr.so (raises OSError if it is missing: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"{path} not found; build it with `python -m paper_2404_19075_b200.build`")
    if "DINR_NCCL_LIB" not in os.environ:
        # reuse the NCCL that torch bundles (a second, older libnccl.so.2 would break torch)
        try:
            import nvidia.nccl  # noqa: F401

            cand = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["DINR_NCCL_LIB"] = cand
        except Exception:
            pass
    lib = C.CDLL(path)
    vp, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)
    st = C.c_int
    sig = {
        "dinr_param_count": (i64, [i32, i32]),
        "dinr_create": (st, [C.c_int, C.POINTER(vp)]),
        "dinr_destroy": (st, [vp]),
        "dinr_last_error": (C.c_char_p, [vp]),
        "dinr_status_string": (C.c_char_p, [st]),
        "dinr_set_geometry": (st, [vp, C.POINTER(Geometry), d, d, i64]),
        "dinr_set_sampling": (st, [vp, C.c_int, C.c_uint64, C.c_uint32]),
        "dinr_default_grid": (st, [vp, C.POINTER(VoxelGrid)]),
        "dinr_train_path": (st, [vp, i64, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "dinr_train_gemm_layers": (st, [vp, i64, C.POINTER(C.c_int32)]),
        "dinr_iterations_per_epoch": (st, [vp, C.POINTER(TrainDesc), C.POINTER(C.c_int64)]),
        "dinr_sample_batch": (st, [vp, C.POINTER(TrainDesc), i64, i64, vp, vp, vp, vp]),
        "dinr_train_iterations": (st, [vp, C.POINTER(TrainDesc), i64, i64, vp, vp, vp, vp, vp, vp, vp]),
        "dinr_voxelize": (st, [vp, C.POINTER(VoxelGrid), C.c_double, i64, i64, vp, vp]),
        "dinr_voxelize_to_file": (st, [vp, C.POINTER(VoxelGrid), i64, i64, C.c_char_p, i64]),
        "dinr_set_field_weights": (st, [vp, C.POINTER(FieldDesc), vp, vp, vp]),
        "dinr_project": (st, [vp, vp, i64, vp, vp, vp, vp, vp]),
        "dinr_project_and_grad": (st, [vp, vp, i64, vp, vp, C.c_int, vp]),
        "dinr_project_and_grad_host": (st, [vp, vp, i64, vp, vp, C.c_int, vp]),
        "dinr_ray_records": (st, [vp, vp, i64, vp, vp]),
        "dinr_nccl_unique_id": (st, [vp]),
        "dinr_comm_init": (st, [vp, vp, C.c_int, C.c_int]),
        "dinr_allreduce_grads": (st, [vp, vp, i64, vp]),
        "dinr_get_device_status": (st, [vp]),
        "dinr_set_timing": (st, [vp, C.c_int]),
        "dinr_read_timing": (st, [vp, C.c_int, d, C.POINTER(C.c_int64), C.c_int]),
        "dinr_launch_count": (i64, [vp]),
        "dinr_adam_step": (st, [vp, vp, vp, vp, vp, i64, C.c_double, C.c_double, C.c_double, C.c_double, i64, vp]),
        "dinr_phantom_project": (st, [vp, vp, i32, vp, i64, i32, C.c_double, C.c_uint64, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(ctx, status):
    if status != 0:
        msg = load().dinr_last_error(ctx).decode() if ctx else ""
        raise DinrError(status, msg)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream, like=None):
    if stream is not None:
        return C.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)
    import torch

    dev = like.device if like is not None else torch.device("cuda", torch.cuda.current_device())
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def param_count(n_freq: int, n_layers: int) -> int:
    return int(load().dinr_param_count(n_freq, n_layers))


def create(device: int = 0):
    ctx = C.c_void_p()
    s = load().dinr_create(device, C.byref(ctx))
    if s != 0:
        raise DinrError(s, "dinr_create failed")
    return ctx


def destroy(ctx):
    _check(ctx, load().dinr_destroy(ctx))


def geometry_struct(g: dict) -> Geometry:
    return Geometry(BEAMS[g["beam"]] if isinstance(g["beam"], str) else g["beam"], g["n_rows"], g["n_cols"],
                    g["sub_x"], g["sub_z"], g["n_s"], g["sod"], g["odd"], g["pixel_dx"], g["pixel_dz"],
                    g["offset_cx"], g["offset_cz"], g["fov_radius"], g["rot_center_x"], g["z_lo"], g["z_hi"],
                    g["t_lo"], g["t_hi"])


def set_geometry(ctx, g: dict, theta, t):
    th = np.ascontiguousarray(theta, dtype=np.float64)
    tt = np.ascontiguousarray(t, dtype=np.float64)
    gs = geometry_struct(g)
    _check(ctx, load().dinr_set_geometry(ctx, C.byref(gs), th.ctypes.data_as(C.POINTER(C.c_double)),
                                         tt.ctypes.data_as(C.POINTER(C.c_double)), len(th)))


def set_sampling(ctx, mode: str = "midpoint", seed: int = 0, step: int = 0):
    """N3 sample placement for the following calls: "midpoint" (R8) or "jitter" (Philox)."""
    _check(ctx, load().dinr_set_sampling(ctx, SAMPLINGS[mode], int(seed) & 0xFFFFFFFFFFFFFFFF,
                                         int(step) & 0xFFFFFFFF))


def train_path(ctx, n: int):
    """(fused kernel: 0 split / 1 one-stream / 2 two-stream, number of TMEM-fused dW layers)."""
    fk, nf = C.c_int32(), C.c_int32()
    _check(ctx, load().dinr_train_path(ctx, int(n), C.byref(fk), C.byref(nf)))
    return fk.value, nf.value


def train_gemm_layers(ctx, n: int) -> dict:
    """Algorithmic H x H GEMMs per sample done by each timed kernel class (sums to 3L - 1)."""
    arr = (C.c_int32 * 8)()
    _check(ctx, load().dinr_train_gemm_layers(ctx, int(n), arr))
    return {k: arr[v] for k, v in TIMERS.items()}


def iterations_per_epoch(ctx, desc: TrainDesc) -> int:
    """N1: ceil(M N / (world * batch))."""
    out = C.c_int64()
    _check(ctx, load().dinr_iterations_per_epoch(ctx, C.byref(desc), C.byref(out)))
    return out.value


def sample_batch(ctx, desc: TrainDesc, epoch: int, iteration: int, idx, y_src=None, y=None, stream=None):
    """N1: the batch of (epoch, iteration) for desc.rank into idx (int64[batch]) and, with a y
    source, the gathered measurements into y (float32[batch])."""
    _check(ctx, load().dinr_sample_batch(ctx, C.byref(desc), int(epoch), int(iteration),
                                         _ptr(y_src) if y_src is not None else None, _ptr(idx),
                                         _ptr(y) if y is not None else None, _stream(stream, idx)))


def train_iterations(ctx, desc: TrainDesc, first: int, count: int, y_src, params, m, v, grad, loss, stream=None):
    """N1: global iterations first .. first + count - 1 of the epoch loop (sample, local loss and
    gradient, all-reduce, Adam at lr0 decay^epoch); loss[count] receives each iteration's mean loss."""
    _check(ctx, load().dinr_train_iterations(ctx, C.byref(desc), int(first), int(count), _ptr(y_src), _ptr(params),
                                             _ptr(m), _ptr(v), _ptr(grad), _ptr(loss), _stream(stream, params)))


def default_grid(ctx) -> dict:
    """N4: the paper's voxel grid (detector pixel / magnification over the FOV box)."""
    gr = VoxelGrid()
    _check(ctx, load().dinr_default_grid(ctx, C.byref(gr)))
    return {k: getattr(gr, k) for k in GRID_KEYS}


def voxelize(ctx, grid: dict, t: float, out, k_begin: int = 0, k_count: int | None = None, stream=None):
    """N4: mu at the voxel centres of z planes [k_begin, k_begin + k_count) into out (device fp32)."""
    k_count = grid["nz"] - k_begin if k_count is None else k_count
    gr = VoxelGrid(*[grid[k] for k in GRID_KEYS])
    _check(ctx, load().dinr_voxelize(ctx, C.byref(gr), float(t), int(k_begin), int(k_count), _ptr(out),
                                     _stream(stream, out)))


def voxelize_to_file(ctx, grid: dict, path: str, view_begin: int = 0, n_views: int = 1, slab_planes: int = 64):
    """N4: volumes at the view times streamed to a raw fp32 file [view][z][y][x]."""
    gr = VoxelGrid(*[grid[k] for k in GRID_KEYS])
    _check(ctx, load().dinr_voxelize_to_file(ctx, C.byref(gr), int(view_begin), int(n_views), path.encode(),
                                             int(slab_planes)))


def set_field_weights(ctx, f: dict, B, params, precision: str = "bf16", stream=None):
    fd = FieldDesc(f["C"], f["L"], 2 * f["C"], COMBINES[f.get("combine", "beer")], PRECISIONS[precision], 0,
                   f["mu0"])
    _check(ctx, load().dinr_set_field_weights(ctx, C.byref(fd), _ptr(B), _ptr(params), _stream(stream, B)))


def project(ctx, idx, fhat, p_sub=None, I0=None, Ihat=None, stream=None):
    _check(ctx, load().dinr_project(ctx, _ptr(idx), idx.numel(), _ptr(fhat), _ptr(p_sub), _ptr(I0), _ptr(Ihat),
                                    _stream(stream, idx)))


def project_and_grad(ctx, idx, y, grad, accumulate: bool = False, stream=None):
    _check(ctx, load().dinr_project_and_grad(ctx, _ptr(idx), idx.numel(), _ptr(y), _ptr(grad), int(accumulate),
                                             _stream(stream, grad)))


def project_and_grad_host(ctx, idx_host, y_host, grad_host, allreduce: bool = False, stream=None):
    """Host-buffer entry point (numpy arrays or pinned CPU tensors)."""
    def hp(a):
        return C.c_void_p(a.data_ptr()) if hasattr(a, "data_ptr") else C.c_void_p(a.ctypes.data)
    n = idx_host.numel() if hasattr(idx_host, "numel") else len(idx_host)
    _check(ctx, load().dinr_project_and_grad_host(ctx, hp(idx_host), n, hp(y_host), hp(grad_host), int(allreduce),
                                                  _stream(stream)))


def adam_step(ctx, params, grad, m, v, lr, step, beta1=0.9, beta2=0.999, eps=1e-8, stream=None):
    """N1: fused Adam update of params (in place) + re-pack of the bf16 weight images."""
    _check(ctx, load().dinr_adam_step(ctx, _ptr(params), _ptr(grad), _ptr(m), _ptr(v), params.numel(), lr, beta1,
                                      beta2, eps, step, _stream(stream, params)))


def phantom_project(ctx, prims, idx, fhat, p_sub=None, combine="beer", noise_frac=0.0, seed=0, stream=None):
    """N2: exact line integrals of an analytic phantom (list of dicts as in synth.phantom), with
    optional transmission-space noise."""
    arr = (Primitive * max(1, len(prims)))()
    for q, pr in enumerate(prims):
        arr[q].kind = PRIM_KINDS[pr["kind"]]
        arr[q].value = pr["value"]
        for k in range(3):
            arr[q].center[k] = pr["center"][k]
            arr[q].velocity[k] = pr.get("velocity", (0, 0, 0))[k]
            arr[q].axes[k] = pr["axes"][k]
            arr[q].axes_rate[k] = pr.get("axes_rate", (0, 0, 0))[k]
    _check(ctx, load().dinr_phantom_project(ctx, arr, len(prims), _ptr(idx), idx.numel(), COMBINES[combine],
                                            float(noise_frac), int(seed), _ptr(fhat), _ptr(p_sub),
                                            _stream(stream, idx)))


def ray_records(ctx, idx, rec, stream=None):
    _check(ctx, load().dinr_ray_records(ctx, _ptr(idx), idx.numel(), _ptr(rec), _stream(stream, idx)))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    s = load().dinr_nccl_unique_id(buf)
    if s != 0:
        raise DinrError(s, "ncclGetUniqueId failed")
    return buf.raw


def comm_init(ctx, uid: bytes, rank: int, world: int):
    buf = C.create_string_buffer(bytes(uid), 128)
    _check(ctx, load().dinr_comm_init(ctx, buf, rank, world))


def allreduce_grads(ctx, grad, stream=None):
    _check(ctx, load().dinr_allreduce_grads(ctx, _ptr(grad), grad.numel(), _stream(stream, grad)))


def get_device_status(ctx) -> int:
    """Returns 0 or the sticky device status (e.g. 2 = DINR_ERANGE) without raising."""
    return int(load().dinr_get_device_status(ctx))


def set_timing(ctx, enable: bool):
    _check(ctx, load().dinr_set_timing(ctx, int(enable)))


def read_timing(ctx, which: str, reset: bool = False):
    ms, n = C.c_double(), C.c_int64()
    _check(ctx, load().dinr_read_timing(ctx, TIMERS[which], C.byref(ms), C.byref(n), int(reset)))
    return ms.value, n.value


def launch_count(ctx) -> int:
    return int(load().dinr_launch_count(ctx))
