"""Seeded synthetic-input generators shared by the tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic (no ray geometry, no quadrature, no
network, no loss).  It only produces plain numbers: scanner/view/field descriptions of the
BASELINE.json workloads (recipe in DESIGN.md "Input recipe"), the frozen GRFF matrix B,
random-init network parameters, pixel batches and phantom descriptions.  Both the CUDA path
(through the C ABI) and the fp64 oracle consume exactly these values.
"""
from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------------------
# Workloads (BASELINE.json "configs"; concrete numbers proposed in SURVEY.md 8(d)).
# Lengths in mm, angles in degrees here (converted to radians by views()).
# ---------------------------------------------------------------------------------------
WORKLOADS = {
    # configs[0]: parallel-beam, 64x64 detector, 60 views, static sphere, 3x64 MLP, 32 samples/ray, 1 sub-ray
    "parallel64": dict(
        beam="parallel", n_rows=64, n_cols=64, sub_x=1, sub_z=1, n_s=32,
        sod=64.0, odd=64.0, pixel_dx=1.0, pixel_dz=1.0, fov_radius=32.0, rot_center_x=0.0,
        n_views=60, dtheta_deg=3.0, dt=0.0, C=32, L=3, mu0=0.05, sigma_s=0.5, sigma_t=0.1,
        batch=131072,
        phantom=[dict(kind="indicator", value=0.05, center=(3.0, -2.0, 0.0), axes=(20.0, 20.0, 20.0))],
    ),
    # configs[1]: fan-beam single slice, 512 cols, 360 views, 2 sub-rays/pixel, 128 samples/ray, 4x128 MLP
    "fan512": dict(
        beam="fan", n_rows=1, n_cols=512, sub_x=2, sub_z=1, n_s=128,
        sod=500.0, odd=500.0, pixel_dx=1.0, pixel_dz=1.0,
        fov_radius=500.0 * math.sin(math.atan(256.0 / 1000.0)), rot_center_x=0.0,
        n_views=360, dtheta_deg=1.0, dt=0.0, C=64, L=4, mu0=0.02, sigma_s=0.5, sigma_t=0.1,
        batch=16384,
        phantom=[
            dict(kind="indicator", value=0.02, center=(0.0, 0.0, 0.0), axes=(90.0, 110.0, 1e3)),
            dict(kind="indicator", value=-0.016, center=(0.0, -2.0, 0.0), axes=(85.0, 104.0, 1e3)),
            dict(kind="indicator", value=0.01, center=(25.0, 10.0, 0.0), axes=(20.0, 35.0, 1e3)),
            dict(kind="indicator", value=0.01, center=(-25.0, 10.0, 0.0), axes=(25.0, 40.0, 1e3)),
            dict(kind="indicator", value=0.005, center=(0.0, -50.0, 0.0), axes=(10.0, 10.0, 1e3)),
        ],
    ),
    # configs[2]: cone-beam static, 512x512 detector, 720 views, 2x2 sub-rays, 256 samples/ray, 6x256 MLP
    "cone512": dict(
        beam="cone", n_rows=512, n_cols=512, sub_x=2, sub_z=2, n_s=256,
        sod=80.0, odd=60.0, pixel_dx=0.13832, pixel_dz=0.13832,
        fov_radius=80.0 * math.sin(math.atan(35.41 / 140.0)), rot_center_x=0.0,
        n_views=720, dtheta_deg=0.5, dt=0.0, C=128, L=6, mu0=0.05, sigma_s=0.5, sigma_t=0.1,
        batch=4096,
        phantom=[
            dict(kind="indicator", value=0.04, center=(0.0, 0.0, 0.0), axes=(15.0, 17.0, 14.0)),
            dict(kind="indicator", value=0.03, center=(4.0, 3.0, 2.0), axes=(3.0, 5.0, 6.0)),
            dict(kind="indicator", value=0.02, center=(-5.0, -2.0, -3.0), axes=(4.0, 2.5, 5.0)),
        ],
    ),
    # configs[3]: cone-beam 4D, 512x512, 1800 views over continuous rotation, t-conditioned MLP
    "cone4d512": dict(
        beam="cone", n_rows=512, n_cols=512, sub_x=2, sub_z=2, n_s=256,
        sod=80.0, odd=60.0, pixel_dx=0.13832, pixel_dz=0.13832,
        fov_radius=80.0 * math.sin(math.atan(35.41 / 140.0)), rot_center_x=0.0,
        n_views=1800, dtheta_deg=1.0, dt=10.0, C=128, L=5, mu0=0.05, sigma_s=0.5, sigma_t=0.1,
        batch=4096,
        phantom=[
            dict(kind="indicator", value=0.04, center=(0.0, 0.0, 0.0), axes=(15.0, 15.0, 12.0),
                 axes_rate=(0.0, 0.0, -0.0003)),
            dict(kind="indicator", value=0.03, center=(3.0, 0.0, 0.0), axes=(2.0, 12.0, 2.0),
                 velocity=(0.0, 0.0, -0.0002)),
        ],
    ),
    # configs[4]: large cone-beam 4D, 2048x2048, 3600 views, 2x2 sub-rays, 512 samples/ray
    "cone4d2048": dict(
        beam="cone", n_rows=2048, n_cols=2048, sub_x=2, sub_z=2, n_s=512,
        sod=80.0, odd=60.0, pixel_dx=0.03458, pixel_dz=0.03458,
        fov_radius=80.0 * math.sin(math.atan(35.41 / 140.0)), rot_center_x=0.0,
        n_views=3600, dtheta_deg=1.0, dt=10.0, C=128, L=5, mu0=0.05, sigma_s=0.5, sigma_t=0.1,
        batch=2048,
        phantom=[
            dict(kind="indicator", value=0.04, center=(0.0, 0.0, 0.0), axes=(15.0, 15.0, 12.0),
                 axes_rate=(0.0, 0.0, -0.00015)),
        ],
    ),
}

BASELINE_CONFIG_NAMES = ["parallel64", "fan512", "cone512", "cone4d512", "cone4d2048"]


def geometry(name: str, **over) -> dict:
    """Plain-number scanner description (keys mirror dinr_geometry / or_geom)."""
    w = dict(WORKLOADS[name])
    w.update(over)
    g = {k: w[k] for k in ("beam", "n_rows", "n_cols", "sub_x", "sub_z", "n_s", "sod", "odd",
                           "pixel_dx", "pixel_dz", "fov_radius", "rot_center_x")}
    # Optical axis at the panel centre: C_x, C_z = half panel extents.
    g["offset_cx"] = w.get("offset_cx", 0.5 * g["n_cols"] * g["pixel_dx"])
    g["offset_cz"] = w.get("offset_cz", 0.5 * g["n_rows"] * g["pixel_dz"])
    # Normalization box (reading R11): detector z extent, scaled for cone beam to the
    # far side of the FOV cylinder; t over the view schedule.
    zlo, zhi = -g["offset_cz"], -g["offset_cz"] + g["n_rows"] * g["pixel_dz"]
    if g["beam"] == "cone":
        mag_far = (g["sod"] + g["fov_radius"]) / (g["sod"] + g["odd"])
        zlo, zhi = zlo * mag_far, zhi * mag_far
    g["z_lo"], g["z_hi"] = w.get("z_lo", zlo), w.get("z_hi", zhi)
    nv = w["n_views"]
    g["t_lo"], g["t_hi"] = 0.0, float((nv - 1) * w["dt"])
    return g


def views(name: str, **over):
    """theta_k = k * dtheta (radians), t_k = k * dt (T_m ~ 10 m s)."""
    w = dict(WORKLOADS[name])
    w.update(over)
    k = np.arange(w["n_views"], dtype=np.float64)
    return np.deg2rad(k * w["dtheta_deg"]), k * float(w["dt"])


def field(name: str, combine: str = "beer", **over) -> dict:
    w = dict(WORKLOADS[name])
    w.update(over)
    return dict(C=int(w["C"]), L=int(w["L"]), mu0=float(w["mu0"]), combine=combine,
                sigma_s=float(w["sigma_s"]), sigma_t=float(w["sigma_t"]))


def bf16_round(x) -> np.ndarray:
    """Round fp32 values to the nearest bf16-representable fp32 (ties to even)."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(a.shape)


def grff_matrix(C: int, sigma_t: float, sigma_s: float, seed: int = 1) -> np.ndarray:
    """B (C x 4, columns t,z,y,x): col 0 ~ N(0, sigma_t^2), cols 1..3 ~ N(0, sigma_s^2)."""
    rng = np.random.default_rng(seed)
    B = rng.standard_normal((C, 4))
    B[:, 0] *= sigma_t
    B[:, 1:] *= sigma_s
    return B.astype(np.float32)


def param_count(C: int, L: int) -> int:
    H = 2 * C
    return L * (H * H + H) + H + 1


def init_params(C: int, L: int, seed: int = 2, bf16: bool = True, head_bias: float | None = None) -> np.ndarray:
    """Flat fp32 gamma in the D5 layout: [W_1, b_1, ..., W_L, b_L, w_o, b_o]; every entry
    ~ U(-1/sqrt(H), 1/sqrt(H)) (PyTorch nn.Linear default, R18); optionally rounded
    to bf16-representable values so the bf16 path sees the same weights as the oracle."""
    H = 2 * C
    rng = np.random.default_rng(seed)
    p = rng.uniform(-1.0, 1.0, size=param_count(C, L)) / math.sqrt(H)
    if head_bias is not None:
        p[-1] = head_bias
    p = p.astype(np.float32)
    return bf16_round(p) if bf16 else p


def pixel_batch(name: str, n: int, seed: int = 3, rank: int = 0, world: int = 1, **over) -> np.ndarray:
    """n distinct flat pixel indices i = m*N + n drawn uniformly without
    replacement from the views owned by `rank` (views k with k % world == rank)."""
    w = dict(WORKLOADS[name])
    w.update(over)
    N = int(w["n_rows"]) * int(w["n_cols"])
    own = np.arange(rank, int(w["n_views"]), world, dtype=np.int64)
    total = len(own) * N
    rng = np.random.default_rng(seed + rank)
    if n > total:
        raise ValueError("batch larger than the shard")
    if total <= 1 << 24:
        flat = rng.choice(total, size=n, replace=False)
    else:
        flat = np.unique(rng.integers(0, total, size=int(n * 1.05) + 16))
        while len(flat) < n:
            flat = np.unique(np.concatenate([flat, rng.integers(0, total, size=n)]))
        flat = rng.permutation(flat)[:n]
    k = own[flat // N]
    return (k * N + flat % N).astype(np.int64)


def synthetic_y(n: int, scale: float, seed: int = 4) -> np.ndarray:
    """Throughput-only measured projections (values do not change the work): U(0, scale)."""
    rng = np.random.default_rng(seed)
    return (rng.uniform(0.0, scale, size=n)).astype(np.float32)


def phantom(name: str):
    return [dict(p) for p in WORKLOADS[name]["phantom"]]
