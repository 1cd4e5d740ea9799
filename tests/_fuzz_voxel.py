"""Randomized N4 voxelization sweep against the fp64 oracle (test infrastructure; run by hand:
python tests/_fuzz_voxel.py [n_cases] [seed]).  Random beams, widths, depths, precisions, grid
shapes / offsets / spacings and z slabs; per case the FOV support must match exactly and the values
meet the N4 tolerances (bf16 L-inf 1.5e-2, RMS 3e-3; fp32 verify 1e-5)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_19075_b200 import _lib as D  # noqa: E402
from paper_2404_19075_b200 import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
dev = torch.device("cuda", 0)
O.lib()
fails = 0
for k in range(n_cases):
    name = str(rng.choice(["parallel64", "fan512", "cone512", "cone4d512"]))
    fover = {"C": int(rng.choice([32, 64, 128])), "L": int(rng.integers(1, 7))}
    prec = "fp32_verify" if rng.random() < 0.25 else "bf16"
    g = synth.geometry(name)
    th, t = synth.views(name)
    f = synth.field(name, **fover)
    B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"], seed=1 + k)
    prm = synth.init_params(f["C"], f["L"], seed=2 + k)
    ctx = D.create(0)
    D.set_geometry(ctx, g, th, t)
    D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev), precision=prec)
    r = g["fov_radius"]
    nx, ny, nz = int(rng.integers(1, 41)), int(rng.integers(1, 41)), int(rng.integers(1, 6))
    vx = 2.2 * r / nx * float(rng.uniform(0.5, 1.2))
    vy = 2.2 * r / ny * float(rng.uniform(0.5, 1.2))
    zlo, zhi = float(g.get("z_lo", -1.0)), float(g.get("z_hi", 1.0))
    vz = float(rng.uniform(0.05, 1.0)) * max(abs(zhi - zlo), 1.0) / nz
    grid = dict(nx=nx, ny=ny, nz=nz, x0=-0.5 * nx * vx + float(rng.uniform(-2, 2)), y0=-0.5 * ny * vy,
                z0=float(rng.uniform(-1, 0)) * nz * vz, vx=vx, vy=vy, vz=vz)
    k0 = int(rng.integers(0, nz))
    kc = int(rng.integers(1, nz - k0 + 1))
    tv = float(t[int(rng.integers(0, len(t)))])
    out = torch.full((nx * ny * kc,), 7.0, device=dev)
    D.voxelize(ctx, grid, tv, out, k_begin=k0, k_count=kc)
    torch.cuda.synchronize()
    ref = O.voxelize(g, f, B, prm, grid, tv, k_begin=k0, k_count=kc).ravel()
    got = out.cpu().numpy().astype(np.float64)
    support_ok = bool(np.array_equal(got == 0.0, ref == 0.0))
    mx = max(float(np.max(np.abs(ref))), 1e-300)
    linf = float(np.max(np.abs(got - ref))) / mx
    nzm = ref != 0
    rms = float(np.sqrt(np.mean((got - ref)[nzm] ** 2)) / mx) if nzm.any() else 0.0
    tol, rtol = (1e-5, 1e-5) if prec == "fp32_verify" else (1.5e-2, 3e-3)
    ok = support_ok and linf <= tol and rms <= rtol
    fails += 0 if ok else 1
    print(json.dumps({"case": k, "ok": ok, "name": name, "field": fover, "prec": prec, "grid": [nx, ny, nz, k0, kc],
                      "support_ok": support_ok, "linf": linf, "rms": rms}), flush=True)
    D.destroy(ctx)
print(f"{n_cases - fails}/{n_cases} cases within tolerance")
sys.exit(1 if fails else 0)
