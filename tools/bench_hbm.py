"""HBM-bound kernels of the hot path measured standalone at a large size: the ray
setup K1 (k_ray_setup) and the pixel combine / loss K4 (k_loss), timed by the library's own CUDA
events on the launch stream inside dinr_project.  Algorithmic bytes per pixel (DESIGN.md "HBM
kernels"):
  K1: 8 (pixel index) + S * (32 (two float4 ray records) + 4 (quadrature weight)) written
  K4: S * (4 (quadrature weight) + 4 * N_s / 32 (ray-chunk sums)) + 4 (f-hat)
    python tools/bench_hbm.py [log2_rays]        # default 2^26 rays
Prints one JSON line per geometry."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_19075_b200 import _lib as D  # noqa: E402
from paper_2404_19075_b200 import synth  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
dev = torch.device("cuda", 0)
with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
    pk = json.load(fh)
hbm = float(pk.get("hbm_gbs", 6555.5))
for name, over in [("parallel64", {}), ("cone512", {"n_s": 32})]:
    g = synth.geometry(name, **over)
    th, t = synth.views(name, **over)
    f = synth.field(name, C=32, L=1)  # tiny MLP: the forward between K1 and K4 is not measured here
    ctx = D.create(0)
    D.set_geometry(ctx, g, th, t)
    D.set_field_weights(ctx, f, torch.tensor(synth.grff_matrix(f["C"], 0.1, 0.5), device=dev),
                        torch.tensor(synth.init_params(f["C"], f["L"]), device=dev))
    S = g["sub_x"] * g["sub_z"]
    ns = g["n_s"]
    n = (1 << lg) // S
    npx = len(th) * g["n_rows"] * g["n_cols"]
    idx = torch.randint(0, npx, (n,), device=dev, dtype=torch.int64)
    fhat = torch.empty(n, device=dev)
    for _ in range(2):
        D.project(ctx, idx, fhat)
    torch.cuda.synchronize()
    D.set_timing(ctx, True)
    for k in D.TIMERS:
        D.read_timing(ctx, k, reset=True)
    reps = 5
    for _ in range(reps):
        D.project(ctx, idx, fhat)
    torch.cuda.synchronize()
    tr, nr = D.read_timing(ctx, "rays", reset=True)
    tl, nl = D.read_timing(ctx, "loss", reset=True)
    D.set_timing(ctx, False)
    b1 = n * (8 + S * 36)
    b4 = n * (S * (4 + 4 * (ns // 32)) + 4)
    r1 = b1 / (tr / max(1, nr) / 1e3) / 1e9
    r4 = b4 / (tl / max(1, nl) / 1e3) / 1e9
    print(json.dumps({"geometry": name, "pixels": n, "rays": n * S, "S": S, "n_s": ns,
                      "k_ray_setup": {"ms": tr / max(1, nr), "bytes": b1, "GB_s": r1, "frac_hbm": r1 / hbm},
                      "k_loss": {"ms": tl / max(1, nl), "bytes": b4, "GB_s": r4, "frac_hbm": r4 / hbm},
                      "hbm_peak_GB_s": hbm}))
    D.destroy(ctx)
