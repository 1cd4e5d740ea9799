"""N4 throughput: voxelize the paper's default grid of a workload at one view time.
    python tools/bench_voxelize.py [workload] [planes]
Prints one JSON line: voxels/s (device-timed, CUDA events on the launch stream), the tensor-core
roofline of the MLP (2 L H^2 FLOP per voxel), and the file-streaming rate through
dinr_voxelize_to_file (host write included)."""
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2404_19075_b200 import _lib as D  # noqa: E402
from paper_2404_19075_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "fan512"
planes = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dev = torch.device("cuda", 0)
g = synth.geometry(name)
th, t = synth.views(name)
f = synth.field(name)
ctx = D.create(0)
D.set_geometry(ctx, g, th, t)
D.set_field_weights(ctx, f, torch.tensor(synth.grff_matrix(f["C"], 0.1, 0.5), device=dev),
                    torch.tensor(synth.init_params(f["C"], f["L"]), device=dev))
grid = D.default_grid(ctx)
kc = min(planes, grid["nz"])
n = grid["nx"] * grid["ny"] * kc
out = torch.empty(n, device=dev)
for _ in range(3):
    D.voxelize(ctx, grid, float(t[0]), out, k_begin=0, k_count=kc)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    D.voxelize(ctx, grid, float(t[0]), out, k_begin=0, k_count=kc)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
ms = ts[len(ts) // 2]
H, L = 2 * f["C"], f["L"]
flop = 2.0 * L * H * H
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
bf16 = peaks.get("bf16_tflops", 1674.3)
vps = n / (ms * 1e-3)
with tempfile.TemporaryDirectory() as d:
    path = os.path.join(d, "vol.f32")
    t0 = time.perf_counter()
    D.voxelize_to_file(ctx, dict(grid, nz=kc), path, view_begin=0, n_views=1, slab_planes=max(1, kc // 4))
    t1 = time.perf_counter()
print(json.dumps({"metric": "voxels/sec (N4 inference)", "workload": name, "grid": [grid["nx"], grid["ny"], kc],
                  "voxels": n, "ms": ms, "value": vps, "unit": "voxels/s",
                  "roofline": {"bound": "tensor", "achieved": vps * flop / 1e12, "peak": bf16, "unit": "TFLOP/s",
                               "frac": vps * flop / 1e12 / bf16},
                  "to_file_voxels_per_s": n / (t1 - t0)}))
