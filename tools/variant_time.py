"""Time the training step (project_and_grad) of one or more library variants on a workload.
    python tools/variant_time.py fan512 libdinr.so libdinr_var_a.so ...
Each variant runs in a fresh subprocess (one libdinr per process)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, sys
sys.path.insert(0, ROOT)
import torch
from paper_2404_19075_b200 import _lib as D, synth
D.load(os.path.join(ROOT, "paper_2404_19075_b200", LIB))
dev = torch.device("cuda", 0)
name = NAME
g = synth.geometry(name); th, t = synth.views(name); f = synth.field(name)
ctx = D.create(0)
D.set_geometry(ctx, g, th, t)
D.set_field_weights(ctx, f, torch.tensor(synth.grff_matrix(f["C"], 0.1, 0.5), device=dev),
                    torch.tensor(synth.init_params(f["C"], f["L"]), device=dev))
n = synth.WORKLOADS[name]["batch"]
idx = torch.tensor(synth.pixel_batch(name, n), device=dev)
y = torch.tensor(synth.synthetic_y(n, 1.0), device=dev)
grad = torch.zeros(synth.param_count(f["C"], f["L"]) + 1, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    D.project_and_grad(ctx, idx, y, grad)
ts = []
for _ in range(10):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); D.project_and_grad(ctx, idx, y, grad); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
D.set_timing(ctx, True)
for k in D.TIMERS:
    D.read_timing(ctx, k, reset=True)
for _ in range(5):
    flush.fill_(1)
    D.project_and_grad(ctx, idx, y, grad)
torch.cuda.synchronize()
D.set_timing(ctx, False)
kt = " ".join(f"{k} {D.read_timing(ctx, k, reset=True)[0] / 5:.2f}" for k in ("forward", "backward", "dw"))
print(f"{LIB:40s} median {ts[len(ts)//2]:.3f} ms  min {ts[0]:.3f} ms  loss {grad[-1].item():.6f}  [{kt}]")
"""

if __name__ == "__main__":
    name = sys.argv[1]
    for lib in sys.argv[2:]:
        code = CHILD.replace("ROOT", repr(ROOT)).replace("LIB", repr(lib)).replace("NAME", repr(name))
        subprocess.run([sys.executable, "-c", code], check=False)
