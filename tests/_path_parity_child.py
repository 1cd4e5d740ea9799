"""Child process of test_gpu_paths.py: one gradient-parity check of the training step against the
fp64 oracle, run with whatever DINR_* path switches the parent put in the environment (the library
reads them once per process).  argv: workload, json of geometry overrides, json of field
overrides, n pixels.  Prints the path the library chose and the worst per-tensor error."""
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

name, over, fover, n = sys.argv[1], json.loads(sys.argv[2]), json.loads(sys.argv[3]), int(sys.argv[4])
dev = torch.device("cuda", 0)
O.lib()
g = synth.geometry(name, **over)
th, t = synth.views(name, **over)
f = synth.field(name, **fover)
B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"], seed=1)
prm = synth.init_params(f["C"], f["L"], seed=2)
ctx = D.create(0)
D.set_geometry(ctx, g, th, t)
D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev))
idx = synth.pixel_batch(name, n, seed=8, **over)
y, _, _ = O.project_exact(g, th, t, synth.phantom(name), idx, f["combine"])
y = y.astype(np.float32)
P = synth.param_count(f["C"], f["L"])
grad = torch.zeros(P + 1, device=dev)
D.project_and_grad(ctx, torch.tensor(idx, device=dev), torch.tensor(y, device=dev), grad)
torch.cuda.synchronize()
ref, rc = O.project_and_grad(g, th, t, f, B, prm, idx, y)
assert rc == 0
got = grad.cpu().numpy().astype(np.float64)
H, off, errs = 2 * f["C"], 0, []
for _ in range(f["L"]):
    for m in (H * H, H):
        errs.append(float(np.max(np.abs(got[off:off + m] - ref[off:off + m])) / np.max(np.abs(ref[off:off + m]))))
        off += m
for m in (H, 1):
    errs.append(float(np.max(np.abs(got[off:off + m] - ref[off:off + m])) / max(np.max(np.abs(ref[off:off + m])), 1e-300)))
    off += m
print(json.dumps({"path": list(D.train_path(ctx, n)), "max_err": max(errs), "loss_rel": abs(got[P] - ref[P]) / abs(ref[P])}))
