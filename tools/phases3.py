"""Run cone4d2048 training steps with the DINR_PHASES library variant and print k_tc_fwd3's
per-role cycle counters (stderr).  python tools/phases3.py [workload]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2404_19075_b200 import _lib as D  # noqa: E402
from paper_2404_19075_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cone4d2048"
D.load(os.path.join(ROOT, "paper_2404_19075_b200", os.environ.get("DINR_PHASES_LIB", "libdinr_phases.so")))
dev = torch.device("cuda", 0)
g = synth.geometry(name)
th, t = synth.views(name)
f = synth.field(name)
ctx = D.create(0)
D.set_geometry(ctx, g, th, t)
D.set_field_weights(ctx, f, torch.tensor(synth.grff_matrix(f["C"], 0.1, 0.5), device=dev),
                    torch.tensor(synth.init_params(f["C"], f["L"]), device=dev))
n = synth.WORKLOADS[name]["batch"]
idx = torch.tensor(synth.pixel_batch(name, n), device=dev)
y = torch.tensor(synth.synthetic_y(n, 1.0), device=dev)
grad = torch.zeros(synth.param_count(f["C"], f["L"]) + 1, device=dev)
for _ in range(3):
    D.project_and_grad(ctx, idx, y, grad)
torch.cuda.synchronize()
