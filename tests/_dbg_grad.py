"""Debug helper: per-tensor gradient errors (GPU vs oracle) for one parity case."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2404_19075_b200 import _lib as D  # noqa: E402
from paper_2404_19075_b200 import synth  # noqa: E402
from test_gpu_parity import CASES, setup_case, tensor_errs  # noqa: E402

dev = torch.device("cuda", 0)
for case in [int(a) for a in sys.argv[1:]] or [0, 1]:
    name, over, fover, n = CASES[case]
    ctx = D.create(0)
    g, th, t, f, B, prm = setup_case(ctx, dev, name, over, fover, "bf16", "beer")
    idx = synth.pixel_batch(name, n, seed=8, **over)
    y, _, _ = O.project_exact(g, th, t, synth.phantom(name), idx, "beer")
    y = y.astype(np.float32)
    P = synth.param_count(f["C"], f["L"])
    grad = torch.zeros(P + 1, device=dev)
    D.project_and_grad(ctx, torch.tensor(idx, device=dev), torch.tensor(y, device=dev), grad)
    torch.cuda.synchronize()
    ref, rc = O.project_and_grad(g, th, t, f, B, prm, idx, y)
    errs = tensor_errs(grad.cpu().numpy()[:P], ref[:P], f["C"], f["L"])
    print(name, "path", D.train_path(ctx, n), ["%.2e" % e for e in errs], "loss", grad[P].item(), ref[P])
    D.destroy(ctx)
