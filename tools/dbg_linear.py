"""Debug: batch linearity of the training gradient (full batch vs 4 exact quarters)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2404_19075_b200 import _lib as D, synth
if os.environ.get("DINR_LIB"): D.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2404_19075_b200", os.environ["DINR_LIB"]))
dev = torch.device("cuda", 0)
name = sys.argv[1]
prec = sys.argv[3] if len(sys.argv) > 3 else "bf16"
for n in [int(x) for x in sys.argv[2].split(",")]:
    g = synth.geometry(name); th, t = synth.views(name); f = synth.field(name)
    ctx = D.create(0)
    D.set_geometry(ctx, g, th, t)
    D.set_field_weights(ctx, f, torch.tensor(synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"], seed=1), device=dev),
                        torch.tensor(synth.init_params(f["C"], f["L"], seed=2), device=dev), precision=prec)
    idx = torch.tensor(synth.pixel_batch(name, n, seed=5), device=dev)
    y = torch.tensor(synth.synthetic_y(n, 1.0, seed=6), device=dev)
    P = synth.param_count(f["C"], f["L"])
    full = torch.zeros(P + 1, device=dev)
    D.project_and_grad(ctx, idx, y, full)
    acc = torch.zeros(P + 1, dtype=torch.float64, device=dev)
    for k in range(4):
        a, b = k * n // 4, (k + 1) * n // 4
        part = torch.zeros(P + 1, device=dev)
        D.project_and_grad(ctx, idx[a:b].contiguous(), y[a:b].contiguous(), part)
        acc += part.double() * 0.25
    full, acc = full.double().cpu().numpy(), acc.cpu().numpy()
    H = 2 * f["C"]; off = 0; errs = []
    for l in range(f["L"]):
        for m in (H * H, H):
            d = full[off:off + m] - acc[off:off + m]
            errs.append(float(np.max(np.abs(d)) / np.max(np.abs(acc[off:off + m]))))
            off += m
    print(name, prec, n, "loss", full[P], acc[P], "max tensor err", ["%.1e" % e for e in errs])
    D.destroy(ctx)
