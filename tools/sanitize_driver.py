"""One small call of every kernel family through the C ABI, for compute-sanitizer
(tools/sanitize.sh): k_fused2 + k_dw01 (fan512), k_fused2 at H = 64 (parallel64), the H = 256
split path (k_tc_fwd2, k_loss, k_tc_bwd2, k_tc_dw), the one-tile K2/K3 (k_tc_mlp), the fp32 verify
path, k_adam_pack, the N1 sampler, N2 phantom projector and N4 voxelizer.  Sizes are config-1
scale so the instrumented run takes minutes, not hours."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2404_19075_b200 import _lib as D  # noqa: E402
from paper_2404_19075_b200 import synth  # noqa: E402

dev = torch.device("cuda", 0)
which = sys.argv[1] if len(sys.argv) > 1 else "all"


def step(name, n, over=None, fover=None, precision="bf16", extra=False):
    over, fover = over or {}, fover or {}
    g = synth.geometry(name, **over)
    th, t = synth.views(name, **over)
    f = synth.field(name, **fover)
    B = torch.tensor(synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"]), device=dev)
    prm = torch.tensor(synth.init_params(f["C"], f["L"]), device=dev)
    ctx = D.create(0)
    D.set_geometry(ctx, g, th, t)
    D.set_field_weights(ctx, f, B, prm, precision=precision)
    P = synth.param_count(f["C"], f["L"])
    idx = torch.tensor(synth.pixel_batch(name, n, seed=5, **over), device=dev)
    y = torch.rand(n, device=dev)
    grad = torch.zeros(P + 1, device=dev)
    D.project_and_grad(ctx, idx, y, grad)
    fh = torch.zeros(n, device=dev)
    D.project(ctx, idx, fh)
    if extra:
        m, v = torch.zeros(P, device=dev), torch.zeros(P, device=dev)
        D.adam_step(ctx, prm, grad, m, v, lr=1e-3, step=1)
        desc = D.train_desc(seed=3, batch=n)
        ys = torch.rand(len(th) * g["n_rows"] * g["n_cols"], device=dev)
        loss = torch.zeros(2, device=dev)
        D.train_iterations(ctx, desc, 0, 2, ys, prm, m, v, grad, loss)
        D.phantom_project(ctx, synth.phantom(name), idx, fh, combine="beer", noise_frac=1e-3, seed=1)
        gr = D.default_grid(ctx)
        gr = dict(gr, nz=2)
        vox = torch.zeros(gr["nx"] * gr["ny"] * 2, device=dev)
        D.voxelize(ctx, gr, 0.0, vox, 0, 2)
    torch.cuda.synchronize()
    st = D.get_device_status(ctx)
    assert st == 0, (st, D.load().dinr_last_error(ctx))
    D.destroy(ctx)
    print("ok", name, n, over, fover, precision, flush=True)


if which in ("all", "fused"):
    step("fan512", 300, extra=True)                                  # k_fused2 + k_dw01, Adam, N1, N2, N4 (k_infer)
    step("parallel64", 2400, fover=dict(L=1))                        # k_fused2 H = 64, per-stream loss mode
if which in ("all", "split"):
    step("cone512", 40, over=dict(n_s=64), extra=True)               # k_tc_fwd2, k_tc_bwd2, k_tc_dw, K2 grid mode
    step("fan512", 60, fover=dict(L=5))                              # one-tile k_tc_mlp MODE 1 / 2 (H = 128)
if which in ("all", "verify"):
    step("fan512", 20, precision="fp32_verify")
