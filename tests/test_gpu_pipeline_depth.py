"""H = 256 split path (k_tc_fwd3 / k_tc_bwd3 on CTA pairs, K5) against the fp64 oracle at batch
sizes where every CTA pair runs two or more pair-iterations, at the depths that exercise the
weight rings' schedules: L = 1 (no dX layer: K3's MMA and W-ring threads idle), L = 2, and L = 6
(the envelope's deepest H = 256 network: 24 K-half weight loads per forward iteration and 20 per
backward iteration, so the five-buffer rings start every iteration at a different buffer).
Inputs follow the conditioned recipe of tests/_fuzz_parity.py (R23): a positive head
bias and measured data above the model.  Tolerances as tests/test_gpu_parity.py (north_star):
projections 2e-3, gradients 1e-2 relative L-inf per parameter tensor."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2404_19075_b200 import _lib as D  # noqa: E402
from paper_2404_19075_b200 import synth  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2404_19075_b200 import build

    build.build()
    return torch.device("cuda", 0)


def rel_linf(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


# 80 pixels x 4 sub-rays x 256 samples = 81 920 samples = 640 tiles = 160 pair-iterations over
# at most 74 CTA pairs (148 SMs): every pair runs two or three iterations
N_PX = 80


@pytest.mark.parametrize("L", [1, 2, 6])
def test_split_path_multi_iteration_parity(dev, O, L):
    name = "cone512"
    g = synth.geometry(name)
    th, t = synth.views(name)
    f = synth.field(name, L=L)
    assert 2 * f["C"] == 256
    B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"], seed=11 + L)
    prm = synth.init_params(f["C"], f["L"], seed=12 + L, head_bias=0.5)
    ctx = D.create(0)
    try:
        D.set_geometry(ctx, g, th, t)
        D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev))
        path = D.train_path(ctx, N_PX)
        assert path[0] == 0, path  # the split path (H = 256)
        idx = synth.pixel_batch(name, N_PX, seed=13 + L)
        rf, _, rc = O.project(g, th, t, f, B, prm, idx)
        assert rc == 0
        y = (rf + np.random.default_rng(14 + L).uniform(0.05, 0.5, N_PX) * max(np.max(np.abs(rf)), 1e-3))
        y = y.astype(np.float32)
        P = synth.param_count(f["C"], f["L"])
        grad = torch.zeros(P + 1, device=dev)
        fhat = torch.zeros(N_PX, device=dev)
        D.project_and_grad(ctx, torch.tensor(idx, device=dev), torch.tensor(y, device=dev), grad)
        D.project(ctx, torch.tensor(idx, device=dev), fhat)
        torch.cuda.synchronize()
        assert D.get_device_status(ctx) == 0
    finally:
        D.destroy(ctx)
    assert rel_linf(fhat.cpu().numpy(), rf) <= 2e-3
    ref, rc = O.project_and_grad(g, th, t, f, B, prm, idx, y)
    assert rc == 0
    got = grad.cpu().numpy()
    H, off, errs = 2 * f["C"], 0, []
    for _ in range(f["L"]):
        for m in (H * H, H):
            errs.append(rel_linf(got[off:off + m], ref[off:off + m]))
            off += m
    for m in (H, 1):
        errs.append(rel_linf(got[off:off + m], ref[off:off + m]))
        off += m
    assert max(errs) <= 1e-2, errs
    assert abs(got[-1] - ref[-1]) <= 1e-2 * abs(ref[-1]), (got[-1], ref[-1])  # the loss slot


def test_deep_h256_falls_back_and_bounds(dev):
    """At H = 256 the forward kernel is chosen by shared-memory fit: L = 12 runs k_tc_fwd3, L = 16
    and L = 27 k_tc_fwd2 (k_tc_fwd3's K-half weight ring leaves room for the biases of 12 layers);
    L = 28 is refused at dinr_set_field_weights (the forward-only k_tc_mlp no longer fits;
    include/dinr.h).  Deep networks
    are outside the bf16 accuracy envelope, so this checks the launch, the status and a finite,
    batch-consistent result: the loss is the batch mean, so the gradient of a batch equals half the
    sum of its two equal halves' gradients (accumulate mode) to fp32 reduction-order precision."""
    name = "cone512"
    g = synth.geometry(name, n_s=32)
    th, t = synth.views(name, n_s=32)
    for L in (12, 16, 27):
        f = synth.field(name, L=L)
        B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"], seed=21)
        prm = synth.init_params(f["C"], f["L"], seed=22, head_bias=0.5)
        ctx = D.create(0)
        try:
            D.set_geometry(ctx, g, th, t)
            D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev))
            n = 24
            idx = torch.tensor(synth.pixel_batch(name, n, seed=23, n_s=32), device=dev)
            y = torch.full((n,), 0.5, device=dev)
            P = synth.param_count(f["C"], f["L"])
            g_all = torch.zeros(P + 1, device=dev)
            D.project_and_grad(ctx, idx, y, g_all)
            g_half = torch.zeros(P + 1, device=dev)
            D.project_and_grad(ctx, idx[: n // 2], y[: n // 2], g_half)
            D.project_and_grad(ctx, idx[n // 2:], y[n // 2:], g_half, accumulate=True)
            torch.cuda.synchronize()
            assert D.get_device_status(ctx) == 0
        finally:
            D.destroy(ctx)
        a, b = g_all[:-1].cpu().numpy(), 0.5 * g_half[:-1].cpu().numpy()
        assert np.all(np.isfinite(a)) and np.max(np.abs(a)) > 0, L
        assert rel_linf(b, a) <= 1e-4, (L, rel_linf(b, a))
    f = synth.field(name, L=28)
    ctx = D.create(0)
    try:
        D.set_geometry(ctx, g, th, t)
        B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"], seed=21)
        prm = synth.init_params(f["C"], f["L"], seed=22)
        with pytest.raises(D.DinrError):
            D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev))
    finally:
        D.destroy(ctx)
