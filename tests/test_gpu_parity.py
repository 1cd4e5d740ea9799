"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs (paper_2404_19075_b200.synth).  Tolerances (north_star / DESIGN.md "Parity"):
  ray records (K1, fp64)             bit-identical
  projections, bf16 tensor-core path  relative L-inf <= 2e-3
  gradients, bf16 tensor-core path    relative L-inf <= 1e-2 per parameter tensor
  projections, fp32 verify path       relative L-inf <= 1e-5
  gradients, fp32 verify path         relative L-inf <= 1e-4 per parameter tensor
relative L-inf = max|gpu - oracle| / max|oracle| (R23)."""
import math

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


@pytest.fixture()
def ctx(dev):
    c = D.create(0)
    yield c
    D.destroy(c)


def rel_linf(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def tensor_errs(g, ref, C_, L):
    H = 2 * C_
    out, off = [], 0
    for _ in range(L):
        for n in (H * H, H):
            out.append(rel_linf(g[off:off + n], ref[off:off + n]))
            off += n
    for n in (H, 1):
        out.append(rel_linf(g[off:off + n], ref[off:off + n]))
        off += n
    return out


def small(name, **over):
    """A reduced-size copy of a BASELINE workload (same geometry, fewer views/smaller batch)."""
    g = synth.geometry(name, **over)
    th, t = synth.views(name, **over)
    return g, th, t


CASES = [
    # (workload, overrides, field overrides, n pixels)  -- chosen to span several tiles + ragged tails
    ("parallel64", {}, {}, 45),
    ("fan512", {}, {}, 13),
    ("cone512", dict(n_s=64), dict(C=64, L=3), 9),
    ("cone4d512", dict(n_s=32), dict(C=32, L=2), 11),
    ("cone512", dict(n_s=32), {}, 5),          # H = 256, streamed weights
]


def setup_case(ctx, dev, name, over, fover, precision, combine, seed=0):
    g, th, t = small(name, **over)
    f = synth.field(name, combine=combine, **fover)
    B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"], seed=1 + seed)
    prm = synth.init_params(f["C"], f["L"], seed=2 + seed)
    D.set_geometry(ctx, g, th, t)
    D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev), precision=precision)
    return g, th, t, f, B, prm


@pytest.mark.parametrize("beam", ["parallel", "fan", "cone"])
def test_ray_records_bit_identical(ctx, dev, O, beam):
    rng = np.random.default_rng(5)
    g = dict(beam=beam, n_rows=37, n_cols=53, sub_x=2, sub_z=3 if beam == "cone" else 1, n_s=32, sod=31.0,
             odd=17.5, pixel_dx=0.37, pixel_dz=0.41, offset_cx=9.7, offset_cz=7.3, fov_radius=10.1,
             rot_center_x=0.61, z_lo=-8.0, z_hi=8.0, t_lo=0.0, t_hi=10.0)
    M = 97
    th = rng.uniform(-7, 7, M)
    t = np.sort(rng.uniform(0, 10, M))
    D.set_geometry(ctx, g, th, t)
    idx = rng.integers(0, M * g["n_rows"] * g["n_cols"], 5000)
    idx[:3] = [0, M * g["n_rows"] * g["n_cols"] - 1, g["n_cols"] - 1]
    S = g["sub_x"] * g["sub_z"]
    rec = torch.zeros(len(idx) * S * 9, dtype=torch.float64, device=dev)
    D.ray_records(ctx, torch.tensor(idx, device=dev), rec)
    torch.cuda.synchronize()
    ref, rc = O.rays(g, th, idx)
    assert rc == 0
    got = rec.cpu().numpy().reshape(len(idx), S, 9)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), np.argwhere(got != ref)[:5]
    if beam == "parallel":  # column 0 lies outside the FOV: misses are in the bit-match too
        assert np.any(ref[:, :, 8] == 0) and np.any(ref[:, :, 8] > 0)


@pytest.mark.parametrize("precision,tol", [("bf16", 2e-3), ("fp32_verify", 1e-5)])
@pytest.mark.parametrize("combine", ["beer", "linear"])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_projection_parity(ctx, dev, O, precision, tol, combine, case):
    name, over, fover, n = CASES[case]
    g, th, t, f, B, prm = setup_case(ctx, dev, name, over, fover, precision, combine)
    idx = synth.pixel_batch(name, n, seed=7, **over)
    S = g["sub_x"] * g["sub_z"]
    fhat = torch.zeros(n, device=dev)
    psub = torch.zeros(n * S, device=dev)
    D.project(ctx, torch.tensor(idx, device=dev), fhat, psub)
    torch.cuda.synchronize()
    rf, rp, rc = O.project(g, th, t, f, B, prm, idx)
    assert rc == 0
    ep = rel_linf(psub.cpu().numpy().reshape(n, S), rp)
    ef = rel_linf(fhat.cpu().numpy(), rf)
    assert ep <= tol and ef <= tol, (ep, ef)


@pytest.mark.parametrize("precision,tol", [("bf16", 1e-2), ("fp32_verify", 1e-4)])
@pytest.mark.parametrize("combine", ["beer", "linear"])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_gradient_parity(ctx, dev, O, precision, tol, combine, case):
    name, over, fover, n = CASES[case]
    g, th, t, f, B, prm = setup_case(ctx, dev, name, over, fover, precision, combine)
    idx = synth.pixel_batch(name, n, seed=8, **over)
    # measured data = exact (noiseless) line integrals of the workload phantom (DESIGN.md input recipe)
    y, _, _ = O.project_exact(g, th, t, synth.phantom(name), idx, combine)
    y = y.astype(np.float32)
    P = synth.param_count(f["C"], f["L"])
    grad = torch.zeros(P + 1, device=dev)
    D.project_and_grad(ctx, torch.tensor(idx, device=dev), torch.tensor(y, device=dev), grad)
    torch.cuda.synchronize()
    ref, rc = O.project_and_grad(g, th, t, f, B, prm, idx, y)
    assert rc == 0
    got = grad.cpu().numpy()
    errs = tensor_errs(got[:P], ref[:P], f["C"], f["L"])
    assert max(errs) <= tol, errs
    assert abs(got[P] - ref[P]) <= max(tol, 1e-6) * abs(ref[P])


def test_constant_field_chord(ctx, dev, O):
    """w_o = 0, b_o = 1, mu0 = 2^-4: p_s = mu0 chord_s, only fp32 rounding of chord/N_s."""
    g, th, t = small("fan512")
    f = synth.field("fan512", combine="beer", mu0=0.0625)
    prm = synth.init_params(f["C"], f["L"])
    H = 2 * f["C"]
    prm[f["L"] * (H * H + H):-1] = 0.0
    prm[-1] = 1.0
    B = synth.grff_matrix(f["C"], 0.1, 0.5)
    D.set_geometry(ctx, g, th, t)
    D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev))
    idx = synth.pixel_batch("fan512", 300, seed=3)
    fhat = torch.zeros(300, device=dev)
    psub = torch.zeros(600, device=dev)
    D.project(ctx, torch.tensor(idx, device=dev), fhat, psub)
    rec, _ = O.rays(g, th, idx)
    assert rel_linf(psub.cpu().numpy().reshape(300, 2), 0.0625 * rec[:, :, 8]) <= 5e-7


def test_edge_cases(ctx, dev, O):
    g, th, t, f, B, prm = setup_case(ctx, dev, "parallel64", {}, {}, "bf16", "beer")
    P = synth.param_count(f["C"], f["L"])
    # n = 0: zeros, and accumulate leaves the buffer alone
    grad = torch.full((P + 1,), 3.0, device=dev)
    D.project_and_grad(ctx, torch.zeros(0, dtype=torch.int64, device=dev), torch.zeros(0, device=dev), grad)
    assert torch.count_nonzero(grad).item() == 0
    # accumulate = 1 doubles
    idx = torch.tensor(synth.pixel_batch("parallel64", 7, seed=1), device=dev)
    y = torch.rand(7, device=dev)
    g1 = torch.zeros(P + 1, device=dev)
    D.project_and_grad(ctx, idx, y, g1)
    g2 = g1.clone()
    D.project_and_grad(ctx, idx, y, g2, accumulate=True)
    assert torch.allclose(g2, 2 * g1)
    # out-of-range index -> fhat 0 and sticky DINR_ERANGE
    bad = torch.tensor([5, 10**9], dtype=torch.int64, device=dev)
    fh = torch.full((2,), 7.0, device=dev)
    D.project(ctx, bad, fh)
    assert D.get_device_status(ctx) == 2
    assert fh[1].item() == 0.0
    assert D.get_device_status(ctx) == 0
    # invalid geometry is rejected with no side effects
    g_bad = dict(g, fov_radius=1e6)
    with pytest.raises(D.DinrError):
        D.set_geometry(ctx, g_bad, th, t)
    D.project(ctx, idx, torch.zeros(7, device=dev))


def test_host_entry_point_matches_device(ctx, dev, O):
    g, th, t, f, B, prm = setup_case(ctx, dev, "fan512", {}, {}, "bf16", "beer")
    P = synth.param_count(f["C"], f["L"])
    idx = synth.pixel_batch("fan512", 64, seed=4)
    y = synth.synthetic_y(64, 1.0)
    g_dev = torch.zeros(P + 1, device=dev)
    D.project_and_grad(ctx, torch.tensor(idx, device=dev), torch.tensor(y, device=dev), g_dev)
    g_host = np.zeros(P + 1, dtype=np.float32)
    D.project_and_grad_host(ctx, np.ascontiguousarray(idx), np.ascontiguousarray(y), g_host)
    assert np.array_equal(g_host, g_dev.cpu().numpy())


def test_allreduce_world1_identity(ctx, dev):
    g, th, t, f, B, prm = setup_case(ctx, dev, "parallel64", {}, {}, "bf16", "beer")
    D.comm_init(ctx, D.nccl_unique_id(), 0, 1)
    x = torch.randn(1000, device=dev)
    x0 = x.clone()
    D.allreduce_grads(ctx, x)
    torch.cuda.synchronize()
    assert torch.equal(x, x0)


@pytest.mark.parametrize("name", ["fan512", "cone512"])
def test_full_size_batch_sampled(ctx, dev, O, name):
    """BASELINE batch size in the bench launch configuration; sampled pixels checked against
    the oracle one by one (bf16 tolerance)."""
    g, th, t, f, B, prm = setup_case(ctx, dev, name, {}, {}, "bf16", "beer")
    n = synth.WORKLOADS[name]["batch"]
    idx = synth.pixel_batch(name, n, seed=11)
    fhat = torch.zeros(n, device=dev)
    D.project(ctx, torch.tensor(idx, device=dev), fhat)
    torch.cuda.synchronize()
    pick = np.random.default_rng(0).choice(n, 24, replace=False)
    rf, _, _ = O.project(g, th, t, f, B, prm, idx[pick])
    assert rel_linf(fhat.cpu().numpy()[pick], rf) <= 2e-3
    assert np.all(np.isfinite(fhat.cpu().numpy()))


@pytest.mark.parametrize("name", ["fan512", "cone512"])
def test_full_size_gradient_is_batch_linear(ctx, dev, name):
    """The training step at the BASELINE batch, in the bench launch configuration (every CTA busy,
    full K-splits, the fused path's ring and stashes at full size), against the same step run as
    four quarter batches: the loss and the gradient are means over pixels, so the full-batch values
    must be the means of the quarters.  Exact quarters scale the upstream factors (and so every
    bf16-rounded delta) by exactly 4, so per-sample arithmetic is identical up to that power of two
    and only the fp32 reduction order differs (tolerance 1e-4 of the largest entry per tensor;
    uneven splits would re-round every delta in bf16: ~1e-3 after the pixel sum's cancellation)."""
    g, th, t, f, B, prm = setup_case(ctx, dev, name, {}, {}, "bf16", "beer")
    n = synth.WORKLOADS[name]["batch"]
    idx = torch.tensor(synth.pixel_batch(name, n, seed=5), device=dev)
    y = torch.tensor(synth.synthetic_y(n, 1.0, seed=6), device=dev)
    P = synth.param_count(f["C"], f["L"])
    full = torch.zeros(P + 1, device=dev)
    D.project_and_grad(ctx, idx, y, full)
    acc = torch.zeros(P + 1, dtype=torch.float64, device=dev)
    assert n % 4 == 0
    for k in range(4):
        a, b = k * n // 4, (k + 1) * n // 4
        part = torch.zeros(P + 1, device=dev)
        D.project_and_grad(ctx, idx[a:b].contiguous(), y[a:b].contiguous(), part)
        acc += part.double() * 0.25
    torch.cuda.synchronize()
    full, acc = full.double().cpu().numpy(), acc.cpu().numpy()
    assert np.all(np.isfinite(full))
    assert abs(full[P] - acc[P]) <= 1e-4 * abs(acc[P])  # loss
    errs = tensor_errs(full[:P], acc[:P], f["C"], f["L"])
    assert max(errs) <= 1e-4, errs


def test_adam_step_parity_and_repack(ctx, dev, O):
    """N1: the fused Adam + re-pack kernel matches the oracle's Adam (fp32 tolerance) and the
    re-packed bf16 images equal those of dinr_set_field_weights on the updated parameters."""
    g, th, t, f, B, prm = setup_case(ctx, dev, "fan512", {}, {}, "bf16", "beer")
    P = synth.param_count(f["C"], f["L"])
    rng = np.random.default_rng(12)
    grad = rng.standard_normal(P + 1).astype(np.float32) * 1e-3
    m0 = rng.standard_normal(P).astype(np.float32) * 1e-4
    v0 = np.abs(rng.standard_normal(P)).astype(np.float32) * 1e-6
    pt, mt, vt = (torch.tensor(a, device=dev) for a in (prm, m0, v0))
    D.adam_step(ctx, pt, torch.tensor(grad, device=dev), mt, vt, lr=1e-3, step=3)
    rp, rm, rv = O.adam_step(prm, grad[:P], m0, v0, lr=1e-3, step=3)
    assert np.allclose(pt.cpu().numpy(), rp, rtol=1e-5, atol=1e-7)
    # fp32 arithmetic on |m| ~ 1e-4, |v| ~ 1e-6: absolute rounding ~ 1e-11 / 1e-13 near cancellation
    assert np.allclose(mt.cpu().numpy(), rm, rtol=1e-5, atol=1e-10)
    assert np.allclose(vt.cpu().numpy(), rv, rtol=1e-5, atol=1e-12)
    idx = torch.tensor(synth.pixel_batch("fan512", 200, seed=5), device=dev)
    f1 = torch.zeros(200, device=dev)
    D.project(ctx, idx, f1)
    D.set_field_weights(ctx, f, torch.tensor(B, device=dev), pt.clone())
    f2 = torch.zeros(200, device=dev)
    D.project(ctx, idx, f2)
    assert torch.equal(f1, f2)


# Fused-kernel variants (k_fused2 + k_dw01 / K5): pixel-group layouts (S N_s = 256 or 128, 1 or 2
# pixels per group), depths (nu = 0, 1, 2 unfused layers), tiny and ragged batches.
FUSED_SHAPES = [
    ("fan512", dict(sub_x=1, n_s=256), {}, 7),            # one ray = one group, nu = 2 (k_dw01)
    ("fan512", dict(sub_x=2, n_s=64), {}, 9),             # two pixels per group
    ("fan512", dict(sub_x=4, n_s=32), {}, 5),             # four sub-rays, two pixels per group
    ("fan512", {}, dict(L=3), 6),                         # nu = 1: K5 with layer-0 feature recompute
    ("fan512", {}, dict(L=2), 6),                         # nu = 0: every dW fused
    ("cone512", dict(n_s=64), dict(C=64, L=4), 3),        # cone, 2 x 2 sub-rays, H = 128
    ("fan512", {}, {}, 1),                                # a single pixel (ragged last group)
]


@pytest.mark.parametrize("case", range(len(FUSED_SHAPES)))
def test_fused_path_shapes(ctx, dev, O, case):
    name, over, fover, n = FUSED_SHAPES[case]
    g, th, t, f, B, prm = setup_case(ctx, dev, name, over, fover, "bf16", "beer")
    kind, _ = D.train_path(ctx, n)
    assert kind == 2  # the two-stream fused kernel
    idx = synth.pixel_batch(name, n, seed=21 + case, **over)
    S = g["sub_x"] * g["sub_z"]
    fhat = torch.zeros(n, device=dev)
    psub = torch.zeros(n * S, device=dev)
    D.project(ctx, torch.tensor(idx, device=dev), fhat, psub)
    rf, rp, rc = O.project(g, th, t, f, B, prm, idx)
    assert rel_linf(fhat.cpu().numpy(), rf) <= 2e-3
    y, _, _ = O.project_exact(g, th, t, synth.phantom(name), idx, "beer")
    y = y.astype(np.float32)
    P = synth.param_count(f["C"], f["L"])
    grad = torch.zeros(P + 1, device=dev)
    D.project_and_grad(ctx, torch.tensor(idx, device=dev), torch.tensor(y, device=dev), grad)
    torch.cuda.synchronize()
    ref, rc = O.project_and_grad(g, th, t, f, B, prm, idx, y)
    got = grad.cpu().numpy()
    assert max(tensor_errs(got[:P], ref[:P], f["C"], f["L"])) <= 1e-2
    assert abs(got[P] - ref[P]) <= 1e-2 * abs(ref[P])


@pytest.mark.parametrize("L", [5, 6])
def test_deep_h128_network_takes_a_path_that_fits(ctx, dev, O, L):
    """H = 128 with L >= 5: W_1..W_{L-1} no longer fit either fused kernel's shared memory; the
    step must take the split path (it used to fail in cudaFuncSetAttribute) and stay in tolerance."""
    g, th, t, f, B, prm = setup_case(ctx, dev, "fan512", {}, dict(L=L), "bf16", "beer")
    n = 6
    assert D.train_path(ctx, n)[0] == 0
    idx = synth.pixel_batch("fan512", n, seed=8)
    y, _, _ = O.project_exact(g, th, t, synth.phantom("fan512"), idx, "beer")
    y = y.astype(np.float32)
    P = synth.param_count(f["C"], f["L"])
    grad = torch.zeros(P + 1, device=dev)
    D.project_and_grad(ctx, torch.tensor(idx, device=dev), torch.tensor(y, device=dev), grad)
    torch.cuda.synchronize()
    ref, rc = O.project_and_grad(g, th, t, f, B, prm, idx, y)
    got = grad.cpu().numpy()
    assert max(tensor_errs(got[:P], ref[:P], f["C"], f["L"])) <= 1e-2


@pytest.mark.parametrize("name", ["fan512", "cone512"])
def test_training_step_is_deterministic(ctx, dev, name):
    """Every reduction has a fixed order (per-CTA partials, fixed-order assembly): the same step
    twice gives bit-identical gradients and loss."""
    over = dict(n_s=32) if name == "cone512" else {}
    g, th, t, f, B, prm = setup_case(ctx, dev, name, over, {}, "bf16", "beer")
    n = 257
    idx = torch.tensor(synth.pixel_batch(name, n, seed=31, **over), device=dev)
    y = torch.tensor(synth.synthetic_y(n, 1.0), device=dev)
    P = synth.param_count(f["C"], f["L"])
    g1 = torch.zeros(P + 1, device=dev)
    g2 = torch.zeros(P + 1, device=dev)
    D.project_and_grad(ctx, idx, y, g1)
    D.project_and_grad(ctx, idx, y, g2)
    torch.cuda.synchronize()
    assert torch.equal(g1, g2)


@pytest.mark.parametrize("name", ["fan512", "cone4d512"])
def test_nan_normalization_box_is_derived(ctx, dev, name):
    """NaN z_lo / z_hi / t_lo / t_hi are derived from the geometry exactly as the input recipe
    derives them (R11): same projections bit for bit."""
    over = dict(n_s=32) if name.startswith("cone") else {}
    g, th, t, f, B, prm = setup_case(ctx, dev, name, over, {}, "bf16", "beer")
    idx = torch.tensor(synth.pixel_batch(name, 64, seed=41, **over), device=dev)
    a = torch.zeros(64, device=dev)
    D.project(ctx, idx, a)
    gn = dict(g, z_lo=float("nan"), z_hi=float("nan"), t_lo=float("nan"), t_hi=float("nan"))
    D.set_geometry(ctx, gn, th, t)
    b = torch.zeros(64, device=dev)
    D.project(ctx, idx, b)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.parametrize("n_s", [7, 48])
def test_fp32_verify_any_samples_per_ray(ctx, dev, O, n_s):
    """the fp32 verify path accepts any N_s >= 1 (per-ray sums instead of 32-sample
    chunks); the bf16 path keeps N_s a multiple of 32 and rejects the combination."""
    g, th, t, f, B, prm = setup_case(ctx, dev, "fan512", dict(n_s=n_s), dict(C=32, L=2), "fp32_verify", "beer")
    idx = synth.pixel_batch("fan512", 9, seed=3)
    y = synth.synthetic_y(9, 1.0)
    fhat = torch.zeros(9, device=dev)
    D.project(ctx, torch.tensor(idx, device=dev), fhat)
    P = synth.param_count(f["C"], f["L"])
    grad = torch.zeros(P + 1, device=dev)
    D.project_and_grad(ctx, torch.tensor(idx, device=dev), torch.tensor(y, device=dev), grad)
    torch.cuda.synchronize()
    rf, _, rc = O.project(g, th, t, f, B, prm, idx)
    assert rc == 0 and rel_linf(fhat.cpu().numpy(), rf) <= 1e-5
    ref, rc = O.project_and_grad(g, th, t, f, B, prm, idx, y)
    assert max(tensor_errs(grad.cpu().numpy()[:P], ref[:P], f["C"], f["L"])) <= 1e-4
    with pytest.raises(D.DinrError):
        D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev), precision="bf16")
