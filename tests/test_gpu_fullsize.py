"""GPU parity at the sizes and in the corners the small cases of test_gpu_parity.py do not reach.

- Persistent multi-group k_fused2 (every CTA runs >= 8 pixel groups, so the lazily consumed
  accumulator commit, the per-CTA ring reuse and the flush after many groups are all exercised):
  fan512 at 1 200 px and parallel64 at 12 000 px, per parameter tensor against the fp64 oracle.
- The H = 256 split path at the BASELINE sample count per ray (cone512, N_s = 256, 600 px: K2 runs
  many tile pairs per CTA and every K5 CTA chains hundreds of tiles through its 64-tile restarts).
- H = 64, L = 1 (per-stream loss mode, no backward MMA chain to hold stream 0 back) with more
  groups than CTAs.
- Config 5 pixel indices (i >= 2^32: the 64-bit batch decode): ray records bit for bit
  and projections.
- A panel that overhangs the FOV cylinder: sub-rays that hit, miss (disc < 0) and touch it
  (disc = 0 exactly, chord 0) inside one pixel, and whole pixels that miss (R21, eq:deltaminmax
  P:2812-2839), in BEER and LINEAR, through the fused and the split kernels and fp32 verify.
- Weights that are not bf16-representable (after three Adam steps): the bf16 path rounds them when
  it packs the tensor-core images; the error is reported (SURVEY 8(c) asks for it separately from
  the parity fixtures, which round the weights first, R18).

Tolerances are the north_star's (projection 2e-3, gradient 1e-2 per tensor; fp32 verify 1e-5 /
1e-4), relative L-inf (R23)."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2404_19075_b200 import _lib as D  # noqa: E402
from paper_2404_19075_b200 import synth  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


def report(key, value):
    """Append a measured number to gpurun_out/parity_report.jsonl (read back into DESIGN.md)."""
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_report.jsonl"), "a") as fh:
        fh.write(json.dumps({"case": key, **value}) + "\n")


def run_step(ctx, dev, O, g, th, t, f, B, prm, idx, y, precision="bf16"):
    D.set_geometry(ctx, g, th, t)
    D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev), precision=precision)
    n = len(idx)
    S = g["sub_x"] * g["sub_z"]
    P = synth.param_count(f["C"], f["L"])
    grad = torch.zeros(P + 1, device=dev)
    fhat = torch.zeros(n, device=dev)
    psub = torch.zeros(n * S, device=dev)
    it, yt = torch.tensor(idx, device=dev), torch.tensor(y, device=dev)
    D.project_and_grad(ctx, it, yt, grad)
    D.project(ctx, it, fhat, psub)
    torch.cuda.synchronize()
    ref, rc = O.project_and_grad(g, th, t, f, B, prm, idx, y)
    assert rc == 0
    rf, rp, rc = O.project(g, th, t, f, B, prm, idx)
    assert rc == 0
    got = grad.cpu().numpy()
    ge = tensor_errs(got[:P], ref[:P], f["C"], f["L"])
    pe = max(rel_linf(fhat.cpu().numpy(), rf), rel_linf(psub.cpu().numpy().reshape(n, S), rp))
    le = abs(got[P] - ref[P]) / abs(ref[P])
    return ge, pe, le, rp


FULL = [
    # (workload, geometry overrides, field overrides, pixels): >= 8 groups per k_fused2 CTA
    ("fan512", {}, {}, 1200),
    ("parallel64", {}, {}, 12000),
    ("parallel64", {}, dict(L=1), 12000),    # per-stream loss mode with L = 1 (no MMA chain ordering)
    ("cone512", {}, {}, 600),                # H = 256 split path at N_s = 256
]


@pytest.mark.parametrize("case", range(len(FULL)))
def test_full_size_training_step_vs_oracle(ctx, dev, O, case):
    name, over, fover, n = FULL[case]
    g = synth.geometry(name, **over)
    th, t = synth.views(name, **over)
    f = synth.field(name, **fover)
    B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"])
    prm = synth.init_params(f["C"], f["L"])
    idx = synth.pixel_batch(name, n, seed=61 + case, **over)
    y, _, _ = O.project_exact(g, th, t, synth.phantom(name), idx, "beer")
    y = y.astype(np.float32)
    ge, pe, le, _ = run_step(ctx, dev, O, g, th, t, f, B, prm, idx, y)
    kind, nf = D.train_path(ctx, n)
    S, ns = g["sub_x"] * g["sub_z"], g["n_s"]
    if kind == 2:
        assert n * S * ns // 256 >= 8 * 148  # every CTA of the persistent kernel runs >= 8 groups
    report(f"full_{name}_{n}px_L{f['L']}", {"path": kind, "grad_err": max(ge), "proj_err": pe, "loss_err": le})
    assert max(ge) <= 1e-2, ge
    assert pe <= 2e-3 and le <= 1e-2, (pe, le)


def test_config5_indices_beyond_2_pow_32(ctx, dev, O):
    """cone4d2048 (configs[4]): M N = 3600 * 2048^2 = 1.5e10 pixels, so batch indices pass 2^32 and
    K1 takes its 64-bit decode (k = i / N, n = i mod N) -- bit-identical records, then projections."""
    name = "cone4d2048"
    g = synth.geometry(name)
    th, t = synth.views(name)
    MN = len(th) * g["n_rows"] * g["n_cols"]
    assert MN > 1 << 33
    rng = np.random.default_rng(17)
    idx = np.concatenate([
        np.array([MN - 1, (1 << 32), (1 << 32) - 1, (1 << 32) + 2047, MN - g["n_cols"]], np.int64),
        rng.integers(1 << 32, MN, 2043, dtype=np.int64)])
    D.set_geometry(ctx, g, th, t)
    S = g["sub_x"] * g["sub_z"]
    rec = torch.zeros(len(idx) * S * 9, dtype=torch.float64, device=dev)
    D.ray_records(ctx, torch.tensor(idx, device=dev), rec)
    torch.cuda.synchronize()
    ref, rc = O.rays(g, th, idx)
    assert rc == 0
    got = rec.cpu().numpy().reshape(len(idx), S, 9)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), np.argwhere(got != ref)[:5]
    # projections of a few of them through the H = 256 forward (N_s = 512)
    f = synth.field(name)
    B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"])
    prm = synth.init_params(f["C"], f["L"])
    D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev))
    sel = idx[:12]
    fhat = torch.zeros(len(sel), device=dev)
    D.project(ctx, torch.tensor(sel, device=dev), fhat)
    torch.cuda.synchronize()
    rf, _, rc = O.project(g, th, t, f, B, prm, sel)
    assert rc == 0
    assert rel_linf(fhat.cpu().numpy(), rf) <= 2e-3


def overhang_geometry(sub_x):
    """parallel64 with the FOV radius cut to 20.5 mm about x_s0 = 0.125 mm while the panel still
    spans +-32 mm.  With 4 sub-rays per pixel at x = col - 32 + {1,3,5,7}/8, pixel 52 holds a hit
    (20.125), a hit (20.375), an exact tangent (20.625: |x - x_s0| = r, disc = 0 in fp64) and a
    miss (20.875); pixel 11 mirrors it; pixels 0..10 and 53..63 miss completely."""
    return synth.geometry("parallel64", fov_radius=20.5, rot_center_x=0.125, sub_x=sub_x)


def overhang_pixels(g, n_views, rng, n):
    cols = np.array([0, 5, 10, 11, 12, 20, 31, 32, 45, 51, 52, 53, 60, 63])
    N = g["n_rows"] * g["n_cols"]
    k = rng.integers(0, n_views, n)
    row = rng.integers(0, g["n_rows"], n)
    col = cols[np.arange(n) % len(cols)]
    idx = k * N + row * g["n_cols"] + col
    return np.unique(idx)


OVERHANG = [
    # (field overrides, precision, expected path kind): fused (H = 64), split (H = 256), fp32 verify
    (dict(C=32, L=3), "bf16", 2),
    (dict(C=128, L=2), "bf16", 0),
    (dict(C=32, L=3), "fp32_verify", 0),
]


@pytest.mark.parametrize("combine", ["beer", "linear"])
@pytest.mark.parametrize("case", range(len(OVERHANG)))
def test_fov_overhang_hits_misses_tangents(ctx, dev, O, case, combine):
    fover, precision, kind = OVERHANG[case]
    g = overhang_geometry(sub_x=4)
    th, t = synth.views("parallel64")
    f = synth.field("parallel64", combine=combine, **fover)
    B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"])
    prm = synth.init_params(f["C"], f["L"])
    idx = overhang_pixels(g, len(th), np.random.default_rng(3 + case), 300)
    rec, rc = O.rays(g, th, idx)
    assert rc == 0
    chord = rec[:, :, 8]
    # the batch really holds every kind of sub-ray and of pixel
    assert np.any(chord > 0) and np.any((chord == 0) & (rec[:, :, 7] == 0) & (rec[:, :, 6] == 0))  # hits, misses
    assert np.any((chord == 0) & (rec[:, :, 6] == rec[:, :, 7]) & (rec[:, :, 6] > 0))  # tangents: delta_min = delta_max
    assert np.any(np.all(chord == 0, axis=1)) and np.any((chord > 0).any(axis=1) & (chord == 0).any(axis=1))
    y, _, _ = O.project_exact(g, th, t, synth.phantom("parallel64"), idx, combine)
    y = y.astype(np.float32) + np.float32(0.05)  # no pixel with a zero residual
    ge, pe, le, rp = run_step(ctx, dev, O, g, th, t, f, B, prm, idx, y, precision=precision)
    assert D.train_path(ctx, len(idx))[0] == kind
    gtol, ptol = (1e-4, 1e-5) if precision == "fp32_verify" else (1e-2, 2e-3)
    report(f"overhang_{case}_{combine}", {"grad_err": max(ge), "proj_err": pe, "loss_err": le})
    assert max(ge) <= gtol, ge
    assert pe <= ptol and le <= gtol, (pe, le)
    # non-contributing sub-rays give exactly p_s = 0 (R21)
    assert np.all(rp[chord == 0] == 0)


@pytest.mark.parametrize("name", ["fan512", "cone512"])
def test_unrounded_weights_after_adam(ctx, dev, O, name):
    """Weights after three Adam steps (lr 1e-3) are not bf16-representable; the bf16 path
    rounds them once when it packs the tensor-core images (the fp32 head and biases stay exact).
    The oracle keeps them exact.  Reported separately, outside the parity contract
    (whose fixtures are bf16-representable, R18): the weight rounding is a 2^-9 relative
    perturbation of the model itself, so it adds about the bf16 tolerance again (measured on the
    B200: fan512 projection 1.4e-3, gradient 8.0e-3; cone512 2.1e-3, 9.2e-3).  Regression bound:
    twice the north_star tolerances."""
    over = dict(n_s=64) if name == "cone512" else {}
    g = synth.geometry(name, **over)
    th, t = synth.views(name, **over)
    f = synth.field(name)
    B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"])
    prm = synth.init_params(f["C"], f["L"])
    P = synth.param_count(f["C"], f["L"])
    m, v = np.zeros(P, np.float32), np.zeros(P, np.float32)
    for s in range(1, 4):  # three Adam steps on oracle gradients of a small batch (fp64 -> fp32)
        idx = synth.pixel_batch(name, 8, seed=70 + s, **over)
        y, _, _ = O.project_exact(g, th, t, synth.phantom(name), idx, "beer")
        gr, rc = O.project_and_grad(g, th, t, f, B, prm, idx, y.astype(np.float32))
        prm, m, v = (np.asarray(a, np.float32) for a in O.adam_step(prm, gr[:P].astype(np.float32), m, v,
                                                                    lr=1e-3, step=s))
    assert not np.array_equal(prm, synth.bf16_round(prm))
    idx = synth.pixel_batch(name, 24, seed=77, **over)
    y, _, _ = O.project_exact(g, th, t, synth.phantom(name), idx, "beer")
    ge, pe, le, _ = run_step(ctx, dev, O, g, th, t, f, B, prm, idx, y.astype(np.float32))
    report(f"adam3_unrounded_{name}", {"grad_err": max(ge), "proj_err": pe, "loss_err": le})
    assert max(ge) <= 2e-2, ge
    assert pe <= 4e-3, pe
