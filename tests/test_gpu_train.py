"""N1 epoch loop on the GPU (dinr_sample_batch / dinr_train_iterations) against the fp64 oracle's
sampler and training loop (oracle.sample_batch / oracle.train, pinned in test_oracle_sampler.py):
- the sampler's batches (pixel indices and gathered measurements) are identical to the oracle's,
  for view shards and the global split, including a config-5-sized shard (D > 2^32, h = 17);
- a three-epoch training run on a small parallel-beam problem tracks the oracle's loss trajectory
  (fp32 verify tightly, bf16 within the bf16 gradient tolerance) and the loss goes down;
- the learning rate is lr0 0.95^epoch, read off |delta gamma| with beta1 = beta2 = 0;
- K = 2 processes of n/2 pixels (global split) draw exactly the pixels of K = 1 with n, and their
  averaged gradient equals the single process's (SPEC acceptance 2)."""
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


def report(key, value):
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_report.jsonl"), "a") as fh:
        fh.write(json.dumps({"case": key, **value}) + "\n")


SAMPLER_CASES = [
    # (workload, overrides, world, rank, n, sharding, epoch, iteration)
    ("fan512", {}, 1, 0, 1000, "views", 0, 0),
    ("fan512", {}, 3, 2, 777, "views", 5, 91),
    ("parallel64", {}, 4, 1, 4096, "views", 2, 3),        # last iteration wraps around the shard
    ("parallel64", {}, 2, 1, 300, "global", 1, 409),
    ("cone4d2048", {}, 1, 0, 2048, "views", 7, 123456),   # D = 1.5e10 > 2^32
    ("cone4d2048", {}, 8, 5, 2048, "views", 0, 917503),   # the last iteration of an epoch at G = 8
]


@pytest.mark.parametrize("case", range(len(SAMPLER_CASES)))
def test_sampler_matches_oracle(ctx, dev, O, case):
    name, over, world, rank, n, sharding, epoch, it = SAMPLER_CASES[case]
    g = synth.geometry(name, **over)
    th, t = synth.views(name, **over)
    D.set_geometry(ctx, g, th, t)
    M, N = len(th), g["n_rows"] * g["n_cols"]
    desc = D.train_desc(seed=2**35 + 17, batch=n, rank=rank, world=world, sharding=sharding)
    ipe = D.iterations_per_epoch(ctx, desc)
    assert ipe == O.iterations_per_epoch(M, N, world, n)
    ref_idx, ref_src = O.sample_batch(M, N, 2**35 + 17, epoch, it, rank, world, n, sharding)
    # a small y source (the shard would be GBs at config 5): gather only when it fits
    src_len = (len(range(rank, M, world)) * N) if sharding == "views" else M * N
    y_src = torch.arange(src_len, dtype=torch.float32, device=dev) if src_len <= 1 << 26 else None
    idx = torch.zeros(n, dtype=torch.int64, device=dev)
    y = torch.zeros(n, device=dev) if y_src is not None else None
    D.sample_batch(ctx, desc, epoch, it, idx, y_src, y)
    torch.cuda.synchronize()
    assert np.array_equal(idx.cpu().numpy(), ref_idx)
    if y is not None:
        assert np.array_equal(y.cpu().numpy(), ref_src.astype(np.float32))
    assert len(np.unique(ref_idx)) == n  # without replacement inside a batch


def small_problem(precision):
    name = "parallel64"
    over = dict(n_rows=8, n_cols=16, n_views=12)
    g = synth.geometry(name, **over)
    th, t = synth.views(name, **over)
    f = synth.field(name)
    B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"])
    prm = synth.init_params(f["C"], f["L"])
    return name, g, th, t, f, B, prm


@pytest.mark.parametrize("precision,tol", [("fp32_verify", 1e-3), ("bf16", 3e-2)])
def test_three_epochs_track_the_oracle(ctx, dev, O, precision, tol):
    name, g, th, t, f, B, prm = small_problem(precision)
    M, N = len(th), g["n_rows"] * g["n_cols"]
    allpix = np.arange(M * N, dtype=np.int64)
    y_full, _, _ = O.project_exact(g, th, t, synth.phantom(name), allpix, "beer")
    y_full = y_full.astype(np.float32)
    n, seed = 128, 21
    ipe = O.iterations_per_epoch(M, N, 1, n)
    iters = 3 * ipe
    _, ref_loss = O.train(g, th, t, f, B, prm, [y_full], seed=seed, n=n, world=1, iterations=iters)
    D.set_geometry(ctx, g, th, t)
    D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev), precision=precision)
    P = synth.param_count(f["C"], f["L"])
    params = torch.tensor(prm, device=dev)
    m, v = torch.zeros(P, device=dev), torch.zeros(P, device=dev)
    grad = torch.zeros(P + 1, device=dev)
    loss = torch.zeros(iters, device=dev)
    desc = D.train_desc(seed=seed, batch=n)
    assert D.iterations_per_epoch(ctx, desc) == ipe
    D.train_iterations(ctx, desc, 0, iters, torch.tensor(y_full, device=dev), params, m, v, grad, loss)
    torch.cuda.synchronize()
    got = loss.cpu().numpy().astype(np.float64)
    err = float(np.max(np.abs(got - ref_loss) / ref_loss))
    ep = [float(np.mean(ref_loss[e * ipe:(e + 1) * ipe])) for e in range(3)]
    report(f"train3_{precision}", {"loss_traj_rel_err": err, "epoch_mean_loss": ep, "iterations": iters})
    assert err <= tol, (err, got[:5], ref_loss[:5])
    assert ep[2] < ep[0]  # it trains


def test_learning_rate_schedule(ctx, dev, O):
    """beta1 = beta2 = 0, eps tiny: each Adam step moves every parameter with a nonzero gradient
    by exactly lr, so |delta gamma| over iteration g reads lr0 0.95^(g // I)."""
    name, g, th, t, f, B, prm = small_problem("fp32_verify")
    M, N = len(th), g["n_rows"] * g["n_cols"]
    y_src = torch.rand(M * N, device=dev, generator=torch.Generator(device=dev).manual_seed(3))
    D.set_geometry(ctx, g, th, t)
    D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev), precision="fp32_verify")
    P = synth.param_count(f["C"], f["L"])
    params = torch.tensor(prm, device=dev)
    m, v = torch.zeros(P, device=dev), torch.zeros(P, device=dev)
    grad = torch.zeros(P + 1, device=dev)
    loss = torch.zeros(1, device=dev)
    desc = D.train_desc(seed=5, batch=512, beta1=0.0, beta2=0.0, eps=1e-30)
    ipe = D.iterations_per_epoch(ctx, desc)
    assert ipe == 3
    for gi in range(2 * ipe + 1):
        before = params.clone()
        D.train_iterations(ctx, desc, gi, 1, y_src, params, m, v, grad, loss)
        torch.cuda.synchronize()
        step = (params - before).abs().double().cpu().numpy()
        moved = step > 0
        lr = 1e-3 * 0.95 ** (gi // ipe)
        assert moved.sum() > 0.9 * P
        assert np.allclose(step[moved], lr, rtol=2e-3), (gi, lr, step[moved][:4])


def test_two_processes_equal_one(ctx, dev, O):
    """Global split: K = 2 processes of b pixels together draw the 2b pixels of K = 1, and the
    average of their local gradients equals the single-process gradient (exact power-of-two
    scaling of the upstream factors: identical per-sample arithmetic, fp32 sum order only)."""
    name = "fan512"
    g = synth.geometry(name)
    th, t = synth.views(name)
    f = synth.field(name)
    B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"])
    prm = synth.init_params(f["C"], f["L"])
    D.set_geometry(ctx, g, th, t)
    D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev))
    M, N = len(th), g["n_rows"] * g["n_cols"]
    y_src = torch.rand(M * N, device=dev, generator=torch.Generator(device=dev).manual_seed(4))
    P = synth.param_count(f["C"], f["L"])
    b = 1024
    one = D.train_desc(seed=9, batch=2 * b, sharding="global")
    idx1, y1 = torch.zeros(2 * b, dtype=torch.int64, device=dev), torch.zeros(2 * b, device=dev)
    D.sample_batch(ctx, one, 0, 7, idx1, y_src, y1)
    g1 = torch.zeros(P + 1, device=dev)
    D.project_and_grad(ctx, idx1, y1, g1)
    acc = torch.zeros(P + 1, dtype=torch.float64, device=dev)
    parts = []
    for r in range(2):
        two = D.train_desc(seed=9, batch=b, rank=r, world=2, sharding="global")
        idx, y = torch.zeros(b, dtype=torch.int64, device=dev), torch.zeros(b, device=dev)
        D.sample_batch(ctx, two, 0, 7, idx, y_src, y)
        parts.append(idx)
        gr = torch.zeros(P + 1, device=dev)
        D.project_and_grad(ctx, idx, y, gr)
        acc += gr.double() * 0.5
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts), idx1)
    a, c = g1.double().cpu().numpy(), acc.cpu().numpy()
    H, off, worst = 2 * f["C"], 0, 0.0
    for _ in range(f["L"]):
        for k in (H * H, H):
            worst = max(worst, np.max(np.abs(a[off:off + k] - c[off:off + k])) / np.max(np.abs(c[off:off + k])))
            off += k
    assert worst <= 1e-4, worst
    assert abs(a[P] - c[P]) <= 1e-5 * abs(c[P])


def test_world_without_communicator_is_rejected(ctx, dev):
    name, g, th, t, f, B, prm = small_problem("bf16")
    D.set_geometry(ctx, g, th, t)
    D.set_field_weights(ctx, f, torch.tensor(B, device=dev), torch.tensor(prm, device=dev))
    P = synth.param_count(f["C"], f["L"])
    z = torch.zeros(P + 1, device=dev)
    desc = D.train_desc(seed=1, batch=8, rank=0, world=2)
    with pytest.raises(D.DinrError) as e:
        D.train_iterations(ctx, desc, 0, 1, torch.zeros(10**5, device=dev), z[:P].clone(), z[:P].clone(),
                           z[:P].clone(), z.clone(), torch.zeros(1, device=dev))
    assert e.value.status == 6  # DINR_ESTATE
