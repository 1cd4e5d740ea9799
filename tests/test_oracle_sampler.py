"""Pins of the oracle's N1 sampler and epoch loop (oracle/dinr_oracle.c or_perm / or_sample_batch,
oracle.train) against what the paper and the mathematics fix:
- each epoch visits a bijection of the shard (brute force over many shard sizes, seeds, epochs);
  "without replacement": one epoch of ceil(MN / Omega*) iterations
  covers every pixel exactly once when Omega* divides MN, and at most twice otherwise (R27 wrap);
- view sharding: rank r only ever draws views k = r mod K, and its y-source
  positions address its own view-by-view shard;
- the global split is contiguous, so K processes of n/K pixels draw exactly the
  pixels one process of n draws, and the averaged-gradient trajectory is the same (SPEC
  acceptance 2: K=2, |Omega_k|=3 vs K=1, |Omega_k|=6 to 1e-12);
- the learning rate decays by 0.95 after each epoch: with beta1 = beta2 = 0 Adam's
  step is lr * g / (|g| + eps), so |delta gamma| reads the lr of each iteration;
- permutations are uniform: over many epochs each position of a small shard lands on each pixel
  about equally often (chi-square)."""
import numpy as np
import pytest

from paper_2404_19075_b200 import synth


def test_perm_is_a_bijection(O):
    for D in list(range(1, 70)) + [255, 256, 257, 1000, 4097]:
        for seed, epoch in ((0, 0), (7, 3), (2**40 + 11, 2**33 + 5)):
            p = [O.perm(D, seed, epoch, q) for q in range(D)]
            assert sorted(p) == list(range(D)), (D, seed, epoch)


def test_perm_depends_on_seed_and_epoch(O):
    D = 1000
    a = [O.perm(D, 1, 0, q) for q in range(D)]
    assert a == [O.perm(D, 1, 0, q) for q in range(D)]  # reproducible
    assert a != [O.perm(D, 1, 1, q) for q in range(D)]  # a new order every epoch
    assert a != [O.perm(D, 2, 0, q) for q in range(D)]
    assert a != list(range(D))


@pytest.mark.parametrize("D", [5, 8, 13])
def test_perm_is_uniform(O, D):
    """Over many epochs position q lands on every pixel about equally often: chi-square over the
    D x D table ((D - 1)^2 degrees of freedom, rows and columns fixed) within 6 sd."""
    E = 4000
    counts = np.zeros((D, D))
    for e in range(E):
        for q in range(D):
            counts[q, O.perm(D, 99, e, q)] += 1
    exp = E / D
    chi2 = ((counts - exp) ** 2 / exp).sum()
    dof = (D - 1) ** 2
    assert chi2 < dof + 6 * np.sqrt(2 * dof), chi2


@pytest.mark.parametrize("M,N,world,n", [(12, 20, 1, 40), (12, 20, 3, 16), (12, 20, 3, 20), (7, 9, 2, 5), (5, 4, 1, 7)])
def test_epoch_covers_the_shard(O, M, N, world, n):
    ipe = O.iterations_per_epoch(M, N, world, n)
    assert ipe == -(-(M * N) // (world * n))
    for r in range(world):
        D = len(range(r, M, world)) * N  # the rank's shard
        seen = np.zeros(M * N, dtype=int)
        for it in range(ipe):
            idx, src = O.sample_batch(M, N, 5, 2, it, r, world, n)
            assert len(idx) == n
            views = idx // N
            assert np.all(views % world == r) and np.all((views >= 0) & (views < M))
            # src is the position in the rank's shard, stored view by view
            assert np.array_equal(idx, (r + world * (src // N)) * N + src % N)
            assert np.all((src >= 0) & (src < D))
            np.add.at(seen, idx, 1)
        own = np.array([k * N + p for k in range(r, M, world) for p in range(N)])
        assert seen.sum() == seen[own].sum()  # nothing outside the shard
        if D <= ipe * n:  # the epoch reaches the end of the shard's permutation
            assert seen[own].min() >= 1 and seen[own].max() <= 2
            if D == ipe * n:
                assert np.all(seen[own] == 1)  # without replacement


def test_global_split_is_contiguous(O):
    M, N = 9, 10
    for it in range(4):
        one, _ = O.sample_batch(M, N, 3, 1, it, 0, 1, 6, "global")
        two = np.concatenate([O.sample_batch(M, N, 3, 1, it, r, 2, 3, "global")[0] for r in range(2)])
        assert np.array_equal(one, two)
        idx, src = O.sample_batch(M, N, 3, 1, it, 1, 2, 3, "global")
        assert np.array_equal(idx, src)
    # exactly once per epoch when Omega* divides MN
    allx = np.concatenate([O.sample_batch(M, N, 3, 0, it, r, 2, 5, "global")[0]
                           for it in range(O.iterations_per_epoch(M, N, 2, 5)) for r in range(2)])
    assert sorted(allx.tolist()) == list(range(M * N))


def tiny_problem():
    name = "parallel64"
    over = dict(n_rows=4, n_cols=8, n_views=6, n_s=8)
    g = synth.geometry(name, **over)
    th, t = synth.views(name, **over)
    f = synth.field(name, C=2, L=2)
    B = synth.grff_matrix(2, 0.1, 0.5)
    prm = synth.init_params(2, 2)
    return g, th, t, f, B, prm


def test_k_invariance_of_the_training_trajectory(O):
    """SPEC acceptance 2: K = 2 processes of 3 pixels vs one of 6, same seed and permutation."""
    g, th, t, f, B, prm = tiny_problem()
    MN = len(th) * g["n_rows"] * g["n_cols"]
    y = np.random.default_rng(0).uniform(0.0, 2.0, MN)
    p1, l1 = O.train(g, th, t, f, B, prm, [y], seed=4, n=6, world=1, iterations=10, sharding="global")
    p2, l2 = O.train(g, th, t, f, B, prm, [y, y], seed=4, n=3, world=2, iterations=10, sharding="global")
    assert np.max(np.abs(p1 - p2)) <= 1e-12 * np.max(np.abs(p1))
    assert np.allclose(l1, l2, rtol=1e-12, atol=0)


def test_learning_rate_decays_per_epoch(O):
    g, th, t, f, B, prm = tiny_problem()
    M, N = len(th), g["n_rows"] * g["n_cols"]
    y = np.random.default_rng(1).uniform(0.0, 2.0, M * N)
    n = 48
    ipe = O.iterations_per_epoch(M, N, 1, n)
    assert ipe == 4
    prev = np.asarray(prm, np.float64)
    for gi in range(2 * ipe + 1):
        p, _ = O.train(g, th, t, f, B, prev, [y], seed=8, n=n, world=1, iterations=1, sharding="global", b1=0.0,
                       b2=0.0, eps=1e-30, first=gi)
        step = np.abs(p - prev)
        lr = 1e-3 * 0.95 ** (gi // ipe)
        moved = step > 0
        assert moved.sum() > 0.9 * len(p)
        assert np.allclose(step[moved], lr, rtol=1e-9), (gi, step[moved][:4], lr)
        prev = p


def test_view_shards_feed_the_rank_y(O):
    """Mode "views": rank r's y source is its own shard (views r, r + K, ...), and the gathered
    values are the ones stored at the sampled pixels."""
    M, N, world, n = 7, 6, 3, 5
    y_full = np.arange(M * N, dtype=np.float64)
    for r in range(world):
        shard = np.concatenate([y_full[k * N:(k + 1) * N] for k in range(r, M, world)])
        for it in range(3):
            idx, src = O.sample_batch(M, N, 2, 0, it, r, world, n)
            assert np.array_equal(shard[src], y_full[idx])
