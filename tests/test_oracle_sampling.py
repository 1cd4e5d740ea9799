"""Pins for the oracle's N3 randomized sampling (P:290-295 eq:estforwmod,
P:2115-2117 "randomly sampled coordinates"): the Philox4x32-10 generator against its published
known-answer vectors, the stratification of every jittered sample / sub-ray, the distribution of
the uniforms, and the unbiasedness of the stratified estimator against exact line integrals."""
import numpy as np
import pytest

# Known-answer vectors of Philox4x32-10 from the Random123 distribution (kat_vectors,
# Salmon et al., SC'11): (counter, key) -> output.
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers(O, ctr, key, want):
    assert O.philox4x32(ctr, key) == list(want)


def _geom(beam, **over):
    g = dict(beam=beam, n_rows=8, n_cols=12, sub_x=2, sub_z=2, n_s=16, sod=40.0, odd=30.0,
             pixel_dx=1.5, pixel_dz=1.5, offset_cx=9.0, offset_cz=6.0, fov_radius=12.0,
             rot_center_x=0.4, z_lo=-6, z_hi=6, t_lo=0.0, t_hi=100.0, sampling="jitter", seed=1234, step=7)
    if beam != "cone":
        g.update(sub_z=1)
    g.update(over)
    return g


def test_midpoint_offsets_are_one_half(O):
    g = _geom("cone", sampling="midpoint")
    u, uxz = O.sample_offsets(g, np.arange(20))
    assert np.all(u == 0.5) and np.all(uxz == 0.5)


def test_jitter_offsets_uniform_and_keyed(O):
    g = _geom("cone", n_s=64)
    idx = np.arange(0, 96 * 8, 3)
    u, uxz = O.sample_offsets(g, idx)
    x = np.concatenate([u.ravel(), uxz.ravel()])
    assert np.all((x >= 0) & (x < 1))
    # u01 = (x >> 8) 2^-24: multiples of 2^-24
    assert np.all(x * 2**24 == np.floor(x * 2**24))
    n = x.size
    assert abs(x.mean() - 0.5) < 4 * np.sqrt(1 / 12 / n)
    assert abs(x.var() - 1 / 12) < 0.01
    # neighbouring strata are uncorrelated
    a, b = u[..., :-1].ravel(), u[..., 1:].ravel()
    assert abs(np.corrcoef(a, b)[0, 1]) < 4 / np.sqrt(a.size)
    # reproducible; a different seed or step changes every stream
    u2, _ = O.sample_offsets(g, idx)
    assert np.array_equal(u, u2)
    u3, _ = O.sample_offsets(dict(g, seed=1235), idx)
    u4, _ = O.sample_offsets(dict(g, step=8), idx)
    assert np.mean(u3 == u) < 0.01 and np.mean(u4 == u) < 0.01
    # keyed by the global ray id, not by the batch position
    u5, _ = O.sample_offsets(g, idx[::-1])
    assert np.array_equal(u5[::-1], u)


@pytest.mark.parametrize("beam", ["parallel", "fan", "cone"])
def test_jittered_subrays_stay_in_their_subpixel(O, beam):
    """At theta = 0 the detector end of every sub-ray (delta = 1) lies in its sub-pixel cell,
    at the offset the generator drew (P:53-69 pixel area, P:366-370 sub-pixel grid)."""
    g = _geom(beam)
    N = g["n_rows"] * g["n_cols"]
    idx = np.arange(N)
    rec, _ = O.rays(g, np.zeros(1), idx)
    _, uxz = O.sample_offsets(g, idx)
    row, col = idx // g["n_cols"], idx % g["n_cols"]
    for s in range(g["sub_x"] * g["sub_z"]):
        u, v = s % g["sub_x"], s // g["sub_x"]
        xd = rec[:, s, 0] + rec[:, s, 3]
        zd = rec[:, s, 2] + rec[:, s, 5]
        lo_x = -g["offset_cx"] + (col + u / g["sub_x"]) * g["pixel_dx"]
        lo_z = -g["offset_cz"] + (row + v / g["sub_z"]) * g["pixel_dz"]
        assert np.all(xd >= lo_x - 1e-12) and np.all(xd < lo_x + g["pixel_dx"] / g["sub_x"] + 1e-12)
        assert np.all(zd >= lo_z - 1e-12) and np.all(zd < lo_z + g["pixel_dz"] / g["sub_z"] + 1e-12)
        np.testing.assert_allclose(xd, lo_x + uxz[:, s, 0] * g["pixel_dx"] / g["sub_x"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(zd, lo_z + uxz[:, s, 1] * g["pixel_dz"] / g["sub_z"], rtol=0, atol=1e-12)


def test_stratified_estimator_is_unbiased(O):
    """eq:estforwmod with one uniform sample per stratum is an unbiased estimate of the line
    integral: averaged over seeds, (quadrature - exact) of a Gaussian blob vanishes within its
    standard error, while the midpoint rule at the same coarse N_s keeps a systematic error."""
    g = _geom("fan", n_s=3, sub_x=1)
    prims = [dict(kind="gaussian", value=0.2, center=(0.5, 0.3, 0.0), axes=(1.2, 0.9, 1.0))]
    theta, t = np.array([0.3]), np.zeros(1)
    idx = np.arange(3 * 12, 4 * 12)  # a detector row through the blob
    K = 400
    diffs = []
    for seed in range(K):
        gs = dict(g, seed=seed)
        _, pq, _ = O.project_analytic(gs, theta, t, prims, idx, combine="linear")
        _, pe, _ = O.project_exact(gs, theta, t, prims, idx, combine="linear")
        diffs.append(pq[:, 0] - pe[:, 0])
    d = np.array(diffs)
    mean, se = d.mean(0), d.std(0) / np.sqrt(K)
    assert np.all(np.abs(mean) <= 4.5 * se + 1e-12)
    gm = dict(g, sampling="midpoint")
    _, pm, _ = O.project_analytic(gm, theta, t, prims, idx, combine="linear")
    _, pem, _ = O.project_exact(gm, theta, t, prims, idx, combine="linear")
    big = np.abs(pem[:, 0]) > 0.1
    assert big.sum() >= 3
    assert np.max(np.abs(pm[big, 0] - pem[big, 0])) > 10 * np.max(se[big])


def test_constant_field_ignores_sample_jitter(O):
    """M = mu0 b_o everywhere (all weights zero): p_s = chord_s mu0 b_o for any jitter, with the
    chord of the jittered sub-ray (eq:weightfactors P:1434-1450)."""
    g = _geom("cone")
    f = dict(C=4, L=2, mu0=0.7, combine="linear")
    P = O.param_count(4, 2)
    params = np.zeros(P)
    params[-1] = 0.3
    B = np.random.default_rng(0).normal(size=(4, 4))
    theta, t = np.array([0.0, 1.0]), np.array([0.0, 50.0])
    idx = np.arange(0, 2 * 96, 5)
    fhat, psub, rc = O.project(g, theta, t, f, B, params, idx)
    rec, _ = O.rays(g, theta, idx)
    np.testing.assert_allclose(psub, rec[:, :, 8] * 0.7 * 0.3, rtol=1e-13, atol=1e-15)
