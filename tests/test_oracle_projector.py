"""Pins for the oracle's projector (O5, O9, O10, O14): quadrature against closed-form
line integrals, per-view mass conservation, and the BEER/LINEAR combine identities."""
import math

import numpy as np
import pytest

from conftest import golden_geom


def _geom(beam, **over):
    g = dict(beam=beam, n_rows=8, n_cols=12, sub_x=2, sub_z=2, n_s=64, sod=40.0, odd=30.0,
             pixel_dx=1.5, pixel_dz=1.5, offset_cx=9.0, offset_cz=6.0, fov_radius=12.0,
             rot_center_x=0.4, z_lo=-6, z_hi=6, t_lo=0.0, t_hi=100.0)
    if beam != "cone":
        g.update(sub_z=1)
    g.update(over)
    return g


@pytest.mark.parametrize("beam", ["parallel", "fan", "cone"])
def test_indicator_quadrature_within_bound(O, beam):
    """Midpoint quadrature of an indicator ellipsoid differs from the exact chord integral
    by at most 2 mu chord/N_s per ellipsoid crossing (two discontinuities)."""
    g = _geom(beam)
    prims = [dict(kind="indicator", value=0.05, center=(1.0, -0.5, 0.3), axes=(5.0, 6.0, 4.0),
                  velocity=(0.01, 0.0, -0.005), axes_rate=(0.0, 0.002, 0.0))]
    rng = np.random.default_rng(7)
    M = 10
    theta, t = rng.uniform(0, 2 * np.pi, M), np.linspace(0, 100, M)
    idx = rng.choice(M * g["n_rows"] * g["n_cols"], 300, replace=False)
    _, pq, _ = O.project_analytic(g, theta, t, prims, idx)
    _, pe, _ = O.project_exact(g, theta, t, prims, idx)
    rec, _ = O.rays(g, theta, idx)
    bound = 2 * 0.05 * rec[:, :, 8] / g["n_s"] + 1e-14
    assert np.all(np.abs(pq - pe) <= bound)
    assert np.max(pe) > 0.1  # the rays do cross the object


@pytest.mark.parametrize("beam", ["parallel", "fan", "cone"])
def test_smooth_ellipsoid_second_order(O, beam):
    """mu_c (1-rho^2)^2 has a continuous first derivative: midpoint error O(h^2);
    <= 1e-6 relative at N_s = 1024."""
    prims = [dict(kind="smooth", value=0.08, center=(0.5, 0.2, -0.4), axes=(6.0, 4.5, 5.0))]
    rng = np.random.default_rng(8)
    M = 6
    theta, t = rng.uniform(0, 2 * np.pi, M), np.zeros(M)
    errs = []
    for ns in (256, 1024):
        g = _geom(beam, n_s=ns)
        idx = np.arange(0, M * g["n_rows"] * g["n_cols"], 7)
        _, pq, _ = O.project_analytic(g, theta, t, prims, idx)
        _, pe, _ = O.project_exact(g, theta, t, prims, idx)
        errs.append(np.max(np.abs(pq - pe)) / np.max(pe))
    assert errs[1] <= 1e-6
    assert errs[0] / errs[1] > 8.0  # ~16x per 4x refinement: second order


@pytest.mark.parametrize("beam", ["parallel", "fan", "cone"])
def test_gaussian_spectral(O, beam):
    prims = [dict(kind="gaussian", value=0.3, center=(0.5, -0.7, 0.2), axes=(1.0, 1.2, 0.9))]
    g = _geom(beam, n_s=128)
    rng = np.random.default_rng(9)
    M = 5
    theta, t = rng.uniform(0, 2 * np.pi, M), np.zeros(M)
    idx = np.arange(0, M * g["n_rows"] * g["n_cols"], 3)
    _, pq, _ = O.project_analytic(g, theta, t, prims, idx)
    _, pe, _ = O.project_exact(g, theta, t, prims, idx)
    assert np.max(np.abs(pq - pe)) <= 1e-12 * np.max(pe)


@pytest.mark.parametrize("mode", ["exact", "quadrature"])
def test_mass_conservation_parallel(O, mode):
    """North-star pin: parallel beam, every view, sum_px Dx Dz fhat = total mass
    A (2 pi)^{3/2} sx sy sz of Gaussian blobs to 1e-9 relative."""
    g = dict(beam="parallel", n_rows=64, n_cols=64, sub_x=1, sub_z=1, n_s=96, sod=64.0, odd=64.0,
             pixel_dx=1.0, pixel_dz=1.0, offset_cx=32.0, offset_cz=32.0, fov_radius=32.0,
             rot_center_x=0.0, z_lo=-32, z_hi=32, t_lo=0, t_hi=0)
    prims = [dict(kind="gaussian", value=0.05, center=(3.0, -2.0, 1.0), axes=(3.0, 4.0, 3.5)),
             dict(kind="gaussian", value=0.02, center=(-2.0, 1.5, -2.0), axes=(3.2, 3.0, 3.0))]
    mass = sum(p["value"] * (2 * math.pi) ** 1.5 * np.prod(p["axes"]) for p in prims)
    theta = np.deg2rad(np.array([0.0, 17.0, 45.0, 90.0, 133.0, 251.0]))
    N = 64 * 64
    for k in range(len(theta)):
        idx = np.arange(k * N, (k + 1) * N)
        fn = O.project_exact if mode == "exact" else O.project_analytic
        fhat, _, rc = fn(g, theta, np.zeros(len(theta)), prims, idx, "linear")
        assert rc == 0
        total = fhat.sum() * g["pixel_dx"] * g["pixel_dz"]
        assert abs(total - mass) <= 1e-9 * mass, (k, total, mass)


def test_combine_identities(O):
    """R5: S=1 => BEER == LINEAR exactly; Jensen fhat_BEER <= fhat_LINEAR; equal p_s =>
    equal; doubling mu0 doubles p_s exactly."""
    C_, L = 3, 2
    rng = np.random.default_rng(10)
    prm = rng.uniform(-0.5, 0.5, O.param_count(C_, L))
    prm[-1] = 1.0
    B = rng.standard_normal((C_, 4)) * 0.5
    theta, t = rng.uniform(0, 6, 4), np.linspace(0, 30, 4)
    f = lambda comb, mu0=0.05: dict(C=C_, L=L, mu0=mu0, combine=comb)
    g1 = _geom("cone", sub_x=1, sub_z=1, n_s=16)
    idx = rng.choice(4 * 96, 40, replace=False)
    fb, pb, _ = O.project(g1, theta, t, f("beer"), B, prm, idx)
    fl, pl, _ = O.project(g1, theta, t, f("linear"), B, prm, idx)
    assert np.array_equal(fb, fl) and np.array_equal(fb, pb[:, 0])
    g4 = _geom("cone", n_s=16)
    fb, pb, _ = O.project(g4, theta, t, f("beer"), B, prm, idx)
    fl, pl, _ = O.project(g4, theta, t, f("linear"), B, prm, idx)
    assert np.array_equal(pb, pl)
    assert np.all(fb <= fl + 1e-15)
    assert np.max(fl - fb) > 0
    assert np.allclose(fl, pl.mean(1), atol=1e-15)
    # BEER closed form -log(mean exp(-p))
    assert np.allclose(fb, -np.log(np.mean(np.exp(-pb), axis=1)), rtol=1e-13, atol=1e-15)
    _, p2, _ = O.project(g4, theta, t, f("beer", 0.1), B, prm, idx)
    assert np.array_equal(p2, 2 * pb)


def test_constant_field_chord(O):
    """w_o = 0, b_o = beta => p_s = mu0 beta chord_s exactly (R7)."""
    g = _geom("fan", n_s=32)
    C_, L = 2, 2
    prm = np.random.default_rng(11).uniform(-1, 1, O.param_count(C_, L))
    H = 2 * C_
    prm[L * (H * H + H):-1] = 0.0
    prm[-1] = 0.75
    B = np.ones((C_, 4))
    theta = np.array([0.2, 1.4])
    idx = np.arange(0, 2 * 96)
    _, ps, _ = O.project(g, theta, [0, 0], dict(C=C_, L=L, mu0=0.04, combine="linear"), B, prm, idx)
    rec, _ = O.rays(g, theta, idx)
    assert np.allclose(ps, 0.04 * 0.75 * rec[:, :, 8], rtol=1e-13, atol=1e-16)
