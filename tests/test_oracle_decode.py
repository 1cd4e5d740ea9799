"""Pins for the oracle's batch decode (a1, R13) and normalization (O6, R11/R12).

View decode: i = k N + n selects view k's angle theta_k AND time t_k (R13
"t = T_k for view k = floor(i/N)").  Every other geometry pin is theta-invariant or
single-view; here a moving sphere seen from three views gives a different closed-form chord per
(view, column), so a wrong k, a wrong theta index or a wrong time index fails.

Normalization: r = ((t - c_t)/h_t, (z - c_z)/h_z, y/r, (x - x_s0)/r) ("normalized to
[-1, 1] using the min and max of the cylindrical boundary", R11 explicit box; R12 order t, z, y, x).
The voxelizer evaluates the network at normalize(voxel centre, t); a one-voxel grid placed at the
box centre must give M(0), and a point displaced by half the box along one axis must give M at
the half unit vector of that axis's slot.  A swapped y/x column, a wrong centre or half-width, or
a wrong slot order fails these.
"""
import math

import numpy as np
import pytest

from conftest import golden_geom
from paper_2404_19075_b200 import synth


# ------------------------------------------------------------------------------ view decode
def _sphere_chord_parallel(g, theta, tk, col, c0, vel, R):
    """Closed-form chord of a sphere of radius R (centre c0 + vel t) along the parallel-beam ray of
    detector column `col` (row 0) after the source/detector rotation by +theta about (x_s0, 0)
    (eq:rotxsk-rotydk).  The rotated ray is the line
    {(x_s0 + a cos th - y sin th, a sin th + y cos th)} with a = x_d - x_s0, whose unit normal is
    (cos th, sin th): the signed distance of the centre is (c_x - x_s0) cos th + c_y sin th - a."""
    xd = -g["offset_cx"] + (col + 0.5) * g["pixel_dx"]
    zd = -g["offset_cz"] + 0.5 * g["pixel_dz"]
    cx, cy, cz = (c0[q] + vel[q] * tk for q in range(3))
    xs0 = g["rot_center_x"]
    dist = (cx - xs0) * math.cos(theta) + cy * math.sin(theta) - (xd - xs0)
    h2 = R * R - dist * dist - (zd - cz) ** 2
    return 2.0 * math.sqrt(h2) if h2 > 0 else 0.0


VIEWS_THETA = np.array([1.1, 0.3, -0.7])
VIEWS_T = np.array([0.0, 2.0, 5.0])
C0, VEL, RAD = (0.45, 0.3, 0.0), (-0.06, 0.05, 0.0), 0.9


def _all_pixels(g):
    N = g["n_rows"] * g["n_cols"]
    return np.arange(len(VIEWS_THETA) * N), N


def test_view_decode_moving_sphere_exact(O):
    """Indicator sphere, exact line integrals: f = mu * chord(theta_k, t_k, col) for i = k N + col."""
    g = golden_geom("parallel")
    mu = 0.25
    prims = [dict(kind="indicator", value=mu, center=C0, velocity=VEL, axes=(RAD, RAD, RAD))]
    idx, N = _all_pixels(g)
    fhat, _, rc = O.project_exact(g, VIEWS_THETA, VIEWS_T, prims, idx, combine="linear")
    assert rc == 0
    exp = [mu * _sphere_chord_parallel(g, VIEWS_THETA[i // N], VIEWS_T[i // N], i % N, C0, VEL, RAD) for i in idx]
    assert np.allclose(fhat, exp, rtol=0, atol=1e-12)
    # the three views really differ (the pin discriminates k)
    per_view = np.asarray(exp).reshape(len(VIEWS_THETA), N)
    assert np.min(np.abs(per_view[0] - per_view[1])[per_view[0] + per_view[1] > 0]) > 1e-3
    assert np.min(np.abs(per_view[1] - per_view[2])[per_view[1] + per_view[2] > 0]) > 1e-3


def test_view_decode_moving_smooth_sphere_quadrature(O):
    """Same views through the quadrature projector (O14) with a smooth (1 - rho^2)^2 sphere:
    closed form mu_c 16 a^5 / (15 R^4) with a = half chord; midpoint error O(h^2)."""
    g = golden_geom("parallel", n_s=2048)
    mu_c = 0.3
    prims = [dict(kind="smooth", value=mu_c, center=C0, velocity=VEL, axes=(RAD, RAD, RAD))]
    idx, N = _all_pixels(g)
    fhat, _, rc = O.project_analytic(g, VIEWS_THETA, VIEWS_T, prims, idx, combine="linear")
    assert rc == 0
    exp = []
    for i in idx:
        a = 0.5 * _sphere_chord_parallel(g, VIEWS_THETA[i // N], VIEWS_T[i // N], i % N, C0, VEL, RAD)
        exp.append(mu_c * 16.0 * a ** 5 / (15.0 * RAD ** 4))
    assert np.allclose(fhat, exp, rtol=0, atol=1e-6)


@pytest.mark.parametrize("beam", ["parallel", "fan", "cone"])
def test_view_decode_network_path(O, beam):
    """The network projector with a t-conditioned field: pixel k N + col of a three-view schedule
    equals pixel col of the one-view schedule (theta_k, t_k), bit for bit, and the views differ."""
    g = golden_geom(beam, sub_x=2, n_rows=2, t_lo=0.0, t_hi=5.0, z_lo=-1.0, z_hi=1.5)
    g["offset_cz"] = 1.0
    C_, L = 4, 2
    f = dict(C=C_, L=L, mu0=0.7, combine="beer")
    B = synth.grff_matrix(C_, 0.8, 0.5, seed=11)
    prm = synth.init_params(C_, L, seed=12)
    prm[-1] = 1.0  # head bias: projections of order one
    N = g["n_rows"] * g["n_cols"]
    idx = np.arange(3 * N)
    fh_all, ps_all, rc = O.project(g, VIEWS_THETA, VIEWS_T, f, B, prm, idx)
    assert rc == 0
    for k in range(3):
        fh_k, ps_k, rc = O.project(g, VIEWS_THETA[k:k + 1], VIEWS_T[k:k + 1], f, B, prm, np.arange(N))
        assert rc == 0
        assert np.array_equal(fh_all[k * N:(k + 1) * N], fh_k)
        assert np.array_equal(ps_all[k * N:(k + 1) * N], ps_k)
    # time alone changes the result (t enters through t_k): same angle, other time
    fh_t, _, _ = O.project(g, VIEWS_THETA[1:2], VIEWS_T[2:3], f, B, prm, np.arange(N))
    assert np.max(np.abs(fh_t - fh_all[N:2 * N])) > 1e-4


# ------------------------------------------------------------------------------ normalization
def _norm_geom():
    return dict(beam="cone", n_rows=6, n_cols=9, sub_x=1, sub_z=1, n_s=16, sod=40.0, odd=30.0, pixel_dx=1.0,
                pixel_dz=1.2, offset_cx=4.5, offset_cz=3.6, fov_radius=4.0, rot_center_x=0.7, z_lo=-1.0,
                z_hi=3.0, t_lo=10.0, t_hi=50.0)


def _point_value(O, g, f, B, prm, x, y, z, t):
    """M at one world point via a one-voxel grid centred there."""
    v = 0.25
    grid = dict(nx=1, ny=1, nz=1, x0=x - v / 2, y0=y - v / 2, z0=z - v / 2, vx=v, vy=v, vz=v)
    return O.voxelize(g, f, B, prm, grid, t)[0, 0, 0]


def test_normalize_centre_and_axes(O):
    g = _norm_geom()
    C_, L = 6, 2
    f = dict(C=C_, L=L, mu0=1.3, combine="linear")
    # distinct, well-separated B columns so every slot of rbar changes the output differently
    B = synth.grff_matrix(C_, 0.7, 0.9, seed=21)
    prm = synth.init_params(C_, L, seed=22)
    r, xs0 = g["fov_radius"], g["rot_center_x"]
    zc, hz = 0.5 * (g["z_lo"] + g["z_hi"]), 0.5 * (g["z_hi"] - g["z_lo"])
    tc, ht = 0.5 * (g["t_lo"] + g["t_hi"]), 0.5 * (g["t_hi"] - g["t_lo"])
    a = 0.5
    # (world point, rbar it must map to): slots (t, z, y, x)
    cases = [
        ((xs0, 0.0, zc, tc), (0.0, 0.0, 0.0, 0.0)),
        ((xs0 + a * r, 0.0, zc, tc), (0.0, 0.0, 0.0, a)),
        ((xs0, a * r, zc, tc), (0.0, 0.0, a, 0.0)),
        ((xs0, 0.0, zc + a * hz, tc), (0.0, a, 0.0, 0.0)),
        ((xs0, 0.0, zc, tc + a * ht), (a, 0.0, 0.0, 0.0)),
        ((xs0 - a * r, -a * r, zc - a * hz, tc - a * ht), (-a, -a, -a, -a)),
    ]
    vals = []
    for (x, y, z, t), rb in cases:
        got = _point_value(O, g, f, B, prm, x, y, z, t)
        want = O.mlp_eval(f, B, prm, np.array(rb))[0]
        assert got == pytest.approx(want, rel=1e-13, abs=1e-15), (x, y, z, t, rb)
        vals.append(want)
    # the four axis displacements give four different values (a swapped slot cannot pass)
    axis_vals = vals[1:5]
    assert min(abs(p - q) for i, p in enumerate(axis_vals) for q in axis_vals[i + 1:]) > 1e-6
    assert min(abs(v - vals[0]) for v in axis_vals) > 1e-6


def test_normalize_zero_width_time_maps_to_zero(O):
    """A static schedule (t_lo = t_hi) has h_t = 0: the t slot is 0 for every t (R11)."""
    g = _norm_geom()
    g["t_lo"] = g["t_hi"] = 7.0
    f = dict(C=4, L=1, mu0=1.0, combine="linear")
    B = synth.grff_matrix(4, 0.7, 0.9, seed=3)
    prm = synth.init_params(4, 1, seed=4)
    v1 = _point_value(O, g, f, B, prm, 0.7, 0.0, 1.0, 7.0)
    v2 = _point_value(O, g, f, B, prm, 0.7, 0.0, 1.0, 123.0)
    assert v1 == v2 == pytest.approx(O.mlp_eval(f, B, prm, np.zeros(4))[0], rel=1e-13)
