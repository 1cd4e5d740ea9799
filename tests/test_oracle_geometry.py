"""Pins for the oracle's geometry (O1-O4): rotation, FOV delta bounds, arc length / chord.

Every expectation here comes from outside the oracle: SPEC worked examples, closed-form
chord lengths, invariants of the equations, and the survey's golden tables
(tests/golden/*.txt, each with its citation).
"""
import math

import numpy as np
import pytest

from conftest import golden_geom, read_golden


# --- rotation, eq:rotxsk-rotydk -------------------------------------------
def test_rotate_spec_examples(O):
    # S:60-62 worked examples.
    assert O.rotate_point(1.0, 0.0, 0.0, 5.0) == (1.0, 0.0)
    x, y = O.rotate_point(1.0, 0.0, math.pi / 2, 0.0)
    assert abs(x) < 1e-15 and abs(y - 1.0) < 1e-15
    x, y = O.rotate_point(1.0, 2.0, math.pi, 2.0)
    assert abs(x - 3.0) < 1e-14 and abs(y + 2.0) < 1e-14


def test_rotate_isometry_about_centre(O):
    # distance to (x_s0, 0) preserved; anticlockwise: angle increases by theta.
    rng = np.random.default_rng(0)
    for _ in range(500):
        x, y, th, xs0 = rng.uniform(-50, 50), rng.uniform(-50, 50), rng.uniform(-7, 7), rng.uniform(-5, 5)
        xr, yr = O.rotate_point(x, y, th, xs0)
        r0, r1 = math.hypot(x - xs0, y), math.hypot(xr - xs0, yr)
        assert abs(r1 - r0) <= 1e-12 * max(1.0, r0)
        a0, a1 = math.atan2(y, x - xs0), math.atan2(yr, xr - xs0)
        d = (a1 - a0 - th + math.pi) % (2 * math.pi) - math.pi
        assert abs(d) < 1e-9


# --- FOV bounds, eq:solvquaddelta / eq:deltaminmax ------------------------
def test_delta_bounds_spec_examples(O):
    # a=16, b=-16, c=3 -> (0.25, 0.75); miss; tangent (0.5, 0.5).
    assert O.fov_delta_bounds((0, -2), (0, 2), 0.0, 1.0) == (0.25, 0.75)
    assert O.fov_delta_bounds((5, -2), (5, 2), 0.0, 1.0) is None
    assert O.fov_delta_bounds((1, -2), (1, 2), 0.0, 1.0) == (0.5, 0.5)


def _perp_dist(p1, p2, c):
    (x1, y1), (x2, y2), (cx, cy) = p1, p2, c
    dx, dy = x2 - x1, y2 - y1
    return abs(dx * (y1 - cy) - dy * (x1 - cx)) / math.hypot(dx, dy)


@pytest.mark.parametrize("beam", ["parallel", "fan", "cone"])
def test_chord_closed_form_and_fov_invariants(O, beam):
    """10^5 rays: chord = closed form (SURVEY 8(c) chord pins), every sample inside the
    cylinder, bounds invariant under the joint rotation."""
    rng = np.random.default_rng({"parallel": 1, "fan": 2, "cone": 3}[beam])
    g = dict(beam=beam, n_rows=40, n_cols=160, sub_x=2, sub_z=2, n_s=16, sod=30.0, odd=20.0,
             pixel_dx=0.2, pixel_dz=0.25, offset_cx=16.3, offset_cz=4.9, fov_radius=9.0,
             rot_center_x=0.7, z_lo=-5, z_hi=5, t_lo=0, t_hi=0)
    M = 50
    theta = rng.uniform(-4, 4, size=M)
    idx = rng.integers(0, M * g["n_rows"] * g["n_cols"], size=25000)
    rec, rc = O.rays(g, theta, idx)
    assert rc == 0
    rec = rec.reshape(-1, 9)
    assert rec.shape[0] == 100000
    # unrotated endpoints from the pixel index (P:53-69 sub-pixel centres)
    N = g["n_rows"] * g["n_cols"]
    n = idx % N
    row, col = n // g["n_cols"], n % g["n_cols"]
    u = np.tile(np.array([0, 1, 0, 1]), len(idx))
    v = np.tile(np.array([0, 0, 1, 1]), len(idx))
    row, col = np.repeat(row, 4), np.repeat(col, 4)
    xd = -g["offset_cx"] + (col + (u + 0.5) / 2) * g["pixel_dx"]
    zd = -g["offset_cz"] + (row + (v + 0.5) / 2) * g["pixel_dz"]
    r, xs0 = g["fov_radius"], g["rot_center_x"]
    if beam == "parallel":
        expect = 2 * np.sqrt(np.maximum(r * r - (xd - xs0) ** 2, 0))
    else:
        ys, yd = -g["sod"], g["odd"]
        dperp = np.abs(xd * (ys - 0.0) - (yd - ys) * (0.0 - xs0)) / np.hypot(xd, yd - ys)
        expect = 2 * np.sqrt(np.maximum(r * r - dperp ** 2, 0))
        if beam == "cone":
            sxy = np.hypot(xd, yd - ys)
            expect = expect * np.sqrt(sxy ** 2 + zd ** 2) / sxy
    assert np.max(np.abs(rec[:, 8] - expect)) <= 1e-12 * r
    # samples inside the cylinder, incl. both end points
    for frac in (0.0, 0.37, 1.0):
        dl = rec[:, 6] + frac * (rec[:, 7] - rec[:, 6])
        x = rec[:, 0] + dl * rec[:, 3]
        y = rec[:, 1] + dl * rec[:, 4]
        hit = rec[:, 8] > 0
        assert np.all(((x - xs0) ** 2 + y ** 2)[hit] <= r * r * (1 + 1e-12))
    # bounds from the ROTATED points equal the stored theta-invariant bounds
    for q in rng.choice(len(rec), 2000, replace=False):
        o, d = rec[q, :3], rec[q, 3:6]
        b = O.fov_delta_bounds(o[:2], (o + d)[:2], xs0, r)
        if rec[q, 8] > 0:
            assert b is not None
            assert abs(b[0] - rec[q, 6]) < 1e-12 and abs(b[1] - rec[q, 7]) < 1e-12


def test_index_decode_and_out_of_range(O):
    # i = m N + n; out-of-range index -> error, zeroed record.
    g = golden_geom("parallel")
    theta = np.array([0.0, 0.3])
    rec, rc = O.rays(g, theta, [5])  # view 1, col 1
    assert rc == 0
    assert rec[0, 0, 0] != 0.0
    rec, rc = O.rays(g, theta, [8])
    assert rc == -1 and np.all(rec == 0)


# --- golden tables ----------------------------------------------------------------------
def test_golden_constant_field(O):
    rows = read_golden("constant_field.txt")
    assert len(rows) == 4
    for row in rows:
        head, fb, fl = [p.split() for p in row.split("|")]
        beam, sub_x, col = head[0], int(head[1]), int(head[2])
        p_exp = [float(v) for v in head[3:]]
        g = golden_geom(beam, sub_x=sub_x)
        C_, L = 2, 1
        prm = np.random.default_rng(5).uniform(-1, 1, O.param_count(C_, L))
        H = 2 * C_
        prm[L * (H * H + H):L * (H * H + H) + H] = 0.0   # w_o = 0
        prm[-1] = 1.0                                     # b_o = 1
        B = np.random.default_rng(6).standard_normal((C_, 4))
        for combine, fexp in (("beer", float(fb[0])), ("linear", float(fl[0]))):
            f = dict(C=C_, L=L, mu0=0.25, combine=combine)
            fhat, psub, rc = O.project(g, [0.3], [0.0], f, B, prm, [col])
            assert rc == 0
            assert np.allclose(psub[0], p_exp, rtol=0, atol=1e-12)
            assert abs(fhat[0] - fexp) < 1e-12


def test_golden_rotation_sign(O):
    rows = {r.split()[0]: [float(v) for v in r.split()[1:]] for r in read_golden("rotation_sign.txt")}
    g = golden_geom("parallel")
    sphere = [dict(kind="indicator", value=0.25, center=(0.5, 0.3, 0.0), axes=(1.0, 1.0, 1.0))]
    fhat, _, rc = O.project_exact(g, [0.3], [0.0], sphere, [0, 1, 2, 3])
    assert rc == 0
    assert np.allclose(fhat, rows["plus_theta"], atol=1e-11)
    fneg, _, _ = O.project_exact(g, [-0.3], [0.0], sphere, [0, 1, 2, 3])
    assert np.allclose(fneg, rows["minus_theta"], atol=1e-11)
    assert not np.allclose(fhat, fneg, atol=1e-3)


def test_sphere_chord_examples(O):
    # chord through the centre R=1, mu=0.05 -> 0.1; offset 0.6 with mu=1 -> 1.6.
    s = [dict(kind="indicator", value=0.05, center=(0, 0, 0), axes=(1, 1, 1))]
    assert abs(O.line_integral_exact(s, (0, -3, 0), (0, 6, 0), 0.0, 1.0) - 0.1) < 1e-15
    s1 = [dict(kind="indicator", value=1.0, center=(0, 0, 0), axes=(1, 1, 1))]
    assert abs(O.line_integral_exact(s1, (0.6, -3, 0), (0, 6, 0), 0.0, 1.0) - 1.6) < 1e-14
