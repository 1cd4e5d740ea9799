"""Pins for the oracle's N4 inference voxelization:
the paper's voxel size (pixel / magnification), the FOV support, slab independence, and the
ray/voxel consistency that ties the grid's coordinate mapping to the projector's: along the
central parallel ray the voxel sum times the voxel size IS the midpoint quadrature of eq:estforwmod
when the voxel centres sit on the ray samples."""
import numpy as np
import pytest

from paper_2404_19075_b200 import synth


def _geom(beam, **over):
    g = dict(beam=beam, n_rows=6, n_cols=9, sub_x=1, sub_z=1, n_s=16, sod=40.0, odd=30.0, pixel_dx=1.0,
             pixel_dz=1.2, offset_cx=4.5, offset_cz=3.6, fov_radius=4.0, rot_center_x=0.0, z_lo=-3.0, z_hi=3.0,
             t_lo=0.0, t_hi=50.0)
    g.update(over)
    return g


def _field(C=8, L=2, seed=0):
    f = dict(C=C, L=L, mu0=0.9, combine="linear")
    B = synth.grff_matrix(C, 0.3, 0.6, seed=seed)
    prm = synth.init_params(C, L, seed=seed + 1)
    return f, B, prm


@pytest.mark.parametrize("beam,mag", [("parallel", 1.0), ("fan", 70.0 / 40.0), ("cone", 70.0 / 40.0)])
def test_default_grid_is_pixel_over_magnification(O, beam, mag):
    g = _geom(beam)
    gr = O.default_grid(g)
    assert gr["vx"] == pytest.approx(1.0 / mag, rel=1e-15) and gr["vy"] == gr["vx"]
    assert gr["vz"] == pytest.approx(1.2 / mag, rel=1e-15)
    r = g["fov_radius"]
    assert gr["nx"] == int(np.ceil(2 * r / gr["vx"])) and gr["ny"] == gr["nx"]
    assert gr["nz"] == int(np.ceil(6.0 / gr["vz"]))
    # the grid covers the FOV box and is centred on it
    assert gr["x0"] <= -r and gr["x0"] + gr["nx"] * gr["vx"] >= r
    assert gr["x0"] + 0.5 * gr["nx"] * gr["vx"] == pytest.approx(g["rot_center_x"], abs=1e-12)
    assert gr["z0"] + 0.5 * gr["nz"] * gr["vz"] == pytest.approx(0.0, abs=1e-12)


def test_support_is_the_fov_cylinder(O):
    g = _geom("cone", rot_center_x=0.3)
    f, B, prm = _field()
    gr = O.default_grid(g)
    vol = O.voxelize(g, f, B, prm, gr, t=10.0)
    x = gr["x0"] + (np.arange(gr["nx"]) + 0.5) * gr["vx"]
    y = gr["y0"] + (np.arange(gr["ny"]) + 0.5) * gr["vy"]
    inside = (x[None, :] - 0.3) ** 2 + y[:, None] ** 2 <= 16.0
    assert np.all(vol[:, ~inside] == 0.0)
    assert np.all(vol[:, inside] != 0.0)


def test_slabs_match_the_full_volume(O):
    g = _geom("fan")
    f, B, prm = _field(seed=3)
    gr = O.default_grid(g)
    full = O.voxelize(g, f, B, prm, gr, t=20.0)
    part = O.voxelize(g, f, B, prm, gr, t=20.0, k_begin=2, k_count=3)
    assert np.array_equal(part, full[2:5])


@pytest.mark.parametrize("ns", [8, 33])
def test_voxel_sum_equals_ray_quadrature(O, ns):
    """Parallel beam, view angle 0, detector pixel centred on the rotation axis: its ray runs along
    y through (0, y, z_d) with FOV chord [-r, r] and midpoint samples y_j = -r + (j + 1/2) 2r/N_s.
    A one-voxel-wide column of N_s voxels with vy = 2r/N_s has its centres exactly there, so
    vy sum_j vox_j = (chord/N_s) sum_j M(y_j) = p (eq:estforwmod with R7), for any network."""
    r = 4.0
    g = _geom("parallel", n_s=ns, fov_radius=r)
    f, B, prm = _field(C=8, L=3, seed=5)
    row, col = 2, 4  # col 4 centre: -4.5 + 4.5 = 0
    zd = -g["offset_cz"] + (row + 0.5) * g["pixel_dz"]
    theta, t = np.array([0.0]), np.array([17.0])
    idx = np.array([row * g["n_cols"] + col])
    _, p, rc = O.project(g, theta, t, f, B, prm, idx)
    assert rc == 0
    vy = 2 * r / ns
    grid = dict(nx=1, ny=ns, nz=1, x0=-0.5, y0=-r, z0=zd - 0.5, vx=1.0, vy=vy, vz=1.0)
    vol = O.voxelize(g, f, B, prm, grid, t=17.0)
    assert np.all(vol != 0.0)
    assert vy * vol.sum() == pytest.approx(p[0, 0], rel=1e-12)
