"""GPU tests of the widened rows:
  N2  analytic-phantom projector + transmission-space noise (dinr_phantom_project)
Parity against the fp64 oracle's closed-form projector (or_project_exact); noise checked by its
statistics and determinism."""
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


PRIMS = [
    dict(kind="indicator", value=0.05, center=(1.0, -0.5, 0.3), axes=(5.0, 6.0, 4.0), velocity=(0.01, 0.0, -0.005),
         axes_rate=(0.0, 0.002, 0.0)),
    dict(kind="smooth", value=0.08, center=(0.5, 0.2, -0.4), axes=(6.0, 4.5, 5.0)),
    dict(kind="gaussian", value=0.3, center=(-1.0, 0.7, 0.2), axes=(1.0, 1.2, 0.9)),
]


@pytest.mark.parametrize("beam", ["parallel", "fan", "cone"])
@pytest.mark.parametrize("combine", ["beer", "linear"])
def test_phantom_projection_exact_parity(ctx, dev, O, beam, combine):
    g = dict(beam=beam, n_rows=8, n_cols=12, sub_x=2, sub_z=2 if beam == "cone" else 1, n_s=32, sod=40.0, odd=30.0,
             pixel_dx=1.5, pixel_dz=1.5, offset_cx=9.0, offset_cz=6.0, fov_radius=12.0, rot_center_x=0.4,
             z_lo=-6, z_hi=6, t_lo=0.0, t_hi=100.0)
    rng = np.random.default_rng(3)
    M = 10
    theta, t = rng.uniform(0, 2 * np.pi, M), np.linspace(0, 100, M)
    D.set_geometry(ctx, g, theta, t)
    idx = rng.choice(M * g["n_rows"] * g["n_cols"], 500, replace=False)
    S = g["sub_x"] * g["sub_z"]
    fh = torch.zeros(len(idx), device=dev)
    ps = torch.zeros(len(idx) * S, device=dev)
    D.phantom_project(ctx, PRIMS, torch.tensor(idx, device=dev), fh, ps, combine=combine)
    rf, rp, rc = O.project_exact(g, theta, t, PRIMS, idx, combine)
    assert rc == 0
    # fp32 outputs of fp64 computations: relative L-inf at fp32 rounding
    assert np.max(np.abs(fh.cpu().numpy() - rf)) <= 1e-6 * np.max(np.abs(rf))
    assert np.max(np.abs(ps.cpu().numpy().reshape(-1, S) - rp)) <= 1e-6 * np.max(np.abs(rp))


def test_phantom_workload_data_and_noise(ctx, dev, O):
    name = "fan512"
    g = synth.geometry(name)
    th, t = synth.views(name)
    D.set_geometry(ctx, g, th, t)
    n = 150000  # of the 184 320 fan512 pixels
    idx = torch.tensor(synth.pixel_batch(name, n, seed=2), device=dev)
    clean = torch.zeros(n, device=dev)
    D.phantom_project(ctx, synth.phantom(name), idx, clean)
    pick = np.random.default_rng(0).choice(n, 300, replace=False)
    rf, _, _ = O.project_exact(g, th, t, synth.phantom(name), idx.cpu().numpy()[pick])
    assert np.max(np.abs(clean.cpu().numpy()[pick] - rf)) <= 1e-6 * np.max(np.abs(rf))
    # transmission-space noise: T' - T ~ N(0, (frac sqrt(T))^2)  (eq:forwmod, R24)
    frac = 1e-3
    noisy = torch.zeros(n, device=dev)
    D.phantom_project(ctx, synth.phantom(name), idx, noisy, noise_frac=frac, seed=7)
    T, Tn = torch.exp(-clean.double()), torch.exp(-noisy.double())
    z = ((Tn - T) / (frac * torch.sqrt(T))).cpu().numpy()
    assert abs(z.mean()) < 0.02 and abs(z.std() - 1.0) < 0.05
    again = torch.zeros(n, device=dev)
    D.phantom_project(ctx, synth.phantom(name), idx, again, noise_frac=frac, seed=7)
    assert torch.equal(noisy, again)
    other = torch.zeros(n, device=dev)
    D.phantom_project(ctx, synth.phantom(name), idx, other, noise_frac=frac, seed=8)
    assert not torch.equal(noisy, other)


def test_phantom_mass_conservation_parallel(ctx, dev):
    """Per view, sum_px Dx Dz fhat = A (2 pi)^{3/2} sx sy sz for Gaussian blobs (1e-6: fp32 outputs)."""
    g = dict(beam="parallel", n_rows=64, n_cols=64, sub_x=1, sub_z=1, n_s=32, sod=64.0, odd=64.0, pixel_dx=1.0,
             pixel_dz=1.0, offset_cx=32.0, offset_cz=32.0, fov_radius=32.0, rot_center_x=0.0, z_lo=-32, z_hi=32,
             t_lo=0, t_hi=0)
    prims = [dict(kind="gaussian", value=0.05, center=(3.0, -2.0, 1.0), axes=(3.0, 4.0, 3.5))]
    mass = 0.05 * (2 * np.pi) ** 1.5 * 3.0 * 4.0 * 3.5
    theta = np.deg2rad(np.array([0.0, 33.0, 120.0]))
    D.set_geometry(ctx, g, theta, np.zeros(3))
    N = 64 * 64
    fh = torch.zeros(3 * N, device=dev)
    D.phantom_project(ctx, prims, torch.arange(3 * N, device=dev), fh, combine="linear")
    tot = fh.double().view(3, N).sum(1).cpu().numpy()
    assert np.all(np.abs(tot - mass) <= 1e-6 * mass)
