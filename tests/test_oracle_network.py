"""Pins for the oracle's network (O6-O8, O12) and full gradient.

- GRFF special cases, swish identities.
- MLP forward/backward against torch.autograd in float64 on CPU: an independent library
  reference (the paper itself used PyTorch autograd).
- Full loss gradient (eq:partiald) against central finite differences in fp64 on tiny nets,
  all three beams, BEER and LINEAR: relative L-inf per tensor <= 1e-6 (north_star).
- Linearity, zero residual, n = 0, K-invariance of the gradient average.
"""
import math

import numpy as np
import pytest
import torch

from conftest import golden_geom


def test_param_count(O):
    assert O.param_count(128, 5) == 329217
    assert O.param_count(32, 3) == 12545
    assert O.param_count(64, 4) == 66177
    assert O.param_count(128, 6) == 395009


def test_grff_special_values(O):
    C_ = 5
    B = np.random.default_rng(0).standard_normal((C_, 4))
    f0 = O.grff(B, np.zeros(4))[0]
    assert np.array_equal(f0, np.r_[np.ones(C_), np.zeros(C_)])
    rb = np.random.default_rng(1).uniform(-1, 1, (100, 4))
    f = O.grff(B, rb)
    assert np.all(np.abs(f) <= 1.0)
    assert np.allclose(f[:, :C_] ** 2 + f[:, C_:] ** 2, 1.0, atol=1e-15)
    # quarter period: B row with B . rbar = 0.25 -> (cos, sin) = (0, 1)
    B1 = np.array([[0.25, 0.0, 0.0, 0.0]])
    q = O.grff(B1, np.array([1.0, 0.3, -0.2, 0.9]))[0]
    assert abs(q[0]) < 1e-15 and abs(q[1] - 1.0) < 1e-15


def _torch_mlp(C_, L, mu0, B, prm, rb):
    H = 2 * C_
    Bt = torch.tensor(B, dtype=torch.float64)
    P = torch.tensor(prm, dtype=torch.float64, requires_grad=True)
    r = torch.tensor(rb, dtype=torch.float64)
    phi = r @ Bt.T
    h = torch.cat([torch.cos(2 * math.pi * phi), torch.sin(2 * math.pi * phi)], dim=1)
    off = 0
    for _ in range(L):
        W = P[off:off + H * H].view(H, H)
        b = P[off + H * H:off + H * H + H]
        off += H * H + H
        h = torch.nn.functional.silu(h @ W.T + b)
    wo, bo = P[off:off + H], P[off + H]
    return mu0 * (h @ wo + bo), P


@pytest.mark.parametrize("C_,L", [(2, 1), (4, 2), (8, 3)])
def test_mlp_vs_torch_fp64(O, C_, L):
    rng = np.random.default_rng(C_ * 10 + L)
    B = rng.standard_normal((C_, 4)) * 0.7
    prm = rng.uniform(-1, 1, O.param_count(C_, L)) / math.sqrt(2 * C_)
    rb = rng.uniform(-1, 1, (64, 4))
    f = dict(C=C_, L=L, mu0=0.05)
    mu = O.mlp_eval(f, B, prm, rb)
    mt, P = _torch_mlp(C_, L, 0.05, B, prm, rb)
    assert np.max(np.abs(mu - mt.detach().numpy())) <= 1e-12 * max(1e-300, np.max(np.abs(mu)))
    u = rng.standard_normal(64)
    g = O.mlp_grad(f, B, prm, rb, u)
    (mt * torch.tensor(u)).sum().backward()
    gt = P.grad.numpy()
    assert np.max(np.abs(g - gt)) <= 1e-12 * np.max(np.abs(gt))


def test_swish_identities(O):
    # swish(0) = 0: with W=0, b=0 every hidden unit is 0 -> M = mu0 * b_o.
    C_, L = 2, 2
    prm = np.zeros(O.param_count(C_, L))
    prm[-1] = 3.0
    mu = O.mlp_eval(dict(C=C_, L=L, mu0=0.5), np.ones((C_, 4)), prm, np.random.default_rng(0).uniform(-1, 1, (5, 4)))
    assert np.array_equal(mu, np.full(5, 1.5))


def _tiny_geom(beam):
    g = dict(beam=beam, n_rows=3, n_cols=4, sub_x=2, sub_z=2 if beam == "cone" else 1, n_s=5,
             sod=6.0, odd=5.0, pixel_dx=1.2, pixel_dz=1.1, offset_cx=2.3, offset_cz=1.6,
             fov_radius=2.5, rot_center_x=0.3, z_lo=-2.0, z_hi=2.0, t_lo=0.0, t_hi=20.0)
    return g


def _rel_linf_per_tensor(a, b, C_, L):
    H = 2 * C_
    errs = []
    off = 0
    for _ in range(L):
        for n in (H * H, H):
            sl = slice(off, off + n)
            errs.append(np.max(np.abs(a[sl] - b[sl])) / max(np.max(np.abs(b[sl])), 1e-300))
            off += n
    for n in (H, 1):
        sl = slice(off, off + n)
        errs.append(np.max(np.abs(a[sl] - b[sl])) / max(np.max(np.abs(b[sl])), 1e-300))
        off += n
    return max(errs)


@pytest.mark.parametrize("beam", ["parallel", "fan", "cone"])
@pytest.mark.parametrize("combine", ["beer", "linear"])
@pytest.mark.parametrize("C_,L", [(2, 1), (4, 2), (2, 3)])
def test_gradient_vs_central_fd(O, beam, combine, C_, L):
    g = _tiny_geom(beam)
    # a fixed seed per case (Python's hash() of strings changes from run to run)
    rng = np.random.default_rng(["parallel", "fan", "cone"].index(beam) * 1000 + ["beer", "linear"].index(combine) * 100
                                + C_ * 10 + L)
    M = 3
    theta, t = rng.uniform(0, 6, M), np.array([0.0, 10.0, 20.0])
    idx = rng.choice(M * 12, 4, replace=False)
    B = rng.standard_normal((C_, 4)) * 0.6
    prm = rng.uniform(-1, 1, O.param_count(C_, L)) / math.sqrt(2 * C_)
    prm[-1] = 1.0
    f = dict(C=C_, L=L, mu0=0.3, combine=combine)
    y = rng.uniform(0, 2, len(idx))
    grad, rc = O.project_and_grad(g, theta, t, f, B, prm, idx, y)
    assert rc == 0
    P = len(prm)

    def loss(p):
        fh, _, _ = O.project(g, theta, t, f, B, p, idx)
        return np.mean((y - fh) ** 2)

    assert abs(grad[P] - loss(prm)) <= 1e-14 * abs(grad[P])
    fd = np.zeros(P)
    for q in range(P):
        h = 1e-6 * max(1.0, abs(prm[q]))
        pp, pm = prm.copy(), prm.copy()
        pp[q] += h
        pm[q] -= h
        fd[q] = (loss(pp) - loss(pm)) / (2 * h)
    assert _rel_linf_per_tensor(grad[:P], fd, C_, L) <= 1e-6


def test_gradient_structure(O):
    """Linearity (batch grad = mean of per-pixel grads), y = fhat => zero grad, n = 0,
    and K-invariance of the rank average (R16)."""
    g = _tiny_geom("cone")
    rng = np.random.default_rng(42)
    C_, L = 3, 2
    theta, t = rng.uniform(0, 6, 3), np.array([0.0, 10.0, 20.0])
    B = rng.standard_normal((C_, 4)) * 0.6
    prm = rng.uniform(-1, 1, O.param_count(C_, L)) / math.sqrt(2 * C_)
    f = dict(C=C_, L=L, mu0=0.3, combine="beer")
    idx = rng.choice(36, 8, replace=False)
    y = rng.uniform(0, 1, 8)
    full, _ = O.project_and_grad(g, theta, t, f, B, prm, idx, y)
    per = [O.project_and_grad(g, theta, t, f, B, prm, idx[i:i + 1], y[i:i + 1])[0] for i in range(8)]
    assert np.allclose(full, np.mean(per, axis=0), rtol=1e-12, atol=1e-15)
    # K-invariance: G ranks x (n/G) pixels, averaged == 1 rank x n pixels
    for G in (2, 4):
        parts = [O.project_and_grad(g, theta, t, f, B, prm, idx[r::G], y[r::G])[0] for r in range(G)]
        assert np.allclose(O.allreduce_mean(parts), full, rtol=1e-12, atol=1e-15)
    fh, _, _ = O.project(g, theta, t, f, B, prm, idx)
    z, _ = O.project_and_grad(g, theta, t, f, B, prm, idx, fh)
    assert np.max(np.abs(z)) <= 1e-14
    e, rc = O.project_and_grad(g, theta, t, f, B, prm, idx[:0], y[:0])
    assert rc == 0 and np.all(e == 0)
