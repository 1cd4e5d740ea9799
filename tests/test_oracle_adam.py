"""Pins for the oracle's Adam step (NEXT row N1; "We use the Adam optimizer", SPEC
S:377-383 with bias correction).  Expectations are closed forms, not re-typed formulas."""
import numpy as np


def test_first_step_is_a_sign_step(O):
    # first step, any g != 0 -> per-coordinate |update| ~= lr (mhat = g, vhat = g^2)
    g = np.array([0.5, -2.0, 3e-3, -7.0])
    p, m, v = O.adam_step(np.zeros(4), g, np.zeros(4), np.zeros(4), lr=1e-3)
    assert np.allclose(p, -1e-3 * np.sign(g) * np.abs(g) / (np.abs(g) + 1e-8), rtol=1e-12)


def test_zero_gradient_keeps_parameters(O):
    p, m, v = O.adam_step(np.arange(5.0), np.zeros(5), np.zeros(5), np.zeros(5), lr=1e-2)
    assert np.array_equal(p, np.arange(5.0)) and not m.any() and not v.any()


def test_constant_gradient_closed_form(O):
    # constant g for k steps: mhat_k = g and vhat_k = g^2 exactly -> every update is lr*g/(|g|+eps)
    g = np.array([0.3, -1.5])
    p, m, v = np.zeros(2), np.zeros(2), np.zeros(2)
    for k in range(1, 6):
        p, m, v = O.adam_step(p, g, m, v, lr=0.01, step=k)
    assert np.allclose(m, g * (1 - 0.9 ** 5), rtol=1e-12)
    assert np.allclose(v, g * g * (1 - 0.999 ** 5), rtol=1e-12)
    assert np.allclose(p, -5 * 0.01 * g / (np.abs(g) + 1e-8), rtol=1e-9)
