"""Pins of the tensor-product convolution oracle (oracle/conv_oracle.py)
against closed forms and brute force - no GPU."""
import math

import numpy as np
import pytest

from oracle import dense_from_cp
from oracle.conv_oracle import conv1d, conv3d_canonical, dense_conv3d


def test_impulse_at_centre_returns_h_p():
    n, h = 17, 0.3
    rng = np.random.default_rng(1)
    p = rng.normal(size=n)
    u = np.zeros(n)
    u[n // 2] = 1.0
    assert np.allclose(conv1d(u, p, h), h * p, rtol=0, atol=1e-15)
    n = 16
    p = rng.normal(size=n)
    u = np.zeros(n)
    u[n // 2] = 1.0
    assert np.allclose(conv1d(u, p, h), h * p, rtol=0, atol=1e-15)


def test_commutativity():
    rng = np.random.default_rng(2)
    for n in (8, 9, 33):
        u, p = rng.normal(size=n), rng.normal(size=n)
        assert np.allclose(conv1d(u, p, 0.5), conv1d(p, u, 0.5), rtol=0, atol=1e-13)


def test_box_box_is_hat():
    """Boxes of half-width a and b (centred): the convolution is a trapezoid/hat with
    height h * min(2a+1, 2b+1) at the centre, falling by h per grid step outside."""
    n, h, a, b = 41, 0.1, 5, 3
    c = n // 2
    x = np.arange(n) - c
    u = (np.abs(x) <= a).astype(float)
    p = (np.abs(x) <= b).astype(float)
    # sum_j u_j p_{i + c - j} = #{j : |j - c| <= a, |i - j| <= b}  (p index centred at c)
    expect = np.array([h * np.sum((np.abs(x) <= a) & (np.abs(i - (x + c)) <= b)) for i in range(n)])
    hat = h * np.clip(np.minimum(2 * b + 1, a + b + 1 - np.abs(x)), 0, None)
    assert np.array_equal(conv1d(u, p, h), expect)
    assert np.allclose(expect, hat, rtol=0, atol=1e-15)


def test_gaussian_gaussian_closed_form():
    """int exp(-a y^2) exp(-b (x - y)^2) dy = sqrt(pi / (a + b)) exp(-a b x^2 / (a + b)); the
    Riemann sum of well-resolved Gaussians is spectrally accurate (odd n: grid symmetric)."""
    n = 129
    L = 20.0
    h = L / (n - 1)
    x = (np.arange(n) - n // 2) * h
    a, b = 0.7, 1.9
    got = conv1d(np.exp(-a * x ** 2), np.exp(-b * x ** 2), h)
    ref = math.sqrt(math.pi / (a + b)) * np.exp(-a * b * x ** 2 / (a + b))
    assert np.max(np.abs(got - ref)) <= 1e-12


@pytest.mark.parametrize("n", [6, 7])
def test_separability_against_dense_3d_convolution(n):
    """The canonical tensor-product convolution equals the brute-force dense 3-D
    convolution of the dense reconstructions (exact identity up to rounding)."""
    rng = np.random.default_rng(3 + n)
    h = 0.25
    Fa = [rng.normal(size=(n, 2)) for _ in range(3)]
    ca = rng.normal(size=2)
    Fp = [rng.normal(size=(n, 3)) for _ in range(3)]
    cp = rng.normal(size=3)
    F, w = conv3d_canonical(Fa, ca, Fp, cp, h)
    assert F[0].shape == (n, 6) and w.shape == (6,)
    A = dense_from_cp(Fa[0], Fa[1], Fa[2], ca)
    P = dense_from_cp(Fp[0], Fp[1], Fp[2], cp)
    V = dense_conv3d(A, P, h)
    Vc = dense_from_cp(F[0], F[1], F[2], w)
    assert np.linalg.norm(Vc - V) <= 1e-12 * np.linalg.norm(V)


def test_rank_one_times_rank_one_and_weights():
    n = 9
    rng = np.random.default_rng(5)
    Fa = [rng.normal(size=(n, 1)) for _ in range(3)]
    Fp = [rng.normal(size=(n, 1)) for _ in range(3)]
    F, w = conv3d_canonical(Fa, np.array([2.0]), Fp, np.array([-3.0]), 0.5)
    assert F[0].shape == (n, 1) and w[0] == -6.0
    with pytest.raises(ValueError):
        conv1d(np.ones(4), np.ones(5), 1.0)
