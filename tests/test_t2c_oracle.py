"""Pins of the T2C oracle (oracle/t2c_oracle.py; PAPER.md Remark 2.1)
against what the paper and the mathematics fix - no GPU."""
import math

import numpy as np
import pytest

from oracle import dense_from_tucker, rhosvd as oracle_rhosvd, dense_from_canonical
from oracle.t2c_oracle import t2c, t2c_dense, t2c_threshold, c2c_lift, dense_from_cp
from workloads import make_config, make_random_params


def rand_core(shape, seed, decay=True):
    rng = np.random.default_rng(seed)
    b = rng.normal(size=shape)
    if decay:  # graded like a Tucker core: entries fall off with the index sum
        r1, r2, r3 = shape
        g = np.exp(-0.35 * (np.arange(r1)[:, None, None] + np.arange(r2)[None, :, None] + np.arange(r3)[None, None, :]))
        b = b * g
    return b


@pytest.mark.parametrize("shape,seed,eps_rel", [((6, 5, 4), 1, 1e-2), ((12, 12, 12), 2, 1e-4),
                                                ((9, 14, 7), 3, 1e-6), ((20, 18, 16), 4, 1e-3)])
def test_exact_error_identity_and_paper_bound(shape, seed, eps_rel):
    """Slices are orthogonal in mode 3, so ||beta - beta_(R)||^2 is exactly the sum of the
    discarded sigma^2; the paper's guarantee ||beta - beta_(R)|| <= eps."""
    beta = rand_core(shape, seed)
    eps = eps_rel * np.linalg.norm(beta)
    res = t2c(beta, eps)
    err = np.linalg.norm(beta - t2c_dense(res, shape))
    assert abs(err ** 2 - res.err2) <= 1e-12 * np.linalg.norm(beta) ** 2 + 1e-14 * res.err2
    assert err <= eps
    # rank bound R <= p_1 + ... + p_r <= r3 min(r1, r2)  (r^2 for the cubic core)
    assert res.sigma.shape[0] == int(np.sum(res.p)) <= shape[2] * min(shape[0], shape[1])
    # every kept sigma is above the threshold, every dropped one at or below it
    for m in range(shape[2]):
        s = np.linalg.svd(beta[:, :, m], compute_uv=False)
        assert np.all(s[:res.p[m]] > res.thr) and np.all(s[res.p[m]:] <= res.thr)


def test_threshold_reduces_to_paper_form_for_cubic_core():
    """thr = eps / r^{3/2} for an r x r x r core."""
    for r in (1, 4, 10, 33):
        assert math.isclose(t2c_threshold(0.7, (r, r, r)), 0.7 / r ** 1.5, rel_tol=1e-15)


def test_eps_to_zero_is_exact():
    beta = rand_core((8, 7, 6), 5, decay=False)
    res = t2c(beta, 0.0)
    assert res.sigma.shape[0] == 6 * 7  # every slice keeps its full rank
    assert np.linalg.norm(beta - t2c_dense(res, beta.shape)) <= 1e-13 * np.linalg.norm(beta)


def test_closed_form_rank_one_and_diagonal_cores():
    rng = np.random.default_rng(6)
    a, b, c = rng.normal(size=7), rng.normal(size=5), rng.normal(size=6)
    c[2] = 1e-9
    beta = np.einsum("i,j,k->ijk", a, b, c)
    eps = 1e-6 * np.linalg.norm(beta)
    res = t2c(beta, eps)
    expect = np.abs(c) * np.linalg.norm(a) * np.linalg.norm(b)
    keep = expect > res.thr
    assert res.sigma.shape[0] == int(np.sum(keep))
    assert np.allclose(np.sort(res.sigma), np.sort(expect[keep]), rtol=1e-13)
    for j in range(res.sigma.shape[0]):  # u_k = +-a/||a|| with the sign rule (T4)
        u = res.U[:, j]
        ua = a / np.linalg.norm(a)
        ua = ua if ua[np.argmax(np.abs(ua))] > 0 else -ua
        assert np.allclose(u, ua, atol=1e-13)
    d = np.array([3.0, 1e-3, 0.5, 1e-12])
    D = np.zeros((4, 4, 4))
    for i in range(4):
        D[i, i, i] = d[i]
    res = t2c(D, 1e-6)
    assert res.sigma.shape[0] == 3 and np.allclose(np.sort(res.sigma), np.sort(d[:3]), rtol=1e-15)


def test_lift_matches_tucker_brute_force_and_c2c_bound():
    """C2C: the lifted canonical tensor equals beta_(R) x_l Z_l (brute force on a tiny grid),
    and ||A - A_C2C|| <= ||A - A_Tucker|| + eps (the frames are orthonormal)."""
    p = make_random_params(12, 40, seed=9, eps=1e-4)
    U1, U2, U3, xi = make_config(p)
    o = oracle_rhosvd([U1, U2, U3], xi, eps=p.eps)
    eps = 1e-5 * np.linalg.norm(o.beta)
    res = t2c(o.beta, eps)
    F1, F2, F3, w = c2c_lift(res, o.Z)
    A_c2c = dense_from_cp(F1, F2, F3, w)
    A_t = dense_from_tucker(t2c_dense(res, o.beta.shape), o.Z)
    assert np.linalg.norm(A_c2c - A_t) <= 1e-13 * np.linalg.norm(A_t)
    A = dense_from_canonical([U1, U2, U3], xi)
    A_tucker = dense_from_tucker(o.beta, o.Z)
    assert np.linalg.norm(A - A_c2c) <= np.linalg.norm(A - A_tucker) + eps * (1 + 1e-12)
    # the lifted factors are unit columns (normalized canonical format)
    for F in (F1, F2, F3):
        assert np.allclose(np.linalg.norm(F, axis=0), 1.0, atol=1e-13)


def test_empty_and_degenerate():
    res = t2c(np.zeros((3, 4, 5)), 1e-3)
    assert res.sigma.shape == (0,) and res.U.shape == (3, 0) and res.err2 == 0.0
    res = t2c(np.ones((1, 1, 1)), 0.5)
    assert res.sigma.shape == (1,) and res.sigma[0] == 1.0
