"""Pins of the CPU oracle against what the paper and the mathematics fix
(SURVEY.md 8(c) P1-P13).  None of these re-types the oracle's formula: each
checks it against a closed form, an identity, the paper's theorem/corollary,
brute force on a dense n^3 tensor, a full HOSVD, or an independent LAPACK route.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import (canonical_sign, core_kr, dense_from_canonical, dense_from_tucker,
                    exact_error_telescoped, hosvd_full, mode_svd, normalize, project,
                    rhosvd, select_rank, tucker_diff, orth_error, sigma_rel_err)
from workloads import make_config, make_params, make_random_params

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rand_cp(n, R, seed, signed=True):
    rng = np.random.default_rng(seed)
    Us = [rng.normal(size=(R, n)) for _ in range(3)]
    xi = rng.normal(size=R) if signed else rng.uniform(0.5, 1.5, R)
    return Us, xi


# ---------------------------------------------------------------- P1
def test_p1_normalization_unit_columns_and_dense_invariance():
    Us, xi = rand_cp(7, 9, 1)
    Us[1][3] *= 1e-3
    Uh, xip, s, T = normalize(Us, xi)
    for u in Uh:
        assert np.allclose(np.linalg.norm(u, axis=1), 1.0, atol=4e-16 * 4)
    A = dense_from_canonical(Us, xi)
    Ah = dense_from_canonical(Uh, xip)
    assert np.max(np.abs(A - Ah)) <= 1e-14 * np.max(np.abs(A))
    assert np.allclose(T, [9.0, 9.0, 9.0], rtol=1e-15)


def test_p1_rescaling_invariance():
    Us, xi = rand_cp(8, 12, 2)
    a = rhosvd(Us, xi, ranks=(3, 4, 5))
    c = np.exp(np.linspace(-3, 3, 12))
    Us2 = [Us[0] * c[:, None], Us[1] / c[:, None] ** 2, Us[2]]
    xi2 = xi * c
    b = rhosvd(Us2, xi2, ranks=(3, 4, 5))
    for l in range(3):
        assert sigma_rel_err(b.sigma[l], a.sigma[l]) < 1e-13
    d, nrm = tucker_diff(b.beta, b.Z, a.beta, a.Z)
    assert d <= 1e-13 * nrm


def test_zero_column_stays_zero_and_gets_zero_weight():
    # reading A3
    Us, xi = rand_cp(6, 5, 3)
    Us[2][1] = 0.0
    Uh, xip, s, T = normalize(Us, xi)
    assert np.all(Uh[2][1] == 0.0) and xip[1] == 0.0
    assert abs(T[2] - 4.0) < 1e-14 and abs(T[0] - 5.0) < 1e-14


# ---------------------------------------------------------------- P2, P4
@pytest.mark.parametrize("n,R", [(9, 30), (20, 7), (16, 16)])
def test_p2_trace_identity_and_p4_independent_lapack_routes(n, R):
    Us, xi = rand_cp(n, R, 4 + n)
    Uh, xip, s, T = normalize(Us, xi)
    for l in range(3):
        Z, sg = mode_svd(Uh[l])
        assert abs(np.sum(sg ** 2) - T[l]) <= 1e-13 * T[l]                    # P2
        s_gesdd = np.linalg.svd(Uh[l].T, compute_uv=False)                      # P4
        s_gesvd = sla.svd(Uh[l].T, compute_uv=False, lapack_driver="gesvd")
        k = min(n, R)
        assert sigma_rel_err(sg[:k], s_gesdd[:k]) < 1e-12
        assert sigma_rel_err(sg[:k], s_gesvd[:k]) < 1e-12
        # left singular vectors: Z^T Uhat Uhat^T Z = diag(sigma^2)
        G = Uh[l].T @ Uh[l]
        D = Z.T @ G @ Z
        assert np.max(np.abs(D - np.diag(sg ** 2))) <= 1e-13 * sg[0] ** 2
        assert orth_error(Z) < 1e-14


# ---------------------------------------------------------------- P3
def test_p3_eckart_young_residual():
    p = make_params(1)
    Us = [u[:, :] for u in make_config(p)[:3]]
    xi = p.xi
    res = rhosvd(list(Us), xi, ranks=(10, 10, 10))
    Uh, _, _, _ = normalize(list(Us), xi)
    for l in range(3):
        E = Uh[l].T - res.Z[l] @ res.W[l]
        tail2 = np.sum(res.sigma[l][10:] ** 2)
        assert abs(np.sum(E * E) - tail2) <= 1e-10 * tail2 + 1e-14 * res.T[l]


# ---------------------------------------------------------------- P5, P6, P8
@pytest.mark.parametrize("seed", range(12))
def test_p5_p6_p8_bound_telescoped_error_and_core_bruteforce(seed):
    rng = np.random.default_rng(100 + seed)
    n, R = int(rng.integers(5, 13)), int(rng.integers(3, 30))
    Us, xi = rand_cp(n, R, 200 + seed, signed=bool(seed % 2))
    ranks = tuple(int(x) for x in rng.integers(1, min(n, R) + 1, 3))
    res = rhosvd(Us, xi, ranks=ranks)
    A = dense_from_canonical(Us, xi)
    # P8: the KR core equals the dense projection A x_l Z_l^T entrywise
    core = A
    for l in range(3):
        core = np.moveaxis(np.tensordot(res.Z[l].T, np.moveaxis(core, l, 0), axes=1), 0, l)
    assert np.max(np.abs(core - res.beta)) <= 1e-12 * max(1.0, np.max(np.abs(core)))
    A0 = dense_from_tucker(res.beta, res.Z)
    err = np.linalg.norm(A - A0)
    # P6: telescoped exact error without n^3
    Uh, xip, _, _ = normalize(Us, xi)
    tel = exact_error_telescoped(Uh, xip, res.Z)
    assert abs(tel - err) <= 1e-12 * np.linalg.norm(A) + 1e-12 * err
    # P5: Thm. 2.2 and its tighter orthogonal form (A12)
    bp, bns = res.report["bound_paper"], res.report["bound_ns"]
    slack = 64 * 2.2e-16 * np.linalg.norm(A)
    assert err <= bns + slack
    assert bns <= bp + 1e-15 * bp


def test_p5_error_bounds_hand_values():
    """error_bounds against hand-computed values of Thm. 2.2:
    ||xi'|| = ||(3, 4)|| = 5, tails (1, 2, 2): the paper's sum form 5 (1 + 2 + 2) = 25, the
    orthogonal form (A12) 5 sqrt(1 + 4 + 4) = 15; a single truncated mode makes the two
    equal; no truncation gives 0."""
    from oracle.rhosvd_oracle import error_bounds
    bp, bns = error_bounds(np.array([3.0, 4.0]), np.array([1.0, 2.0, 2.0]))
    assert bp == 25.0 and bns == 15.0
    bp, bns = error_bounds(np.array([0.6, 0.8, 0.0]), np.array([0.0, 0.5, 0.0]))
    assert abs(bp - 0.5) <= 1e-16 and abs(bns - 0.5) <= 1e-16
    assert error_bounds(np.array([1.0, -2.0]), np.zeros(3)) == (0.0, 0.0)


# ---------------------------------------------------------------- P7
def test_p7_cor21_A_orthogonal_first_factor():
    rng = np.random.default_rng(7)
    n, R = 10, 6
    Q, _ = np.linalg.qr(rng.normal(size=(n, R)))
    Us = [Q.T.copy(), rng.normal(size=(R, n)), rng.normal(size=(R, n))]
    xi = rng.normal(size=R)
    Uh, xip, _, _ = normalize(Us, xi)
    A = dense_from_canonical(Us, xi)
    assert abs(np.linalg.norm(xip) - np.linalg.norm(A)) <= 1e-13 * np.linalg.norm(A)
    res = rhosvd(Us, xi, ranks=(3, 3, 3))
    err = np.linalg.norm(A - dense_from_tucker(res.beta, res.Z))
    # (errorRHOSVD_orthog) with C = 1
    assert err <= np.linalg.norm(A) * np.sum(res.tails) * (1 + 1e-12)


def test_p7_cor21_B_monotone():
    # cfg 1 is monotone (xi > 0, u > 0): pairwise products >= 0 => ||xi'|| <= ||A||
    p = make_random_params(12, 40, seed=5, ranks=(4, 4, 4), signed=False)
    Us = list(make_config(p)[:3])
    Uh, xip, _, _ = normalize(Us, p.xi)
    A = dense_from_canonical(Us, p.xi)
    assert np.linalg.norm(xip) <= np.linalg.norm(A) * (1 + 1e-13)


# ---------------------------------------------------------------- P9
def test_p9_hosvd_special_case():
    # U2, U3 with orthonormal columns (R <= n), unit-norm U1 columns, equal |xi|:
    # A_(1) A_(1)^T = xi^2 U1 U1^T, so the HOSVD mode-1 frames are the RHOSVD
    # frames and sigma^HOSVD = |xi| sigma.
    rng = np.random.default_rng(9)
    n, R = 9, 5
    Q2, _ = np.linalg.qr(rng.normal(size=(n, R)))
    Q3, _ = np.linalg.qr(rng.normal(size=(n, R)))
    U1 = rng.normal(size=(R, n))
    U1 /= np.linalg.norm(U1, axis=1)[:, None]
    xi = 1.7 * np.where(rng.random(R) < 0.5, -1.0, 1.0)
    Us = [U1, Q2.T.copy(), Q3.T.copy()]
    r = (3, 2, 2)
    res = rhosvd(Us, xi, ranks=r)
    A = dense_from_canonical(Us, xi)
    _, Zh, sh = hosvd_full(A, r)
    P_r = res.Z[0] @ res.Z[0].T
    P_h = Zh[0] @ Zh[0].T
    assert np.max(np.abs(P_r - P_h)) < 1e-12
    assert sigma_rel_err(sh[0][:R], 1.7 * res.sigma[0][:R]) < 1e-12


# ---------------------------------------------------------------- P10
def test_p10_full_rank_is_exact():
    Us, xi = rand_cp(6, 8, 10)
    res = rhosvd(Us, xi, ranks=(6, 6, 6))
    A = dense_from_canonical(Us, xi)
    assert np.linalg.norm(A - dense_from_tucker(res.beta, res.Z)) <= 1e-13 * np.linalg.norm(A)
    # fixed r > min(n, R) is clamped (reading A17)
    res2 = rhosvd(Us, xi, ranks=(50, 50, 50))
    assert res2.ranks == (6, 6, 6)


# ---------------------------------------------------------------- P11 closed forms
def test_p11_closed_forms():
    g = json.load(open(os.path.join(GOLDEN, "closed_forms.json")))
    # rank-1: sigma_1 = 1, exact reconstruction
    rng = np.random.default_rng(11)
    u = [rng.normal(size=(1, 7)) for _ in range(3)]
    res = rhosvd(u, np.array([2.5]), ranks=(1, 1, 1))
    assert abs(res.sigma[0][0] - g["rank1_sigma1"]) < 1e-15
    A = dense_from_canonical(u, np.array([2.5]))
    assert np.linalg.norm(A - dense_from_tucker(res.beta, res.Z)) < 1e-14 * np.linalg.norm(A)
    # R identical columns: sigma_1 = sqrt(R), rest 0
    R = g["identical_R"]
    v = rng.normal(size=(1, 11))
    Us = [np.repeat(v, R, axis=0) for _ in range(3)]
    res = rhosvd(Us, np.ones(R), eps=1e-8)
    assert abs(res.sigma[0][0] - math.sqrt(R)) < 1e-13 * math.sqrt(R)
    assert res.ranks == (1, 1, 1)
    assert np.all(res.sigma[0][1:] < 1e-13)
    # planted m = 2 spectrum: u_k = Q [cos phi_k; sin phi_k]
    phi = np.array(g["planted_phi"])
    Q, _ = np.linalg.qr(rng.normal(size=(13, 2)))
    U = (Q @ np.vstack([np.cos(phi), np.sin(phi)])).T
    Z, sg = mode_svd(U)
    assert sigma_rel_err(sg[:2], np.sqrt(g["planted_sigma2"])) < 1e-14
    assert np.all(sg[2:] < 1e-14)


# ---------------------------------------------------------------- P12
def test_p12_permutation_and_shard_invariance():
    p = make_random_params(10, 37, seed=12, eps=1e-3)
    Us = list(make_config(p)[:3])
    a = rhosvd(Us, p.xi, eps=1e-3)
    perm = np.random.default_rng(1).permutation(37)
    b = rhosvd([u[perm] for u in Us], p.xi[perm], eps=1e-3)
    assert a.ranks == b.ranks
    for l in range(3):
        assert sigma_rel_err(b.sigma[l], a.sigma[l]) < 1e-13
    d, nrm = tucker_diff(b.beta, b.Z, a.beta, a.Z)
    assert d <= 1e-13 * nrm
    # sharding: partial cores over column blocks sum to the full core
    Uh, xip, _, _ = normalize(Us, p.xi)
    part = sum(core_kr(*(a.W[l][:, s:e] for l in range(3)), xip[s:e]) for s, e in [(0, 13), (13, 30), (30, 37)])
    assert np.max(np.abs(part - a.beta)) <= 1e-13 * np.max(np.abs(a.beta))


# ---------------------------------------------------------------- P13 and rank rule
def test_select_rank_by_hand():
    sig = np.array([3.0, 2.0, 1.0, 0.5])        # sigma^2 = 9, 4, 1, .25; T = 14.25
    T = 14.25
    # tails: r=1 -> 5.25, r=2 -> 1.25, r=3 -> .25, r=4 -> 0
    for eps2, r_exp in [(5.3 / T, 1), (5.2 / T, 2), (1.3 / T, 2), (1.2 / T, 3), (0.2 / T, 4)]:
        r, _, _ = select_rank(sig, T, eps=math.sqrt(eps2))
        assert r == r_exp, (eps2, r)
    r, _, _ = select_rank(sig, T, r_fixed=9)
    assert r == 4


def test_p13_rank_monotone_in_eps():
    p = make_random_params(24, 300, seed=13, eps=1e-4)
    Us = list(make_config(p)[:3])
    last = None
    for eps in [1e-1, 1e-2, 1e-3, 1e-4, 1e-6, 1e-8]:
        r = rhosvd(Us, p.xi, eps=eps).ranks
        if last is not None:
            assert all(x >= y for x, y in zip(r, last))
        last = r


def test_canonical_sign():
    Z = np.array([[0.1, -0.9], [-0.5, 0.2], [0.5, 0.3]])
    Zs, sg = canonical_sign(Z)
    assert list(sg) == [-1.0, -1.0]  # col 0: tie |-.5|=|.5| -> lowest row (row 1, negative)
    assert Zs[1, 0] == 0.5 and Zs[0, 1] == 0.9


def test_tucker_diff_matches_dense():
    Us, xi = rand_cp(8, 10, 21)
    a = rhosvd(Us, xi, ranks=(3, 3, 3))
    b = rhosvd(Us, xi, ranks=(4, 3, 2))
    d, _ = tucker_diff(a.beta, a.Z, b.beta, b.Z)
    D = dense_from_tucker(a.beta, a.Z) - dense_from_tucker(b.beta, b.Z)
    assert abs(d - np.linalg.norm(D)) <= 1e-13 * np.linalg.norm(D)
    # sign flips of frame columns (with the core) do not change the tensor
    Zf = [z * np.where(np.arange(z.shape[1]) % 2, -1.0, 1.0)[None, :] for z in a.Z]
    bf = a.beta
    for l in range(3):
        sh = [1, 1, 1]
        sh[l] = -1
        bf = bf * np.where(np.arange(a.beta.shape[l]) % 2, -1.0, 1.0).reshape(sh)
    d2, nrm = tucker_diff(bf, Zf, a.beta, a.Z)
    assert d2 <= 1e-14 * nrm


def test_r_less_than_n():
    # reading A4: R < n allowed, ranks <= R
    Us, xi = rand_cp(12, 4, 31)
    res = rhosvd(Us, xi, eps=1e-12)
    assert res.ranks == (4, 4, 4)
    A = dense_from_canonical(Us, xi)
    assert np.linalg.norm(A - dense_from_tucker(res.beta, res.Z)) <= 1e-13 * np.linalg.norm(A)


def test_empty_R():
    Us = [np.zeros((0, 5)) for _ in range(3)]
    res = rhosvd(Us, np.zeros(0), eps=1e-3)
    assert res.ranks == (0, 0, 0) and res.beta.size == 0


def test_normalization_no_underflow():
    """A column with entries ~1e-200 has norm ~1e-200, not 0: it is normalized to a unit
    column and xi' = xi ||u|| (closed form; the naive sum of squares underflows)."""
    from oracle import normalize
    u = np.array([[3e-200, 4e-200, 0.0], [1.0, 2.0, 2.0]])
    Uh, xip, s, T = normalize([u, u, u], np.array([1.0, 1.0]))
    assert np.allclose(s[0], [5e-200, 3.0], rtol=1e-15)
    assert np.allclose(Uh[0][0], [0.6, 0.8, 0.0], rtol=1e-15)
    assert np.allclose(T, [2.0, 2.0, 2.0], rtol=1e-15)
    assert xip[0] == 0.0 or xip[0] > 0  # (5e-200)^3 underflows to 0: the weight, not the column
