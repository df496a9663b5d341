"""Pins of the RS long-range front-end oracle (oracle/rs_oracle.py; SURVEY.md 8(f) f3;
PAPER.md section 4).  CPU only.

What fixes each part with no implementation to compare against:
  * the sinc rule reproduces the Slater kernel e^{-lambda r} (closed form) to Lemma 4.3's
    max-error and converges exponentially (Eq. sinc_conv);
  * the RS split is an exact partition (Eq. RS_repres: P_R = P_{R_l} + P_{R_s});
  * the short-range part is localised and the long-range part has no cusp (the reason for
    the split) - both as exact inequalities of Gaussian sums;
  * shift-and-windowing equals direct evaluation of the shifted kernel (Eq.
    Slater_interp_multi) and the lattice tensor equals the dense sum of shifted kernels;
  * Prop. 4.2 (weak rank growth in N) and the bands of Table 2 / Fig. 5:
    bands only - the paper fixes neither the quadrature nodes nor the lattice geometry.
"""
import math

import numpy as np
import pytest

from oracle import (dense_from_canonical, kernel_dense, rhosvd, rs_lattice_dense, rs_long_lattice, rs_split,
                    slater_sinc_rule, t2c, window_reference)
from workloads import make_rs_lattice
from workloads.generators import grid

LAM, H, M, WMIN = 0.5, 0.75, 26, 1e-6   # reading RS1


def _rule():
    return slater_sinc_rule(LAM, H, M, WMIN)


def _G(tau, w, r):
    return (w[None, :] * np.exp(-np.outer(np.asarray(r) ** 2, tau))).sum(1)


def test_rule_reproduces_slater_kernel():
    tau, w = _rule()
    r = np.concatenate([[0.0], np.logspace(-4, np.log10(40.0), 3000)])
    err = np.abs(_G(tau, w, r) - np.exp(-LAM * r))
    assert err.max() <= 2e-5, err.max()          # Lemma 4.3: max-error O(eps), eps_N = 1e-5
    # a different lambda: same construction, same accuracy class
    t2, w2 = slater_sinc_rule(1.0, H, M, WMIN)
    assert np.abs(_G(t2, w2, r) - np.exp(-1.0 * r)).max() <= 5e-5


def test_rule_converges_exponentially():
    """Eq. sinc_conv: error <= C e^{-beta sqrt(M)} - with h = 4 / sqrt(M) the log of the max
    error falls linearly in sqrt(M) (fit slope < 0, every doubling of M at least 10x better)."""
    r = np.linspace(0.0, 30.0, 1201)
    Ms = [8, 16, 32, 64]
    errs = []
    for Mk in Ms:
        tau, w = slater_sinc_rule(LAM, 4.0 / math.sqrt(Mk), Mk, 0.0)
        errs.append(np.abs(_G(tau, w, r) - np.exp(-LAM * r)).max())
    assert all(b < 0.1 * a for a, b in zip(errs, errs[1:])), errs
    slope = np.polyfit(np.sqrt(Ms), np.log(errs), 1)[0]
    assert slope < -1.5, slope


def test_split_is_exact_partition():
    tau, w = _rule()
    kl, ks = rs_split(tau)
    assert len(kl) + len(ks) == len(tau) and not set(kl) & set(ks)
    assert np.all(tau[kl] <= 1.0) and np.all(tau[ks] > 1.0)     # t_k = sqrt(tau_k) <= 1
    assert len(kl) == 8 and len(tau) == 34
    x = grid(12, 3.0)
    full = kernel_dense(tau, w, x)
    parts = kernel_dense(tau[kl], w[kl], x) + kernel_dense(tau[ks], w[ks], x)
    assert np.max(np.abs(full - parts)) <= 1e-15 * np.max(np.abs(full))


def test_short_part_localised_long_part_smooth():
    tau, w = _rule()
    kl, ks = rs_split(tau)
    r = np.linspace(0.0, 20.0, 2001)
    Gs, Gl = _G(tau[ks], w[ks], r), _G(tau[kl], w[kl], r)
    # every short-range Gaussian has tau > 1: |G_s(r)| <= e^{-r^2} sum w_s (exact bound)
    assert np.all(Gs <= np.exp(-r * r) * w[ks].sum() * (1 + 1e-14))
    assert Gs[r >= 4.0].max() <= 1e-6 * Gs[0]
    # no cusp in the long part: 0 <= G_l(0) - G_l(r) <= r^2 sum_k w_k tau_k (1 - e^{-x} <= x)
    d = Gl[0] - Gl
    assert np.all(d >= -1e-15) and np.all(d <= r * r * np.sum(w[kl] * tau[kl]) + 1e-15)
    # while the full kernel has the cusp: its slope at 0 is -lambda
    h = 1e-3
    full = _G(tau, w, [0.0, h])
    assert (full[0] - full[1]) / h > 0.4 * LAM


def test_window_equals_direct_evaluation():
    tau, w = _rule()
    tl = tau[rs_split(tau)[0]]
    n, b = 384, 12.0
    x, h = grid(n, b), 2 * b / n
    for m in (0, 1, 191, 192, 383):
        U = window_reference(tl, n, h, m)
        D = np.exp(-np.outer(tl, (x - x[m]) ** 2))
        assert np.max(np.abs(U - D)) <= 4e-16, m


def test_lattice_tensor_equals_dense_sum_of_shifted_kernels():
    tau, w = _rule()
    kl, _ = rs_split(tau)
    lat = make_rs_lattice((2, 3, 2), n=16, b=3.0, spacing=3)
    U1, U2, U3, xi = rs_long_lattice(tau[kl], w[kl], lat.x, lat.nodes, lat.c)
    assert U1.shape == (lat.N * len(kl), 16) and xi.shape == (lat.N * len(kl),)
    A = dense_from_canonical([U1, U2, U3], xi)
    D = rs_lattice_dense(tau[kl], w[kl], lat.x, lat.nodes, lat.c)
    assert np.max(np.abs(A - D)) <= 1e-13 * np.max(np.abs(D))


# ------------------------------------------------------------------ Prop. 4.2 and the paper's bands
PAPER_TABLE2 = {(4, 4, 4): (13, 13, 13), (6, 6, 6): (15, 15, 15), (8, 8, 8): (19, 19, 19),
                (16, 16, 8): (32, 32, 19)}


def _long_tucker(L, eps=1e-3, **kw):
    tau, w = _rule()
    kl, _ = rs_split(tau)
    lat = make_rs_lattice(L, **kw)
    U1, U2, U3, xi = rs_long_lattice(tau[kl], w[kl], lat.x, lat.nodes, lat.c)
    return rhosvd([U1, U2, U3], xi, eps=eps), len(xi)


@pytest.fixture(scope="module")
def table2():
    return {L: _long_tucker(L) for L in PAPER_TABLE2}


def test_prop42_rank_grows_weakly_in_N(table2):
    """Prop. 4.2: rank_Tuck(G_{N,l}) = C b log^{3/2} log(N / eps) - 32x more nodes (4^3 -> 16x16x8)
    must not even double the Tucker rank, and never exceed ~2.2x log^{3/2} log growth."""
    r0 = max(table2[(4, 4, 4)][0].ranks)
    r1 = max(table2[(16, 16, 8)][0].ranks)
    assert table2[(16, 16, 8)][1] == 32 * table2[(4, 4, 4)][1]
    assert r0 <= r1 < 2 * r0, (r0, r1)
    growth = (math.log(math.log(2048 / 1e-3)) / math.log(math.log(64 / 1e-3))) ** 1.5
    assert r1 / r0 <= 2.2 * growth


def test_table2_tucker_ranks_within_band(table2):
    for L, paper in PAPER_TABLE2.items():
        o, R = table2[L]
        assert R == 8 * L[0] * L[1] * L[2]                  # R_ini = N R_l (R_l = 8 here, 3 in the paper)
        for got, want in zip(o.ranks, paper):
            assert want / 2 <= got <= 2 * want, (L, o.ranks, paper)


def test_fig5_c2c_reduces_long_part():
    """Fig. 5: 12 x 12 x 4 lattice, RHOSVD then T2C at eps = 1e-3:
    the paper reduces R_L = 2304 to 71; here R_ini = 576 x 8 = 4608 must drop >= 10x and
    within 4x of the paper's 71."""
    o, R = _long_tucker((12, 12, 4))
    res = t2c(o.beta, 1e-3 * np.linalg.norm(o.beta))
    Rcc = int(np.sum(res.p))
    assert R == 4608
    assert Rcc * 10 <= R and 71 / 4 <= Rcc <= 71 * 4, Rcc
    assert Rcc <= o.ranks[2] * min(o.ranks[0], o.ranks[1])   # Remark 2.1 rank bound
