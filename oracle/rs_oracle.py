"""CPU oracle for the range-separated (RS) long-range front-end of RHOSVD
(SURVEY.md 8(f) row f3).

TEST INFRASTRUCTURE ONLY (same rules as oracle/rhosvd_oracle.py): only tests/,
__graft_entry__.smoke() and bench.py's baseline legs may import it; the product
package never does and shares no code with it.

Plain fp64 NumPy, following PAPER.md section 4 in its order and notation:

  Slater kernel G(x) = e^{-lambda ||x||} through its Laplace transform
      G(rho) = e^{-2 sqrt(alpha rho)} = sqrt(alpha/pi) int_0^inf tau^{-3/2}
               exp(-alpha/tau - rho tau) dtau,   rho = ||x||^2, alpha = lambda^2 / 4
                                                        (Eq. Slater_Laplace_tr)
  sinc quadrature of that integral -> rank-R canonical tensor
      G_R = sum_k w_k prod_l e^{-tau_k x_l^2}             (Lemma 4.3;
                                                         PAPER.md:1049-1054, Eq. sinc_general)
  RS split  K_l = {k : t_k <= 1},  K_s = {k : t_k > 1},  t_k^2 = tau_k
      G_R = G_{R_l} + G_{R_s}                              (Eq. RS_repres)
  multi-Slater lattice, long-range part by shift-and-windowing
      G_{N,l} = sum_j c_j W_j G_l                          (Eq. Slater_interp_multi)
  then RHOSVD C2T of G_{N,l} (oracle/rhosvd_oracle.py) and T2C (oracle/t2c_oracle.py);
  Prop. 4.2: its Tucker rank grows only as log^{3/2} log(N / eps).

Readings (RS1-RS5):
  RS1 quadrature: trapezoid (sinc) rule in s = ln tau, nodes s_k = k h, |k| <= M, the
      paper leaves the nodes open ("proper choice"); terms whose weight is
      below w_min are dropped (they change G by < w_min everywhere).
  RS2 split: t_k <= 1 with t_k = sqrt(tau_k) (the paper writes the Gaussians as
      e^{-t_k^2 x^2}), i.e. tau_k <= 1.
  RS3 collocation on the cell-centred grid of reading A5; lattice nodes ON grid points,
      so the windowed replica W_j G_l (the reference long part on the doubled grid,
      shifted to node j and cut to the n-grid) is the direct evaluation
      e^{-tau_k (x_i - c_j)^2} at the same points.
  RS4 term order of the lattice tensor: node-major, index j R_l + k.
  RS5 weights c_j and lattice geometry are inputs (workloads/rs_lattice.py).

Pinned by tests/test_rs_oracle.py: the rule reproduces e^{-lambda r} (closed form,
Lemma 4.3's max-error), the split is an exact partition, short-range terms are localised
and the long part has no cusp, windowing equals direct evaluation, the lattice tensor
equals the dense sum of shifted kernels on a tiny grid, and Prop. 4.2 / Table 2 / Fig. 5
rank bands.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = ["slater_sinc_rule", "rs_split", "kernel_dense", "window_reference",
           "rs_long_lattice", "rs_lattice_dense"]


def slater_sinc_rule(lam, h, M, w_min=0.0):
    """Sinc (trapezoid-in-ln tau) rule for G(rho) = e^{-lambda sqrt(rho)}.

    With tau = e^s:  G(rho) = int_R sqrt(alpha/pi) e^{-s/2} e^{-alpha e^{-s}} e^{-rho e^s} ds,
    so  w_k = h sqrt(alpha/pi) e^{-s_k/2} e^{-alpha e^{-s_k}},  tau_k = e^{s_k},  s_k = k h.
    Returns (tau, w) in increasing tau, terms with w < w_min dropped (reading RS1).
    """
    alpha = lam * lam / 4.0
    s = np.arange(-M, M + 1, dtype=np.float64) * h
    w = h * math.sqrt(alpha / math.pi) * np.exp(-s / 2.0) * np.exp(-alpha * np.exp(-s))
    tau = np.exp(s)
    keep = w >= w_min
    return tau[keep], w[keep]


def rs_split(tau):
    """Index sets K_l = {k : t_k <= 1}, K_s = {k : t_k > 1}, t_k = sqrt(tau_k)  (Eq. RS_repres)."""
    t = np.sqrt(np.asarray(tau, dtype=np.float64))
    return np.nonzero(t <= 1.0)[0], np.nonzero(t > 1.0)[0]


def kernel_dense(tau, w, x):
    """Dense n^3 tensor sum_k w_k prod_l e^{-tau_k x_l^2} on the grid x (tiny n only)."""
    E = np.exp(-np.outer(tau, x * x))                   # (R, n)
    return np.einsum("k,ki,kj,kl->ijl", w, E, E, E, optimize=True)


def window_reference(tau, n, h, m):
    """Shift-and-windowing W_j: the reference vectors
    g_k[o] = e^{-tau_k (o h)^2}, o = -(n-1)..(n-1) (the doubled grid centred at the
    origin), cut to the n-grid around node index m: u[i] = g_k[i - m]."""
    o = np.arange(-(n - 1), n, dtype=np.float64)
    g = np.exp(-np.outer(tau, (o * h) ** 2))            # (R, 2n-1)
    i = np.arange(n)
    return g[:, i - m + (n - 1)]                        # (R, n)


def rs_long_lattice(tau_l, w_l, x, nodes, c):
    """Long-range part of the multi-Slater lattice sum as a canonical tensor
    (Eq. Slater_interp_multi), by direct evaluation (reading RS3):
      term j R_l + k : xi = c_j w_k,  u^(l)(x_i) = e^{-tau_k (x_i - X_{j,l})^2}.
    nodes: (N, 3) node coordinates;  c: (N,) amplitudes.
    Returns (U1, U2, U3, xi) with U_l of shape (N R_l, n) (column-major n x R)."""
    tau_l = np.asarray(tau_l, dtype=np.float64)
    N, Rl = nodes.shape[0], tau_l.shape[0]
    xi = (np.asarray(c, dtype=np.float64)[:, None] * np.asarray(w_l)[None, :]).reshape(-1)
    Us = []
    for l in range(3):
        d = x[None, :] - nodes[:, l][:, None]            # (N, n)
        U = np.exp(-tau_l[None, :, None] * (d * d)[:, None, :]).reshape(N * Rl, x.shape[0])
        Us.append(np.ascontiguousarray(U))
    return Us[0], Us[1], Us[2], xi


def rs_lattice_dense(tau, w, x, nodes, c):
    """Dense n^3 sum_j c_j G_R(x - X_j) (tiny grids; pins only)."""
    A = np.zeros((x.shape[0],) * 3)
    for j in range(nodes.shape[0]):
        E = [np.exp(-np.outer(tau, (x - nodes[j, l]) ** 2)) for l in range(3)]
        A += c[j] * np.einsum("k,ki,kj,kl->ijl", w, E[0], E[1], E[2], optimize=True)
    return A
