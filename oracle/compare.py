"""Parity comparison helpers (TEST INFRASTRUCTURE ONLY; see oracle/rhosvd_oracle.py header).

Implements SURVEY.md 8(c)'s sign- and rotation-invariant Tucker comparison
(BASELINE.json: "comparing projectors Z Z^T rather than sign-ambiguous
vectors"; reading A14):

  [Zhat_l, Z_l] = Q_l [Mhat_l, M_l]   (thin QR, Q_l orthonormal n x 2r)
  D = betahat x_l Mhat_l - beta x_l M_l     (2r x 2r x 2r)
  ||That - T||_F = ||D||_F exactly (Q_l orthonormal), with no cancellation.
"""
from __future__ import annotations

import numpy as np

from .rhosvd_oracle import mode_product

__all__ = ["tucker_diff", "orth_error", "sin_theta", "sigma_rel_err"]


def tucker_diff(beta_a, Za, beta_b, Zb):
    """Return (||Ta - Tb||_F, ||Tb||_F) for Tucker tensors (beta, [Z1, Z2, Z3])."""
    Ma, Mb = [], []
    for za, zb in zip(Za, Zb):
        Q, Rm = np.linalg.qr(np.concatenate([za, zb], axis=1))
        ra = za.shape[1]
        Ma.append(Rm[:, :ra])
        Mb.append(Rm[:, ra:])
    Xa, Xb = beta_a, beta_b
    for l in range(len(Ma)):
        Xa = mode_product(Xa, Ma[l], l)
        Xb = mode_product(Xb, Mb[l], l)
    return float(np.linalg.norm(Xa - Xb)), float(np.linalg.norm(beta_b))


def orth_error(Z):
    """max |Z^T Z - I|."""
    if Z.shape[1] == 0:
        return 0.0
    return float(np.max(np.abs(Z.T @ Z - np.eye(Z.shape[1]))))


def sin_theta(Za, Zb):
    """Largest principal-angle sine ||(I - Zb Zb^T) Za||_2 (diagnostic only)."""
    if Za.shape[1] == 0:
        return 0.0
    E = Za - Zb @ (Zb.T @ Za)
    return float(np.linalg.norm(E, 2))


def sigma_rel_err(sa, sb):
    """max_k |sa_k - sb_k| / sb_k over the retained values (reading A13)."""
    sa = np.asarray(sa, dtype=np.float64)
    sb = np.asarray(sb, dtype=np.float64)
    m = min(sa.shape[0], sb.shape[0])
    if m == 0:
        return 0.0
    return float(np.max(np.abs(sa[:m] - sb[:m]) / np.abs(sb[:m])))
