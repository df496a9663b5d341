"""CPU oracle for the canonical-to-Tucker ALS sweep that refines the RHOSVD frames
(SURVEY.md 8(f) row f2).

TEST INFRASTRUCTURE ONLY (same rules as oracle/rhosvd_oracle.py): only tests/,
__graft_entry__.smoke() and bench.py's baseline legs may import it; the product
package never does.

Plain fp64 NumPy/LAPACK, following PAPER.md section 2.1 after Def. 2.1
(Eq. can_A_Tuck_als and Fig. 2) in its order and notation:

  (can_A_Tuck_als)  A = Z^(1) x_1 A_2 x_2 Z^(3),
                    A_2 = xi x_1 D_{1,0} V_0^(1)T x_3 D_{3,0} V_0^(3)T
                    i.e. A_2 = A x_1 Z^(1)T x_3 Z^(3)T (the factors W_l = Z^(l)T U^(l)
                    of Prop. 2.1 contracted into the canonical sum);
  "optimize the orthogonal subspace in the second variable by calculating the best
  rank-r_2 approximation to the r_1 r_3 x n_2 matrix unfolding of A_2"

so the mode-l update is  Z^(l) <- r_l dominant left singular vectors of the n x r_b r_c
unfolding  M_l = Uhat_l diag(xi') (W_c (.) W_b)^T  (column (b, c) of the Khatri-Rao
product = W_b[b, :] * W_c[c, :]), with W_m = Z^(m)T Uhat_m for the two other modes.

Readings:
  * L1 a sweep updates the modes in the order 1, 2, 3, each with the latest frames of
    the others (the paper spells out mode 2 and says "similar" for the rest; SPEC
    S:194-202 fixes the order); the ranks stay those of the RHOSVD start;
  * L2 the core after the sweeps is the projection beta = A x_l Z^(l)T, computed in the
    Prop. 2.1 form xi' x_l (Z^(l)T Uhat_l) (the same formula as the RHOSVD core);
  * L3 sigma of mode l = the singular values of the LAST unfolding M_l of that mode
    (the RHOSVD sigma are the singular values of Uhat_l); signs as reading A9.

Pinned by tests/test_als_oracle.py: the unfolding identity against the dense tensor
(brute force), the fixed point of an exact Tucker tensor, monotonicity of the error over
frame updates, ALS error <= RHOSVD error, the rank-1 closed form, sweeps = 0.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .rhosvd_oracle import canonical_sign, core_kr, normalize, rhosvd

__all__ = ["ALSResult", "als_unfolding", "c2t_als", "tucker_error2"]


@dataclass
class ALSResult:
    Z: list           # frames n x r_l (orthonormal, sign-fixed)
    beta: np.ndarray  # core r1 x r2 x r3
    sigma: list       # singular values of the last mode-l unfolding (r_l each)
    W: list           # r_l x R CP factors of the core (Z_l^T Uhat_l)
    xip: np.ndarray
    beta_norms: list  # ||beta|| after each frame update (projection norm, non-decreasing)


def als_unfolding(Uh, xip, Zs, l):
    """M_l = Uhat_l diag(xi') (W_c (.) W_b)^T : the mode-l unfolding of
    A x_b Z_b^T x_c Z_c^T (columns ordered (b, c), b the lower other mode).  Uh[m] is (R, n)."""
    b, c = [m for m in range(3) if m != l]
    Wb = Zs[b].T @ Uh[b].T                      # r_b x R
    Wc = Zs[c].T @ Uh[c].T                      # r_c x R
    KR = (Wb[:, None, :] * Wc[None, :, :]).reshape(Wb.shape[0] * Wc.shape[0], -1)
    return (Uh[l].T * xip[None, :]) @ KR.T      # n x (r_b r_c)


def _core(Uh, xip, Zs):
    Ws = [Z.T @ u.T for Z, u in zip(Zs, Uh)]
    return core_kr(Ws[0], Ws[1], Ws[2], xip), Ws


def c2t_als(Us, xi, sweeps, eps=None, ranks=None, start=None):
    """RHOSVD (the paper's initial guess) followed by `sweeps` ALS
    sweeps.  Us: list of (R, n) raw side matrices, xi: (R,).  `start` (optional): an
    oracle RHOSVD result to start from (else computed with eps / ranks)."""
    if sweeps < 0:
        raise ValueError("sweeps must be >= 0")
    o = start if start is not None else rhosvd(Us, xi, eps=eps, ranks=ranks)
    Uh, xip, _, _ = normalize(Us, xi)
    Zs = [z.copy() for z in o.Z]
    sig = [o.sigma[l][:Zs[l].shape[1]].copy() for l in range(3)]
    norms = []
    for _ in range(sweeps):
        for l in range(3):
            r = Zs[l].shape[1]
            M = als_unfolding(Uh, xip, Zs, l)
            u, s, _ = np.linalg.svd(M, full_matrices=False)    # LAPACK gesdd
            Zs[l], _ = canonical_sign(u[:, :r])
            sig[l] = s[:r].copy()
            beta, _ = _core(Uh, xip, Zs)
            norms.append(float(np.linalg.norm(beta)))
    beta, Ws = _core(Uh, xip, Zs)
    return ALSResult(Z=Zs, beta=beta, sigma=sig, W=Ws, xip=xip, beta_norms=norms)


def tucker_error2(A_dense, beta, Zs):
    """||A - beta x_l Z_l||_F^2 by brute force on a dense tensor (tiny grids only)."""
    X = beta
    for l, Z in enumerate(Zs):
        Xm = np.moveaxis(X, l, 0)
        shp = Xm.shape
        X = np.moveaxis((Z @ Xm.reshape(shp[0], -1)).reshape((Z.shape[0],) + shp[1:]), 0, l)
    return float(np.sum((A_dense - X) ** 2))
