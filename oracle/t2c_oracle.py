"""CPU oracle for the Tucker-to-canonical (T2C) step that completes the canonical
rank reduction C2C = T2C o C2T.

TEST INFRASTRUCTURE ONLY (same rules as oracle/rhosvd_oracle.py): only tests/,
__graft_entry__.smoke() and bench.py's baseline legs may import it; the product
package never does.

Plain fp64 NumPy/LAPACK, following PAPER.md section 2.3 (Remark 2.1)
in its order and notation:

  (T2C_slice)  beta = sum_{m=1}^{r} B_m (x) z_m,   z_m the m-th unit vector
  p_m = minimal p with sigma_k^(m) <= eps / r^{3/2} for k = p+1..r
  B_{p_m} = sum_{k<=p_m} sigma_k^(m) u_k (x) v_k   (truncated SVD)
  (beta_R)     beta_(R) = sum_m B_{p_m} (x) z_m,   R = p_1 + ... + p_r <= r^2
  ||beta - beta_(R)|| <= sum_m ||B_m - B_{p_m}|| <= eps

The canonical output of C2C lifts the core's CP factors through the Tucker frames
(Lemma 2.1; mixed format PAPER.md:531-545):
  A ~ sum_m sum_{k<=p_m} sigma_k^(m) (Z_1 u_k) (x) (Z_2 v_k) (x) (Z_3 e_m).

Readings:
  * T1 slices are taken in mode 3 (the paper: "in each fixed mode", any of the d
    decompositions is allowed; mode 3 is the contiguous one in C order).
  * T2 the core is r1 x r2 x r3 (not cubic): r3 slices of size r1 x r2 with
    q = min(r1, r2) singular values each; the threshold that keeps the paper's proof
    (sum_m sqrt(q thr^2) <= eps) is thr = eps / (r3 sqrt(q)), which is eps / r^{3/2}
    for the cubic core.
  * T3 eps is absolute, as in the paper (||beta - beta_(R)|| <= eps); the ABI takes
    eps_rel and uses eps = eps_rel ||beta||_F.
  * T4 singular values are compared with "<= thr" exactly as printed (a value equal
    to thr is dropped); the signs of (u_k, v_k) are fixed so that the largest-|.|
    entry of u_k is positive (lowest index on ties).

Pinned by tests/test_t2c_oracle.py: the exact error identity (slices are orthogonal
in mode 3, so ||beta - beta_(R)||^2 = sum_m sum_{k>p_m} sigma_k^2), the paper's bound,
the rank bound, exact reconstruction as eps -> 0, closed-form rank-1 and
diagonal cores, and brute-force dense reconstruction of the lifted tensor.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["T2CResult", "t2c_threshold", "t2c", "t2c_dense", "c2c_lift", "dense_from_cp"]


@dataclass
class T2CResult:
    U: np.ndarray        # r1 x R  left factors u_k (unit columns)
    V: np.ndarray        # r2 x R  right factors v_k (unit columns)
    slice_of: np.ndarray  # R      slice index m of each term (mode-3 unit vector z_m)
    sigma: np.ndarray    # R      weights sigma_k^(m)
    p: np.ndarray        # r3     kept count per slice
    thr: float
    eps: float
    err2: float          # sum of the discarded sigma^2 = ||beta - beta_(R)||^2 (exact)
    near_tie: bool       # some sigma within 1e-8 (relative) of thr


def t2c_threshold(eps, shape):
    """thr = eps / (r3 sqrt(min(r1, r2)))  (reading T2)."""
    r1, r2, r3 = shape
    q = min(r1, r2)
    return eps / (r3 * math.sqrt(q)) if r3 > 0 and q > 0 else 0.0


def t2c(beta, eps):
    """Remark 2.1: canonical approximation of the core beta (r1 x r2 x r3) within eps."""
    r1, r2, r3 = beta.shape
    thr = t2c_threshold(eps, beta.shape)
    Us, Vs, sl, sg, ps = [], [], [], [], []
    err2 = 0.0
    tie = False
    for m in range(r3):
        Bm = beta[:, :, m]                                  # B_m (T2C_slice)
        u, s, vt = np.linalg.svd(Bm, full_matrices=False)   # LAPACK gesdd
        keep = s > thr                                      # sigma_k <= thr dropped (T4)
        # p_m = minimal p with sigma_k <= thr for all k > p (s is descending)
        p = int(np.max(np.nonzero(keep)[0]) + 1) if np.any(keep) else 0
        tie |= bool(np.any(np.abs(s - thr) <= 1e-8 * max(thr, 1e-300)))
        err2 += float(np.sum(s[p:] ** 2))
        for k in range(p):
            uk, vk = u[:, k], vt[k, :]
            i = int(np.argmax(np.abs(uk)))
            if uk[i] < 0:
                uk, vk = -uk, -vk
            Us.append(uk)
            Vs.append(vk)
            sl.append(m)
            sg.append(s[k])
        ps.append(p)
    R = len(sg)
    return T2CResult(U=np.array(Us).T.reshape(r1, R), V=np.array(Vs).T.reshape(r2, R),
                     slice_of=np.array(sl, dtype=np.int64), sigma=np.array(sg), p=np.array(ps),
                     thr=thr, eps=eps, err2=err2, near_tie=tie)


def t2c_dense(res: T2CResult, shape):
    """beta_(R) = sum_m B_{p_m} (x) z_m  (Eq. beta_R) as a dense r1 x r2 x r3 array."""
    out = np.zeros(shape)
    for j in range(res.sigma.shape[0]):
        out[:, :, res.slice_of[j]] += res.sigma[j] * np.outer(res.U[:, j], res.V[:, j])
    return out


def c2c_lift(res: T2CResult, Zs):
    """Canonical factors of the lifted tensor: (Z1 U, Z2 V, Z3[:, slice]), weights sigma."""
    F1 = Zs[0] @ res.U
    F2 = Zs[1] @ res.V
    F3 = Zs[2][:, res.slice_of]
    return F1, F2, F3, res.sigma.copy()


def dense_from_cp(F1, F2, F3, w):
    """sum_j w_j F1[:,j] (x) F2[:,j] (x) F3[:,j] (brute force, tiny sizes only)."""
    return np.einsum("j,aj,bj,cj->abc", w, F1, F2, F3, optimize=True)
