"""CPU oracle for the RHOSVD canonical-to-Tucker (C2T) hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import or call anything under
oracle/.  The product path (paper_2201_12663_b200/) never imports it and shares
no code with it; the two meet only at the seeded generators in workloads/.

Plain, slow, obviously-correct fp64 NumPy/LAPACK implementation of the
definition, following PAPER.md section 2.1 in the paper's order and notation:

  (can_A3)   A = sum_nu xi_nu u_nu^(1) (x) u_nu^(2) (x) u_nu^(3) with
             normalized canonical vectors ||u_nu^(l)|| = 1
  (SVD_Ul)   U^(l) = Z^(l) D_l V^(l)^T
  (svdr)     rank-r_l truncated SVD, Z_0^(l) = first r_l left
             singular vectors, D_{l,0} = leading sigma
  Def. 2.1   A_(r)^0 = (xi x_l [D_{l,0} V_0^(l)^T]) x_l Z_0^(l)
  Prop. 2.1  core beta_0 = xi x_l U_0^(l)^T with U_0^(l)^T = D_{l,0} V_0^(l)^T
             = Z_0^(l)^T U^(l)  (rank-R CP core)
  Thm. 2.2   ||A - A_(r)^0|| <= ||xi|| sum_l (sum_{k>r_l} sigma_{l,k}^2)^{1/2}
                                                              

Where the paper is silent the oracle takes SURVEY.md 8(c)'s readings, listed in
DESIGN.md: A1 (relative Frobenius tail rule for epsilon), A2 (normalisation
absorbed into xi), A3 (zero columns stay zero, xi' = 0), A4 (R < n allowed),
A9 (canonical sign: largest-|.| entry of each frame column positive, lowest
row index on ties), A12 (the tighter bound ||xi|| (sum_l tail_l^2)^{1/2} is
reported beside the paper's), A17 (fixed r clamped to min(n, R)).

Pinned by tests/test_oracle_pins.py: closed forms,
exact identities, the paper's theorem and corollary, brute force against a
dense n^3 tensor and a full HOSVD on tiny grids, and an independent LAPACK
route.  Every function below is pinned; none is "parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "normalize", "mode_svd", "select_rank", "canonical_sign", "project",
    "core_kr", "rhosvd", "OracleResult", "dense_from_canonical",
    "dense_from_tucker", "mode_product", "hosvd_full", "exact_error_telescoped",
    "error_bounds",
]


# --------------------------------------------------------------------------
# O2  normalisation ("normalized canonical vectors"; reading A2/A3)
# --------------------------------------------------------------------------
def normalize(Us, xi):
    """Normalize the canonical vectors; absorb the norms into the weights.

    Us: list of d arrays of shape (R, n) (row k = u_k^(l)); xi: (R,).
    Returns (Uhat list, xi' (R,), s (d, R) column norms, T (d,) = ||Uhat_l||_F^2).
    Zero columns stay zero and get xi'_k = 0 (reading A3).  The 2-norm is evaluated
    as m ||u / m||_2 with m = max_i |u_i| (the plain definition without the underflow
    of sum u_i^2: a column with entries ~1e-200 is NOT zero).
    """
    d = len(Us)
    R = xi.shape[0]
    s = np.zeros((d, R))
    Uh = []
    for l, U in enumerate(Us):
        mx = np.max(np.abs(U), axis=1) if U.shape[1] else np.zeros(U.shape[0])
        safe = np.where(mx > 0, mx, 1.0)
        Us_ = U / safe[:, None]                     # entries in [-1, 1]
        nr = np.linalg.norm(Us_, axis=1)
        sl = np.where(mx > 0, mx * nr, 0.0)         # ||u_k^(l)||_2
        s[l] = sl
        inv = np.where(mx > 0, 1.0 / np.where(nr > 0, nr, 1.0), 0.0)
        Uh.append(Us_ * inv[:, None])
    xip = xi * np.prod(s, axis=0)                  # xi'_k = xi_k prod_l s_{l,k}
    T = np.array([np.sum(u * u) for u in Uh])      # T_l (reading A19)
    return Uh, xip, s, T


# --------------------------------------------------------------------------
# O3  SVD of the side matrices (Eq. SVD_Ul)
# --------------------------------------------------------------------------
def mode_svd(Uh):
    """Left singular vectors and singular values of the n x R side matrix.

    Uh: (R, n) array = column-major n x R matrix Uhat^(l).
    If R >= n: R-factor of QR(Uhat^T) (n x n), then SVD of its transpose -
    the textbook QR-first SVD of a wide matrix (avoids the n x R right factor).
    If R < n: SVD of Uhat directly (reading A4).
    Returns (Z (n x min(n,R)), sigma (min(n,R),) descending).
    """
    R, n = Uh.shape
    M = Uh.T                                        # n x R
    if R >= n:
        Rf = np.linalg.qr(M.T, mode="r")            # M^T = Q Rf, Rf n x n
        Z, sig, _ = np.linalg.svd(Rf.T)             # M = Rf^T Q^T
    else:
        Z, sig, _ = np.linalg.svd(M, full_matrices=False)
    return Z, sig


# --------------------------------------------------------------------------
# O4  rank selection (reading A1 relative tail rule)
# --------------------------------------------------------------------------
def select_rank(sigma, T, eps=None, r_fixed=None):
    """r = min{r >= 1 : sum_{k>r} sigma_k^2 <= eps^2 T} (eps mode), or
    min(r_fixed, len(sigma)) (fixed mode, reading A17).

    Tails are summed smallest-first.  Returns (r, tail2 array over r=0..m,
    margins (m_l, m'_l)) with m_l = tail(r)/(eps^2 T) - 1 <= 0 and
    m'_l = tail(r-1)/(eps^2 T) - 1 > 0 (None in fixed mode).
    """
    m = sigma.shape[0]
    sq = sigma.astype(np.float64) ** 2
    tail2 = np.zeros(m + 1)                         # tail2[r] = sum_{k>r} sigma_k^2
    acc = 0.0
    for r in range(m - 1, -1, -1):                  # smallest-first summation
        acc += sq[r]
        tail2[r] = acc
    if m == 0:
        return 0, tail2, (None, None)
    if r_fixed is not None:
        return int(min(r_fixed, m)), tail2, (None, None)
    thr = eps * eps * T
    r = m
    for cand in range(1, m + 1):
        if tail2[cand] <= thr:
            r = cand
            break
    mar = tail2[r] / thr - 1.0 if thr > 0 else None
    marp = tail2[r - 1] / thr - 1.0 if thr > 0 and r >= 1 else None
    return r, tail2, (mar, marp)


def canonical_sign(Z):
    """Make the largest-|.| entry of each column positive (lowest row on ties).
    Returns (Z signed, sign vector).  Reading A9 - for determinism only."""
    if Z.shape[1] == 0:
        return Z.copy(), np.ones(0)
    idx = np.argmax(np.abs(Z), axis=0)              # argmax returns the first max
    sgn = np.sign(Z[idx, np.arange(Z.shape[1])])
    sgn[sgn == 0] = 1.0
    return Z * sgn[None, :], sgn


# --------------------------------------------------------------------------
# O6  projection  U_0^(l)^T = Z_0^(l)^T Uhat^(l)
# --------------------------------------------------------------------------
def project(Z, Uh):
    """W^(l) = Z^T Uhat (r x R).  Uh is (R, n)."""
    return Z.T @ Uh.T


# --------------------------------------------------------------------------
# O7  core (Prop. 2.1; Def. 2.1 second line)
# --------------------------------------------------------------------------
def core_kr(W1, W2, W3, xip, chunk=None):
    """beta[a,b,c] = sum_k xi'_k W1[a,k] W2[b,k] W3[c,k], summed over R-chunks.

    Each chunk evaluates the Khatri-Rao block KR(W1, W2)[:, chunk] explicitly
    and multiplies it by (xi' o W3)[:, chunk]^T (one LAPACK/BLAS GEMM).
    Returns beta (r1, r2, r3), C order.
    """
    r1, R = W1.shape
    r2, r3 = W2.shape[0], W3.shape[0]
    beta = np.zeros((r1 * r2, r3))
    if chunk is None:
        # keep the explicit KR block <= ~256 MB
        chunk = max(1, min(R, (1 << 25) // max(1, r1 * r2)))
    for s in range(0, R, chunk):
        e = min(R, s + chunk)
        KR = (W1[:, None, s:e] * W2[None, :, s:e]).reshape(r1 * r2, e - s)
        beta += KR @ (xip[None, s:e] * W3[:, s:e]).T
    return beta.reshape(r1, r2, r3)


def error_bounds(xip, tails):
    """Thm. 2.2 and the tighter orthogonal-sum form (A12).

    tails[l] = (sum_{k>r_l} sigma_{l,k}^2)^{1/2}.
    Returns (bound_paper, bound_ns)."""
    xn = float(np.linalg.norm(xip))
    return xn * float(np.sum(tails)), xn * float(math.sqrt(np.sum(np.asarray(tails) ** 2)))


@dataclass
class OracleResult:
    Z: list            # frames n x r_l, orthonormal, sign-fixed
    beta: np.ndarray   # core r1 x r2 x r3
    sigma: list        # FULL spectrum per mode (descending)
    ranks: tuple
    W: list            # r_l x R CP factors of the core (Prop. 2.1)
    xip: np.ndarray
    T: np.ndarray
    tails: np.ndarray  # (sum_{k>r_l} sigma^2)^{1/2} per mode
    margins: list      # (m_l, m'_l) per mode
    report: dict = field(default_factory=dict)


def rhosvd(Us, xi, eps=None, ranks=None, with_W=True, with_core=True, timings=None):
    """RHOSVD canonical-to-Tucker transform (O1-O8), d = len(Us) (3 here).

    Us: list of (R, n_l) arrays (raw, unnormalized); xi: (R,).
    Exactly one of eps (relative tail rule A1) or ranks (fixed) is given.
    with_core=False stops after O6 (frames, sigma, ranks, W; beta = None): the
    Tucker tensor is then fixed by the frames through Def. 2.1, and the full-size
    parity fixtures need only those.
    timings: optional dict; receives the wall seconds of each step (normalize, svd,
    rank_frames, projection, core) for the CPU baseline report.  No effect on results.
    """
    import time
    clock = time.perf_counter
    tm = timings if timings is not None else {}
    for key in ("normalize", "svd", "rank_frames", "projection", "core"):
        tm[key] = 0.0
    t0 = clock()
    d = len(Us)
    if (eps is None) == (ranks is None):
        raise ValueError("give exactly one of eps or ranks")
    if eps is not None and not (0.0 < eps < 1.0):
        raise ValueError("eps must lie in (0, 1)")
    R = xi.shape[0]
    Uh, xip, s, T = normalize(Us, xi)
    tm["normalize"] += clock() - t0
    Zs, sig, rs, tails, margins, Ws = [], [], [], [], [], []
    for l in range(d):
        n = Uh[l].shape[1]
        if R == 0:
            Z_full, sg = np.zeros((n, 0)), np.zeros(0)
        else:
            t0 = clock()
            Z_full, sg = mode_svd(Uh[l])
            tm["svd"] += clock() - t0
        t0 = clock()
        r, tail2, mar = select_rank(sg, T[l], eps=eps,
                                    r_fixed=None if ranks is None else ranks[l])
        Z, _ = canonical_sign(Z_full[:, :r])
        Zs.append(Z)
        sig.append(sg)
        rs.append(r)
        tails.append(math.sqrt(max(tail2[r], 0.0)) if sg.shape[0] else 0.0)
        margins.append(mar)
        tm["rank_frames"] += clock() - t0
        t0 = clock()
        Ws.append(project(Z, Uh[l]))
        tm["projection"] += clock() - t0
    if not with_core:
        beta = None
    elif d == 3:
        t0 = clock()
        beta = core_kr(Ws[0], Ws[1], Ws[2], xip)
        tm["core"] += clock() - t0
    else:
        raise NotImplementedError("hot path is d = 3")
    bp, bns = error_bounds(xip, tails)
    rep = dict(
        ranks=list(rs), trace=[float(t) for t in T], tail=[float(t) for t in tails],
        xi_norm=float(np.linalg.norm(xip)), bound_paper=bp, bound_ns=bns,
        beta_norm=None if beta is None else float(np.linalg.norm(beta)),
        margins=[[None if v is None else float(v) for v in m] for m in margins],
        near_tie=[bool(m[0] is not None and (abs(m[0]) < 1e-6 or abs(m[1]) < 1e-6)) for m in margins],
    )
    return OracleResult(Z=Zs, beta=beta, sigma=sig, ranks=tuple(rs),
                        W=Ws if with_W else None, xip=xip, T=T,
                        tails=np.array(tails), margins=margins, report=rep)


# --------------------------------------------------------------------------
# Dense helpers for tiny grids (brute force pins P1, P8, P9, P10)
# --------------------------------------------------------------------------
def dense_from_canonical(Us, xi):
    """A[i,j,k] = sum_nu xi_nu u1[nu,i] u2[nu,j] u3[nu,k] (Eq. can_A3)."""
    return np.einsum("r,ri,rj,rk->ijk", xi, Us[0], Us[1], Us[2], optimize=True)


def mode_product(X, M, mode):
    """X x_mode M : contract tensor index `mode` with the columns of M."""
    Xm = np.moveaxis(X, mode, 0)
    shp = Xm.shape
    Y = (M @ Xm.reshape(shp[0], -1)).reshape((M.shape[0],) + shp[1:])
    return np.moveaxis(Y, 0, mode)


def dense_from_tucker(beta, Zs):
    """beta x_1 Z1 x_2 Z2 x_3 Z3."""
    X = beta
    for l, Z in enumerate(Zs):
        X = mode_product(X, Z, l)
    return X


def hosvd_full(A, ranks):
    """Truncated HOSVD of a dense tensor: frames = dominant left singular
    vectors of the mode unfoldings; core = projection (test oracle only)."""
    Zs, sigs = [], []
    for l in range(A.ndim):
        Al = np.moveaxis(A, l, 0).reshape(A.shape[l], -1)
        Z, sg, _ = np.linalg.svd(Al, full_matrices=False)
        Zs.append(Z[:, :ranks[l]])
        sigs.append(sg)
    core = A
    for l, Z in enumerate(Zs):
        core = mode_product(core, Z.T, l)
    return core, Zs, sigs


def exact_error_telescoped(Uh, xip, Zs):
    """Exact ||A - A_(r)^0||_F without forming n^3 (pin P6).

    ||A - A0||^2 = sum_l ||B_l||^2 (the telescoping terms of the proof of
    Thm. 2.2, are mutually orthogonal, reading A12) with
    B_l = xi' x_{m<l} Uhat_m x_l E_l x_{m>l} P_m Uhat_m, E_l = (I - P_l) Uhat_l,
    P_m = Z_m Z_m^T.  ||B_l||^2 = xi'^T [ (o_{m<l} Uhat_m^T Uhat_m)
    o (E_l^T E_l) o (o_{m>l} W_m^T W_m) ] xi', W_m = Z_m^T Uhat_m.
    Cost O(R^2 (n + r)) - only for R <= ~8000.
    """
    d = len(Uh)
    M = [u.T for u in Uh]                              # n x R
    Ws = [Z.T @ m for Z, m in zip(Zs, M)]
    tot = 0.0
    for l in range(d):
        H = np.ones((xip.shape[0], xip.shape[0]))
        for m in range(l):
            H *= M[m].T @ M[m]
        E = M[l] - Zs[l] @ Ws[l]
        H *= E.T @ E
        for m in range(l + 1, d):
            H *= Ws[m].T @ Ws[m]
        tot += float(xip @ H @ xip)
    return math.sqrt(max(tot, 0.0))
