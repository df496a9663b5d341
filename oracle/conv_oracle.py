"""CPU oracle for the 3-D tensor-product convolution of canonical tensors
(SURVEY.md 8(f) row f4).

TEST INFRASTRUCTURE ONLY (same rules as oracle/rhosvd_oracle.py): only tests/,
__graft_entry__.smoke() and bench.py's baseline legs may import it; the product
package never does.

PAPER.md section 3: with a canonical density Theta' (rank R_rho) and a
canonical kernel P_R (rank R_N) on the same n x n x n grid,
    V = Theta' * P_R = sum_m sum_q c_m (u_m^(1) * p_q^(1)) (x) (u_m^(2) * p_q^(2))
                                        (x) (u_m^(3) * p_q^(3)),
"a sum of tensor products of 1D convolutions" (separability of the convolution of
separable functions).  The output is a canonical tensor of rank R_rho R_N.

Readings:
  * C1 the 1-D convolution is the Riemann-sum quadrature of the continuous one on the
    common grid x_i = x_0 + i h:  (u * p)_i = h sum_j u_j p_{i + s - j},  s = floor(n/2),
    p_k = 0 outside 0..n-1 (the central n samples of the full discrete convolution;
    SPEC S:489-496 fixes the same: an impulse at the centre returns h p);
  * C2 output term (m, q) is column m R_N + q of each factor, weight c_m w_q (the kernel's
    CP weights w_q; 1 when the kernel carries its weights in the factors);
  * C3 the three modes share n and h (cubic grid, as in the paper).

Pinned by tests/test_conv_oracle.py: impulse identity, commutativity, box * box = hat
(closed form), Gaussian * Gaussian = Gaussian with summed variances (analytic), and the
separability identity against a brute-force dense 3-D convolution on a tiny grid.
"""
from __future__ import annotations

import numpy as np

__all__ = ["conv1d", "conv3d_canonical", "dense_conv3d"]


def conv1d(u, p, h):
    """(u * p)_i = h sum_j u_j p_{i + s - j}, s = n // 2 (reading C1)."""
    n = u.shape[0]
    if p.shape[0] != n:
        raise ValueError("length mismatch")
    s = n // 2
    full = np.convolve(u, p)              # full[k] = sum_j u_j p_{k - j}, k = 0..2n-2
    return h * full[s:s + n]


def conv3d_canonical(Fa, ca, Fp, cp, h):
    """Theta' * P: Fa[l] (n x R_a) factors and ca (R_a) weights of the density; Fp[l]
    (n x R_p), cp (R_p) of the kernel.  Returns (F[l] (n x R_a R_p), w (R_a R_p)) with
    column m R_p + q = u_m^(l) * p_q^(l) and w = c_m w_q (reading C2)."""
    Ra, Rp = Fa[0].shape[1], Fp[0].shape[1]
    F = []
    for l in range(3):
        n = Fa[l].shape[0]
        out = np.zeros((n, Ra * Rp))
        for m in range(Ra):
            for q in range(Rp):
                out[:, m * Rp + q] = conv1d(Fa[l][:, m], Fp[l][:, q], h)
        F.append(out)
    w = (ca[:, None] * cp[None, :]).reshape(-1)
    return F, w


def dense_conv3d(A, P, h):
    """Brute force: V[i,j,k] = h^3 sum_{a,b,c} A[a,b,c] P[i+s-a, j+s-b, k+s-c] (tiny grids)."""
    n = A.shape[0]
    s = n // 2
    V = np.zeros_like(A)
    for a in range(n):
        for b in range(n):
            for c in range(n):
                if A[a, b, c] == 0.0:
                    continue
                # P index i + s - a for output i: valid for 0 <= i + s - a < n
                i0, i1 = max(0, a - s), min(n, n + a - s)
                j0, j1 = max(0, b - s), min(n, n + b - s)
                k0, k1 = max(0, c - s), min(n, n + c - s)
                V[i0:i1, j0:j1, k0:k1] += A[a, b, c] * P[i0 + s - a:i1 + s - a, j0 + s - b:j1 + s - b,
                                                         k0 + s - c:k1 + s - c]
    return h ** 3 * V
