"""Full-size Tucker-tensor comparison for the parity tests (TEST INFRASTRUCTURE ONLY).

The oracle's Tucker tensor of Def. 2.1 is fixed by its frames:
with W_l = Z_l^T Uhat_l (the oracle's projection, O6) and xi' (its normalisation, O2),

    T = beta x_1 Z_1 x_2 Z_2 x_3 Z_3,   beta = sum_k xi'_k W1[:,k] (x) W2[:,k] (x) W3[:,k]
                                                                  (Prop. 2.1).

SURVEY.md 8(c)'s cancellation-free comparison takes the thin QR [Zhat_l, Z_l] = Q_l
[Mhat_l, M_l] and compares D = betahat x_l Mhat_l - beta x_l M_l (an isometric image of
That - T).  Here beta x_l M_l is evaluated directly from the oracle's CP factors,

    beta x_l M_l = sum_k xi'_k (M_1 W1[:,k]) (x) (M_2 W2[:,k]) (x) (M_3 W3[:,k]),

i.e. a Khatri-Rao contraction in the (r_hat + r)^3 comparison basis, so the oracle's
dense core (2.2 GB on cfg 4, three hours of host BLAS) is never needed.  This is the
"(2r)^3 core products in torch fp64 on one GPU inside the test harness" of SURVEY.md
8(c); the CUDA library under test is not used.  The same code runs on CPU torch, where
tests/test_fullsize_compare.py pins it against oracle.compare.tucker_diff (explicit dense
oracle core) on small cases.
"""
from __future__ import annotations

import math


def tucker_diff_cp(beta_hat, Z_hat, Z, W, xip, device="cpu", chunk_bytes=4 << 30):
    """Return (||That - T||_F, ||T||_F).

    beta_hat : torch (r1', r2', r3') core under test;  Z_hat : 3 torch (n, r_l') frames
    Z        : 3 (n, r_l) oracle frames;  W : 3 (r_l, R) oracle CP factors Z_l^T Uhat_l
    xip      : (R,) oracle weights xi'.   Arrays may be numpy or torch; all work in fp64
    on `device`.
    """
    import torch

    f64 = torch.float64

    def t(x):
        return torch.as_tensor(x, dtype=f64).to(device)

    Mh, M = [], []
    for zh, z in zip(Z_hat, Z):
        zh, z = t(zh), t(z)
        _, Rm = torch.linalg.qr(torch.cat([zh, z], dim=1), mode="reduced")
        Mh.append(Rm[:, :zh.shape[1]])
        M.append(Rm[:, zh.shape[1]:])
    # Xhat = beta_hat x_1 Mh1 x_2 Mh2 x_3 Mh3   (mode 3, 2, 1 in turn)
    X = t(beta_hat)
    X = torch.tensordot(X, Mh[2], dims=([2], [1]))                    # (r1', r2', q3)
    X = torch.tensordot(X, Mh[1], dims=([1], [1])).permute(0, 2, 1)    # (r1', q2, q3)
    X = torch.tensordot(Mh[0], X, dims=([1], [0]))                    # (q1, q2, q3)
    X = X.contiguous()
    q1, q2, q3 = X.shape
    # subtract sum_k xi'_k y1_k (x) y2_k (x) y3_k,  y_l = M_l W_l, chunked over k
    Y = [M[l] @ t(W[l]) for l in range(3)]                            # (q_l, R)
    x = t(xip)
    R = x.shape[0]
    kc = max(1, min(R, int(chunk_bytes // (8 * q1 * q2))))
    Xf = X.view(q1 * q2, q3)
    Tn2 = 0.0
    for s in range(0, R, kc):
        e = min(R, s + kc)
        KR = (Y[0][:, None, s:e] * Y[1][None, :, s:e]).reshape(q1 * q2, e - s)
        Xf.addmm_(KR, (x[s:e, None] * Y[2][:, s:e].T), alpha=-1.0)
        del KR
    d = float(torch.linalg.vector_norm(Xf))
    # ||T|| = ||beta x_l M_l|| (Q_l orthonormal): rebuild from the CP factors in norm form
    # ||T||^2 = xi'^T [(Y1^T Y1) o (Y2^T Y2) o (Y3^T Y3)] xi', chunked over column blocks
    for s in range(0, R, kc):
        e = min(R, s + kc)
        H = (Y[0].T @ Y[0][:, s:e]) * (Y[1].T @ Y[1][:, s:e]) * (Y[2].T @ Y[2][:, s:e])
        Tn2 += float(x @ (H @ x[s:e]))
    return d, math.sqrt(max(Tn2, 0.0))
