"""Pins of the C2T ALS oracle (oracle/als_oracle.py, Eq.
can_A_Tuck_als, Fig. 2) against what the paper and the mathematics fix - no GPU."""
import numpy as np
import pytest

from oracle import dense_from_canonical, hosvd_full, rhosvd as oracle_rhosvd
from oracle.als_oracle import als_unfolding, c2t_als, tucker_error2
from oracle.rhosvd_oracle import normalize


def rand_canonical(n, R, seed, decay=0.0):
    rng = np.random.default_rng(seed)
    Us = [rng.normal(size=(R, n)) for _ in range(3)]
    xi = rng.normal(size=R) * np.exp(-decay * np.arange(R))
    return Us, xi


def proj(Z):
    return Z @ Z.T


def test_unfolding_is_the_dense_contraction():
    """M_l equals the mode-l unfolding of A x_b Z_b^T x_c Z_c^T built from the dense tensor
    (brute force; the (b, c) column order of the Khatri-Rao product)."""
    Us, xi = rand_canonical(7, 11, 1)
    A = dense_from_canonical(Us, xi)
    Uh, xip, _, _ = normalize(Us, xi)
    rng = np.random.default_rng(2)
    Zs = [np.linalg.qr(rng.normal(size=(7, r)))[0] for r in (3, 4, 2)]
    for l in range(3):
        b, c = [m for m in range(3) if m != l]
        X = np.moveaxis(A, l, 0)                      # l, b, c
        Y = np.einsum("ibc,bp,cq->ipq", X, Zs[b], Zs[c])
        M_dense = Y.reshape(7, -1)                    # columns (p, q), q fastest
        assert np.allclose(als_unfolding(Uh, xip, Zs, l), M_dense, atol=1e-12 * np.abs(M_dense).max())


def test_exact_tucker_tensor_is_a_fixed_point():
    """A = C x_l Q_l written as a CP sum (R = r^3 terms, canonical vectors = frame columns):
    one sweep from the RHOSVD start recovers the frames and the error is ~0."""
    rng = np.random.default_rng(3)
    n, r = 9, 3
    Q = [np.linalg.qr(rng.normal(size=(n, r)))[0] for _ in range(3)]
    C = rng.normal(size=(r, r, r))
    idx = [(a, b, c) for a in range(r) for b in range(r) for c in range(r)]
    Us = [np.array([Q[m][:, t[m]] for t in idx]) for m in range(3)]
    xi = np.array([C[t] for t in idx])
    A = dense_from_canonical(Us, xi)
    res = c2t_als(Us, xi, 1, ranks=(r, r, r))
    assert tucker_error2(A, res.beta, res.Z) <= 1e-24 * np.sum(A ** 2)
    for l in range(3):
        assert np.abs(proj(res.Z[l]) - proj(Q[l])).max() <= 1e-12


@pytest.mark.parametrize("seed,ranks", [(4, (3, 4, 3)), (5, (2, 2, 5)), (6, (4, 4, 4))])
def test_error_non_increasing_over_frame_updates(seed, ranks):
    """Each frame update maximises ||A x_l Z_l^T|| over Z_l with the others fixed, so the
    projection norm ||beta|| never decreases and ||A - A_r||^2 = ||A||^2 - ||beta||^2 never
    increases (checked densely after every update)."""
    Us, xi = rand_canonical(10, 30, seed, decay=0.05)
    A = dense_from_canonical(Us, xi)
    o = oracle_rhosvd(Us, xi, ranks=ranks)
    errs = [tucker_error2(A, o.beta, o.Z)]
    Zs = [z.copy() for z in o.Z]
    for sw in range(3):
        res = c2t_als(Us, xi, 1, start=type(o)(**{**o.__dict__, "Z": Zs}))
        Zs = res.Z
        errs.append(tucker_error2(A, res.beta, res.Z))
        nrm = [np.linalg.norm(o.beta)] + res.beta_norms
        assert all(b >= a * (1 - 1e-12) for a, b in zip(nrm, nrm[1:]))
    assert all(b <= a * (1 + 1e-12) + 1e-28 for a, b in zip(errs, errs[1:]))
    # exact identity ||A - A_r||^2 = ||A||^2 - ||beta||^2 (orthogonal projection)
    assert abs(errs[-1] - (np.sum(A ** 2) - np.linalg.norm(res.beta) ** 2)) <= 1e-10 * np.sum(A ** 2)


def test_als_not_worse_than_rhosvd_and_not_better_than_hosvd_bound():
    """Over seeds: ALS(1 sweep) error <= RHOSVD error (the start) - the paper's use of
    RHOSVD as the initial guess."""
    for seed in range(10, 20):
        Us, xi = rand_canonical(8, 10, seed)
        A = dense_from_canonical(Us, xi)
        o = oracle_rhosvd(Us, xi, ranks=(4, 4, 4))
        res = c2t_als(Us, xi, 1, start=o)
        e_r, e_a = tucker_error2(A, o.beta, o.Z), tucker_error2(A, res.beta, res.Z)
        assert e_a <= e_r * (1 + 1e-12) + 1e-28
        # and no better than the best rank-(4,4,4) error lower bound: max_l tail of unfolding
        lb = max(np.sum(np.linalg.svd(np.moveaxis(A, l, 0).reshape(8, -1), compute_uv=False)[4:] ** 2)
                 for l in range(3))
        assert e_a >= lb * (1 - 1e-10)


def test_rank_one_closed_form_and_zero_sweeps():
    rng = np.random.default_rng(21)
    a, b, c = rng.normal(size=6), rng.normal(size=5), rng.normal(size=7)
    Us = [a[None, :], b[None, :], c[None, :]]
    xi = np.array([2.5])
    res = c2t_als(Us, xi, 2, ranks=(1, 1, 1))
    for Z, v in zip(res.Z, (a, b, c)):
        vv = v / np.linalg.norm(v)
        vv = vv if vv[np.argmax(np.abs(vv))] > 0 else -vv
        assert np.allclose(Z[:, 0], vv, atol=1e-14)
    assert np.isclose(abs(res.beta.item()), 2.5 * np.linalg.norm(a) * np.linalg.norm(b) * np.linalg.norm(c),
                      rtol=1e-14)
    # sweeps = 0: the RHOSVD frames and core unchanged
    Us, xi = rand_canonical(8, 12, 22)
    o = oracle_rhosvd(Us, xi, ranks=(3, 3, 3))
    r0 = c2t_als(Us, xi, 0, start=o)
    assert all(np.array_equal(z0, z1) for z0, z1 in zip(r0.Z, o.Z))
    assert np.allclose(r0.beta, o.beta, rtol=0, atol=1e-14 * np.abs(o.beta).max())


def test_sigma_are_unfolding_singular_values_and_hooi_stationary():
    """sigma_l = singular values of the last unfolding; after many sweeps the frames are
    stationary (HOOI fixed point): another sweep moves the projectors by < 1e-9."""
    Us, xi = rand_canonical(9, 25, 23, decay=0.1)
    res = c2t_als(Us, xi, 40, ranks=(3, 3, 3))
    Uh, xip, _, _ = normalize(Us, xi)
    for l in range(3):
        s = np.linalg.svd(als_unfolding(Uh, xip, res.Z, l), compute_uv=False)
        assert np.allclose(res.sigma[l], s[:3], rtol=1e-6)
    o = oracle_rhosvd(Us, xi, ranks=(3, 3, 3))
    more = c2t_als(Us, xi, 41, start=o)
    for l in range(3):
        assert np.abs(proj(more.Z[l]) - proj(res.Z[l])).max() <= 1e-9
    # HOSVD of the dense tensor starts elsewhere but the converged ALS objective is at
    # least the HOSVD projection norm (HOOI improves on HOSVD)
    A = dense_from_canonical(Us, xi)
    core_h, _, _ = hosvd_full(A, (3, 3, 3))
    assert np.linalg.norm(more.beta) >= np.linalg.norm(core_h) * (1 - 1e-12)
