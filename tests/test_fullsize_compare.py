"""Pins for tests/fullsize_compare.tucker_diff_cp (CPU torch, no GPU): it must agree with
the explicit-core comparison oracle.compare.tucker_diff and with a dense
n^3 difference on tiny grids, and give ||T|| = ||beta||_F of the oracle's core."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import dense_from_tucker, rhosvd, tucker_diff  # noqa: E402
from workloads import make_config, make_random_params  # noqa: E402

from fullsize_compare import tucker_diff_cp  # noqa: E402


def _case(n, R, seed, ranks):
    p = make_random_params(n, R, seed=seed, ranks=ranks)
    U1, U2, U3, xi = make_config(p)
    return rhosvd([U1, U2, U3], xi, ranks=ranks)


@pytest.mark.parametrize("n,R,seed", [(12, 30, 1), (20, 90, 2), (33, 150, 3)])
def test_matches_explicit_core_comparison(n, R, seed):
    o = _case(n, R, seed, (5, 6, 4))
    h = _case(n, R, seed, (4, 6, 5))        # a different Tucker tensor of the same A
    d_ref, n_ref = tucker_diff(h.beta, h.Z, o.beta, o.Z)
    d, nrm = tucker_diff_cp(h.beta, h.Z, o.Z, o.W, o.xip, chunk_bytes=1 << 12)  # many k-chunks
    assert d_ref > 1e-6 * n_ref              # the two tensors really differ
    assert abs(d - d_ref) <= 1e-12 * n_ref
    assert abs(nrm - np.linalg.norm(o.beta)) <= 1e-13 * nrm
    if n <= 20:  # dense n^3 check of the same number
        dd = np.linalg.norm(dense_from_tucker(h.beta, h.Z) - dense_from_tucker(o.beta, o.Z))
        assert abs(d - dd) <= 1e-12 * n_ref


def test_identical_tensors_give_zero_and_rotation_invariance():
    o = _case(24, 100, 7, (6, 5, 7))
    d, nrm = tucker_diff_cp(o.beta, o.Z, o.Z, o.W, o.xip)
    assert d <= 1e-13 * nrm
    # the same Tucker tensor in rotated / sign-flipped frames: Z Q, beta x_l Q^T
    rng = np.random.default_rng(0)
    Qs = [np.linalg.qr(rng.normal(size=(z.shape[1], z.shape[1])))[0] for z in o.Z]
    Zr = [z @ q for z, q in zip(o.Z, Qs)]
    b = o.beta
    b = np.einsum("abc,ai,bj,ck->ijk", b, Qs[0], Qs[1], Qs[2])
    d2, _ = tucker_diff_cp(b, Zr, o.Z, o.W, o.xip)
    assert d2 <= 1e-13 * nrm


def test_a_perturbed_core_entry_is_seen():
    o = _case(16, 60, 9, (4, 4, 4))
    b = o.beta.copy()
    b[1, 2, 3] += 1e-7 * np.linalg.norm(b)
    d, nrm = tucker_diff_cp(b, o.Z, o.Z, o.W, o.xip)
    assert abs(d - 1e-7 * nrm) <= 1e-12 * nrm
