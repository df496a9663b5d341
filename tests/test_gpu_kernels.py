"""Kernel-level parity on the GPU (through the C ABI): DMMA GEMM engine, Gram,
Jacobi eigensolver, Khatri-Rao core - each against NumPy/LAPACK fp64 (or the
oracle's own core routine) on identical seeded inputs, at sizes spanning
several tiles and ragged tails."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rh():
    from paper_2201_12663_b200 import rhosvd
    rhosvd.lib()
    return rhosvd


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


# (1000, 730, 2048), (147, 3000, 2048), (3000, 147, 2500), (200, 300, 5000): 128-tiles plus a
# narrower column-edge launch where the wave model takes it, with and without split-K
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (64, 64, 16), (130, 67, 301), (200, 300, 5000),
                                   (513, 129, 1000), (31, 33, 20000), (1000, 730, 2048), (147, 3000, 2048),
                                   (3000, 147, 2500)])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_dgemm(rh, M, N, K, ta, tb):
    rng = np.random.default_rng(M * 7 + N * 13 + K)
    A = rng.normal(size=(K, M) if ta else (M, K))
    B = rng.normal(size=(N, K) if tb else (K, N))
    C = rh.dgemm(dev(A), dev(B), transa=ta, transb=tb).cpu().numpy()
    ref = (A.T if ta else A) @ (B.T if tb else B)
    scale = np.sqrt(K) * 8
    assert np.max(np.abs(C - ref)) <= 1e-14 * scale * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("n,R", [(1, 5), (37, 200), (64, 1000), (130, 3001), (512, 2400), (1000, 7)])
def test_gram(rh, n, R):
    rng = np.random.default_rng(n + R)
    U = rng.normal(size=(R, n))
    G = rh.gram(dev(U)).cpu().numpy()
    ref = U.T @ U
    assert np.max(np.abs(G - ref)) <= 1e-14 * np.sqrt(R) * 8 * np.max(np.abs(ref))
    assert np.array_equal(G, G.T)  # mirrored exactly


def test_gram_deterministic(rh):
    rng = np.random.default_rng(3)
    U = dev(rng.normal(size=(20000, 300)))
    G1 = rh.gram(U)
    G2 = rh.gram(U)
    assert torch.equal(G1, G2)


@pytest.mark.parametrize("b", [1, 2, 3, 16, 33, 97, 150, 161, 300, 707])
def test_syevj_random(rh, b):
    rng = np.random.default_rng(b)
    A = rng.normal(size=(b, b))
    A = A + A.T
    lam, V, sw = rh.syevj(dev(A))
    lam = lam.cpu().numpy()
    V = V.cpu().numpy()
    ref = np.linalg.eigvalsh(A)[::-1]
    nrm = np.max(np.abs(ref))
    assert sw > 0
    assert np.max(np.abs(lam - ref)) <= 1e-13 * b * nrm
    assert np.all(np.diff(lam) <= 0)
    assert np.max(np.abs(V.T @ V - np.eye(b))) <= 1e-13 * b
    assert np.max(np.abs(A @ V - V * lam[None, :])) <= 1e-13 * b * nrm


@pytest.mark.parametrize("b", [20, 130, 400, 715])
def test_syevj_graded_high_relative_accuracy(rh, b):
    """D A D with A well conditioned, D graded over 12 decades: Jacobi with the
    relative stopping rule resolves even the smallest eigenvalues to high
    relative accuracy (the property the one-sided Rayleigh-Ritz relies on).
    Reference: squared singular values of (D L)^T = L^T D (L = chol(A)) from
    LAPACK dgejsv (preconditioned one-sided Jacobi SVD, high relative accuracy
    for column-scaled well-conditioned matrices)."""
    rng = np.random.default_rng(b)
    E = rng.normal(size=(b, b)) * 0.01
    A = np.eye(b) + E + E.T
    d = np.logspace(0, -6, b)
    H = d[:, None] * A * d[None, :]
    lam, V, sw = rh.syevj(dev(H))
    lam = lam.cpu().numpy()
    import scipy.linalg.lapack as lapack
    L = np.linalg.cholesky(A)
    sva, _, _, work, _, info = lapack.dgejsv((d[:, None] * L).T)  # column-graded: dgejsv is accurate
    assert info == 0
    ref = np.sort((sva * (work[0] / work[1])) ** 2)[::-1]
    assert np.max(np.abs(lam - ref) / ref) < 1e-11


@pytest.mark.parametrize("b,band", [(300, 40), (715, 90), (400, 3)])
def test_syevj_graded_banded(rh, b, band):
    """The block Jacobi's banded pre-phase (csrc/small_dense.cu): couplings confined to
    |i - j| <= band, as in the Rayleigh-Ritz matrices W W^T of the pipeline, so the band
    sweeps run before the round-robin sweeps (no coupling beyond D ~ b/96 blocks).  Same
    high-relative-accuracy reference as the dense graded case; the result must not depend on
    the schedule (RHOSVD_JAC_BAND=0 is covered by the subprocess below)."""
    rng = np.random.default_rng(b + band)
    E = rng.normal(size=(b, b)) * 0.03
    i, j = np.indices((b, b))
    E[np.abs(i - j) > band] = 0.0
    A = np.eye(b) + np.triu(E, 1) + np.triu(E, 1).T
    d = np.logspace(0, -6, b)
    H = d[:, None] * A * d[None, :]
    lam, V, sw = rh.syevj(dev(H))
    lam = lam.cpu().numpy()
    V = V.cpu().numpy()
    import scipy.linalg.lapack as lapack
    L = np.linalg.cholesky(A)
    sva, _, _, work, _, info = lapack.dgejsv((d[:, None] * L).T)
    assert info == 0
    ref = np.sort((sva * (work[0] / work[1])) ** 2)[::-1]
    assert np.max(np.abs(lam - ref) / ref) < 1e-11
    assert np.max(np.abs(V.T @ V - np.eye(b))) <= 1e-13 * b


def test_syevj_band_schedule_invariant():
    """Eigenvalues with and without the banded pre-phase agree to high relative accuracy
    (different rotation sequences, same converged decomposition)."""
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, sys; sys.path.insert(0, %r);"
        "from paper_2201_12663_b200 import rhosvd as rh;"
        "b=500; rng=np.random.default_rng(5); E=rng.normal(size=(b,b))*0.03; i,j=np.indices((b,b));"
        "E[np.abs(i-j)>48]=0; A=np.eye(b)+np.triu(E,1)+np.triu(E,1).T; d=np.logspace(0,-6,b);"
        "H=torch.as_tensor(d[:,None]*A*d[None,:],device='cuda');"
        "np.save(sys.argv[1], rh.syevj(H)[0].cpu().numpy())"
    ) % ROOT
    import tempfile
    out = {}
    for v in ("0", "1"):
        with tempfile.NamedTemporaryFile(suffix=".npy", delete=False) as t:
            path = t.name
        env = dict(os.environ, RHOSVD_JAC_BAND=v)
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env, timeout=300)
        out[v] = np.load(path)
        os.unlink(path)
    assert np.max(np.abs(out["0"] - out["1"]) / out["0"]) < 1e-12


# (6, 7, 270) and (3, 40, 652): BN 128 with a <= 16-column leftover -> the 144-wide edge tile
@pytest.mark.parametrize("r,R", [((1, 1, 1), 1), ((3, 5, 7), 50), ((10, 10, 10), 200), ((70, 129, 33), 1500),
                                 ((20, 20, 20), 40001), ((5, 130, 97), 3000), ((4, 3, 130), 777),
                                 ((2, 1, 65), 100), ((40, 200, 300), 2000), ((130, 131, 97), 513),
                                 ((30, 30, 60), 10), ((9, 256, 200), 4099),
                                 ((6, 7, 270), 300), ((3, 40, 652), 1000)])
def test_core(rh, r, R):
    from oracle import core_kr
    rng = np.random.default_rng(sum(r) + R)
    W = [rng.normal(size=(rl, R)) for rl in r]
    xi = rng.normal(size=R)
    beta = rh.core(dev(W[0]), dev(W[1]), dev(W[2]), dev(xi)).cpu().numpy()
    ref = core_kr(W[0], W[1], W[2], xi)
    assert np.max(np.abs(beta - ref)) <= 1e-13 * np.sqrt(R) * np.max(np.abs(ref)) * 8


# b <= 160: the one-CTA register kernel (every 32-block count and its edges); larger b:
# the cooperative blocked kernel
@pytest.mark.parametrize("b", [1, 5, 31, 32, 33, 64, 65, 96, 127, 128, 129, 130, 159, 160, 161, 298, 449, 707, 873])
def test_chol_inv(rh, b):
    """Bp = D L^{-T} (scaled Cholesky inverse) against LAPACK; Q = M Bp orthonormal."""
    rng = np.random.default_rng(b + 11)
    M = rng.normal(size=(3 * b + 7, b)) * np.logspace(0, -3, b)[None, :]
    S = M.T @ M
    Bp = rh.chol_inv(dev(S)).cpu().numpy()
    d = 1.0 / np.sqrt(np.diag(S))
    L = np.linalg.cholesky(d[:, None] * S * d[None, :])
    ref = d[:, None] * np.linalg.inv(L).T
    assert np.max(np.abs(Bp - ref)) <= 1e-11 * np.max(np.abs(ref))
    Q = M @ Bp
    assert np.max(np.abs(Q.T @ Q - np.eye(b))) <= 1e-12


# dependent column in the second / first 32-half of a diagonal block and in a later
# panel (blocked kernel), and in the one-CTA kernel
@pytest.mark.parametrize("b,col", [(100, 40), (200, 40), (200, 10), (300, 130)])
def test_chol_inv_dependent_column(rh, b, col):
    """A numerically dependent column gets a unit pivot and a zero sub-column: the
    remaining columns stay orthonormal and no NaN appears (one-CTA and blocked kernels)."""
    rng = np.random.default_rng(5)
    M = rng.normal(size=(3 * b, b))
    M[:, col] = M[:, 3] + 1e-9 * M[:, col]
    S = M.T @ M
    Bp = rh.chol_inv(dev(S)).cpu().numpy()
    assert np.all(np.isfinite(Bp))
    Q = M @ Bp
    keep = [i for i in range(b) if i != col]
    G = Q[:, keep].T @ Q[:, keep]
    assert np.max(np.abs(G - np.eye(b - 1))) <= 1e-8
