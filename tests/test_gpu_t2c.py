"""T2C / C2C on the GPU (rhosvd_t2c through the C ABI) against the T2C oracle
(oracle/t2c_oracle.py, Remark 2.1) applied to the SAME core beta
(the library is deterministic: rhosvd.c2t and rhosvd.c2c return bitwise-identical
cores), so the comparison isolates the T2C step:
  * identical per-slice kept counts p_m and total rank R (integer, exact) except for
    singular values within the sigma tolerance of the threshold (either side may keep them);
  * kept sigma within 1e-12 sigma_1(B_m) + 1e-10 sigma (one-sided Jacobi vs LAPACK);
  * beta_(R) from the GPU factors equal to the oracle's within 1e-11 ||beta||;
  * ||beta - beta_(R)|| <= eps and err2 equal to the oracle's discarded energy;
  * lifted factors: unit columns, F1 = Z1 u, F2 = Z2 v, F3 = Z3 e_slice.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.t2c_oracle import t2c as oracle_t2c, t2c_dense  # noqa: E402
from workloads import make_config, make_params, make_random_params  # noqa: E402


@pytest.fixture(scope="module")
def rh():
    from paper_2201_12663_b200 import rhosvd
    rhosvd.lib()
    return rhosvd


def dev_inputs(p):
    U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
    return [U1, U2, U3], xi


def beta_from_gpu(cp, shape):
    r1, r2, r3 = shape
    U = cp.U.cpu().numpy()
    V = cp.V.cpu().numpy()
    w = cp.w.cpu().numpy()
    sl = cp.slice_of.cpu().numpy()
    out = np.zeros(shape)
    for j in range(cp.R):
        out[:, :, sl[j]] += w[j] * np.outer(U[:, j], V[:, j])
    return out


def check_case(rh, Us, xi, eps, ranks, t2c_eps):
    g = rh.c2t(Us, xi, eps=eps, ranks=ranks, keep_w=False)
    beta = g.beta.cpu().numpy()
    cp = rh.c2c(Us, xi, t2c_eps, eps=eps, ranks=ranks)
    o = oracle_t2c(beta, t2c_eps * np.linalg.norm(beta))
    assert abs(cp.thr - o.thr) <= 1e-12 * o.thr
    # A singular value within the sigma tolerance (1e-12 sigma_1(B_m) + 1e-10 sigma) of the
    # threshold may be kept by one side and dropped by the other: such "ambiguous" values are
    # the only allowed difference in the per-slice counts, and each adds at most ~thr to the
    # difference of the truncated cores and ~thr^2 to the discarded energy.
    sl = cp.slice_of.cpu().numpy()
    w = cp.w.cpu().numpy()
    pg = np.bincount(sl, minlength=beta.shape[2])
    amb_tot = 0
    for m in range(beta.shape[2]):
        sv = np.linalg.svd(beta[:, :, m], compute_uv=False)
        s1 = sv[0] if sv.size else 0.0
        amb = int(np.sum(np.abs(sv - o.thr) <= 1e-12 * s1 + 1e-10 * o.thr))
        amb_tot += amb
        assert abs(int(pg[m]) - int(o.p[m])) <= amb, (m, pg[m], o.p[m])
        k = min(pg[m], o.p[m])  # the unambiguous leading values agree
        wg, wo = np.sort(w[sl == m])[::-1][:k], o.sigma[o.slice_of == m][:k]
        assert np.all(np.abs(wg - wo) <= 1e-12 * s1 + 1e-10 * wo)
    assert abs(cp.R - o.sigma.shape[0]) <= amb_tot
    bR = beta_from_gpu(cp, beta.shape)
    nb = np.linalg.norm(beta)
    assert np.linalg.norm(bR - t2c_dense(o, beta.shape)) <= 1e-11 * nb + 1.01 * np.sqrt(amb_tot) * o.thr
    err = np.linalg.norm(beta - bR)
    assert err <= cp.eps * (1 + 1e-12) + 1e-12 * nb  # + rounding (columns below 16 u ||B|| are zero)
    assert abs(cp.err2 - o.err2) <= 1e-10 * o.err2 + 1e-13 * nb ** 2 + 1.03 * amb_tot * o.thr ** 2
    # lifted factors
    Z = [z.cpu().numpy() for z in g.Z]
    F = [f.cpu().numpy() for f in cp.F]
    sl = cp.slice_of.cpu().numpy()
    assert np.allclose(F[0], Z[0] @ cp.U.cpu().numpy(), atol=1e-13)
    assert np.allclose(F[1], Z[1] @ cp.V.cpu().numpy(), atol=1e-13)
    assert np.array_equal(F[2], Z[2][:, sl])
    for f in F:
        if f.shape[1]:
            assert np.max(np.abs(np.linalg.norm(f, axis=0) - 1.0)) <= 1e-12
    return cp, o


@pytest.mark.parametrize("n,R,seed,eps,ranks,t2c_eps", [
    (30, 200, 1, None, (8, 9, 7), 1e-4),
    (48, 300, 2, 1e-6, None, 1e-6),
    (40, 257, 3, 1e-5, None, 0.0),
    (64, 500, 4, None, (33, 17, 40), 1e-3),
])
def test_t2c_random(rh, n, R, seed, eps, ranks, t2c_eps):
    p = make_random_params(n, R, seed=seed, eps=eps, ranks=ranks)
    Us, xi = dev_inputs(p)
    cp, o = check_case(rh, Us, xi, p.eps, p.ranks, t2c_eps)
    if t2c_eps == 0.0:  # exact: every slice keeps its numerical rank
        assert cp.err2 <= 1e-20 * np.sum(o.sigma ** 2) + 1e-300


@pytest.mark.parametrize("k,t2c_eps", [(1, 1e-6), (3, 1e-6), (5, 1e-5)])
def test_t2c_baseline_configs(rh, k, t2c_eps):
    """cfg 1 (r = 10), cfg 3 (r ~ 130), cfg 5 (r = 108): slices fit shared memory."""
    p = make_params(k)
    Us, xi = dev_inputs(p)
    cp, o = check_case(rh, Us, xi, p.eps, p.ranks, t2c_eps)
    r1, r2, r3 = cp.U.shape[0], cp.V.shape[0], len(o.p)
    assert cp.R <= r3 * min(r1, r2)


@pytest.mark.parametrize("n,R,ranks,t2c_eps", [(400, 600, (170, 170, 4), 1e-6), (300, 900, (257, 190, 9), 1e-5)])
def test_t2c_large_slices_block_kernel(rh, n, R, ranks, t2c_eps):
    """Slices too large for shared memory take the block one-sided Jacobi path."""
    p = make_random_params(n, R, seed=5, ranks=ranks)
    Us, xi = dev_inputs(p)
    check_case(rh, Us, xi, None, p.ranks, t2c_eps)


def test_t2c_cfg2(rh):
    """cfg 2 (r = 278 / 282 / 282): 282 slices of 278 x 282 through the block path."""
    p = make_params(2)
    Us, xi = dev_inputs(p)
    check_case(rh, Us, xi, p.eps, p.ranks, 1e-6)


def test_t2c_plain_kernel_subprocess():
    """Both paths (shared-memory slices and the global-memory block path for large slices)
    default to the QR-preconditioned kernels; RHOSVD_T2C_QR=0 selects the plain one-sided
    Jacobi kernels (read once per process), so the random, baseline, large-slice and cfg 2
    cases run once more with them in a subprocess."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, RHOSVD_T2C_QR="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.join(here, "test_gpu_t2c.py"),
                        "-k", "random or baseline_configs or large_slices or cfg2"], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-2000:])
