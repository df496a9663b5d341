"""C2T ALS on the GPU (rhosvd_c2t_als through the C ABI) against the ALS oracle
(oracle/als_oracle.py) on the same seeded inputs:
  * ranks identical (those of the RHOSVD start);
  * frames: projectors Z Z^T within 1e-9 (max entry) - the GPU takes the dominant
    subspace of the unfolding's Gram (Gram-domain accuracy u kappa^2 / gap, reading L3),
    the oracle LAPACK's SVD of the unfolding;
  * sigma (singular values of the last unfolding): |d sigma| <= 1e-12 sigma_1 + 1e-9 sigma;
  * the Tucker tensor beta x_l Z_l (basis-free) within 1e-9 relative Frobenius (dense);
  * the projection norm ||beta|| never below the RHOSVD one (monotone ALS);
  * sweeps = 0 is bitwise rhosvd_c2t.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import dense_from_tucker, rhosvd as oracle_rhosvd  # noqa: E402
from oracle.als_oracle import c2t_als  # noqa: E402
from workloads import make_config, make_params, make_random_params  # noqa: E402


@pytest.fixture(scope="module")
def rh():
    from paper_2201_12663_b200 import rhosvd
    rhosvd.lib()
    return rhosvd


def test_als_both_routes_subprocess():
    """The two routes to the unfolding Gram (direct Khatri-Rao contraction / blocked
    R x R middle factor) are chosen by FLOP count; RHOSVD_ALS_ROUTE forces each one
    (read once per process, so each runs this module's parity cases in a subprocess)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for route in ("direct", "block"):
        env = dict(os.environ, RHOSVD_ALS_ROUTE=route)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.join(here, "test_gpu_als.py"),
                            "-k", "random or cfg1 or medium"], env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, (route, r.stdout[-3000:], r.stderr[-2000:])


def run_case(rh, p, sweeps, dense=True):
    U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
    g0 = rh.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, keep_w=False)
    g = rh.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, keep_w=False, als_sweeps=sweeps)
    Us = [u.cpu().numpy() for u in (U1, U2, U3)]
    x = xi.cpu().numpy()
    o0 = oracle_rhosvd(Us, x, eps=p.eps, ranks=p.ranks)
    assert tuple(g0.ranks) == tuple(o0.ranks)
    o = c2t_als(Us, x, sweeps, start=o0)
    assert tuple(g.ranks) == tuple(o0.ranks)
    Zg = [z.cpu().numpy() for z in g.Z]
    for l in range(3):
        sg, so = g.sigma[l].cpu().numpy(), o.sigma[l]
        # unique part: singular directions with sigma > 0 (an unfolding of rank < r_l,
        # e.g. r_l > r_b r_c, has a null part any orthonormal completion spans)
        k = int(np.sum(so > 1e-10 * so[0])) if so.size else 0
        Pg, Po = Zg[l][:, :k] @ Zg[l][:, :k].T, o.Z[l][:, :k] @ o.Z[l][:, :k].T
        assert np.abs(Pg - Po).max() <= 1e-9, (l, np.abs(Pg - Po).max())
        assert np.all(np.abs(sg[:k] - so[:k]) <= 1e-12 * so[0] + 1e-9 * so[:k]), (l, np.abs(sg - so).max())
        assert np.all(np.abs(sg[k:]) <= 1e-7 * so[0])  # Gram-domain zeros: sqrt(u) sigma_1
        assert np.abs(Zg[l].T @ Zg[l] - np.eye(Zg[l].shape[1])).max() <= 1e-12
    bg = g.beta.cpu().numpy()
    assert np.linalg.norm(bg) >= np.linalg.norm(g0.beta.cpu().numpy()) * (1 - 1e-12)
    assert abs(np.linalg.norm(bg) - np.linalg.norm(o.beta)) <= 1e-10 * np.linalg.norm(o.beta)
    if dense:
        Tg = dense_from_tucker(bg, Zg)
        To = dense_from_tucker(o.beta, o.Z)
        assert np.linalg.norm(Tg - To) <= 1e-9 * np.linalg.norm(To)
    return g, o


@pytest.mark.parametrize("n,R,seed,eps,ranks,sweeps", [
    (40, 120, 1, None, (6, 7, 5), 1),
    (40, 120, 1, None, (6, 7, 5), 2),
    (48, 300, 2, 1e-3, None, 1),
    (33, 257, 3, None, (1, 4, 9), 1),
])
def test_als_random(rh, n, R, seed, eps, ranks, sweeps):
    run_case(rh, make_random_params(n, R, seed=seed, eps=eps, ranks=ranks), sweeps)


def test_als_cfg1(rh):
    run_case(rh, make_params(1), 1)


def test_als_medium_blocked_K(rh):
    """n = 256, R = 3000: the R x R middle factor goes through several column blocks."""
    run_case(rh, make_random_params(256, 3000, seed=4, ranks=(24, 20, 28)), 1, dense=False)


def test_als_zero_sweeps_is_c2t(rh):
    p = make_random_params(50, 200, seed=5, ranks=(5, 5, 5))
    U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
    a = rh.c2t([U1, U2, U3], xi, ranks=p.ranks, keep_w=False)
    b = rh.c2t([U1, U2, U3], xi, ranks=p.ranks, keep_w=False, als_sweeps=0)
    assert torch.equal(a.beta, b.beta)
    assert all(torch.equal(x, y) for x, y in zip(a.Z, b.Z))


def test_als_rejects_negative_sweeps(rh):
    p = make_random_params(16, 20, seed=6, ranks=(2, 2, 2))
    U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
    with pytest.raises(rh.RhosvdError):
        rh.c2t([U1, U2, U3], xi, ranks=p.ranks, als_sweeps=-1)
