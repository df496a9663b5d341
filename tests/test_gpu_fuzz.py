"""Seeded fuzz over the public entry points on small random problems: every call succeeds
(or fails with the documented status), and the cross-API invariants hold -
  * ranks <= min(n, R); frames orthonormal;
  * rhosvd_c2t_host bitwise equal to rhosvd_c2t;
  * rhosvd_c2t_als: same ranks, projection norm ||beta|| not below the RHOSVD one;
  * rhosvd_t2c on the C2T core: ||beta - beta_(R)|| <= eps (Remark 2.1) and R <= r3 min(r1, r2).
Oracle parity for these paths is in the dedicated test files; this sweeps shapes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import make_config, make_random_params  # noqa: E402


@pytest.fixture(scope="module")
def rh():
    from paper_2201_12663_b200 import rhosvd
    rhosvd.lib()
    return rhosvd


def _cases():
    rng = np.random.default_rng(4242)
    out = []
    for i in range(16):
        n = int(rng.choice([1, 2, 7, 16, 33, 64, 70]))
        R = int(rng.choice([1, 4, 30, 129, 300]))
        if rng.random() < 0.5:
            eps, ranks = float(rng.choice([1e-3, 1e-6, 1e-9])), None
        else:
            m = min(n, R)
            eps, ranks = None, tuple(int(x) for x in rng.integers(1, m + 2, size=3))
        out.append((i, n, R, eps, ranks))
    return out


@pytest.mark.parametrize("i,n,R,eps,ranks", _cases())
def test_fuzz_entry_points(rh, i, n, R, eps, ranks):
    p = make_random_params(n, R, seed=100 + i, eps=eps, ranks=ranks)
    U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
    g = rh.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, keep_w=False)
    m = min(n, R)
    assert all(0 <= r <= m for r in g.ranks)
    for z in g.Z:
        zz = z.cpu().numpy()
        if zz.shape[1]:
            assert np.abs(zz.T @ zz - np.eye(zz.shape[1])).max() <= 1e-12
    # host-buffer twin
    h = rh.c2t_host([u.cpu().pin_memory() for u in (U1, U2, U3)], xi.cpu().pin_memory(), eps=p.eps, ranks=p.ranks)
    try:
        assert h.ranks == g.ranks
        assert torch.equal(h.beta, g.beta.cpu())
    finally:
        h.close()
    # one ALS sweep
    a = rh.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, keep_w=False, als_sweeps=1)
    assert a.ranks == g.ranks
    nb, na = float(np.linalg.norm(g.beta.cpu().numpy())), float(np.linalg.norm(a.beta.cpu().numpy()))
    assert na >= nb * (1 - 1e-10) - 1e-300
    # C2C
    if all(r > 0 for r in g.ranks):
        cp = rh.c2c([U1, U2, U3], xi, 1e-4, eps=p.eps, ranks=p.ranks)
        r1, r2, r3 = g.ranks
        assert cp.R <= r3 * min(r1, r2)
        assert cp.err2 ** 0.5 <= cp.eps * (1 + 1e-10) + 1e-14 * nb
