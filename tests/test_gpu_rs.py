"""GPU parity of the RS long-range front-end (section 4.5):
rhosvd_rs_lattice (shift-and-windowing on the device) against the oracle's direct
evaluation of the lattice tensor, then RHOSVD C2T of the long-range part (rhosvd_c2t)
against the CPU oracle on the same tensor - ranks, sigma 1e-10, Tucker 1e-9 (BJ
criteria) - and the C2C rank of the GPU T2C against the oracle T2C of the same core."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import rhosvd as oracle_rhosvd, rs_long_lattice, rs_split, sigma_rel_err, slater_sinc_rule, t2c, tucker_diff  # noqa: E402,E501
from workloads import make_rs_lattice  # noqa: E402

DEV = torch.device("cuda:0")


def _gpu_lattice(rh, lat):
    t, w = rh.sinc_slater(lat.lam, 0.75, 26, 1e-6)
    (tl, wl), _ = rh.rs_split(t, w)
    idx = torch.as_tensor(lat.node_idx, device=DEV)
    c = torch.as_tensor(lat.c, device=DEV)
    return rh.rs_lattice(tl, wl, lat.h, lat.n, idx, c), len(tl)


def _oracle_lattice(lat):
    tau, w = slater_sinc_rule(lat.lam, 0.75, 26, 1e-6)
    kl, _ = rs_split(tau)
    return rs_long_lattice(tau[kl], w[kl], lat.x, lat.nodes, lat.c)


@pytest.fixture(scope="module")
def rh():
    from paper_2201_12663_b200 import rhosvd
    rhosvd.lib()
    return rhosvd


@pytest.mark.parametrize("L,kw", [((4, 4, 4), {}), ((3, 2, 5), dict(n=97, b=6.0, spacing=13)),
                                  ((1, 1, 1), dict(n=33, b=2.0, spacing=1))])
def test_window_matches_direct_evaluation(rh, L, kw):
    lat = make_rs_lattice(L, **kw)
    (U1, U2, U3, xi), Rl = _gpu_lattice(rh, lat)
    O = _oracle_lattice(lat)
    for g, o in zip((U1, U2, U3), O[:3]):
        assert g.shape == o.shape
        # (i - m) h on the device vs x_i - x_m on the host, and device vs host exp: a few ulps
        assert np.max(np.abs(g.cpu().numpy() - o)) <= 2e-15
    assert np.max(np.abs(xi.cpu().numpy() - O[3]) / np.abs(O[3])) <= 2e-15   # w_k: libm vs numpy exp


def test_window_edge_nodes(rh):
    """Nodes at grid indices 0 and n - 1 (the window touches both ends of the doubled table)."""
    lat = make_rs_lattice((2, 2, 2), n=40, b=4.0, spacing=39, first=0)
    assert lat.node_idx.min() == 0 and lat.node_idx.max() == 39
    (U1, U2, U3, xi), _ = _gpu_lattice(rh, lat)
    O = _oracle_lattice(lat)
    assert np.max(np.abs(U3.cpu().numpy() - O[2])) <= 2e-15


@pytest.mark.parametrize("L", [(4, 4, 4), (8, 8, 8), (16, 16, 8)])
def test_long_range_c2t_parity(rh, L):
    lat = make_rs_lattice(L)
    (U1, U2, U3, xi), Rl = _gpu_lattice(rh, lat)
    g = rh.c2t([U1, U2, U3], xi, eps=1e-3)
    O = _oracle_lattice(lat)
    o = oracle_rhosvd(list(O[:3]), O[3], eps=1e-3)
    assert tuple(g.ranks) == tuple(o.ranks), (g.ranks, o.ranks)
    for l in range(3):
        assert sigma_rel_err(g.sigma[l].cpu().numpy(), o.sigma[l][:o.ranks[l]]) <= 1e-10
    d, nrm = tucker_diff(g.beta.cpu().numpy(), [z.cpu().numpy() for z in g.Z], o.beta, o.Z)
    assert d <= 1e-9 * nrm, d / nrm
    # C2C (Table 2's R_comp step): the GPU T2C keeps exactly the slices' terms the oracle T2C
    # keeps on the same core
    cp = rh.c2c([U1, U2, U3], xi, 1e-5, eps=1e-3)
    ref = t2c(g.beta.cpu().numpy(), cp.eps)   # rhosvd_c2t is deterministic: c2c's core is g.beta
    assert cp.R == int(np.sum(ref.p))
    print(f"{L}: R_ini {xi.numel()} Tucker {g.ranks} R_comp {cp.R}")
