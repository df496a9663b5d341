"""Error semantics of rhosvd_c2t (include/rhosvd.h): the library fails
loudly (RHOSVD_ENOCONV = -3) instead of returning a rank that violates the eps rule or a
frame from an unconverged subspace iteration.

Forcing case: BASELINE.json config 1 (fixed r = 10) with oversample p = 1, i.e. block
b = 11.  Its spectrum decays slowly at the cut (sigma_11 / sigma_10 ~ 0.87, SURVEY.md
Appendix A.1: relative gap 0.10-0.19), so the block-edge rate rho = lambda_11 / lambda_10
~ 0.76 needs ~60 subspace steps for sin(theta) ~ 1e-7.  With max_iters = 2 the iteration
stops far short and the call must return -3; with max_iters = 100 the same input
converges and matches the CPU oracle.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _cfg1():
    from workloads import make_config, make_params
    p = make_params(1)
    U1, U2, U3, xi = make_config(p)
    dev = torch.device("cuda:0")
    return p, (U1, U2, U3, xi), [torch.as_tensor(u, device=dev) for u in (U1, U2, U3)], torch.as_tensor(xi, device=dev)


def test_enoconv_when_iteration_cap_too_small():
    from paper_2201_12663_b200 import rhosvd
    p, _, Ud, xid = _cfg1()
    with pytest.raises(rhosvd.RhosvdError) as ei:
        rhosvd.c2t(Ud, xid, ranks=p.ranks, oversample=1, max_iters=2)
    assert ei.value.status == -3
    assert "max_iters" in str(ei.value)


def test_same_input_converges_with_enough_iterations():
    from oracle import rhosvd as oracle_rhosvd, sigma_rel_err, tucker_diff
    from paper_2201_12663_b200 import rhosvd
    p, host, Ud, xid = _cfg1()
    g = rhosvd.c2t(Ud, xid, ranks=p.ranks, oversample=1, max_iters=100)
    o = oracle_rhosvd(list(host[:3]), host[3], ranks=p.ranks)
    assert tuple(g.ranks) == tuple(o.ranks)
    for l in range(3):
        assert sigma_rel_err(g.sigma[l].cpu().numpy(), o.sigma[l][:o.ranks[l]]) <= 1e-10
    d, nrm = tucker_diff(g.beta.cpu().numpy(), [z.cpu().numpy() for z in g.Z], o.beta, o.Z)
    assert d <= 1e-9 * nrm


def test_library_usable_after_enoconv():
    """A failed call leaves no state behind: the next default call is bitwise the usual one."""
    from paper_2201_12663_b200 import rhosvd
    p, _, Ud, xid = _cfg1()
    a = rhosvd.c2t(Ud, xid, ranks=p.ranks)
    with pytest.raises(rhosvd.RhosvdError):
        rhosvd.c2t(Ud, xid, ranks=p.ranks, oversample=1, max_iters=2)
    b = rhosvd.c2t(Ud, xid, ranks=p.ranks)
    assert torch.equal(a.beta, b.beta)
    assert all(torch.equal(x, y) for x, y in zip(a.Z, b.Z))
