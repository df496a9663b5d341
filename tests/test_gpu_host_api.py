"""rhosvd_c2t_host (host buffers in, host buffers out; include/rhosvd.h) against
rhosvd_c2t on the same inputs: the same kernels in the same order per output element
(the row-chunked core launch and the early per-mode Gram only change scheduling), so the
outputs must be BITWISE identical - and therefore inherit rhosvd_c2t's oracle parity
(tests/test_gpu_parity.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import make_config, make_params, make_random_params  # noqa: E402


@pytest.fixture(scope="module")
def rh():
    from paper_2201_12663_b200 import rhosvd
    rhosvd.lib()
    return rhosvd


def run_both(rh, p, pinned=True):
    U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
    g = rh.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, keep_w=False)
    hU = [u.cpu() for u in (U1, U2, U3)]
    hx = xi.cpu()
    if pinned:
        hU = [u.pin_memory() for u in hU]
        hx = hx.pin_memory()
    h = rh.c2t_host(hU, hx, eps=p.eps, ranks=p.ranks)
    try:
        assert h.ranks == g.ranks
        assert torch.equal(h.beta, g.beta.cpu())
        for l in range(3):
            assert torch.equal(h.Z[l], g.Z[l].cpu())
            assert torch.equal(h.sigma[l], g.sigma[l].cpu())
        for k in ("ranks", "block", "iters"):
            assert list(h.report[k]) == list(g.report[k])
    finally:
        h.close()
    return g


@pytest.mark.parametrize("n,R,seed,eps,ranks", [
    (64, 300, 1, 1e-6, None),
    (96, 513, 2, None, (7, 12, 9)),
])
def test_host_api_random(rh, n, R, seed, eps, ranks):
    run_both(rh, make_random_params(n, R, seed=seed, eps=eps, ranks=ranks))


def test_host_api_chunked_core(rh):
    """r = 200: 626 core tiles, no split-K -> the core runs as 8 row chunks with the D2H
    of each chunk overlapped; the host beta must still equal the device one bit for bit."""
    run_both(rh, make_random_params(256, 2000, seed=3, ranks=(200, 200, 200)))


def test_host_api_pageable_inputs(rh):
    run_both(rh, make_random_params(80, 400, seed=4, eps=1e-5), pinned=False)


def test_host_api_cfg1(rh):
    run_both(rh, make_params(1))


def test_host_api_device_result_has_no_host_outputs(rh):
    p = make_random_params(32, 50, seed=5, ranks=(3, 3, 3))
    U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
    opts = rh.make_opts(ranks=p.ranks)
    h = rh.c2t_raw((U1, U2, U3), xi, opts)
    try:
        import ctypes as C
        b = C.c_void_p()
        assert rh.lib().rhosvd_result_host_core(h, C.byref(b)) == -1  # EINVAL
    finally:
        rh.lib().rhosvd_result_free(h)


@pytest.mark.parametrize("where", ["U2", "xi"])
def test_host_api_nonfinite_rejected(rh, where):
    """Streamed host path: a NaN in a side matrix (caught by that mode's own flag) or an
    Inf in xi (caught after the modes) fails the call with ENONFINITE; the library stays
    usable afterwards."""
    p = make_random_params(40, 90, seed=7, ranks=(3, 3, 3))
    U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
    hU = [u.cpu().pin_memory() for u in (U1, U2, U3)]
    hx = xi.cpu().pin_memory()
    if where == "U2":
        hU[1][5, 3] = float("nan")
    else:
        hx[7] = float("inf")
    with pytest.raises(rh.RhosvdError) as ei:
        rh.c2t_host(hU, hx, ranks=p.ranks)
    assert ei.value.status == -2  # ENONFINITE
    ok = rh.c2t_host([u.cpu().pin_memory() for u in (U1, U2, U3)], xi.cpu().pin_memory(), ranks=p.ranks)
    assert ok.ranks == (3, 3, 3)
    ok.close()


def test_host_api_empty_and_tiny(rh):
    """R_local = 0 (empty Tucker tensor) and n = 1 through the host-buffer entry point."""
    import ctypes as C
    e = [torch.zeros(0, 8, dtype=torch.float64) for _ in range(3)]
    h = rh.c2t_host(e, torch.zeros(0, dtype=torch.float64), eps=1e-6)
    assert h.ranks == (0, 0, 0)
    h.close()
    p = make_random_params(1, 5, seed=9, ranks=(1, 1, 1))
    run_both(rh, p)
