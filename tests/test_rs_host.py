"""The RS front-end's host-side entry points of librhosvd.so (rhosvd_sinc_slater,
rhosvd_rs_split: O(M) scalar work, no GPU) against the oracle (oracle/rs_oracle.py)."""
import numpy as np
import pytest

from oracle import rs_split as o_split, slater_sinc_rule


@pytest.fixture(scope="module")
def rh():
    from paper_2201_12663_b200 import rhosvd
    rhosvd.lib()
    return rhosvd


@pytest.mark.parametrize("lam,h,M,wmin", [(0.5, 0.75, 26, 1e-6), (1.0, 0.5, 40, 0.0), (2.0, 1.0, 5, 1e-3)])
def test_sinc_rule_matches_oracle(rh, lam, h, M, wmin):
    t, w = rh.sinc_slater(lam, h, M, wmin)
    to, wo = slater_sinc_rule(lam, h, M, wmin)
    assert t.shape == to.shape
    # libm vs numpy exp: a few ulps (w is a product of two exponentials)
    assert np.all(np.abs(t - to) <= 4e-16 * to) and np.all(np.abs(w - wo) <= 1e-15 * wo + 1e-300)


def test_split_matches_oracle(rh):
    t, w = rh.sinc_slater(0.5, 0.75, 26, 1e-6)
    (tl, wl), (ts, ws) = rh.rs_split(t, w)
    kl, ks = o_split(t)
    assert np.array_equal(tl, t[kl]) and np.array_equal(wl, w[kl])
    assert np.array_equal(ts, t[ks]) and np.array_equal(ws, w[ks])


def test_rule_capacity_and_args(rh):
    import ctypes as C
    tau = np.zeros(3)
    w = np.zeros(3)
    R = C.c_int64()
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    assert rh.lib().rhosvd_sinc_slater(0.5, 0.75, 26, 0.0, P(tau), P(w), 3, C.byref(R)) == -1
    assert rh.lib().rhosvd_sinc_slater(-1.0, 0.75, 26, 0.0, P(tau), P(w), 3, C.byref(R)) == -1
