"""Tensor-product convolution on the GPU (rhosvd_conv3d through the C ABI) against the
oracle (oracle/conv_oracle.py): every output factor column
u_m^(l) * p_q^(l) elementwise within the rounding of an n-term dot product
(1e-13 n h max|u| max|p|), weights exactly c_m w_q; plus the C2C -> convolution chain on
a Gaussian density against the analytic Gaussian * Gaussian result."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.conv_oracle import conv3d_canonical  # noqa: E402


@pytest.fixture(scope="module")
def rh():
    from paper_2201_12663_b200 import rhosvd
    rhosvd.lib()
    return rhosvd


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


def test_conv3d_both_routes_subprocess():
    """The FFT route (n <= 2730) and the dense Toeplitz-GEMM route are picked by size;
    RHOSVD_CONV_ROUTE forces each (read once per process), so this module's parity cases
    run once per route in a subprocess."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for route in ("dense", "fft"):
        env = dict(os.environ, RHOSVD_CONV_ROUTE=route)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.join(here, "test_gpu_conv.py"),
                            "-k", "random or gaussians or edge"], env=env, capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, (route, r.stdout[-3000:], r.stderr[-2000:])


@pytest.mark.parametrize("n,Ra,Rp,seed", [(64, 5, 3, 1), (65, 7, 4, 2), (300, 20, 9, 3), (129, 1, 1, 4),
                                          (512, 33, 12, 5)])
def test_conv3d_random(rh, n, Ra, Rp, seed):
    rng = np.random.default_rng(seed)
    h = 0.37
    Fa = [rng.normal(size=(n, Ra)) for _ in range(3)]
    Fp = [rng.normal(size=(n, Rp)) * np.exp(-np.abs(np.arange(n) - n // 2) / 20.0)[:, None] for _ in range(3)]
    ca, cp = rng.normal(size=Ra), rng.normal(size=Rp)
    F, w = rh.conv3d([dev(f.T) for f in Fa], dev(ca), [dev(f.T) for f in Fp], dev(cp), h)
    Fo, wo = conv3d_canonical(Fa, ca, Fp, cp, h)
    assert np.array_equal(w.cpu().numpy(), wo)
    for l in range(3):
        got = F[l].cpu().numpy().T  # n x Ra Rp
        scale = np.repeat(np.abs(Fa[l]).max(axis=0), Rp) * np.tile(np.abs(Fp[l]).max(axis=0), Ra)
        assert np.all(np.abs(got - Fo[l]) <= 1e-13 * n * h * scale[None, :] + 1e-300)


def test_conv3d_gaussians_analytic(rh):
    """A rank-3 sum of Gaussians convolved with a rank-2 Gaussian kernel: each factor column is
    sqrt(pi / (a + b)) exp(-a b x^2 / (a + b)) to spectral accuracy (odd n, symmetric grid)."""
    n = 257
    L = 24.0
    h = L / (n - 1)
    x = (np.arange(n) - n // 2) * h
    a_s, b_s = [0.5, 1.3, 2.2], [0.8, 3.0]
    Fa = [np.stack([np.exp(-a * x ** 2) for a in a_s], axis=1) for _ in range(3)]
    Fp = [np.stack([np.exp(-b * x ** 2) for b in b_s], axis=1) for _ in range(3)]
    F, w = rh.conv3d([dev(f.T) for f in Fa], dev(np.ones(3)), [dev(f.T) for f in Fp], dev(np.ones(2)), h)
    for l in range(3):
        got = F[l].cpu().numpy()
        for m, a in enumerate(a_s):
            for q, b in enumerate(b_s):
                ref = math.sqrt(math.pi / (a + b)) * np.exp(-a * b * x ** 2 / (a + b))
                assert np.max(np.abs(got[m * 2 + q] - ref)) <= 1e-12


def test_conv3d_empty_and_errors(rh):
    F, w = rh.conv3d([dev(np.zeros((0, 8)))] * 3, dev(np.zeros(0)), [dev(np.ones((2, 8)))] * 3, dev(np.ones(2)), 1.0)
    assert F[0].shape == (0, 8) and w.shape == (0,)


@pytest.mark.parametrize("n", [1, 2, 3, 2730, 2731, 5000, 6000])
def test_conv3d_edge_sizes(rh, n):
    """Degenerate grids and the route boundaries (N = 2^k >= 1.5 n: 2730 -> 4096 one-CTA FFT,
    2731 -> 8192 and 5000 -> 8192, 6000 -> 16384: four-step FFT)."""
    rng = np.random.default_rng(n)
    Ra, Rp, h = 3, 2, 0.5
    Fa = [rng.normal(size=(n, Ra)) for _ in range(3)]
    Fp = [rng.normal(size=(n, Rp)) for _ in range(3)]
    ca, cp = rng.normal(size=Ra), rng.normal(size=Rp)
    F, w = rh.conv3d([dev(f.T) for f in Fa], dev(ca), [dev(f.T) for f in Fp], dev(cp), h)
    Fo, wo = conv3d_canonical(Fa, ca, Fp, cp, h)
    for l in range(3):
        got = F[l].cpu().numpy().T
        scale = np.repeat(np.abs(Fa[l]).max(axis=0), Rp) * np.tile(np.abs(Fp[l]).max(axis=0), Ra)
        assert np.all(np.abs(got - Fo[l]) <= 1e-13 * max(n, 8) * h * scale[None, :])
