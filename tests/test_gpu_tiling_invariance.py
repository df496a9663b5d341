"""Tile shapes never change the arithmetic: every output element of the core and of the
GEMM engine is accumulated over the same k order whatever column segment computes it, so
the outputs with the narrow / wide edge launches and without them are BITWISE equal.
The knobs are read once per process, so each setting runs in its own subprocess:
  RHOSVD_CORE_WIDE_EDGE=0  (r3 = 652 / 270: 16-wide edge instead of the 144-wide tile),
  RHOSVD_CORE_EDGE=0       (padded last 128-tile instead of any edge launch),
  RHOSVD_GEMM_EDGE=0       (padded last 128-column tile instead of a 32/64/96-wide launch),
and a full C2T on a cfg-3-sized problem (b ~ 147: the refinement GEMMs take the column
edge) must give bitwise-identical ranks, sigma, frames and core."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[2])
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_params
out = {}
rng = np.random.default_rng(7)
dev = lambda x: torch.as_tensor(np.ascontiguousarray(x), device="cuda")
for i, (r, R) in enumerate([((6, 7, 270), 300), ((3, 40, 652), 1000), ((5, 9, 300), 700)]):
    W = [rng.normal(size=(rl, R)) for rl in r]
    xi = rng.normal(size=R)
    out[f"core{i}"] = rhosvd.core(dev(W[0]), dev(W[1]), dev(W[2]), dev(xi)).cpu().numpy()
for i, (M, N, K) in enumerate([(3000, 147, 2500), (147, 3000, 2048), (1000, 730, 4096)]):
    A, B = rng.normal(size=(M, K)), rng.normal(size=(K, N))
    out[f"gemm{i}"] = rhosvd.dgemm(dev(A), dev(B)).cpu().numpy()
p = make_params(3)
U1, U2, U3, x = make_config(p, backend="torch", device=torch.device("cuda"))
g = rhosvd.c2t([U1, U2, U3], x, eps=p.eps, ranks=p.ranks, keep_w=False)
out["ranks"] = np.array(g.ranks)
out["beta"] = g.beta.cpu().numpy()
for l in range(3):
    out[f"Z{l}"] = g.Z[l].cpu().numpy()
    out[f"s{l}"] = g.sigma[l].cpu().numpy()
np.savez(sys.argv[1], **out)
'''


def _run(tmp_path, name, env_extra):
    path = str(tmp_path / f"{name}.npz")
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, path, ROOT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, (name, r.stdout[-2000:], r.stderr[-3000:])
    return dict(np.load(path))


def test_edge_launches_bitwise_invariant(tmp_path):
    base = _run(tmp_path, "default", {})
    for name, env in [("no_wide_edge", {"RHOSVD_CORE_WIDE_EDGE": "0"}), ("no_core_edge", {"RHOSVD_CORE_EDGE": "0"}),
                      ("no_gemm_edge", {"RHOSVD_GEMM_EDGE": "0"})]:
        other = _run(tmp_path, name, env)
        assert base.keys() == other.keys()
        for k in base:
            assert np.array_equal(base[k], other[k]), (name, k)
