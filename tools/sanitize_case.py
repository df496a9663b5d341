"""Small end-to-end run for compute-sanitizer: one C2T (eps mode, ragged sizes), one T2C,
and the kernel-level entry points."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_random_params

dev = torch.device("cuda")
p = make_random_params(70, 333, seed=5, eps=1e-6)
U1, U2, U3, xi = make_config(p, backend="torch", device=dev)
g = rhosvd.c2t([U1, U2, U3], xi, eps=p.eps)
cp = rhosvd.c2c([U1, U2, U3], xi, 1e-6, eps=p.eps)
rng = np.random.default_rng(1)
A = torch.as_tensor(rng.normal(size=(130, 67)), device=dev)
B = torch.as_tensor(rng.normal(size=(67, 45)), device=dev)
rhosvd.dgemm(A, B)
S = torch.as_tensor(rng.normal(size=(200, 200)), device=dev)
rhosvd.syevj(S + S.t())
M = torch.as_tensor(rng.normal(size=(300, 97)), device=dev)
rhosvd.chol_inv(M.t() @ M)
W = [torch.as_tensor(rng.normal(size=(r, 500)), device=dev) for r in (5, 130, 97)]
rhosvd.core(W[0], W[1], W[2], torch.as_tensor(rng.normal(size=500), device=dev))
# 144-wide edge tile (r3 = 652 -> 4 x 128 + 144), ring wrapping (R / 32 > stages)
W = [torch.as_tensor(rng.normal(size=(r, 700)), device=dev) for r in (3, 40, 652)]
rhosvd.core(W[0], W[1], W[2], torch.as_tensor(rng.normal(size=700), device=dev))
# host-buffer entry point, ALS sweep, convolution
h = rhosvd.c2t_host([u.cpu().pin_memory() for u in (U1, U2, U3)], xi.cpu().pin_memory(), eps=p.eps)
h.close()
rhosvd.c2t([U1, U2, U3], xi, eps=p.eps, als_sweeps=1)
F = [torch.as_tensor(rng.normal(size=(4, 100)), device=dev) for _ in range(3)]
P = [torch.as_tensor(rng.normal(size=(2, 100)), device=dev) for _ in range(3)]
rhosvd.conv3d(F, torch.ones(4, dtype=torch.float64, device=dev), P, torch.ones(2, dtype=torch.float64, device=dev), 0.5)
# round-2 kernels: the Gram's diagonal-strip path and snake deal (n >= 128 tiles, K >= 2048),
# the register-resident column normalisation (512 <= n <= 4096, odd n), the block Jacobi's
# banded pre-phase and mark-driven sweeps (the pipeline's W W^T, b > 112)
p2 = make_random_params(521, 2600, seed=11, eps=1e-6)
V1, V2, V3, xi2 = make_config(p2, backend="torch", device=dev)
g2 = rhosvd.c2t([V1, V2, V3], xi2, eps=p2.eps)
b = 300
Eb = rng.normal(size=(b, b)) * 0.03
ii, jj = np.indices((b, b))
Eb[np.abs(ii - jj) > 40] = 0.0
Ab = np.eye(b) + np.triu(Eb, 1) + np.triu(Eb, 1).T
db = np.logspace(0, -6, b)
rhosvd.syevj(torch.as_tensor(db[:, None] * Ab * db[None, :], device=dev))
torch.cuda.synchronize()
print("ok", g.ranks, cp.R, g2.ranks, g2.report["block"])
