import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_random_params
n, R, eps = 100, 1000, 1e-5
p = make_random_params(n, R, seed=n * 1000 + R, eps=eps)
U1, U2, U3, xi = make_config(p)
Ud = [torch.as_tensor(u, device="cuda") for u in (U1, U2, U3)]
g = rhosvd.c2t(Ud, torch.as_tensor(xi, device="cuda"), eps=eps)
print("ranks", g.ranks, g.report["block"], g.report["iters"])
