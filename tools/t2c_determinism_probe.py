import hashlib, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_params
p = make_params(3)
U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
for i in range(5):
    cp = rhosvd.c2c([U1, U2, U3], xi, 1e-6, eps=p.eps, ranks=p.ranks)
    print(i, cp.R, hashlib.sha1(cp.w.cpu().numpy().tobytes()).hexdigest()[:10], cp.sweeps, flush=True)
