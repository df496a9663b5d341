"""Does a call's result depend on what ran before it in the process (stale workspace)?
cfg 3 alone vs cfg 3 after other shapes, bitwise."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_params, make_random_params


def run(p, als=None):
    U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
    g = rhosvd.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, keep_w=False, als_sweeps=als)
    return g.ranks, hashlib.sha1(g.beta.cpu().numpy().tobytes()).hexdigest()[:12], \
        [hashlib.sha1(s.cpu().numpy().tobytes()).hexdigest()[:8] for s in g.sigma]


p3 = make_params(3)
print("cfg3 first :", run(p3), flush=True)
for q in [make_random_params(400, 600, seed=5, ranks=(170, 170, 4)), make_random_params(300, 900, seed=5, ranks=(257, 190, 9)),
          make_params(2), make_random_params(64, 500, seed=4, ranks=(33, 17, 40)), make_params(5)]:
    run(q)
    run(q, als=1)
    print("cfg3 after", q.n, q.R, ":", run(p3), flush=True)
