"""Repeated rhosvd_c2t calls on a BASELINE config: are beta / Z / sigma bitwise identical?"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_params

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
p = make_params(k)
U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
seen = {}
for i in range(reps):
    g = rhosvd.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, keep_w=False)
    hb = hashlib.sha1(g.beta.cpu().numpy().tobytes()).hexdigest()[:12]
    hz = [hashlib.sha1(z.cpu().numpy().tobytes()).hexdigest()[:8] for z in g.Z]
    hs = [hashlib.sha1(s.cpu().numpy().tobytes()).hexdigest()[:8] for s in g.sigma]
    key = (hb, tuple(hz), tuple(hs))
    seen[key] = seen.get(key, 0) + 1
    print(i, g.ranks, hb, hz, hs, flush=True)
print("distinct results:", len(seen))
