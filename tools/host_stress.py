"""Repeated rhosvd_c2t_host calls (host buffers, streamed path): ranks and beta bitwise
equal to the device-buffer call every time."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2201_12663_b200 import rhosvd  # noqa: E402
from workloads import make_config, make_params  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = make_params(k)
U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
g = rhosvd.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, keep_w=False)
ref_beta = g.beta.cpu()
hU = [u.cpu().pin_memory() for u in (U1, U2, U3)]
hx = xi.cpu().pin_memory()
bad = 0
for i in range(reps):
    h = rhosvd.c2t_host(hU, hx, eps=p.eps, ranks=p.ranks)
    ok = h.ranks == g.ranks and torch.equal(h.beta, ref_beta)
    h.close()
    if not ok:
        bad += 1
        print("call", i, "differs: ranks", h.ranks, flush=True)
print("host calls differing from the device call:", bad, "of", reps)
