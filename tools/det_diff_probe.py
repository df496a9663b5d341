"""Repeated rhosvd_c2t calls: size of the difference of each mode's sigma / Z and of beta
from the first call's (diagnoses run-to-run differences)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2201_12663_b200 import rhosvd  # noqa: E402
from workloads import make_config, make_params  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
p = make_params(k)
U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
ref = None
nd = 0
for i in range(reps):
    g = rhosvd.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, keep_w=True)
    cur = ([s.clone() for s in g.sigma], [z.clone() for z in g.Z], [w.clone() for w in g.W], g.beta.clone(),
           [float(x) for x in g.report["tail"]])
    if ref is None:
        ref = cur
        continue
    if all(torch.equal(a, b) for a, b in zip(cur[0] + cur[1] + cur[2] + [cur[3]], ref[0] + ref[1] + ref[2] + [ref[3]])):
        continue
    nd += 1
    ds = [float(((a - b).abs() / b.abs()).max()) for a, b in zip(cur[0], ref[0])]
    dz = [float((a.abs() - b.abs()).abs().max()) for a, b in zip(cur[1], ref[1])]
    dw = [float((a - b).abs().max() / b.abs().max()) for a, b in zip(cur[2], ref[2])]
    db = float((cur[3] - ref[3]).abs().max() / ref[3].abs().max())
    print(i, "dsigma", ds, "d|Z|", dz, "dW", dw, "dbeta", db, "tail", cur[4], ref[4], flush=True)
print("calls differing from the first:", nd)
