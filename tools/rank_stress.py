"""Repeated rhosvd_c2t on a BASELINE config; prints the report of every call whose ranks
differ from the expected ones (diagnoses intermittent rank errors)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2201_12663_b200 import rhosvd  # noqa: E402
from workloads import make_config, make_params  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
keep_w = len(sys.argv) > 3 and sys.argv[3] == "keep_w"
p = make_params(k)
U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
first = None
bad = 0
for i in range(reps):
    g = rhosvd.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, keep_w=keep_w)
    hold = [s.clone() for s in g.sigma] + [z.clone() for z in g.Z] + ([w.clone() for w in g.W] if keep_w else [])
    rep = g.report
    if first is None:
        first = (tuple(g.ranks), [float(s[-1]) for s in g.sigma])
        print("first", first, rep["tail"], rep["rho"], rep["block"], flush=True)
        continue
    if tuple(g.ranks) != first[0]:
        bad += 1
        print(i, "ranks", g.ranks, "block", rep["block"], "tail", rep["tail"], "rho", rep["rho"], "iters", rep["iters"],
              "sigma_last", [float(s[-1]) for s in g.sigma], "sigma_first", [float(s[0]) for s in g.sigma],
              flush=True)
print("bad calls:", bad, "of", reps - 1)
