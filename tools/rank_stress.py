"""Repeated rhosvd_c2t on a BASELINE config; prints the report of every call whose ranks
differ from the expected ones or that fails (RHOSVD_ENOCONV etc.), and counts calls whose
sigma / frames are not bitwise equal to the first call's (diagnoses intermittent errors).

    python tools/rank_stress.py 4 200"""
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
bad = errors = nonbitwise = 0
ref = None
for i in range(reps):
    try:
        g = rhosvd.c2t([U1, U2, U3], xi, eps=p.eps, ranks=p.ranks, keep_w=keep_w)
    except rhosvd.RhosvdError as e:
        errors += 1
        print(i, "error", e, flush=True)
        continue
    if ref is None:
        ref = ([s.clone() for s in g.sigma], [z.clone() for z in g.Z], g.beta.clone())
    elif not (all(torch.equal(a, b) for a, b in zip(ref[0], g.sigma)) and
              all(torch.equal(a, b) for a, b in zip(ref[1], g.Z)) and torch.equal(ref[2], g.beta)):
        nonbitwise += 1
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
print("bad calls:", bad, "of", reps - 1, "errors:", errors, "not bitwise equal to the first:", nonbitwise)
