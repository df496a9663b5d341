"""Debug helper: GPU vs oracle sigma per index for stress cases (development only)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2201_12663_b200 import rhosvd
from oracle import rhosvd as orh
from workloads import make_config, make_random_params

sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_gpu_parity import _stress_cases  # noqa: E402

want = [int(x) for x in sys.argv[1:]]
for (i, n, R, eps, ranks, wide) in _stress_cases():
    if i not in want:
        continue
    p = make_random_params(n, R, seed=7000 + i, eps=eps, ranks=ranks,
                           a_range=(0.05, 400.0) if wide else (0.5, 20.0), signed=bool(i % 2))
    U1, U2, U3, xi = make_config(p)
    o = orh([U1, U2, U3], xi, eps=eps, ranks=ranks)
    g = rhosvd.c2t([torch.as_tensor(u, device="cuda") for u in (U1, U2, U3)], torch.as_tensor(xi, device="cuda"),
                   eps=eps, ranks=ranks)
    print("case", i, n, R, eps, ranks, "ranks", g.ranks, o.ranks, "blocks", g.report["block"], "iters", g.report["iters"])
    for l in range(3):
        sg = g.sigma[l].cpu().numpy()
        so = o.sigma[l][: o.ranks[l]]
        err = np.abs(sg - so) / so
        k = int(np.argmax(err))
        print("  mode", l, "max rel err %.2e at k=%d sigma %.3e (sigma_1 %.3e, T %.1f)" % (err[k], k, so[k], so[0], o.T[l]))
