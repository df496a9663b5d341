"""Wider seeded parity sweep at mid sizes (n 100-1100, R 200-6000, eps 1e-3..1e-7 or fixed
ranks, narrow / wide exponents, signed weights) against the CPU oracle: ranks, sigma (with
the any-fp64-SVD floor of reading A13) and the Tucker tensor.  Prints one line per case and
a summary; ENOCONV is reported separately (allowed only when eps^2 T is below the squared
resolution)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_random_params
from oracle import rhosvd as orh, sigma_rel_err, tucker_diff, orth_error

N = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 99)
bad = 0
for i in range(N):
    n = int(rng.integers(100, 1100)); R = int(rng.integers(200, 6000))
    if rng.random() < 0.7:
        eps, ranks = float(rng.choice([1e-3, 1e-4, 1e-5, 1e-6, 1e-7])), None
    else:
        eps, ranks = None, tuple(int(x) for x in rng.integers(1, min(n, R, 200), size=3))
    wide = bool(rng.random() < 0.5)
    p = make_random_params(n, R, seed=50000 + i, eps=eps, ranks=ranks,
                           a_range=(0.05, 400.0) if wide else (0.5, 20.0), signed=bool(i % 2))
    U1, U2, U3, xi = make_config(p)
    o = orh([U1, U2, U3], xi, eps=eps, ranks=ranks)
    try:
        g = rhosvd.c2t([torch.as_tensor(u, device="cuda") for u in (U1, U2, U3)], torch.as_tensor(xi, device="cuda"),
                       eps=eps, ranks=ranks)
    except rhosvd.RhosvdError as e:
        print(f"{i:3d} n {n} R {R} eps {eps} ranks {ranks}: ENOCONV/err {e.status} {str(e)[:100]}", flush=True)
        bad += 1
        continue
    msg = []
    if tuple(g.ranks) != tuple(o.ranks):
        if any(o.report["near_tie"]):
            msg.append("near-tie")
        else:
            msg.append(f"RANKS {g.ranks} vs {o.ranks}")
    else:
        for l in range(3):
            so = o.sigma[l][:o.ranks[l]]; sg = g.sigma[l].cpu().numpy()
            if len(so):
                tol = np.maximum(1e-10, 16 * 1.11e-16 * so[0] / so)
                if not np.all(np.abs(sg - so) <= tol * so):
                    msg.append(f"SIGMA mode {l} {np.max(np.abs(sg - so) / so):.2e}")
            if orth_error(g.Z[l].cpu().numpy()) > 1e-13:
                msg.append("ORTH")
        d, nrm = tucker_diff(g.beta.cpu().numpy(), [z.cpu().numpy() for z in g.Z], o.beta, o.Z)
        if nrm > 0 and d > 1e-9 * nrm:
            msg.append(f"TUCKER {d / nrm:.2e}")
    ok = not [m for m in msg if m != "near-tie"]
    bad += 0 if ok else 1
    print(f"{i:3d} n {n} R {R} eps {eps} ranks {ranks} -> {g.ranks} {'ok' if ok else 'FAIL'} {' '.join(msg)}", flush=True)
print("cases", N, "not ok", bad)
