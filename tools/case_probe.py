"""Where does a parity-sweep case's Tucker error come from?  (GPU probe)

For one tools/parity_sweep.py case: the GPU result against the oracle per mode - frame
orthonormality, projector distance ||Z_g Z_g^T - Z_o Z_o^T||_2 (sin theta), sigma - and the
Tucker distance of (a) the GPU tensor, (b) the oracle core recomputed on the CPU from the
GPU frames (W = Z_g^T Uhat, beta = core_kr) and (c) the GPU core against (b): (b) isolates
the frames, (c) the projection + core.

Usage: python tools/case_probe.py SWEEP_SEED CASE"""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tools")
from cut_conditioning import sweep_params
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_random_params
from oracle import rhosvd as orh, tucker_diff, orth_error
from oracle.rhosvd_oracle import normalize, project, core_kr

seed, case = int(sys.argv[1]), int(sys.argv[2])
n, R, eps, ranks, wide, i = sweep_params(seed, case)[case]
p = make_random_params(n, R, seed=50000 + i, eps=eps, ranks=ranks,
                       a_range=(0.05, 400.0) if wide else (0.5, 20.0), signed=bool(i % 2))
U1, U2, U3, xi = make_config(p)
o = orh([U1, U2, U3], xi, eps=eps, ranks=ranks)
Uh, xip = normalize([U1, U2, U3], xi)[:2]
print(f"case {case}: n {n} R {R} eps {eps} ranks {ranks} oracle ranks {tuple(o.ranks)}", flush=True)
for rep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 1):
    g = rhosvd.c2t([torch.as_tensor(u, device="cuda") for u in (U1, U2, U3)], torch.as_tensor(xi, device="cuda"),
                   eps=eps, ranks=ranks)
    Zg = [z.cpu().numpy() for z in g.Z]
    bg = g.beta.cpu().numpy()
    print(f" rep {rep} gpu ranks {tuple(g.ranks)} block {getattr(g, 'block', None)}")
    for l in range(3):
        r = min(g.ranks[l], o.ranks[l])
        Pg, Po = Zg[l] @ Zg[l].T, o.Z[l] @ o.Z[l].T
        st = np.linalg.norm(Pg - Po, 2)
        sg, so = g.sigma[l].cpu().numpy()[:r], o.sigma[l][:r]
        print(f"  mode {l}: orth {orth_error(Zg[l]):.2e}  sin theta {st:.2e}  sigma rel max {np.max(np.abs(sg - so) / so):.2e}"
              f"  (at k: {int(np.argmax(np.abs(sg - so) / so))})  sigma_r/sigma_1 {so[-1] / so[0]:.2e}")
    bc = core_kr(*[project(Zg[l], Uh[l]) for l in range(3)], xip)
    da, na = tucker_diff(bg, Zg, o.beta, o.Z)
    db, _ = tucker_diff(bc, Zg, o.beta, o.Z)
    dc = float(np.linalg.norm(bg - bc))
    print(f"  Tucker: gpu {da / na:.2e}  cpu-core-on-gpu-frames {db / na:.2e}  gpu core vs cpu core {dc / na:.2e}", flush=True)
