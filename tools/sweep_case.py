"""Re-run one case of tools/parity_sweep.py (same seeds) and print per-column diagnostics."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_random_params
from oracle import rhosvd as orh

target = int(sys.argv[1]); seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 99
rng = np.random.default_rng(seed0)
for i in range(target + 1):
    n = int(rng.integers(100, 1100)); R = int(rng.integers(200, 6000))
    if rng.random() < 0.7:
        eps, ranks = float(rng.choice([1e-3, 1e-4, 1e-5, 1e-6, 1e-7])), None
    else:
        eps, ranks = None, tuple(int(x) for x in rng.integers(1, min(n, R, 200), size=3))
    wide = bool(rng.random() < 0.5)
p = make_random_params(n, R, seed=50000 + target, eps=eps, ranks=ranks,
                       a_range=(0.05, 400.0) if wide else (0.5, 20.0), signed=bool(target % 2))
U1, U2, U3, xi = make_config(p)
o = orh([U1, U2, U3], xi, eps=eps, ranks=ranks)
g = rhosvd.c2t([torch.as_tensor(u, device="cuda") for u in (U1, U2, U3)], torch.as_tensor(xi, device="cuda"), eps=eps, ranks=ranks)
print("case", target, "n", n, "R", R, "eps", eps, "ranks", ranks, "gpu", g.ranks, "block", g.report["block"], "refines", g.report.get("refines"))
for l in range(3):
    Z = g.Z[l].cpu().numpy(); sg = g.sigma[l].cpu().numpy(); so = o.sigma[l][:o.ranks[l]]
    C = Z.T @ Z - np.eye(Z.shape[1])
    colerr = np.max(np.abs(C), axis=0)
    badc = np.where(colerr > 1e-13)[0]
    rel = np.abs(sg - so) / np.maximum(so, 1e-300)
    print(f" mode {l}: orth max {np.abs(C).max():.2e}, bad cols {badc[:10]} (n={len(badc)}), sigma rel max {rel.max():.2e} at {rel.argmax()}, "
          f"sigma_g[-3:] {sg[-3:]}, sigma_o[-3:] {so[-3:]}, sigma_o[0] {so[0]:.3e}, numerical rank (oracle sigma > 1e-14 s1) {(o.sigma[l] > 1e-14*o.sigma[l][0]).sum()}")
