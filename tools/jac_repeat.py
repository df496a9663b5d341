"""Bitwise repeatability of the block Jacobi on a dense graded matrix (~20 sweeps)."""
import hashlib, os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2201_12663_b200 import rhosvd
b = int(sys.argv[1]) if len(sys.argv) > 1 else 600
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rng = np.random.default_rng(b)
Q, _ = np.linalg.qr(rng.normal(size=(b, b)))
lam = np.logspace(0, -9, b)
A = torch.as_tensor(((Q * lam) @ Q.T + ((Q * lam) @ Q.T).T) / 2, device="cuda")
out = {}
for i in range(reps):
    l, V, sw = rhosvd.syevj(A)
    h = hashlib.sha1(l.cpu().numpy().tobytes() + V.cpu().numpy().tobytes()).hexdigest()[:12]
    out[(h, sw)] = out.get((h, sw), 0) + 1
print(os.environ.get("RHOSVD_COOP_MAX", "-"), b, out, flush=True)
