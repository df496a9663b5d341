"""Bitwise repeatability of the blocked Cholesky inverse on a rank-deficient Gram (many
dependent columns: pivots below delta)."""
import hashlib, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2201_12663_b200 import rhosvd
b = int(sys.argv[1]) if len(sys.argv) > 1 else 600
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
rng = np.random.default_rng(b)
M = rng.normal(size=(2 * b, b // 2)) @ rng.normal(size=(b // 2, b))   # rank b/2
M += 1e-9 * rng.normal(size=M.shape)
S = torch.as_tensor(M.T @ M, device="cuda")
out = {}
for i in range(reps):
    Bp = rhosvd.chol_inv(S)
    h = hashlib.sha1(Bp.cpu().numpy().tobytes()).hexdigest()[:12]
    out[h] = out.get(h, 0) + 1
print(b, out, flush=True)
