import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2201_12663_b200 import rhosvd
for b in [732, 1500, 2048]:
    rng = np.random.default_rng(b)
    M = torch.as_tensor(rng.normal(size=(4096, b)), device="cuda")
    S = M.t() @ M
    rhosvd.chol_inv(S)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): rhosvd.chol_inv(S)
    e1.record(); torch.cuda.synchronize()
    print("b", b, "chol_inv ms", e0.elapsed_time(e1) / 3)
