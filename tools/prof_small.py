"""One syevj (b=707 dense) and one chol_inv (b=707) call, for ncu captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2201_12663_b200 import rhosvd

b = int(sys.argv[1]) if len(sys.argv) > 1 else 707
rng = np.random.default_rng(b)
A = rng.normal(size=(b, b))
A = torch.as_tensor(A + A.T, device="cuda")
rhosvd.syevj(A)
M = torch.as_tensor(rng.normal(size=(2048, b)), device="cuda")
rhosvd.chol_inv(M.t() @ M)
torch.cuda.synchronize()
print("ok")
