"""Block Jacobi timing probe: RHOSVD_TS=1 prints per-phase times of jacobi_block_kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2201_12663_b200 import rhosvd

for b in [int(x) for x in sys.argv[1:]] or [64, 300, 732]:
    rng = np.random.default_rng(b)
    # graded spectrum like W W^T: eigenvalues over 7 decades, random eigenvectors
    Q, _ = np.linalg.qr(rng.normal(size=(b, b)))
    lam = np.logspace(0, -7, b)
    A = (Q * lam) @ Q.T
    A = torch.as_tensor((A + A.T) / 2, device="cuda")
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lam_g, V, sw = rhosvd.syevj(A)
        e1.record()
        torch.cuda.synchronize()
        print(f"b={b} rep {rep}: {e0.elapsed_time(e1):.3f} ms sweeps {sw}", flush=True)
