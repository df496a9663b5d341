"""Time the b x b kernels (Jacobi eigensolver, scaled Cholesky + inverse) through the
C ABI at the block sizes of the BASELINE configs (CUDA events, warm)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2201_12663_b200 import rhosvd
    rhosvd.lib()
    out = []
    for b in [124, 147, 298, 707]:
        rng = np.random.default_rng(b)
        A = rng.normal(size=(b, b))
        A = torch.as_tensor(A + A.T, device="cuda")
        E = rng.normal(size=(b, b)) * 0.01
        d = np.logspace(0, -5, b)
        Hg = torch.as_tensor(d[:, None] * (np.eye(b) + E + E.T) * d[None, :], device="cuda")
        for name, M in (("dense", A), ("graded_near_diag", Hg)):
            rhosvd.syevj(M)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            reps = 3
            for _ in range(reps):
                lam, V, sw = rhosvd.syevj(M)
            e1.record()
            torch.cuda.synchronize()
            out.append({"kernel": "syevj", "b": b, "input": name, "ms": e0.elapsed_time(e1) / reps, "sweeps": sw})
            print(json.dumps(out[-1]), flush=True)
        M = torch.as_tensor(rng.normal(size=(2048, b)), device="cuda")
        S = M.t() @ M
        rhosvd.chol_inv(S)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            rhosvd.chol_inv(S)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"kernel": "chol_inv", "b": b, "ms": e0.elapsed_time(e1) / 10}), flush=True)


if __name__ == "__main__":
    main()
