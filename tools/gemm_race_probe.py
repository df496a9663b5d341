"""Bitwise repeatability of the GEMM engine: the cfg-3 refinement shapes (column edge +
split-K) issued back to back on ONE stream (the kernel-level entry points share one
split-K scratch, so they must not run on several streams at once) while a cuBLAS DGEMM
loop on a second stream contends for the SMs; compared with a result computed alone."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2201_12663_b200 import rhosvd  # noqa: E402

torch.manual_seed(0)
dev = torch.device("cuda")
# (M_py, K, N_py): the library sees M = N_py, N = M_py (145 / 147: the column edge), every
# transpose combination (all four operand layouts of the engine)
shapes = [(145, 7260, 2048), (145, 2048, 7260), (147, 7260, 2048)]
ops = []
for (M, K, N) in shapes:
    for ta in (False, True):
        for tb in (False, True):
            A = torch.randn(*((K, M) if ta else (M, K)), dtype=torch.float64, device=dev)
            B = torch.randn(*((N, K) if tb else (K, N)), dtype=torch.float64, device=dev)
            ops.append((A, B, ta, tb, rhosvd.dgemm(A, B, transa=ta, transb=tb)))
torch.cuda.synchronize()
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
X = torch.randn(4096, 4096, dtype=torch.float64, device=dev)
bad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    outs = []
    with torch.cuda.stream(s1):
        for _ in range(it % 3):
            X @ X
    with torch.cuda.stream(s0):
        for (A, B, ta, tb, _) in ops:
            outs.append(rhosvd.dgemm(A, B, transa=ta, transb=tb, stream=s0))
    torch.cuda.synchronize()
    for q, (o, (_, _, _, _, ref)) in enumerate(zip(outs, ops)):
        if not torch.equal(o, ref):
            bad += 1
            d = (o - ref).abs()
            print("iter", it, "op", q, "differs: max", float(d.max()), "count", int((d > 0).sum()),
                  "first", [int(x) for x in (d > 0).nonzero()[0]], flush=True)
print("mismatches:", bad)
