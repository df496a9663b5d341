"""Time the DMMA GEMM engine at the refinement shapes of cfg 4 / cfg 5 (CUDA events)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2201_12663_b200 import rhosvd

L = rhosvd.lib()


def run(name, ta, tb, M, N, K, lda, ldb, ldc, a_el, b_el, reps=5):
    A = torch.randn(a_el, dtype=torch.float64, device="cuda")
    B = torch.randn(b_el, dtype=torch.float64, device="cuda")
    Cm = torch.empty(ldc * N, dtype=torch.float64, device="cuda")
    args = (ta, tb, M, N, K, 1.0, C.c_void_p(A.data_ptr()), lda, C.c_void_p(B.data_ptr()), ldb, 0.0,
            C.c_void_p(Cm.data_ptr()), ldc, rhosvd._stream_ptr(None))
    L.rhosvd_dgemm(*args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        L.rhosvd_dgemm(*args)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "ms": ms, "tflops": 2.0 * M * N * K / ms / 1e9}), flush=True)


n, b, R = 2048, 712, 48000
run("cfg4 W = Uh^T Z", b"T", b"N", R, b, n, n, n, R, n * R, n * b)
run("cfg4 M = Uh W^T", b"N", b"N", n, b, R, n, R, n, n * R, R * b)
run("cfg4 resid-shape Z W", b"N", b"T", n, R, b, n, R, n, n * b, b * R)
run("cfg4 G Z", b"N", b"N", n, b, n, n, n, n, n * n, n * b)
run("cfg4 SYRK Y^T Y", b"T", b"N", b, b, n, n, n, b, n * b, n * b)
n, b, R = 4096, 124, 100000
run("cfg5 W = Uh^T Z", b"T", b"N", R, b, n, n, n, R, n * R, n * b)
run("cfg5 M = Uh W^T", b"N", b"N", n, b, R, n, R, n, n * R, R * b)
