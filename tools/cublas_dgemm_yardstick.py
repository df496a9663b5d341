"""cuBLAS DGEMM 8192^3 yardstick (SURVEY.md 8(d) Metric 2 (iii)): torch.matmul on fp64 CUDA
tensors, CUDA events, clocks logged.  Never linked into the library - a reference point
for the FP64 tensor peak beside tools/fp64_peak.cu."""
import json
import subprocess

import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record()
for _ in range(reps):
    c = a @ b
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                     capture_output=True, text=True).stdout.strip()
print(json.dumps({"gemm": "cuBLAS DGEMM 8192^3 (torch.matmul fp64)", "ms": ms, "tflops": 2 * n ** 3 / ms / 1e9,
                  "sm_mhz_power_w_after": clk}))
