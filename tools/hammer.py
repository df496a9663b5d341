"""GPU load generator for race hunting: fp64 GEMMs in a loop for N seconds."""
import sys
import time
import torch
t_end = time.time() + float(sys.argv[1] if len(sys.argv) > 1 else 60)
a = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
while time.time() < t_end:
    a = (a @ a) * 1e-4
    torch.cuda.synchronize()
