"""3-D tensor-product convolution timing (the paper's Table 1 "C*C" row analog):
rhosvd_conv3d of a rank-Ra density with a rank-Rp kernel on n^3 grids, CUDA events.
Ranks (reading C4): Ra = 100 (a reduced density, "R_rho ~ 10^2"),
Rp = 40 (a sinc-quadrature Newton kernel rank of the order the paper cites)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2201_12663_b200 import rhosvd

Ra, Rp = 100, 40
# warm the GPU (an idle B200 sits at 120 MHz; the first milliseconds run below max clock)
_w = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
for _ in range(20):
    _w = _w @ _w * 1e-3
torch.cuda.synchronize()
del _w
for n in [int(a) for a in sys.argv[1:]] or [1024, 2048, 4096, 8192, 16384]:
    g = torch.Generator(device="cuda").manual_seed(n)
    Fa = [torch.randn(Ra, n, dtype=torch.float64, device="cuda", generator=g) for _ in range(3)]
    Fp = [torch.randn(Rp, n, dtype=torch.float64, device="cuda", generator=g) for _ in range(3)]
    ca = torch.randn(Ra, dtype=torch.float64, device="cuda", generator=g)
    cp = torch.randn(Rp, dtype=torch.float64, device="cuda", generator=g)
    rhosvd.conv3d(Fa, ca, Fp, cp, 0.01)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        F, w = rhosvd.conv3d(Fa, ca, Fp, cp, 0.01)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 3 * 2.0 * n * n * Ra * Rp
    print(json.dumps({"n": n, "Ra": Ra, "Rp": Rp, "ms": ms, "tflops": fl / ms / 1e9}), flush=True)
    del F, w, Fa, Fp
    torch.cuda.empty_cache()
