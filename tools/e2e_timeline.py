"""Per-mode event timeline of rhosvd_c2t_host on a BASELINE config (RHOSVD_TIMELINE=1
prints it): where the host path's extra time over the device path goes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2201_12663_b200 import rhosvd  # noqa: E402
from workloads import make_config, make_params  # noqa: E402

p = make_params(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
U1, U2, U3, xi = make_config(p, backend="torch", device=torch.device("cuda"))
hU = [u.cpu().pin_memory() for u in (U1, U2, U3)]
hx = xi.cpu().pin_memory()
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h = rhosvd.c2t_host(hU, hx, eps=p.eps, ranks=p.ranks)
    e1.record()
    torch.cuda.synchronize()
    print(f"[rep {rep}] c2t_host {e0.elapsed_time(e1):.1f} ms", file=sys.stderr, flush=True)
    h.close()
