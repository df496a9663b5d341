"""Per-call overhead outside the library's own phase timer: CUDA events on the caller's
stream around each rhosvd_c2t call vs the reported total, plus host wall time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_params

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p = make_params(k)
dev = torch.device("cuda:0")
U1, U2, U3, xi = make_config(p, backend="torch", device=dev)
lib = rhosvd.lib()
opts = rhosvd.make_opts(eps=p.eps, ranks=p.ranks)
st = torch.cuda.current_stream(dev)
for i in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    h = rhosvd.c2t_raw((U1, U2, U3), xi, opts, None, st)
    t1 = time.perf_counter()
    rep = rhosvd.Report()
    lib.rhosvd_result_report(h, rhosvd.C.byref(rep))
    lib.rhosvd_result_free(h)
    t2 = time.perf_counter()
    e1.record(st)
    torch.cuda.synchronize()
    d = rhosvd._report_dict(rep)
    print(f"cfg {k} call {i}: events {e0.elapsed_time(e1):.1f} ms, reported total {d['ms']['total']:.1f} ms, "
          f"host c2t {1e3 * (t1 - t0):.1f} ms, free {1e3 * (t2 - t1):.1f} ms", flush=True)
