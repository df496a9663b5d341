"""Where the e2e time goes on cfg 4: pinned H2D / D2H bandwidth, c2t_raw vs the Python c2t."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2201_12663_b200 import rhosvd
from workloads import make_config, make_params

dev = torch.device("cuda", 0)
p = make_params(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
U1, U2, U3, xi = make_config(p, backend="torch", device=dev)
hU = [u.cpu().pin_memory() for u in (U1, U2, U3)]
st = torch.cuda.current_stream(dev)


def tm(f, reps=2):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(reps):
        f()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) * 1e3 / reps


nb = sum(u.numel() * 8 for u in hU)
ms, w = tm(lambda: [u.to(dev, non_blocking=True) for u in hU])
print(f"H2D pinned {nb / 1e9:.2f} GB: {ms:.1f} ms ({nb / ms / 1e6:.1f} GB/s) wall {w:.1f}")
big = torch.empty(2_245_000_000 // 8, dtype=torch.float64, device=dev)
hb = torch.empty(big.shape, dtype=torch.float64, pin_memory=True)
ms, w = tm(lambda: hb.copy_(big, non_blocking=True))
print(f"D2H pinned {big.numel() * 8 / 1e9:.2f} GB: {ms:.1f} ms ({big.numel() * 8 / ms / 1e6:.1f} GB/s) wall {w:.1f}")
del big
opts = rhosvd.make_opts(eps=p.eps, ranks=p.ranks)
L = rhosvd.lib()
ms, w = tm(lambda: L.rhosvd_result_free(rhosvd.c2t_raw((U1, U2, U3), xi, opts, None, st)))
print(f"c2t_raw: {ms:.1f} ms wall {w:.1f}")
ms, w = tm(lambda: rhosvd.c2t((U1, U2, U3), xi, eps=p.eps, ranks=p.ranks, keep_w=False))
print(f"c2t (python, outputs copied to torch): {ms:.1f} ms wall {w:.1f}")

# the bench's e2e step, piece by piece
hx = xi.cpu().pin_memory()
pinned = {}


def to_host(t, key):
    h = pinned.get(key)
    if h is None or h.shape != t.shape:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        pinned[key] = h
    h.copy_(t, non_blocking=True)
    return h


def e2e_step(parts):
    t0 = time.perf_counter()
    dU = [u.to(dev, non_blocking=True) for u in hU]
    dx = hx.to(dev, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    res = rhosvd.c2t(dU, dx, eps=p.eps, ranks=p.ranks, keep_w=False)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    outs = [to_host(res.beta, "beta")] + [to_host(z, f"Z{i}") for i, z in enumerate(res.Z)] + \
           [to_host(s, f"s{i}") for i, s in enumerate(res.sigma)]
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    parts.append((t1 - t0, t2 - t1, t3 - t2))


for i in range(3):
    parts = []
    e2e_step(parts)
    print("e2e step h2d %.1f ms, c2t %.1f ms, d2h %.1f ms" % tuple(1e3 * x for x in parts[0]))
