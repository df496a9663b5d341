"""Measurement of the RS long-range front-end on the
multi-Slater lattices of PAPER.md Table 2 (n = 384): the device window kernel against the
HBM roofline, then RHOSVD C2T (eps_Tuck = 1e-3) and C2C (eps_T2C = 1e-5) of the long part.

    python tools/bench_rs.py [--reps 5]

One JSON line per lattice: R_ini, Tucker ranks, R_comp, the window kernel's time and
bandwidth (algorithmic bytes: the N R_l columns of three n-row side matrices written once +
xi, the (2n-1) R_l reference table written and read), and the C2T / C2C times (CUDA events).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    from paper_2201_12663_b200 import rhosvd
    from workloads import TABLE2_LATTICES, make_rs_lattice
    dev = torch.device("cuda:0")
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs")
    for L in TABLE2_LATTICES + [(12, 12, 4)]:
        lat = make_rs_lattice(L)
        t, w = rhosvd.sinc_slater(lat.lam, 0.75, 26, 1e-6)
        (tl, wl), _ = rhosvd.rs_split(t, w)
        idx = torch.as_tensor(lat.node_idx, device=dev)
        c = torch.as_tensor(lat.c, device=dev)
        # window kernel alone
        U = rhosvd.rs_lattice(tl, wl, lat.h, lat.n, idx, c)  # warm-up / allocation
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            U = rhosvd.rs_lattice(tl, wl, lat.h, lat.n, idx, c)
        e1.record()
        torch.cuda.synchronize()
        win_ms = e0.elapsed_time(e1) / args.reps
        Rl = len(tl)
        R = lat.N * Rl
        nbytes = 3 * R * lat.n * 8 + R * 8 + 2 * (2 * lat.n - 1) * Rl * 8 + lat.N * (12 + 8)
        # C2T and C2C of the long part
        g = rhosvd.c2t(list(U[:3]), U[3], eps=1e-3)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.reps):
            g = rhosvd.c2t(list(U[:3]), U[3], eps=1e-3)
        e1.record()
        torch.cuda.synchronize()
        c2t_ms = e0.elapsed_time(e1) / args.reps
        cp = rhosvd.c2c(list(U[:3]), U[3], 1e-5, eps=1e-3)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.reps):
            cp = rhosvd.c2c(list(U[:3]), U[3], 1e-5, eps=1e-3)
        e1.record()
        torch.cuda.synchronize()
        c2c_ms = e0.elapsed_time(e1) / args.reps
        print(json.dumps({"lattice": list(L), "N": lat.N, "R_l": Rl, "R_ini": R, "tucker": list(g.ranks),
                          "R_comp": cp.R, "window_ms": win_ms, "window_bytes": nbytes,
                          "window_GBps": nbytes / (win_ms * 1e-3) / 1e9,
                          "window_frac_hbm": (nbytes / (win_ms * 1e-3) / 1e9 / hbm) if hbm else None,
                          "hbm_peak_GBps": hbm, "c2t_ms": c2t_ms, "c2c_ms": c2c_ms}), flush=True)


if __name__ == "__main__":
    main()
