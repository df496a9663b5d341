"""Per-config table: GPU rhosvd_c2t time (median of reps, CUDA events inside the library)
and the CPU oracle on the same host (one run, wall clock), terms/s for both.

    python tools/config_table.py --configs 1 2 3 5 --reps 5
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 5])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2201_12663_b200 import rhosvd
    from workloads import make_config, make_params
    lib = rhosvd.lib()
    for k in args.configs:
        p = make_params(k)
        dev = torch.device("cuda:0")
        U1, U2, U3, xi = make_config(p, backend="torch", device=dev)
        opts = rhosvd.make_opts(eps=p.eps, ranks=p.ranks)
        ts = []
        for i in range(args.reps + 2):
            h = rhosvd.c2t_raw((U1, U2, U3), xi, opts)
            rep = rhosvd.Report()
            lib.rhosvd_result_report(h, rhosvd.C.byref(rep))
            lib.rhosvd_result_free(h)
            if i >= 2:
                ts.append(rep.ms[8])
        gms = float(np.median(ts))
        line = {"config": k, "name": p.name, "n": p.n, "R": p.R, "ranks": list(rep.ranks), "gpu_ms": gms,
                "gpu_terms_per_s": p.R / (gms * 1e-3)}
        if not args.no_oracle:
            from oracle import rhosvd as oracle_rhosvd
            Uh = make_config(p)
            t0 = time.perf_counter()
            o = oracle_rhosvd(list(Uh[:3]), Uh[3], eps=p.eps, ranks=p.ranks)
            dt = time.perf_counter() - t0
            line.update({"oracle_s": dt, "oracle_terms_per_s": p.R / dt, "oracle_ranks": list(o.ranks),
                         "host_cores": len(os.sched_getaffinity(0)), "speedup": dt / (gms * 1e-3)})
        print(json.dumps(line), flush=True)
        del U1, U2, U3, xi
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
