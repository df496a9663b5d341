"""Run rhosvd_c2t on a BASELINE.json config (inputs generated on the GPU) and
print the per-phase report; used for ncu launch lists and quick timing.

    python tools/run_config.py --config 2 --reps 2
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
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--block0", type=int, default=0)
    ap.add_argument("--oversample", type=int, default=16)
    ap.add_argument("--t2c", type=float, default=None, help="also time rhosvd_t2c with this eps_rel")
    ap.add_argument("--als", type=int, default=None, help="call rhosvd_c2t_als with this many sweeps")
    args = ap.parse_args()
    import torch
    from paper_2201_12663_b200 import rhosvd
    from workloads import make_config, make_params
    p = make_params(args.config)
    dev = torch.device("cuda:0")
    U1, U2, U3, xi = make_config(p, backend="torch", device=dev)
    lib = rhosvd.lib()
    opts = rhosvd.make_opts(eps=p.eps, ranks=p.ranks, block0=args.block0, oversample=args.oversample)
    for i in range(args.reps):
        t0 = time.perf_counter()
        h = rhosvd.c2t_raw((U1, U2, U3), xi, opts, als_sweeps=args.als)
        rep = rhosvd.Report()
        lib.rhosvd_result_report(h, rhosvd.C.byref(rep))
        t2c = None
        if args.t2c is not None:
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cp = rhosvd.C.c_void_p()
            e0.record()
            st = lib.rhosvd_t2c(h, args.t2c, rhosvd._stream_ptr(None), rhosvd.C.byref(cp))
            e1.record()
            torch.cuda.synchronize()
            if st == 0:
                Rc = rhosvd.C.c_int64()
                lib.rhosvd_cp_rank(cp, rhosvd.C.byref(Rc))
                ea, th, e2, sw = (rhosvd.C.c_double(), rhosvd.C.c_double(), rhosvd.C.c_double(), rhosvd.C.c_int32())
                lib.rhosvd_cp_info(cp, rhosvd.C.byref(ea), rhosvd.C.byref(th), rhosvd.C.byref(e2), rhosvd.C.byref(sw))
                t2c = {"ms": e0.elapsed_time(e1), "R": int(Rc.value), "eps_abs": ea.value, "thr": th.value,
                       "err": e2.value ** 0.5, "max_sweeps": int(sw.value)}
                lib.rhosvd_cp_free(cp)
            else:
                t2c = {"error": lib.rhosvd_last_error().decode()}
        lib.rhosvd_result_free(h)
        torch.cuda.synchronize()
        d = rhosvd._report_dict(rep)
        d["wall_s"] = time.perf_counter() - t0
        print(json.dumps({"config": args.config, "rep": i, "als": args.als, **{k: d[k] for k in
                          ("ranks", "block", "iters", "grow_events", "ms", "core_ms", "gram_ms", "launches",
                           "gemm_flops", "wall_s", "tail", "beta_norm")}, "t2c": t2c}), flush=True)


if __name__ == "__main__":
    main()
