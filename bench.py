#!/usr/bin/env python
"""Benchmark of the RHOSVD canonical-to-Tucker hot path (BASELINE.json metric:
"RHOSVD canonical terms/s and FP64 tensor-pipe % of peak at 1/2/4/8 B200").

One "step" = one full rhosvd_c2t call (normalize, Gram, eigensolve, one-sided
Rayleigh-Ritz + refinement, rank selection, projection, core, and the NCCL
all-reduces when R-sharded) on the BASELINE.json workload (default cfg 4:
n = 2048, R = 48 000 multi-particle Newton potential, eps = 1e-5), inputs
resident in HBM (2.36 GB > L2, so no L2 flush is needed between steps).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (R-sharded, strong scaling)

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (the
reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RHOSVD canonical terms/s"
UNIT = "terms/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="terms in the oracle sample (0 = auto)")
    ap.add_argument("--cpu-full", action="store_true", help="time the oracle on the FULL configuration (minutes)")
    ap.add_argument("--cpu-only", action="store_true", help="only the cpu_baseline leg (writes its JSON)")
    ap.add_argument("--report", default="", help="write per-phase report JSON here (rank 0)")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    # nvidia-smi in loop mode during the timed region.  The period is 1 s: at 200 ms the
    # driver queries cost ~17 ms per 965-ms step (host launches of the latency-bound
    # eigensolver stall behind them); RHOSVD_BENCH_CLOCK_MS overrides it.
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", os.environ.get("RHOSVD_BENCH_CLOCK_MS", "1000")],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm_sorted = sorted(sm)
        med = sm_sorted[len(sm_sorted) // 2] if sm_sorted else None
        return {"sm_mhz": med, "sm_max_mhz": max(mx) if mx else None, "samples": len(sm),
                "power_w_max": max(pw) if pw else None, "reasons": sorted(reasons)}


# ---------------------------------------------------------------- FP64 peak
def fp64_peak():
    """Measured DMMA (mma.sync.m8n8k4.f64) peak from tools/fp64_peak.cu."""
    exe = os.path.join(ROOT, "build", "fp64_peak")
    try:
        if not os.path.exists(exe):
            from paper_2201_12663_b200.build import build_tools
            build_tools()
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as e:  # pragma: no cover
        return {"error": str(e)}


# ---------------------------------------------------------------- oracle sample (cpu_baseline / reference arm)
def oracle_ranks(cfg):
    """The full problem's eps-ranks as the ORACLE found them (tests/golden/oracle_cfg{k}.json,
    written by tools/make_oracle_fixtures.py from oracle/ only); None if not recorded."""
    try:
        return tuple(json.load(open(os.path.join(ROOT, "tests", "golden", f"oracle_cfg{cfg}.json")))["ranks"])
    except Exception:
        return None


def oracle_sample(cfg, sample_terms, full=False):
    """Time the CPU oracle (oracle.rhosvd as it stands) on config `cfg`.

    full=False: the first `sample_terms` terms with the ranks FIXED to the full problem's
    oracle eps-ranks, so the per-term work (the core's 2 r1 r2 r3 FLOP per term, 96 % of
    cfg 4) matches the full configuration; an eps-mode run on a sample would pick smaller
    ranks (cfg 4, 4000 terms: [499, 501, 502]) and about half the per-term work.
    Returns (terms, seconds, ranks, per-phase seconds, how)."""
    from oracle import rhosvd as oracle_rhosvd
    from workloads import make_config, make_params
    p = make_params(cfg)
    Rs = p.R if full else min(p.R, sample_terms)
    U1, U2, U3, xi = make_config(p, 0, Rs)
    ranks, eps = p.ranks, p.eps
    how = "eps mode (the configuration's own rule)" if p.eps is not None else "the configuration's fixed ranks"
    # untimed tiny oracle call: LAPACK's first-call set-up (~1 s) is not the oracle's work
    from workloads import make_random_params
    q = make_random_params(96, 300, seed=1, ranks=(3, 3, 3))  # large enough for threaded BLAS
    oracle_rhosvd(list(make_config(q)[:3]), make_config(q)[3], ranks=q.ranks)
    if not full and Rs < p.R and p.eps is not None and oracle_ranks(cfg):
        ranks, eps = oracle_ranks(cfg), None
        how = f"ranks fixed to the full problem's oracle eps-ranks {list(ranks)} (per-term work matched)"
    tm = {}
    t0 = time.perf_counter()
    o = oracle_rhosvd([U1, U2, U3], xi, eps=eps, ranks=ranks, timings=tm)
    dt = time.perf_counter() - t0
    return Rs, dt, o.ranks, tm, how


def default_sample(cfg):
    return {1: 200, 2: 2400, 3: 7260, 4: 4000, 5: 4000}[cfg]


def host_info():
    info = {"nproc": os.cpu_count(), "affinity": cpu_cores()}
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                info["cpu_model"] = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [{k: d.get(k) for k in ("internal_api", "version", "num_threads", "threading_layer")}
                        for d in threadpool_info() if d.get("user_api") == "blas"]
    except Exception:
        pass
    return info


def cpu_baseline_entry(cfg, sample_terms, full=False):
    from workloads import make_params
    p = make_params(cfg)
    Rs, dt, oranks, tm, how = oracle_sample(cfg, sample_terms, full=full)
    what = "all" if Rs == p.R else f"first {Rs} of"
    return {"value": Rs / dt, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
            "sample": f"{what} {p.R} terms of {p.name} (n={p.n}); {how}; oracle ranks {list(oranks)}; {dt:.2f} s",
            "phase_s": {k: round(v, 3) for k, v in tm.items()}, "seconds": dt, "terms": Rs, "host": host_info()}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args):
    """Reference arm of this tier: the CPU oracle as it stands, on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from workloads import make_params
    p = make_params(args.config)
    Rs = args.cpu_sample or default_sample(args.config)
    for _ in range(max(0, min(args.warmup, 1))):
        oracle_sample(args.config, Rs, full=args.cpu_full)
    times = []
    for _ in range(args.steps):
        Rs_, dt, ranks, tm, how = oracle_sample(args.config, Rs, full=args.cpu_full)
        times.append(dt)
    tot = sum(times)
    val = Rs_ * args.steps / tot
    what = "all" if Rs_ == p.R else f"first {Rs_} of"
    sample = f"{what} {p.R} terms of {p.name} (n={p.n}); {how}; oracle ranks {list(ranks)}"
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": p.name, "config_index": args.config, "n": p.n,
                                        "R": p.R, "eps": p.eps, "sample_terms": Rs_},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle", "sample": sample,
                         "phase_s_last": {k: round(v, 3) for k, v in tm.items()}, "host": host_info()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def max_over_ranks(ms, dev=None):
    """Max of a per-rank time over all ranks (bench contract: max over ranks)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(ms)], dtype=torch.float64, device=dev)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2201_12663_b200 import rhosvd
    from workloads import make_config, make_params, shard_bounds

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, (world, args.gpus)
    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = world > 1
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
    lib = rhosvd.lib()
    p = make_params(args.config)
    k0, k1 = shard_bounds(p.R, world, rank)
    U1, U2, U3, xi = make_config(p, k0, k1, backend="torch", device=dev)
    comm = rhosvd.Comm.nccl() if distributed else None
    opts = rhosvd.make_opts(eps=p.eps, ranks=p.ranks)
    stream = torch.cuda.current_stream(dev)

    def step():
        h = rhosvd.c2t_raw((U1, U2, U3), xi, opts, comm, stream)
        return h

    def report_of(h):
        rep = rhosvd.Report()
        lib.rhosvd_result_report(h, rhosvd.C.byref(rep))
        return rhosvd._report_dict(rep)

    cold_ms = None
    for wi in range(args.warmup):
        if wi == 0:  # the cold first call (workspace / output allocation) reported separately
            torch.cuda.synchronize(dev)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
        h = step()
        if wi == 0:
            c1.record(stream)
        last = report_of(h)
        lib.rhosvd_result_free(h)
        if wi == 0:
            torch.cuda.synchronize(dev)
            cold_ms = c0.elapsed_time(c1)
    torch.cuda.synchronize(dev)
    if distributed:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = []
    # inputs smaller than 2x the 126 MB L2 (cfg 1 / 2): flush L2 before every timed step by
    # writing a 512 MB buffer, outside the step's events (the steps' times are summed)
    in_bytes = 3 * p.n * (k1 - k0) * 8
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev) if in_bytes < 2 * 126 * 2 ** 20 else None
    st_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    en_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e0.record(stream)
    for i in range(args.steps):
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.fill_(float(i))
        st_ev[i].record(stream)
        h = step()
        en_ev[i].record(stream)
        reps.append(report_of(h))
        lib.rhosvd_result_free(h)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    step_seq = [st_ev[i].elapsed_time(en_ev[i]) for i in range(args.steps)]
    per_step = sorted(step_seq)
    clk = clocks.stop()
    ms_max = max_over_ranks(sum(step_seq) if flush is not None else e0.elapsed_time(e1), dev)
    value = p.R * args.steps / (ms_max * 1e-3)

    # dominant kernel roofline (FP64 DMMA pipe): the one with the larger share of the step
    # (the core K7 on cfg 2/4, the Gram K1 on cfg 3/5)
    rep = reps[-1]
    r1, r2, r3 = rep["ranks"]
    Rl = k1 - k0
    core_flops = 2.0 * r1 * r2 * r3 * Rl
    gram_flops = 3.0 * p.n * (p.n + 1) * Rl  # upper-triangle Gram, 3 modes
    core_ms = sum(r["core_ms"] for r in reps) / len(reps)
    gram_ms = sum(r["gram_ms"] for r in reps) / len(reps)
    if core_ms >= gram_ms:
        dom, fl, kms = "core_kr (K7)", core_flops, core_ms
    else:
        dom, fl, kms = "gram (K1)", gram_flops, gram_ms
    peak = fp64_peak() if rank == 0 else {}
    peak_tf = peak.get("dmma_tflops")
    achieved = fl / (kms * 1e-3) / 1e12 if kms > 0 else None
    traffic, traffic_src = None, None
    try:  # DRAM bytes per launch of the dominant kernel from the committed ncu capture
        tj = json.load(open(os.path.join(ROOT, "profiles", "r1_traffic.json")))
        key = "core (K7) cfg4" if dom.startswith("core") else "tma_gemm_kernel<128,128,0,0> (Gram)"
        if key in tj and (args.config == 4 if dom.startswith("core") else args.config == 5):
            traffic, traffic_src = tj[key]["bytes"], tj[key]["capture"]
    except Exception:
        pass
    roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
            "frac": (achieved / peak_tf) if (achieved and peak_tf) else None, "traffic": traffic,
            "traffic_unit": "bytes per call of the dominant kernel (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                            "summed over its launches in one call, like achieved)",
            "traffic_source": traffic_src,
            "peak_source": "measured DMMA m8n8k4.f64 microbenchmark (tools/fp64_peak.cu) on this GPU; "
                           "MEASURED_PEAKS.json has no FP64 entry",
            "peak_detail": peak, "algorithmic_flop_per_launch": fl, "kernel_ms": kms,
            "other": {"gram_tflops": gram_flops / (gram_ms * 1e-3) / 1e12 if gram_ms > 0 else None,
                      "core_tflops": core_flops / (core_ms * 1e-3) / 1e12 if core_ms > 0 else None,
                      "gram_ms": gram_ms, "core_ms": core_ms}}

    # ---- e2e: host buffers through the C-ABI host entry point rhosvd_c2t_host (H2D of the
    # inputs from pinned memory and D2H of beta / Z / sigma inside the timed region; the
    # library overlaps both with compute)
    e2e = None
    if not args.no_e2e:
        hU = [u.cpu().pin_memory() for u in (U1, U2, U3)]
        hx = xi.cpu().pin_memory()
        h2d = sum(u.numel() * 8 for u in hU) + hx.numel() * 8
        d2h = 0
        dbg = os.environ.get("RHOSVD_E2E_DEBUG") == "1"
        sink = []

        def e2e_step():
            nonlocal d2h
            t0 = time.perf_counter()
            res = rhosvd.c2t_host(hU, hx, eps=p.eps, ranks=p.ranks, comm=comm, device=dev)
            # read the results on the host (the call returns once they are there)
            sink.append(float(res.beta.view(-1)[-1]) + sum(float(s.sum()) for s in res.sigma))
            d2h = res.beta.numel() * 8 + sum(z.shape[0] * z.shape[1] * 8 for z in res.Z) + \
                sum(s.numel() * 8 for s in res.sigma)
            res.close()
            if dbg:
                print(f"[e2e] step {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr)

        e2e_step()
        torch.cuda.synchronize(dev)
        if distributed:
            dist.barrier()
        ks = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        q0 = torch.cuda.Event(enable_timing=True)
        q1 = torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for _ in range(ks):
            e2e_step()
        q1.record(stream)
        torch.cuda.synchronize(dev)
        ems = max_over_ranks(q0.elapsed_time(q1), dev)
        e2e = {"value": p.R * ks / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": ks, "wall_s": time.perf_counter() - t0,
               "api": "rhosvd_c2t_host (C ABI, host buffers)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_entry(args.config, args.cpu_sample or default_sample(args.config), full=args.cpu_full)
        # the full-configuration oracle run of the same workload on this pool's host cores,
        # measured once by `bench.py --cpu-full` (profiles/r2_oracle_full_cfg{k}.json): context
        try:
            full = json.load(open(os.path.join(ROOT, "profiles", f"r2_oracle_full_cfg{args.config}.json")))
            cpu["full_config_run"] = {k: full.get(k) for k in ("value", "seconds", "sample", "phase_s", "host")}
            cpu["full_config_run"]["source"] = f"profiles/r2_oracle_full_cfg{args.config}.json (bench.py --cpu-full)"
        except Exception:
            pass

    if rank == 0:
        launches = sum(r["launches"] for r in reps)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": p.name, "config_index": args.config, "n": p.n, "R": p.R,
                       "eps": p.eps, "ranks": p.ranks, "parallelism": f"R-sharded x{world}",
                       "l2": ("inputs (3 n R fp64 = %.3f GB per rank) smaller than 2x L2: L2 flushed (512 MB "
                              "write) before every timed step, outside the timed steps" if flush is not None else
                              "inputs (3 n R fp64 = %.2f GB per rank) larger than L2; no flush") % (in_bytes / 1e9)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "step_ms": {"median": per_step[len(per_step) // 2], "min": per_step[0], "max": per_step[-1],
                        "cold_first_call": cold_ms, "in_order": [round(x, 2) for x in step_seq],
                        "note": "this rank's per-step CUDA-event times"},
            "clocks": clk,
            "result": {"ranks": rep["ranks"], "block": rep["block"], "iters": rep["iters"],
                       "tail": rep["tail"], "beta_norm": rep["beta_norm"], "phase_ms": rep["ms"],
                       "gemm_tflop_executed": rep["gemm_flops"] / 1e12},
        }
        print(json.dumps(line), flush=True)
        if args.report:
            with open(args.report, "w") as f:
                json.dump({"reports": reps, "line": line}, f, indent=1)
    if comm is not None:
        comm.close()
    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_ranks(args):
    """`bench.py --gpus N` without a torchrun environment: start N ranks (one process per
    GPU, NCCL) through torch.distributed.run on 127.0.0.1 with the same arguments, and
    return its exit code.  Rank 0 prints the JSON line; NCCL_DEBUG=INFO (unless set) puts
    each rank's communicator lines on stderr."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "0") or 0)
    if args.gpus > 1 and world == 0:
        return launch_ranks(args)
    if world and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    if args.cpu_only:
        print(json.dumps(cpu_baseline_entry(args.config, args.cpu_sample or default_sample(args.config),
                                            full=args.cpu_full)), flush=True)
        return 0
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
