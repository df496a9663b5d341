"""Summarise an ncu --set full report (.ncu-rep) into the counters this repo's
roofline uses: duration, DRAM bytes, FP64 tensor-pipe (DMMA) utilisation,
issue activity, occupancy and the top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [algorithmic_flop_per_launch ...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read BW"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active % (of active cycles)"),
    ("sm__ops_path_tensor_src_fp64.sum", "FP64 tensor ops (FMA x2 incl. padding)"),
    ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "FP64 tensor ops % of peak (elapsed)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1/smem throughput %"),
]


def main(path, flops):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for li, r in enumerate(rows[2:]):
        d = dict(zip(h, r))
        un = dict(zip(h, u))
        name = d.get("Kernel Name", "?")
        print(f"== launch {li}: {name[:110]}")
        for k, lab in KEYS:
            if k in d:
                print(f"   {lab:45s} {d[k]:>20s} {un.get(k, '')}")
        st = [(k, float(d[k])) for k in d if k.startswith("smsp__average_warps_issue_stalled_")
              and k.endswith("_per_issue_active.ratio") and d[k] not in ("", "n/a")]
        st.sort(key=lambda x: -x[1])
        print("   top stalls (warps per issue):", ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
            for k, v in st[:6]))
        if li < len(flops) and "gpu__time_duration.sum" in d:
            t = float(d["gpu__time_duration.sum"])
            scale = {"s": 1.0, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9}
            t *= scale.get(un.get("gpu__time_duration.sum", "s"), 1.0)
            print(f"   algorithmic TFLOP/s (cold, under ncu)            {flops[li] / t / 1e12:20.2f}")


if __name__ == "__main__":
    main(sys.argv[1], [float(x) for x in sys.argv[2:]])
