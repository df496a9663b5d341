#!/bin/bash
# r1o: bench line, launch list and ncu --set full of both core segments (BN 128 + 144-wide edge) on cfg 4
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/o_bench.json 2> gpurun_out/o_bench.err; echo "bench $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/o_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/o_ncu1.log 2>&1; echo "ncu1 $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:core_kr_tma -c 2 \
   -o gpurun_out/o_core_cfg4 python tools/run_config.py --config 4 --reps 1 > gpurun_out/o_ncu2.log 2>&1; echo "ncu2 $?"
