#!/bin/bash
# r1u: launch list of the bench and ncu --set full of both core launches (main, then edge alone)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/u_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/u_ncu1.log 2>&1; echo "ncu1 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:core_kr_tma -c 1 \
   -o gpurun_out/u_core_main python tools/run_config.py --config 4 --reps 1 > gpurun_out/u_ncu2.log 2>&1; echo "ncu2 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:core_kr_tma --launch-skip 1 -c 1 \
   -o gpurun_out/u_core_edge python tools/run_config.py --config 4 --reps 1 > gpurun_out/u_ncu3.log 2>&1; echo "ncu3 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tma_gemm_kernel -c 1 \
   -o gpurun_out/u_gram_cfg5 python tools/run_config.py --config 5 --reps 1 > gpurun_out/u_ncu4.log 2>&1; echo "ncu4 $?"
