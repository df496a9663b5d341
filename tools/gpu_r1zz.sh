#!/bin/bash
# r1zz: final bench line, launch list and core ncu captures after the ring fix
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/zz_bench.json 2> gpurun_out/zz_bench.err; echo "bench $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/zz_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/zz_ncu1.log 2>&1; echo "ncu1 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:core_kr_tma -c 1 \
   -o gpurun_out/zz_core_main python tools/run_config.py --config 4 --reps 1 > gpurun_out/zz_ncu2.log 2>&1; echo "ncu2 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:core_kr_tma --launch-skip 1 -c 1 \
   -o gpurun_out/zz_core_edge python tools/run_config.py --config 4 --reps 1 > gpurun_out/zz_ncu3.log 2>&1; echo "ncu3 $?"
