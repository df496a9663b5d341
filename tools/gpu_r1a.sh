#!/bin/bash
# round-1 GPU session A: env + FP64 peak, GPU tests, per-config timing, bench line,
# launch list of the bench command, one ncu --set full capture of the core kernel.
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
(nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv; nproc; lscpu | grep -E "Model name|^CPU\(s\)") > gpurun_out/a_env.txt 2>&1
timeout 120 ./build/fp64_peak > gpurun_out/a_fp64_peak.json 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/a_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/a_tests.log
for k in 1 2 3 4 5; do timeout 600 python tools/run_config.py --config $k --reps 3 > gpurun_out/a_cfg$k.log 2>&1; done
timeout 900 python bench.py > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err; echo "bench exit $?" >> gpurun_out/a_bench.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/a_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/a_launches_bench.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/a_ncu_launch.log 2>&1
timeout 600 python tools/run_config.py --config 4 --reps 1 > gpurun_out/a_plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:core_kr_kernel -c 1 \
   -o gpurun_out/a_core_cfg4 python tools/run_config.py --config 4 --reps 1 > gpurun_out/a_ncu_full.log 2>&1
timeout 600 python tools/run_config.py --config 5 --reps 1 > gpurun_out/a_plain3.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dmma_gemm_kernel -s 0 -c 2 \
   -o gpurun_out/a_gemm_cfg5 python tools/run_config.py --config 5 --reps 1 > gpurun_out/a_ncu_full5.log 2>&1
tail -3 gpurun_out/a_tests.log; for k in 1 2 3 4 5; do tail -1 gpurun_out/a_cfg$k.log | cut -c1-600; done; cat gpurun_out/a_bench.json | cut -c1-3000; cat gpurun_out/a_fp64_peak.json
