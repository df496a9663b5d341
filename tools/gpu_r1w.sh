#!/bin/bash
# fresh evidence for profiles/: launch list of the bench command, full captures of core + Gram
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/w_bench.json 2> gpurun_out/w_bench.err; echo "bench exit $?"; cut -c1-300 gpurun_out/w_bench.json
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/w_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/w_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/w_ncu1.log 2>&1; echo "ncu1 $?"
python tools/run_config.py --config 4 --reps 1 > gpurun_out/w_plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"core_kr_tma|tma_gemm_kernel" -c 4 \
   -o gpurun_out/w_full_cfg4 python tools/run_config.py --config 4 --reps 1 > gpurun_out/w_ncu2.log 2>&1; echo "ncu2 $?"
python tools/run_config.py --config 5 --reps 1 > gpurun_out/w_plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tma_gemm_kernel" -c 1 \
   -o gpurun_out/w_gram_cfg5 python tools/run_config.py --config 5 --reps 1 > gpurun_out/w_ncu3.log 2>&1; echo "ncu3 $?"
