#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/p_tests.log
tail -3 gpurun_out/p_tests.log
for k in 1 2 3 4 5; do timeout 600 python tools/run_config.py --config $k --reps 3 > gpurun_out/p_cfg$k.log 2>&1; tail -1 gpurun_out/p_cfg$k.log | cut -c1-330; done
timeout 900 python bench.py > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err; echo "bench exit $?"; cut -c1-600 gpurun_out/p_bench.json
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_ncu.log 2>&1; echo "ncu $?"
