#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/n_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/n_tests.log
tail -3 gpurun_out/n_tests.log
for k in 1 2 3 4 5; do timeout 600 python tools/run_config.py --config $k --reps 3 > gpurun_out/n_cfg$k.log 2>&1; tail -1 gpurun_out/n_cfg$k.log | cut -c1-330; done
timeout 900 python bench.py > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err; echo "bench exit $?"; cut -c1-1500 gpurun_out/n_bench.json
