#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/s2_kernels.log 2>&1; echo "kernels exit $?" >> gpurun_out/s2_kernels.log
timeout 600 python tools/run_config.py --config 2 --reps 2 > gpurun_out/s2_cfg2.log 2>&1
timeout 900 python tools/run_config.py --config 4 --reps 2 > gpurun_out/s2_cfg4.log 2>&1
timeout 900 python tools/run_config.py --config 5 --reps 2 > gpurun_out/s2_cfg5.log 2>&1
timeout 600 python tools/run_config.py --config 2 --reps 1 > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_launches_cfg2.csv python tools/run_config.py --config 2 --reps 1 > gpurun_out/s2_ncu.log 2>&1
tail -3 gpurun_out/s2_kernels.log; cat gpurun_out/s2_cfg2.log gpurun_out/s2_cfg4.log gpurun_out/s2_cfg5.log | cut -c1-600
