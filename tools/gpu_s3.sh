#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q > gpurun_out/s3_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/s3_tests.log
for k in 1 2 3 4 5; do timeout 600 python tools/run_config.py --config $k --reps 2 > gpurun_out/s3_cfg$k.log 2>&1; done
timeout 600 python tools/run_config.py --config 4 --reps 1 > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_launches_cfg4.csv python tools/run_config.py --config 4 --reps 1 > gpurun_out/s3_ncu.log 2>&1
tail -3 gpurun_out/s3_tests.log; for k in 1 2 3 4 5; do tail -1 gpurun_out/s3_cfg$k.log | cut -c1-700; done
