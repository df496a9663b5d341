#!/bin/bash
# session C: core kernel v2 (TMA + mbarrier ring, flattened KR rows, persistent)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k core > gpurun_out/d_core_tests.log 2>&1; echo "core tests exit $?" >> gpurun_out/d_core_tests.log
tail -5 gpurun_out/d_core_tests.log
grep -q "exit 0" gpurun_out/d_core_tests.log || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/d_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/d_tests.log
tail -3 gpurun_out/d_tests.log
for k in 2 4 5; do timeout 600 python tools/run_config.py --config $k --reps 2 > gpurun_out/d_cfg$k.log 2>&1; tail -1 gpurun_out/d_cfg$k.log | cut -c1-500; done
timeout 600 python tools/run_config.py --config 4 --reps 1 > gpurun_out/d_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:core_kr_tma -c 1 \
   -o gpurun_out/d_core_cfg4 python tools/run_config.py --config 4 --reps 1 > gpurun_out/d_ncu.log 2>&1
echo ncu $?
