#!/bin/bash
# first GPU session: peaks, kernel unit tests, parity
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
(nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv; nproc; lscpu | grep -E "Model name|^CPU\(s\)") > gpurun_out/s1_env.txt 2>&1
timeout 120 ./build/fp64_peak > gpurun_out/s1_fp64_peak.json 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/s1_kernels.log 2>&1
echo "kernels exit $?" >> gpurun_out/s1_kernels.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not full_size" -s > gpurun_out/s1_parity.log 2>&1
echo "parity exit $?" >> gpurun_out/s1_parity.log
tail -5 gpurun_out/s1_kernels.log gpurun_out/s1_parity.log
cat gpurun_out/s1_fp64_peak.json
