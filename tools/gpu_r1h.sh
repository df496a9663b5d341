mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "syevj or chol" > gpurun_out/h_k.log 2>&1; tail -3 gpurun_out/h_k.log
timeout 300 python tools/bench_small.py
echo "--- smem kernel up to 160"
RHOSVD_JAC_SMEM_MAXB=160 timeout 300 python tools/bench_small.py 2>&1 | grep -E '"b": 1[24]'
