#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python tools/run_config.py --config 4 --reps 1 > gpurun_out/z_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:core_kr_tma -c 1 \
   -o gpurun_out/z_core_cfg4 python tools/run_config.py --config 4 --reps 1 > gpurun_out/z_ncu.log 2>&1; echo "ncu $?"
