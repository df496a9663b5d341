#!/bin/bash
# r1p2: per-phase timeline of cfg 4 and ncu --set full of the 144-wide core edge launch alone
mkdir -p gpurun_out
RHOSVD_TIMELINE=1 timeout 600 python tools/run_config.py --config 4 --reps 3 > gpurun_out/p2_timeline.log 2>&1; echo "tl $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:core_kr_tma --launch-skip 1 -c 1 \
   -o gpurun_out/p2_core144 python tools/run_config.py --config 4 --reps 1 > gpurun_out/p2_ncu.log 2>&1; echo "ncu $?"
