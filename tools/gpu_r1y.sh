#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/y_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/y_tests.log
tail -3 gpurun_out/y_tests.log
for k in 1 2 3 4 5; do timeout 600 python tools/run_config.py --config $k --reps 3 > gpurun_out/y_cfg$k.log 2>&1; tail -1 gpurun_out/y_cfg$k.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], d['ranks'], {k: round(v,1) for k,v in d['ms'].items()})"; done
for k in 2 4; do RHOSVD_SERIAL_MODES=1 timeout 600 python tools/run_config.py --config $k --reps 3 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('serial', d['config'], round(d['ms']['total'],1))"; done
