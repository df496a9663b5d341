#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/t_tests.log
tail -3 gpurun_out/t_tests.log
for k in 1 3 5; do timeout 600 python tools/run_config.py --config $k --reps 2 --t2c 1e-6 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], d['ranks'], d['t2c'])"; done
