#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/bb_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/bb_tests.log
tail -3 gpurun_out/bb_tests.log
timeout 900 python bench.py > gpurun_out/bb_bench.json 2> gpurun_out/bb_bench.err; echo "bench exit $?"
python3 -c "import json; d=json.load(open('gpurun_out/bb_bench.json')); print({k: d[k] for k in ['value','ms_per_step','gpu_launches']}, d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bb_ref.json 2>&1; echo "ref exit $?"; cut -c1-400 gpurun_out/bb_ref.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bb_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/bb_smoke.log
