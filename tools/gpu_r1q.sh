#!/bin/bash
# r1q: per-step times vs nvidia-smi sampling period
mkdir -p gpurun_out
for ms in 1000 5000 250 1000; do
  RHOSVD_BENCH_CLOCK_MS=$ms timeout 600 python bench.py --steps 8 --no-cpu-baseline --no-e2e > gpurun_out/q_$ms.json 2>/dev/null
  python -c "import json,sys;d=json.load(open('gpurun_out/q_$ms.json'));print($ms, round(d['value']), d['step_ms']['in_order'], d['clocks'].get('samples'))"
done
