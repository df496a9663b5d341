#!/bin/bash
# r1r: cfg 4 start-block sweep (total / eigensolve / iterations / ranks)
for b0 in 0 256 384 512 640; do
  timeout 600 python tools/run_config.py --config 4 --reps 3 --block0 $b0 2>/dev/null | tail -1 | \
   python -c "import json,sys;d=json.loads(sys.stdin.read());print($b0, d['ranks'], d['block'], d['iters'], d['grow_events'], round(d['ms']['total'],1), round(d['ms']['eigensolve'],1), d['beta_norm'])"
done
