#!/bin/bash
# r1s: mode-stream priorities x GEMM grid waves (cfg 4 and 5 totals)
for cfg in 4 5; do
for pr in 0 1; do for wv in 1 0 3; do
  RHOSVD_MODE_PRIO=$pr RHOSVD_GEMM_WAVES=$wv timeout 600 python tools/run_config.py --config $cfg --reps 3 2>/dev/null | tail -1 | \
   python -c "import json,sys;d=json.loads(sys.stdin.read());print($cfg, 'prio', $pr, 'waves', $wv, d['ranks'], round(d['ms']['total'],1), 'gram', round(d['gram_ms'],1), 'eig', round(d['ms']['eigensolve'],1), 'core', round(d['core_ms'],1))"
done; done; done
