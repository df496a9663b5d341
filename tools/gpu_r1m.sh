#!/bin/bash
# eigensolver restructure: parity + per-config timing
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/m_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/m_tests.log
tail -4 gpurun_out/m_tests.log
for k in 1 2 3 4 5; do RHOSVD_DEBUG=0 timeout 600 python tools/run_config.py --config $k --reps 2 > gpurun_out/m_cfg$k.log 2>&1; tail -1 gpurun_out/m_cfg$k.log | cut -c1-420; done
