#!/bin/bash
# k_direct_tc: parity tests, then timing ablations (ASX_DTC_DBG bits; results wrong, timing only)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_direct_tc.py -x -q > gpurun_out/pytest_dtc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dtc.log
for d in ${DBGS:-0 1 2 3}; do
  echo "dbg=$d $(ASX_DTC_DBG=$d timeout 120 python scripts/sweep.py --configs 3 --methods direct | cut -c1-120)"
done > gpurun_out/dtc_ab.log 2>&1
