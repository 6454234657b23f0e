#!/bin/bash
# packed-FP32x2 A/B: device-time sweep of variant builds (VARIANTS="_nopk _pk1 ...")
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in ${VARIANTS:-_nopk _pk1}; do
  echo "== lib$v" >> gpurun_out/pk_sweep.log
  ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx$v.so timeout 600 python scripts/sweep.py --configs ${CONFIGS:-3,4} --methods ${METHODS:-chirp} >> gpurun_out/pk_sweep.log 2>&1
done
