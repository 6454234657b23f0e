#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in $VARIANTS; do
  [ "$v" = "default" ] && v=""
  echo "== libasx$v" >> gpurun_out/acc.log
  ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx$v.so python scripts/diag_c64_fullbatch.py >> gpurun_out/acc.log 2>&1
  ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx$v.so python scripts/sweep.py --configs 4 --methods chirp,fft >> gpurun_out/acc.log 2>&1
done
