#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-v}
rm -f gpurun_out/sweep_$TAG.log
for v in $VARIANTS; do
  echo "== $v" >> gpurun_out/sweep_$TAG.log
  ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx$v.so timeout 600 python scripts/sweep.py --configs ${CONFIGS:-1a,1b,3,4} --methods ${METHODS:-fft,chirp} >> gpurun_out/sweep_$TAG.log 2>&1
done
echo done
