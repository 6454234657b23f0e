#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in "" _v2; do
  echo "== variant libasx$v" >> gpurun_out/sweep_variants.log
  ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx$v.so timeout 600 python scripts/sweep.py --configs 1a,1b,3,4 --methods fft,chirp >> gpurun_out/sweep_variants.log 2>&1
done
echo done
