#!/bin/bash
# A/B of library variants: full-batch complex64 accuracy (config 4) and the
# device-time sweep, per variant; then the GPU parity suite on the default lib.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-ab}
rm -f gpurun_out/ab_$TAG.log
for v in $VARIANTS; do
  [ "$v" = "default" ] && v=""
  echo "== variant '$v'" >> gpurun_out/ab_$TAG.log
  export ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx$v.so
  [ "${ACC_BATCH:-65536}" != 0 ] && timeout 300 python scripts/diag_c64_fullbatch.py ${ACC_BATCH:-65536} >> gpurun_out/ab_$TAG.log 2>&1
  timeout 600 python scripts/sweep.py --configs ${CONFIGS:-1a,1b,3,4} --methods ${METHODS:-fft,chirp} >> gpurun_out/ab_$TAG.log 2>&1
done
unset ASX_LIB_PATH
if [ -n "$PYTEST" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
fi
echo done
