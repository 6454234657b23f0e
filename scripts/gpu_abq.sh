#!/bin/bash
# quick A/B of library variants on one config/method (device-time sweep)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-abq}
rm -f gpurun_out/abq_$TAG.log
for v in $VARIANTS; do
  [ "$v" = "default" ] && v=""
  echo "== variant '$v'" >> gpurun_out/abq_$TAG.log
  ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx$v.so timeout 300 python scripts/sweep.py --configs ${CONFIGS:-1a} --methods ${METHODS:-fft} --reps ${REPS:-20} --batch ${BATCH:-0} >> gpurun_out/abq_$TAG.log 2>&1
done
if [ -n "$PYTEST" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu $PYTEST_ARGS > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
fi
echo done
