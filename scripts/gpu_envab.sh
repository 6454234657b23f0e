#!/bin/bash
# A/B of an environment switch (ENVVAR=1 vs unset) on one sweep, then the GPU tests
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-envab}
rm -f gpurun_out/envab_$TAG.log
for r in 1 2; do
  timeout 300 python scripts/sweep.py --configs ${CONFIGS:-1b} --methods ${METHODS:-chirp} --reps ${REPS:-20} >> gpurun_out/envab_$TAG.log 2>&1
  env ${ENVVAR:-ASX_NO_LOCAL}=1 timeout 300 python scripts/sweep.py --configs ${CONFIGS:-1b} --methods ${METHODS:-chirp} --reps ${REPS:-20} | sed 's/^/B /' >> gpurun_out/envab_$TAG.log 2>&1
done
if [ -n "$PYTEST" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu $PYTEST_ARGS > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
fi
echo done
