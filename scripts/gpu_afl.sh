#!/bin/bash
# k_afft_local A/B: config 1a device time with / without the group-local
# kernel, then the GPU parity tests that exercise it.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-afl}
timeout 300 python scripts/sweep.py --configs 1a --methods fft > gpurun_out/afl_$TAG.log 2>&1
ASX_NO_AFFT_LOCAL=1 timeout 300 python scripts/sweep.py --configs 1a --methods fft >> gpurun_out/afl_$TAG.log 2>&1
timeout 600 python -m pytest tests -x -q -m gpu ${PYK:-} > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
echo done
