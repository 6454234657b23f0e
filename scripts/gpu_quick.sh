#!/bin/bash
# tests + sweep of the main configs (fast iteration loop)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python scripts/sweep.py --configs ${CONFIGS:-1a,1b,2,3,4} --methods ${METHODS:-fft,chirp} > gpurun_out/sweep_$TAG.log 2>&1
echo done
