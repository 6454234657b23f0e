#!/bin/bash
# tensor-core direct kernel: parity tests + config-3 timing (direct vs chirp)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-dtc}
timeout 240 python -m pytest tests/test_gpu_direct_tc.py -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 240 python -m pytest tests/test_gpu_direct.py -x -q >> gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python scripts/sweep.py --configs 3 --methods chirp,direct > gpurun_out/sweep_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_$TAG.log
