#!/bin/bash
# round-end style session: GPU tests, smoke, ncu of k_direct_tc (config 3), bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
CMD="python scripts/sweep.py --configs 3 --methods direct --reps 2"
$CMD > gpurun_out/ncu_plain_dtc.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_direct_tc -s 2 -c 1 -o gpurun_out/prof_dtc_final $CMD > gpurun_out/ncu_dtc_final.log 2>&1
echo done
