#!/bin/bash
# ncu launch list (gpu__time_duration only) of one config/method sweep run, after it ran clean without ncu
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-list}
CMD="python scripts/sweep.py --configs ${CFG:-2} --methods ${METHOD:-chirp} --reps 1"
$CMD > gpurun_out/list_plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/list_$TAG.csv $CMD > gpurun_out/list_ncu_$TAG.log 2>&1
echo done
