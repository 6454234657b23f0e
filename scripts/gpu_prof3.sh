#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out

CMD="python scripts/sweep.py --configs 4 --methods chirp --batch 2048 --reps 1"
$CMD > gpurun_out/plain_p3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_persist -s 3 -c 1 -o gpurun_out/prof_chirp4_v3 $CMD > gpurun_out/ncu_p3.log 2>&1
echo done
