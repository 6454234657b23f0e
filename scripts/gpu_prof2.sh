#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in "" _v2; do
CMD="python scripts/sweep.py --configs 4 --methods chirp --batch 2048 --reps 1"
ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx$v.so $CMD > gpurun_out/plain$v.log 2>&1 && \
ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx$v.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_persist -s 3 -c 1 -o gpurun_out/prof_chirp4$v $CMD > gpurun_out/ncu$v.log 2>&1
done
CMD="python scripts/sweep.py --configs 1a --methods fft --batch 1024 --reps 1"
$CMD > gpurun_out/plain_1a.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft_persist -s 3 -c 1 -o gpurun_out/prof_afft1a $CMD > gpurun_out/ncu_1a.log 2>&1
echo done
