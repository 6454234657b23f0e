#!/bin/bash
# ncu --set full of one launch of the persistent kernel for one config/method
# (after the same command ran clean without ncu).  CFG, METHOD, TAG, LIBV.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-cfg}
[ -n "$LIBV" ] && export ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx$LIBV.so
CMD="python scripts/sweep.py --configs ${CFG:-1a} --methods ${METHOD:-fft} --reps 2"
$CMD > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_fft_persist} -s ${SKIP:-3} -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo done
