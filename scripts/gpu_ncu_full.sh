#!/bin/bash
# ncu --set full of the bench's dominant kernel, after the same command ran
# clean without ncu (a separate gpurun call from gpu_measure.sh).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-r1}
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-alt --no-other-configs ${BENCH_ARGS:-}"
$CMD > gpurun_out/plain2_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_fft_persist} -s 3 -c 1 -o gpurun_out/prof_bench_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
