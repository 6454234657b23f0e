#!/bin/bash
# k_direct_tc with / without the scale warps' L2 prefetch (time + DRAM bytes), then the all-config sweep
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for d in 0 8 0 8; do
  echo "dbg=$d $(ASX_DTC_DBG=$d timeout 120 python scripts/sweep.py --configs 3 --methods direct | cut -c1-120)"
done > gpurun_out/dtc_pf.log 2>&1
for d in 0 8; do
  ASX_DTC_DBG=$d timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_direct_tc -s 2 -c 1 python scripts/sweep.py --configs 3 --methods direct --reps 2 > gpurun_out/dtc_pf_ncu_$d.log 2>&1
done
timeout 600 python scripts/sweep.py > gpurun_out/sweep_all.log 2>&1
