#!/bin/bash
# Round-2 ncu captures of the hot kernels (one GPU, each only after the plain run exited 0):
#   gpurun --timeout 1500 -- bash scripts/gpu_profile.sh
# Writes text summaries (raw-page summary, details CSV, hottest SASS lines) into gpurun_out/; copy them into profiles/.
set -u
mkdir -p gpurun_out
cap() {  # name config method kernel-regex [extra run_config args]
  local name=$1 cfg=$2 method=$3 kre=$4; shift 4
  python scripts/run_config.py --config $cfg --method $method --reps 2 "$@" > gpurun_out/${name}_plain.log 2>&1 || { echo "$name plain run failed"; return; }
  ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 -f -o gpurun_out/$name \
      python scripts/run_config.py --config $cfg --method $method --reps 2 "$@" > gpurun_out/${name}_ncu.log 2>&1
  python scripts/ncu_summary.py gpurun_out/$name.ncu-rep > gpurun_out/${name}_ncu_full_summary.txt 2>&1
  ncu -i gpurun_out/$name.ncu-rep --page details --csv > gpurun_out/${name}_ncu_details.csv 2>/dev/null
  python scripts/ncu_hot.py gpurun_out/$name.ncu-rep 25 > gpurun_out/${name}_ncu_hot.txt 2>&1
  rm -f gpurun_out/$name.ncu-rep  # the reports exceed gpurun's 64 MiB return limit; the text exports stay
  head -4 gpurun_out/${name}_ncu_full_summary.txt
}
cap r2_c4_chirp_r32 4 chirp k_chirp_r32
cap r2_c1a_afft_local 1a fft k_afft_local
cap r2_c1b_chirp_local128 1b chirp k_chirp_local128
cap r2_c3_direct_tc 3 direct k_direct_tc
cap r2_c2_large_rows 2 chirp k_large_rows
cap r2_c4_fft_recursion 4 fft k_fft_persist
