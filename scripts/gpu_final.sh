bash scripts/gpu_round.sh > gpurun_out/final_round.log 2>&1
tail -3 gpurun_out/r2_pytest_gpu.log
python scripts/run_config.py --config 1a --method fft --reps 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_afft_local -s 1 -c 1 -f -o gpurun_out/r2_c1a_afft_local python scripts/run_config.py --config 1a --method fft --reps 2 > gpurun_out/r2_c1a_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/r2_c1a_afft_local.ncu-rep > gpurun_out/r2_c1a_afft_local_ncu_full_summary.txt 2>&1
ncu -i gpurun_out/r2_c1a_afft_local.ncu-rep --page details --csv > gpurun_out/r2_c1a_afft_local_ncu_details.csv 2>/dev/null
python scripts/ncu_hot.py gpurun_out/r2_c1a_afft_local.ncu-rep 25 > gpurun_out/r2_c1a_afft_local_ncu_hot.txt 2>&1
rm -f gpurun_out/*.ncu-rep
python scripts/run_config.py --config 3 --method direct --reps 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_direct_tc -s 1 -c 1 -f -o gpurun_out/r2_c3_direct_tc python scripts/run_config.py --config 3 --method direct --reps 2 > gpurun_out/r2_c3_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/r2_c3_direct_tc.ncu-rep > gpurun_out/r2_c3_direct_tc_ncu_full_summary.txt 2>&1
ncu -i gpurun_out/r2_c3_direct_tc.ncu-rep --page details --csv > gpurun_out/r2_c3_direct_tc_ncu_details.csv 2>/dev/null
python scripts/ncu_hot.py gpurun_out/r2_c3_direct_tc.ncu-rep 25 > gpurun_out/r2_c3_direct_tc_ncu_hot.txt 2>&1
rm -f gpurun_out/*.ncu-rep
head -5 gpurun_out/r2_c1a_afft_local_ncu_full_summary.txt; head -5 gpurun_out/r2_c3_direct_tc_ncu_full_summary.txt
python scripts/sweep.py --configs 2 --methods chirp,fft --reps 10 | cut -c1-160
