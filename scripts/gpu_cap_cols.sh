set -u
mkdir -p gpurun_out
name=${NAME:-r2_c2_large_cols}
python scripts/run_config.py --config 2 --method chirp --reps 2 > gpurun_out/${name}_plain.log 2>&1 || { echo plain failed; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_large_cols -s ${SKIP:-1} -c 1 -f -o gpurun_out/$name python scripts/run_config.py --config 2 --method chirp --reps 2 > gpurun_out/${name}_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/$name.ncu-rep > gpurun_out/${name}_ncu_full_summary.txt 2>&1
ncu -i gpurun_out/$name.ncu-rep --page details --csv > gpurun_out/${name}_ncu_details.csv 2>/dev/null
python scripts/ncu_hot.py gpurun_out/$name.ncu-rep 60 > gpurun_out/${name}_ncu_hot.txt 2>&1
rm -f gpurun_out/$name.ncu-rep
cat gpurun_out/${name}_ncu_full_summary.txt
