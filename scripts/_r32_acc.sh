mkdir -p gpurun_out
P=paper_2403_16665_b200
timeout 900 python -m pytest tests/test_gpu_r32.py -x -q 2>&1 | tail -2
for lib in libasx.so libasx_ptw.so; do
  echo "== $lib"
  ASX_LIB_PATH=$PWD/$P/$lib timeout 300 python scripts/run_config.py --config 4 --method chirp --reps 4 2>&1 | tail -2
  ASX_LIB_PATH=$PWD/$P/$lib timeout 600 python scripts/diag_c64_fullbatch.py 2>&1 | grep chirp
done
