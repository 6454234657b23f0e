# timing-only ablations of k_direct_tc2 (make variant VNAME=abN VFLAGS=-DASX_DTC2_ABLATE=N)
for v in "" $(ls paper_2403_16665_b200/ | sed -n 's/^libasx\(_ab[0-9a-z_]*\)\.so$/\1/p'); do
  echo "variant $v"; ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx$v.so timeout 120 python scripts/run_config.py --config 3 --reps 6 | tail -1
done
