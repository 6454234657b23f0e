#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; tail -3 gpurun_out/t_pytest.log
ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx_tl.so python scripts/timeline.py --config 1a > gpurun_out/tl_1a.txt 2>&1
ASX_LIB_PATH=$PWD/paper_2403_16665_b200/libasx_tl.so python scripts/timeline.py --config 4 --batch 32768 > gpurun_out/tl_4.txt 2>&1
tail -5 gpurun_out/tl_1a.txt; tail -5 gpurun_out/tl_4.txt
