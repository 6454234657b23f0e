#!/bin/bash
# one round-state call: GPU tests, smoke, bench (both arms), launch list
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
python __graft_entry__.py smoke > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
python bench.py > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err; echo "bench rc=$?" >> gpurun_out/r2_bench_c4.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_c4_reference_arm.json 2> gpurun_out/r2_bench_ref.err
# launch list of the library's own kernels (names start with k_): the bench's timed kernel, the
# other-config kernels, the parity check's complex128 plans and the plan-time table kernels
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 400 --csv --log-file gpurun_out/r2_bench_c4_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_list.log 2>&1
tail -3 gpurun_out/r2_pytest_gpu.log; tail -2 gpurun_out/r2_smoke.log; cat gpurun_out/r2_bench_c4.json
