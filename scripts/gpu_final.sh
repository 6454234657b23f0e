#!/bin/bash
# round-end call: the round state (tests, smoke, both bench arms, launch list), then the ncu captures of the shipped build
bash scripts/gpu_round.sh > gpurun_out/r2_round.log 2>&1
bash scripts/gpu_profile.sh > gpurun_out/r2_profile.log 2>&1
tail -3 gpurun_out/r2_pytest_gpu.log; tail -1 gpurun_out/r2_smoke.log; cat gpurun_out/r2_profile.log
