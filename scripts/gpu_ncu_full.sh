#!/bin/bash
# One full ncu capture (with source) of the step kernel at the bench config.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ftcs_march -s 3 -c 1 -o gpurun_out/${NCU_NAME:-march} -f python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e ${NCU_ARGS} > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
