#!/bin/bash
# GPU call: tests, smoke, A/B bench at 512^3, full bench at 2048^3, ncu of the step kernel.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
PD_NO_MARCH=1 timeout 600 python bench.py --n 512 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench512_tile.log 2>&1
timeout 600 python bench.py --n 512 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench512_march.log 2>&1
timeout 1500 python bench.py --n 2048 --steps 10 --warmup 3 > gpurun_out/bench2048.log 2>&1; echo "bench exit $?" >> gpurun_out/bench2048.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ftcs_march -s 3 -c 1 -o gpurun_out/march512 -f python bench.py --n 512 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu512.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches512.csv python bench.py --n 512 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/launches512.log 2>&1
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 600 gpurun_out/bench512_tile.log; tail -c 600 gpurun_out/bench512_march.log; tail -c 1500 gpurun_out/bench2048.log
