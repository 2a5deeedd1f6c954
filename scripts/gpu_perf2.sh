#!/bin/bash
# tests + smoke + occupancy A/B at 512^3 + 2048^3 bench + ncu of the step kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --n 512 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench512_occ4.log 2>&1
PD_MARCH_OCC=3 timeout 600 python bench.py --n 512 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench512_occ3.log 2>&1
timeout 1500 python bench.py --n 2048 --steps 10 --warmup 3 --no-e2e --cpu-sample 192 > gpurun_out/bench2048.log 2>&1; echo "bench exit $?" >> gpurun_out/bench2048.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ftcs_march -s 3 -c 1 -o gpurun_out/march512 -f python bench.py --n 512 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu512.log 2>&1
for f in bench512_occ4 bench512_occ3 bench2048; do python -c "
import json;l=[x for x in open('gpurun_out/$f.log') if x.startswith('{')][-1];d=json.loads(l);print('$f', d['ms_per_step'], d['value'], d['roofline']['achieved'], d['roofline']['frac'])"; done
