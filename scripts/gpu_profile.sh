#!/bin/bash
# Full default bench + launch list + ncu full capture of the step kernel at the bench config.
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_default.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ftcs_march -s 3 -c 1 -o gpurun_out/march2048 -f python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu2048.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_ref.log
grep "^{" gpurun_out/bench_default.log | tail -1; grep "^{" gpurun_out/bench_ref.log | tail -1
