#!/bin/bash
# Round-2 check: new parity tests first, then the whole GPU suite, smoke and
# the default bench (ours + reference arm).
mkdir -p gpurun_out
{ nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,clocks.sm --format=csv; nproc; free -g; } > gpurun_out/env.txt 2>&1
timeout 900 python -m pytest -q -m gpu tests/test_headline_parity.py tests/test_frap.py tests/test_bench_multi.py -x > gpurun_out/pytest_new.log 2>&1; echo "exit $?" >> gpurun_out/pytest_new.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_ref.log
tail -3 gpurun_out/pytest_new.log; tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; grep "^{" gpurun_out/bench_default.log | tail -1 | cut -c1-600; grep "^{" gpurun_out/bench_ref.log | tail -1 | cut -c1-300
