#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for w in 2 4 8; do timeout 900 python scripts/peer_overhead.py --n 2048 --world $w --steps 10 --balance all > gpurun_out/peer_$w.txt 2>&1; done
tail -3 gpurun_out/pytest_gpu.log; grep -h "" gpurun_out/peer_*.txt | tail -20
