#!/bin/bash
# Measurement-only bracketing of the march kernel (PD_MARCH_DBG bits, v31):
# 8 = compute warps skip the arithmetic, 16 = producer copies nothing,
# 32 = producer copies the own slabs only (no halos). Kernel ms under ncu.
mkdir -p gpurun_out
V=${V:-31}; CFG=${CFG:-0}
for d in ${DBGS:-0 8 16 24 32 40}; do
  PD_MARCH_V=$V PD_M31_CFG=$CFG PD_MARCH_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none -k regex:ftcs_march -s 3 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/dbg_${CFG}_$d.csv 2>&1
  echo "dbg $d: $(grep -E '"(gpu__time|dram__bytes_read|smsp__inst)' gpurun_out/dbg_${CFG}_$d.csv | awk -F'","' '{printf "%s=%s ", $(NF-2), $NF}')"
done
