#!/bin/bash
# halo-traffic experiment (measurement only)
mkdir -p gpurun_out
for d in 0 1 2 4 7; do
  PD_MARCH_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct --clock-control none -k regex:ftcs_march -s 3 -c 1 --csv python bench.py --n 512 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/exp_dbg$d.csv 2>&1
done
for d in 0 7; do PD_MARCH_DBG=$d timeout 600 python bench.py --n 512 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/exp_bench$d.log 2>&1; done
grep -h -E "gpu__time|dram__bytes|hit_rate" gpurun_out/exp_dbg*.csv
