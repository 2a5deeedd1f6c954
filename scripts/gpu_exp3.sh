#!/bin/bash
# Halo-class traffic attribution at the bench config (2048^3): PD_MARCH_DBG
# skips x(1) / y(2) / z(4) halo loads (numerically wrong, traffic only),
# plus one full capture with source for the instruction hot spots.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum
for d in 0 1 2 4 7; do
  PD_MARCH_DBG=$d timeout 600 ncu --metrics $M --clock-control none -k regex:ftcs_march -s 3 -c 1 --csv python bench.py ${EXP_ARGS:---steps 2 --warmup 3 --no-cpu --no-e2e} > gpurun_out/exp3_dbg$d.csv 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ftcs_march -s 3 -c 1 -o gpurun_out/march2048 -f python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu2048.log 2>&1
for d in 0 1 2 4 7; do echo "dbg=$d"; grep -h -E "gpu__time|dram__bytes|hit_rate|inst_exec|srcunit" gpurun_out/exp3_dbg$d.csv | awk -F'","' '{print "  ",$(NF-2), $NF}'; done
