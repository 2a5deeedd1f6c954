#!/bin/bash
mkdir -p gpurun_out
for d in 0 1 2 4 7; do
  PD_MARCH_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_ltcfabric.sum --clock-control none -k regex:ftcs_march -s 3 -c 1 --csv python bench.py --n 512 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/exp2_dbg$d.csv 2>&1
done
# also a plain copy kernel reference: torch copy of 1 GiB
python - > gpurun_out/exp2_copy.txt 2>&1 <<'PY'
import torch,time
a=torch.empty(2**27,dtype=torch.float64,device='cuda'); b=torch.empty_like(a)
for _ in range(3): b.copy_(a)
torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(10): b.copy_(a)
e1.record(); e1.synchronize(); ms=e0.elapsed_time(e1)/10
print("copy GB/s", 2*a.numel()*8/ms/1e6)
PY
for d in 0 1 2 4 7; do echo "dbg=$d"; grep -h -E "gpu__time|dram__bytes|hit_rate|srcunit" gpurun_out/exp2_dbg$d.csv | awk -F'","' '{print "  ",$(NF-2), $NF}'; done
cat gpurun_out/exp2_copy.txt
