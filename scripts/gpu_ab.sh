#!/bin/bash
# A/B of march-kernel variants selected by environment settings.
#   VARIANTS="A:PD_MARCH_XSIDE=1 B:" bash scripts/gpu_ab.sh
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/ab_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/ab_pytest.log; tail -2 gpurun_out/ab_pytest.log
fi
for v in $VARIANTS; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5 --no-cpu --no-e2e} > gpurun_out/ab_$name.log 2>&1
  env $envs timeout 600 ncu --metrics $M --clock-control none -k regex:ftcs_march -s 3 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e ${NCU_ARGS} > gpurun_out/ab_${name}_ncu.csv 2>&1
  echo "== $name ($envs)"; grep "^{" gpurun_out/ab_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  ms/step %.3f  GPts/s %.1f  frac %.3f'%(d['ms_per_step'], d['value'], d['roofline']['frac']))"
  grep -h -E "gpu__time|dram__bytes|hit_rate|inst_exec|issue_active" gpurun_out/ab_${name}_ncu.csv | awk -F'","' '{print "  ",$(NF-2), $NF}'
done
