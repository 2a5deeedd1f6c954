#!/bin/bash
# bench-only sweep over environment settings (no ncu): VARIANTS="name:ENV=.. name2:ENV=.."
mkdir -p gpurun_out
for v in $VARIANTS; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5 --no-cpu --no-e2e} > gpurun_out/sw_$name.log 2>&1
  grep "^{" gpurun_out/sw_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', '%.3f ms  %.1f GPts/s  frac %.3f  clk %s' % (d['ms_per_step'], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz']))" || tail -3 gpurun_out/sw_$name.log
done
