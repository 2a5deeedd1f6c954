#!/bin/bash
# A/B of compiled library variants (scripts/build_variant.sh NAME; selected by
# PD_LIB_VARIANT): parity subset on each variant, then interleaved benches and
# one ncu metric pass each. "base" = the in-tree library.
# usage: VARIANTS="base b2 b6" bash scripts/gpu_variants.sh
mkdir -p gpurun_out
VARIANTS=${VARIANTS:-"base"}
run() { if [ "$1" = base ]; then "${@:2}"; else PD_LIB_VARIANT=$1 "${@:2}"; fi; }
OK=""
for v in $VARIANTS; do
  if run $v timeout 120 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/var_probe_$v.log 2>&1; then OK="$OK $v"; else echo "probe $v FAILED"; fi
done
for v in $OK; do
  run $v timeout 300 python -m pytest -q -m gpu -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_headline_parity.py tests/test_fuzz_parity.py > gpurun_out/var_pytest_$v.log 2>&1; echo "pytest $v: $(tail -1 gpurun_out/var_pytest_$v.log)"
done
for rep in 1 2; do for v in $OK; do
  run $v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/var_bench_${v}_$rep.log 2>&1
  echo "$v $rep $(grep '^{' gpurun_out/var_bench_${v}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['kernel_ms_per_step'],3), d['clocks']['sm_mhz'])")"
done; done
for v in $OK; do
  echo "$v ncu: $(run $v timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none -k regex:ftcs_march -s 3 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E '"(gpu__time|smsp__inst|dram__bytes_read)' | awk -F'","' '{printf "%s=%s ", $(NF-2), $NF}')"
done
