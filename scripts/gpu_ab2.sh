#!/bin/bash
# A/B of march kernel versions (PD_MARCH_V): parity subset on the candidate,
# interleaved bench runs, and a short ncu metric capture of each.
# usage: VERS="14 20" bash scripts/gpu_ab2.sh
mkdir -p gpurun_out
VERS=${VERS:-"14 20"}
CAND=${CAND:-20}
PD_MARCH_V=$CAND timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_parity.py tests/test_fuzz_parity.py tests/test_headline_parity.py tests/test_gpu_kats.py tests/test_march32.py tests/test_gpu_shard.py > gpurun_out/ab_pytest.log 2>&1; echo "exit $?" >> gpurun_out/ab_pytest.log
for rep in 1 2; do for v in $VERS; do
  PD_MARCH_V=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/ab_bench_v${v}_$rep.log 2>&1
done; done
M=smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,smsp__warps_eligible.avg.per_cycle_active,launch__registers_per_thread,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
for v in $VERS; do
  PD_MARCH_V=$v timeout 600 ncu --metrics $M --clock-control none -k regex:ftcs_march -s 3 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_ncu_v$v.csv 2>&1
done
tail -3 gpurun_out/ab_pytest.log
for f in gpurun_out/ab_bench_v*; do echo $f $(grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['kernel_ms_per_step'],3), d['clocks']['sm_mhz'])"); done
for v in $VERS; do echo v$v; grep -E '"(smsp__inst|gpu__time|dram__bytes|sm__issue|smsp__warps|launch__reg|l1tex)' gpurun_out/ab_ncu_v$v.csv | awk -F'","' '{print $(NF-2), $NF}'; done
