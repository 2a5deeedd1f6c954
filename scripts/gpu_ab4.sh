#!/bin/bash
# A/B of march variants "V[:CFG]" (PD_MARCH_V with PD_M30_CFG / PD_M31_CFG):
# the parity subset on every CAND entry, then interleaved benches and one ncu
# metric pass per VARS entry.
# usage: VARS="30:5 31:0 31:1" CANDS="31:0 31:1" bash scripts/gpu_ab4.sh
mkdir -p gpurun_out
VARS=${VARS:-"30:5 31:0"}
CANDS=${CANDS:-"31:0"}
run() { local v=${1%%:*}; local st=${1#*:}; [ "$st" = "$1" ] && st=""; PD_MARCH_V=$v PD_M30_CFG=${st:-5} PD_M31_CFG=${st:-0} PD_M43_PF=${st:-3} "${@:2}"; }
# a new kernel that hangs must not eat the call: 2-minute probe first, and
# variants that fail it are dropped from the benches
OK=""
for x in $VARS; do
  if run $x timeout 120 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ab_probe_${x/:/_}.log 2>&1; then OK="$OK $x"; else echo "probe $x FAILED"; fi
done
VARS=$OK
for x in $CANDS; do
  case " $VARS " in *" $x "*) ;; *) continue;; esac
  run $x timeout 300 python -m pytest -q -m gpu -x tests/test_gpu_parity.py tests/test_fuzz_parity.py tests/test_headline_parity.py tests/test_gpu_kats.py tests/test_march32.py tests/test_gpu_shard.py > gpurun_out/ab_pytest_${x/:/_}.log 2>&1; echo "exit $?" >> gpurun_out/ab_pytest_${x/:/_}.log
done
for rep in 1 2; do for x in $VARS; do
  run $x timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/ab_bench_${x/:/_}_$rep.log 2>&1
done; done
M=smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,smsp__warps_eligible.avg.per_cycle_active,launch__registers_per_thread,lts__t_sector_op_read_hit_rate.pct
for x in $VARS; do
  run $x timeout 600 ncu --metrics $M --clock-control none -k regex:ftcs_march -s 3 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_ncu_${x/:/_}.csv 2>&1
done
if [ -n "$NCU_FULL" ]; then
  run $NCU_FULL timeout 900 ncu --set full --clock-control none --import-source on -k regex:ftcs_march -s 3 -c 1 -o gpurun_out/ab_full_${NCU_FULL/:/_} -f python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_full.log 2>&1
fi
for x in $CANDS; do echo "pytest $x: $(tail -2 gpurun_out/ab_pytest_${x/:/_}.log | tr '\n' ' ')"; done
for f in gpurun_out/ab_bench_*; do echo $f $(grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['kernel_ms_per_step'],3), d['clocks']['sm_mhz'])"); done
for x in $VARS; do echo "== $x"; grep -E '"(smsp__inst|gpu__time|dram__bytes|sm__issue|smsp__warps|launch__reg|lts__t)' gpurun_out/ab_ncu_${x/:/_}.csv | awk -F'","' '{print $(NF-2), $NF}'; done
