#!/bin/bash
# FP32 march A/B: parity subset on the new kernel (each config), then
# scripts/fp32_timing.py per variant ("V:CFG": PD_MARCH32_V, PD_M32B_CFG).
mkdir -p gpurun_out
N=${N:-1024}
timeout 120 python scripts/fp32_timing.py --n 256 --steps 5 > gpurun_out/fp32_probe.log 2>&1 || { echo "FP32 probe FAILED"; tail -5 gpurun_out/fp32_probe.log; exit 1; }
for c in ${CFGS:-0}; do
  PD_M32B_CFG=$c timeout 400 python -m pytest -q -m gpu -x tests/test_march32.py tests/test_gpu_parity.py tests/test_fuzz_parity.py > gpurun_out/fp32_pytest_$c.log 2>&1; echo "pytest cfg $c: $(tail -1 gpurun_out/fp32_pytest_$c.log)"
done
for x in ${VARS:-"14 43:0"}; do
  v=${x%%:*}; c=${x#*:}; [ "$c" = "$x" ] && c=0
  PD_MARCH32_V=$v PD_M32B_CFG=$c timeout 300 python scripts/fp32_timing.py --n $N --steps 100 > gpurun_out/fp32_t_${v}_$c.log 2>&1
  echo "$x: $(grep float32 gpurun_out/fp32_t_${v}_$c.log)"
done
if [ -n "$NCU32" ]; then
  PD_M32B_CFG=$NCU32 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ftcs_march32 -s 3 -c 1 -o gpurun_out/fp32_ncu_$NCU32 -f python scripts/fp32_timing.py --n $N --steps 5 > gpurun_out/fp32_ncu.log 2>&1
fi
