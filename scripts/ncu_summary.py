"""Summarise an ncu report: key throughput metrics, stall reasons per issue,
and the per-instruction hot spots (needs -lineinfo / --import-source)."""
import csv, subprocess, sys, io

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0  # e.g. chunks per launch
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_op_read_hit_rate.pct", "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
        "smsp__warps_eligible.avg.per_cycle_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second"]
for k, x in zip(h, v):
    if k in want:
        print(f"{k:70s} {x}")
print("-- stalls per issue")
st = [(k, float(x)) for k, x in zip(h, v) if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
for k, x in sorted(st, key=lambda t: -t[1])[:12]:
    print(f"  {k[34:-23]:30s} {x:.3f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
ia, isrc, iss = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
data = [x for x in rows[2:] if len(x) > ia and x[ia].isdigit()]
tot = sum(int(x[ia]) for x in data)
print(f"-- {tot} warp instructions, {tot/units:.1f} per unit")
from collections import Counter
c = Counter()
for x in data:
    o = x[isrc].split()
    op = o[1] if o[0].startswith("@") else o[0]
    c[op.split(".")[0]] += int(x[ia])
print("  " + ", ".join(f"{k} {n/units:.0f}" for k, n in c.most_common(16)))
samp = sorted(data, key=lambda x: -int(x[iss]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 15]
tots = sum(int(x[iss]) for x in data)
print(f"-- top stall-sampled instructions (of {tots} samples)")
for x in samp:
    print(f"  {int(x[iss]):7d} {int(x[ia])/units:6.2f}  {x[isrc][:90]}")
