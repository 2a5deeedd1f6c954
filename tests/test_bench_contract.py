"""bench.py's reference arm runs on the CPU (the reference compiled in place,
oracle/_ref) and must print exactly one JSON line with the contract's keys;
the N > 1 launch is exercised on the GPU by test_bench_multi.py."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line(ref):
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "0",
                        "--box", "256", "--cpu-sample", "24", "--cpu-seconds", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "GPts/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_reference_arm_loads_nothing_from_the_product(ref):
    """the reference arm must not import the product
    package nor map libporediff_b200.so (the driver voids vs_reference if it
    does)."""
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', "
            "'--box', '256', '--cpu-sample', '16', '--cpu-seconds', '0.2']; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "mods = [m for m in sys.modules if m.startswith('paper_2304_11165_b200')]; "
            "maps = open('/proc/self/maps').read(); "
            "print('MODS', mods, 'SO', 'libporediff_b200' in maps, 'REF', 'libporediff_ref' in maps)")
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    assert "MODS [] SO False REF True" in p.stdout, p.stdout[-2000:]
