"""Every march kernel kept in the library (selected per process by
PD_MARCH_V / PD_M31_CFG / PD_M43_PF / PD_SCHED for FP64 and PD_MARCH32_V / PD_M32B_CFG for
FP32) reproduces the golden cases bit for bit. The default kernels run in the
whole suite; the A/B variants run here, each in its own process, on the golden
FTCS cases of test_gpu_parity.py."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

VARIANTS = [
    {"PD_MARCH_V": "14"},
    {"PD_MARCH_V": "20"},
    {"PD_MARCH_V": "30"},
    {"PD_MARCH_V": "31", "PD_M31_CFG": "0"},
    {"PD_MARCH_V": "31", "PD_M31_CFG": "1"},
    {"PD_MARCH_V": "31", "PD_M31_CFG": "2"},
    {"PD_MARCH_V": "41"},
    {"PD_MARCH_V": "43", "PD_M43_PF": "3"},
    {"PD_MARCH_V": "43", "PD_M43_PF": "7"},
    {"PD_MARCH_V": "43", "PD_SCHED": "16,2,2"},  # schedule orders: same bits in any order
    {"PD_MARCH_V": "43", "PD_SCHED": "1,0,0"},
    {"PD_MARCH32_V": "14"},
    {"PD_MARCH32_V": "43", "PD_M32B_CFG": "1"},
    {"PD_MARCH32_V": "43", "PD_M32B_CFG": "2"},
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: "-".join(f"{k[3:]}{v}" for k, v in e.items()))
def test_variant_reproduces_golden_cases(env, cuda):
    e = dict(os.environ, PD_MARCH_MIN_CHUNKS="0", **env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        str(ROOT / "tests" / "test_gpu_parity.py"), "-k", "bitwise_equal_to_reference or against_reference"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
