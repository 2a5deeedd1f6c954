"""CPU check that csrc/pd_libm_exp.h (the device D(phi)'s exp) is the host
libm's exp bit for bit, and that pd_smooth_diffusion reproduces the
reference's smooth_diffusion_coefficient expression (geometry.hpp:182-187).
The header is compiled with gcc and swept over 2.7 * 10^7 arguments covering
every branch (random bit patterns, the overflow / subnormal scalings, tiny
|x|, the D transition band); the same operation sequence runs on the device
(tests/test_headline_parity.py checks it there against libm)."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_restated_exp_matches_host_libm(tmp_path):
    exe = tmp_path / "chk"
    flags = ["-mfma"] if "fma" in Path("/proc/cpuinfo").read_text() else []
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", *flags, f"-I{ROOT / 'paper_2304_11165_b200' / 'csrc'}",
                    str(ROOT / "tests" / "native" / "libm_exp_check.c"), "-o", str(exe), "-lm"], check=True)
    out = subprocess.run([str(exe), "3000000"], capture_output=True, text=True)
    checked, bad = map(int, out.stdout.split()[-2:])
    assert checked > 2 * 10 ** 7 and bad == 0, out.stdout


def test_exp_table_regenerates_identically(tmp_path):
    """pd_exp_table.h is what scripts/gen_exp_table.py derives from first
    principles (80-digit decimal 2^(i/128))."""
    hdr = ROOT / "paper_2304_11165_b200" / "csrc" / "pd_exp_table.h"
    before = hdr.read_text()
    subprocess.run(["python", str(ROOT / "scripts" / "gen_exp_table.py")], check=True, capture_output=True)
    assert hdr.read_text() == before
