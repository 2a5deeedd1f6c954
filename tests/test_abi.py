"""The C-ABI library loads on a CPU-only host and exports exactly what
include/porediff_b200.h declares (no compute calls here)."""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "porediff_b200.h").read_text()
    return sorted(set(re.findall(r"\b(pd_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "pd_stepper_run" in syms and "pd_grid_create" in syms
    assert len(syms) >= 25


def test_library_exports_every_declared_symbol():
    from paper_2304_11165_b200 import _lib
    missing = [s for s in declared_symbols() if not hasattr(_lib.lib, s)]
    assert not missing, missing
    assert sorted(_lib.EXPORTED_SYMBOLS) == declared_symbols()


def test_version_and_device_count_do_not_need_a_gpu():
    from paper_2304_11165_b200 import _lib
    assert b"sm_100a" in _lib.lib.pd_version()
    assert _lib.device_count() >= 0


def test_library_is_built_for_sm_100a():
    import subprocess
    so = ROOT / "paper_2304_11165_b200" / "lib" / "libporediff_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out
