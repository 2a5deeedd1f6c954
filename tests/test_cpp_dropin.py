"""The reference's own GoogleTest suites for the FTCS path and its geometry /
analysis layers (/root/reference/proj/tests/{solver,grid,geometry,levelset,
analysis}_test.cpp), compiled here by
cpp/Makefile against the drop-in headers in include/porediff (whose solver
executes on the B200 through libporediff_b200.so), plus cpp/dropin_test.cpp
(host/device mirror coherence). The binaries are built in this container and
travel to the GPU box under build/cpp/."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "build" / "cpp"


def _ensure_built():
    if Path("/root/reference/proj/tests/solver_test.cpp").exists():
        subprocess.run(["make", "-C", str(ROOT / "cpp"), "-s", "-j4"], check=True, capture_output=True)


def _run(name):
    exe = BIN / name
    if not exe.exists():
        _ensure_built()
    if not exe.exists():
        pytest.skip(f"{name} not built (build() compiles it where /root/reference is present)")
    p = subprocess.run([str(exe)], capture_output=True, text=True, timeout=1200)
    tail = "\n".join(p.stdout.splitlines()[-40:])
    assert p.returncode == 0, f"{name} failed:\n{tail}\n{p.stderr[-2000:]}"
    assert "tests ran" in p.stdout
    return p.stdout


# Host-only suites: the sparse block grid store and the geometry build never
# touch the device, so they run in the CPU suite too.
@pytest.mark.parametrize("suite", ["grid_test", "geometry_test"])
def test_reference_host_suites(suite):
    _run(suite)


@pytest.mark.gpu
def test_reference_solver_suite_on_b200():
    out = _run("solver_test")
    assert "[  PASSED  ]" in out


@pytest.mark.gpu
def test_reference_levelset_suite_on_b200():
    # sussman_redistance runs on the device (pd_field_redistance)
    out = _run("levelset_test")
    assert "[  PASSED  ]" in out


@pytest.mark.gpu
def test_reference_analysis_suite_on_b200():
    # run_frap / fit_effective_D: every FTCS run and the region observer on
    # the device
    out = _run("analysis_test")
    assert "[  PASSED  ]" in out


@pytest.mark.gpu
def test_dropin_mirror_coherence():
    _run("dropin_test")


@pytest.mark.gpu
def test_reference_io_suite_on_b200():
    # scalar text, SBGD/SBGR snapshots (device-assembled records), mask files,
    # VTK (node texts formatted on the device) through the drop-in headers
    out = _run("io_test")
    assert "[  PASSED  ]" in out
