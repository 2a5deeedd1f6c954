"""bench.py's N > 1 path end to end, on one GPU: two and three ranks under torchrun
(both on cuda:0 via the PD_BENCH_SAME_GPU / PD_DIST_BACKEND=gloo test hooks;
the halo exchange is the fused peer push over CUDA IPC exactly as on a
multi-GPU box). The JSON line's exact cross-rank final diagnostics must equal
the single-rank run's bit for bit."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _line(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-3000:]
    return json.loads(lines[-1])


@pytest.mark.parametrize("ranks", [2, 3])
def test_multi_rank_bench_matches_single_rank(ranks):
    args = ["--box", "256", "--steps", "4", "--warmup", "3", "--no-cpu", "--no-e2e"]
    one = subprocess.run([sys.executable, "bench.py", "--gpus", "1"] + args, cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert one.returncode == 0, one.stderr[-3000:]
    env = dict(os.environ, PD_BENCH_SAME_GPU="1", PD_DIST_BACKEND="gloo")
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", str(ranks)] + args,
                         cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert two.returncode == 0, (two.stdout[-2000:], two.stderr[-3000:])
    a, b = _line(one.stdout), _line(two.stdout)
    assert b["n_gpus"] == ranks and b["config"]["parallelism"] == f"zslab{ranks}"
    assert b["active_nodes"] == a["active_nodes"] and b["chunks"] == a["chunks"]
    fa, fb = a["final_diagnostics"], b["final_diagnostics"]
    assert (fa["total_mass"], fa["min_u"], fa["max_u"]) == (fb["total_mass"], fb["min_u"], fb["max_u"])


def test_gpus_flag_self_launches_ranks():
    """`python bench.py --gpus 2` with no torchrun around it re-launches
    itself with two ranks and reports n_gpus 2, per-rank
    timings and the single-rank run's exact final diagnostics."""
    args = ["--box", "256", "--steps", "4", "--warmup", "3", "--no-cpu", "--no-e2e"]
    one = subprocess.run([sys.executable, "bench.py", "--gpus", "1"] + args, cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert one.returncode == 0, one.stderr[-3000:]
    env = dict(os.environ, PD_BENCH_SAME_GPU="1", PD_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    two = subprocess.run([sys.executable, "bench.py", "--gpus", "2"] + args, cwd=ROOT, capture_output=True,
                         text=True, timeout=900, env=env)
    assert two.returncode == 0, (two.stdout[-2000:], two.stderr[-3000:])
    a, b = _line(one.stdout), _line(two.stdout)
    assert b["n_gpus"] == 2 and len(b["per_rank"]) == 2 and b["load_imbalance"] >= 0
    assert sum(r["active_nodes"] for r in b["per_rank"]) == a["active_nodes"]
    fa, fb = a["final_diagnostics"], b["final_diagnostics"]
    assert (fa["total_mass"], fa["min_u"], fa["max_u"]) == (fb["total_mass"], fb["min_u"], fb["max_u"])
