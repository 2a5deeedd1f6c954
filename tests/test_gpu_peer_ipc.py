"""The fused multi-GPU exchange across PROCESSES, as bench.py runs it under
torchrun: two ranks (here both on cuda:0 — this box has one GPU; CUDA IPC
maps the other process's allocations exactly as it maps a peer GPU's over
NVLink), each a shard.Domain with exchange="peer": columns and step
counters exchanged as IPC handles (all_gather_object over gloo), the march
kernel pushing boundary planes into the other process's ghost chunks, step
counters ordering the steps. The gathered owned u equals a single-domain run
bit for bit, and the exact cross-rank diagnostics equal the single run's."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, steps, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    from paper_2304_11165_b200 import shard
    from paper_2304_11165_b200 import synthetic as sy

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pack = sy.SpherePacking.random((0, 0, 0), (1, 1, 1), 40, 0.07, 0.15, 23)
    dom = shard.Domain(n, pack, rank, world, 0, exchange="peer")
    st = dom.stepper(dt_frac=0.4, sink_rate=1.0)
    dom.run(st, 0, steps)
    diag = dom.diagnostics(st)
    u = dom.dev.download(1)
    keys = dom.keys
    own = slice(dom.plan.begin, dom.plan.end)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), u=u[own], keys=keys[own], diag=np.array(diag))
    dist.barrier()
    dom.close_peer()
    dist.destroy_process_group()


def test_two_process_ipc_push_equals_single_domain(cuda, tmp_path):
    import torch.multiprocessing as mp

    from paper_2304_11165_b200 import shard
    from paper_2304_11165_b200 import synthetic as sy
    n, steps, world = 56, 9, 2
    mp.start_processes(_worker, args=(world, _free_port(), n, steps, str(tmp_path)), nprocs=world,
                       start_method="spawn", join=True)
    pack = sy.SpherePacking.random((0, 0, 0), (1, 1, 1), 40, 0.07, 0.15, 23)
    one = shard.Domain(n, pack, 0, 1, 0)
    st = one.stepper(dt_frac=0.4, sink_rate=1.0)
    one.run(st, 0, steps)
    want = one.diagnostics(st)
    u1 = one.dev.download(1)
    cc = (n + 7) // 8
    lin = lambda k: (k[:, 2].astype(np.int64) * cc + k[:, 1]) * cc + k[:, 0]  # noqa: E731
    pos = {int(l): i for i, l in enumerate(lin(one.keys))}
    covered = 0
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        for i, l in enumerate(lin(d["keys"])):
            assert np.array_equal(d["u"][i].view(np.uint64), u1[pos[int(l)]].view(np.uint64)), (r, i)
            covered += 1
        assert tuple(float(x) for x in d["diag"]) == tuple(want)
    assert covered == len(one.keys)
