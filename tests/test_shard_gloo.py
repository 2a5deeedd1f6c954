"""Multi-process (world_size 2 and 3, gloo, CPU) check of the z-slab
decomposition used for multi-GPU runs (paper_2304_11165_b200/shard.py): each
rank steps only its chunk layers plus one ghost layer per side (with the
plain-C oracle standing in for the device step) and exchanges the boundary
face planes with torch.distributed after every step. The owned chunks of all
ranks must equal the unsharded run bit for bit."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200.synthetic import SpherePacking
    n = 40
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pk = SpherePacking.random((0, 0, 0), (1, 1, 1), 30, 0.06, 0.14, 4242)
    grid = pd.build_sparse_grid(pk.fluid_sdf_field(geom), geom, pd.PhaseBand(), pd.solver_channels())
    act = grid.active_bool()
    d = grid.channel_data("D", writable=True)
    phi = grid.channel_data("phi")
    d[act] = 0.05 + 1.0 / (1.0 + np.exp(-40.0 * phi[act]))
    u = grid.channel_data("u", writable=True)
    u[act] = np.array([pd.hash_unit_value(3, int(f)) for f in grid.flat_indices()[act]])
    return grid, geom


def _worker(rank, world, port, steps, out):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import torch.distributed as dist

    from oracle.pyoracle import Port, make_config
    from paper_2304_11165_b200 import shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grid, geom = _case()
    keys = grid.keys()
    cc = (geom.size[2] + 7) // 8
    z0, z1 = shard.slab_bounds(cc, world, rank)
    sel = np.nonzero((keys[:, 2] >= z0 - 1) & (keys[:, 2] <= z1))[0]
    lkeys, lmasks = keys[sel], grid.masks()[sel]
    data = {c: grid.channel_data(c)[sel].copy() for c in ("phi", "u", "D", "u_next")}
    plan = shard.exchange_plan(lkeys, z0, z1, rank, world)
    h = 1.0 / geom.size[0]
    dt = 0.4 * 1.0 / (2.0 * float(grid.channel_data("D")[grid.active_bool()].max())) / (3.0 / (h * h))
    cfg = make_config(dt, 1, reaction="surface_sink", rate=2.0, band_half_width=1.0,
                      bc={0: ("dirichlet", 1.0), 5: ("dirichlet", 0.5)}, enforce_stability=False)
    port = Port()
    u, un = data["u"], data["u_next"]
    for _ in range(steps):
        code, msg, _, u_new, un_new = port.run(geom.size, geom.spacing, lkeys, lmasks, data["phi"], u, data["D"],
                                               un, cfg)
        assert code == 0, msg
        u, un = u_new, un_new
        shard.exchange_numpy(plan, u, rank, world, dist)
    out[rank] = (lkeys[plan.begin:plan.end].copy(), u[plan.begin:plan.end].copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_zslab_exchange_matches_unsharded(world):
    import torch.multiprocessing as mp

    from oracle.pyoracle import Port, make_config
    steps = 6
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, steps, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    grid, geom = _case()
    h = 1.0 / geom.size[0]
    dt = 0.4 * 1.0 / (2.0 * float(grid.channel_data("D")[grid.active_bool()].max())) / (3.0 / (h * h))
    cfg = make_config(dt, steps, reaction="surface_sink", rate=2.0, band_half_width=1.0,
                      bc={0: ("dirichlet", 1.0), 5: ("dirichlet", 0.5)}, enforce_stability=False)
    code, msg, _, u_full, _ = Port().run(geom.size, geom.spacing, grid.keys(), grid.masks(),
                                         grid.channel_data("phi"), grid.channel_data("u"),
                                         grid.channel_data("D"), grid.channel_data("u_next"), cfg)
    assert code == 0, msg
    keys = grid.keys()
    cc = (geom.size[0] + 7) // 8
    lin = (keys[:, 2].astype(np.int64) * cc + keys[:, 1]) * cc + keys[:, 0]
    pos = {int(l): i for i, l in enumerate(lin)}
    covered = 0
    for r in range(world):
        k, u = out[r]
        for i in range(len(k)):
            j = pos[(int(k[i, 2]) * cc + int(k[i, 1])) * cc + int(k[i, 0])]
            assert np.array_equal(u[i].view(np.uint64), u_full[j].view(np.uint64)), (r, k[i])
            covered += 1
    assert covered == len(keys)


def test_slab_bounds_partition_and_balance():
    from paper_2304_11165_b200 import shard
    for layers in (1, 5, 64, 256):
        for world in (1, 2, 3, 8):
            b = [shard.slab_bounds(layers, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == layers
            assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))
    w = np.array([1, 1, 1, 1, 10, 10, 1, 1], float)
    b = [shard.slab_bounds(8, 2, r, w) for r in range(2)]
    assert b[0][1] == b[1][0] and b[1][1] == 8


def test_sub_ranges_split_boundary_layers():
    from paper_2304_11165_b200 import shard
    # chunk layers z = 0..5 with 3 chunks each, ascending linear order
    keys = np.array([(x, 0, z) for z in range(6) for x in range(3)], np.int32)
    plan = shard.exchange_plan(keys, 1, 5, 1, 3)  # owns layers 1..4
    (b0, b1), (t0, t1), (i0, i1) = shard.sub_ranges(keys, plan)
    assert (b0, b1) == (3, 6) and (t0, t1) == (12, 15) and (i0, i1) == (6, 12)
    one = shard.exchange_plan(keys, 2, 3, 1, 3)  # a single owned layer
    (b0, b1), (t0, t1), (i0, i1) = shard.sub_ranges(keys, one)
    assert (b0, b1) == (6, 9) and t0 == t1 and i0 == i1


@pytest.mark.parametrize("world", [2, 3, 5])
def test_peer_push_pairing_maps_identical_chunks(world):
    """Host logic of the fused exchange's pairing (shard.Domain.setup_peer):
    rank r pushes its bottom layer into rank r-1's upper ghost layer and its
    top layer into rank r+1's lower ghost layer, ordinal by ordinal. Every
    pair must name the same global chunk on both sides, and every ghost chunk
    must receive exactly one push."""
    from paper_2304_11165_b200 import shard
    grid, geom = _case()
    keys = grid.keys()
    cc = (geom.size[2] + 7) // 8
    plans, lkeys = [], []
    for r in range(world):
        z0, z1 = shard.slab_bounds(cc, world, r)
        sel = np.nonzero((keys[:, 2] >= z0 - 1) & (keys[:, 2] <= z1))[0]
        lkeys.append(keys[sel])
        plans.append(shard.exchange_plan(keys[sel], z0, z1, r, world))
    for r in range(world):
        got = {}
        for side, nb, src in ((0, r - 1, plans[r].send_down), (1, r + 1, plans[r].send_up)):
            if not 0 <= nb < world:
                assert len(src) == 0
                continue
            dst = plans[nb].recv_up if side == 0 else plans[nb].recv_down
            assert len(dst) == len(src)
            for a, b in zip(src, dst):
                assert tuple(lkeys[r][a]) == tuple(lkeys[nb][b])
                got[(nb, int(b))] = got.get((nb, int(b)), 0) + 1
        for (nb, b), k in got.items():
            assert k == 1
    for r in range(world):  # each ghost chunk is fed by exactly its owner
        fed = set()
        for q in (r - 1, r + 1):
            if 0 <= q < world:
                src = plans[q].send_up if q == r - 1 else plans[q].send_down
                fed |= {tuple(lkeys[q][a]) for a in src}
        ghosts = {tuple(lkeys[r][b]) for b in list(plans[r].recv_down) + list(plans[r].recv_up)}
        assert ghosts == fed
