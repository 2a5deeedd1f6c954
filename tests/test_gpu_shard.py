"""z-slab sharding on ONE GPU: two (or three) shard grids built with their
ghost chunk layers (pd_build_sphere_pack_region), stepped on their owned
ordinal range (pd_stepper_set_range) and exchanging face planes with
pd_grid_pack_face / pd_grid_unpack_face after every step, reproduce the
unsharded run bit for bit. The NCCL transport used by bench.py moves exactly
these buffers (shard.Domain.exchange)."""
import ctypes as C
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _build(pd, lib, geom, centers, radii, lo, hi, dtype=np.float64):
    h = C.c_void_p()
    pd._check(lib.pd_build_sphere_pack_region(
        np.dtype(dtype).itemsize, (C.c_int64 * 3)(*geom.size), (C.c_double * 3)(*geom.spacing), (C.c_double * 3)(*geom.origin),
        len(radii), centers.ctypes.data_as(C.POINTER(C.c_double)), radii.ctypes.data_as(C.POINTER(C.c_double)),
        0.0, math.inf, (C.c_int64 * 3)(*lo), (C.c_int64 * 3)(*hi), 4, 0, 0, C.byref(h)))
    n = C.c_int64()
    lib.pd_grid_info(h, C.byref(n), None)
    dev = pd.DeviceGrid(h, geom, dtype, int(n.value), 4)
    dev.populate_diffusion(0, 2, pd.DiffusionProfile(0.02, 1.0, 0.0, 4.0 * geom.size[0]))
    dev.fill_hash(1, 11)
    return dev


def _stepper(pd, lib, dev, dt, rng=None):
    cfg = pd.SimulationConfig(dt=dt, n_steps=1 << 40, record_every=1 << 40)
    cfg.reaction = pd.ReactionSpec.surface_sink(2.0, 1.0)
    cfg.outer_bc[0] = pd.FaceBc.dirichlet(1.0)
    cc = pd._to_c_config(cfg, -1)
    h = C.c_void_p()
    pd._check(lib.pd_stepper_create(dev.h, C.byref(cc), 0, 1, 2, 3, C.byref(h)))
    if rng is not None:
        pd._check(lib.pd_stepper_set_range(h, *rng))
    return h


@pytest.mark.parametrize("world,n,dtype", [(2, 48, np.float64), (3, 61, np.float64), (2, 56, np.float32)])
def test_sharded_run_equals_unsharded(world, n, dtype, cuda):
    import torch

    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200 import shard
    from paper_2304_11165_b200._lib import lib
    from paper_2304_11165_b200.synthetic import SpherePacking

    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pk = SpherePacking.random((0, 0, 0), (1, 1, 1), 40, 0.06, 0.14, 99)
    centers, radii = pk.arrays()
    cc = (n + 7) // 8
    full = _build(pd, lib, geom, centers, radii, (0, 0, 0), (cc, cc, cc), dtype)
    dmax = full.max_active(2)
    dt = 0.45 * pd.stability_dt(geom, dmax)
    steps = 12

    s_full = _stepper(pd, lib, full, dt)
    rows = (pd._lib.pd_diag * 1)()
    nr = C.c_int64()
    pd._check(lib.pd_stepper_run(s_full, 0, steps, 1 << 40, None, rows, C.byref(nr)))
    u_full = full.download(1)
    keys_full, _ = full.layout()

    shards = []
    for r in range(world):
        z0, z1 = shard.slab_bounds(cc, world, r)
        dev = _build(pd, lib, geom, centers, radii, (0, 0, max(0, z0 - 1)), (cc, cc, min(cc, z1 + 1)), dtype)
        keys, _ = dev.layout()
        plan = shard.exchange_plan(keys, z0, z1, r, world)
        s = _stepper(pd, lib, dev, dt, (plan.begin, plan.end))
        shards.append((dev, plan, s, keys))

    def ords(a):
        return torch.from_numpy(np.ascontiguousarray(a, np.int32)).cuda()

    for step in range(steps):
        for dev, plan, s, _ in shards:
            pd._check(lib.pd_stepper_run(s, step, 1, 1 << 40, None, rows, C.byref(nr)))
        torch.cuda.synchronize()
        # exchange: plane z=0 of my bottom layer -> lower rank's upper ghost
        # (its z=0 plane), plane z=7 of my top layer -> upper rank's lower ghost
        sent = {}
        for r, (dev, plan, s, _) in enumerate(shards):
            for lst, face, to in ((plan.send_down, shard.FACE_ZLO, r - 1), (plan.send_up, shard.FACE_ZHI, r + 1)):
                if len(lst) == 0:
                    continue
                buf = torch.empty((len(lst), 64), dtype=torch.float64 if dtype == np.float64 else torch.float32, device="cuda")
                o = ords(lst)
                pd._check(lib.pd_grid_pack_face(dev.h, 1, C.c_void_p(o.data_ptr()), len(lst), face,
                                                C.c_void_p(buf.data_ptr())))
                sent[(r, to)] = (buf, o)
        torch.cuda.synchronize()
        for r, (dev, plan, s, _) in enumerate(shards):
            for lst, face, frm in ((plan.recv_down, shard.FACE_ZHI, r - 1), (plan.recv_up, shard.FACE_ZLO, r + 1)):
                if len(lst) == 0:
                    continue
                buf, _ = sent[(frm, r)]
                assert buf.shape[0] == len(lst)
                o = ords(lst)
                pd._check(lib.pd_grid_unpack_face(dev.h, 1, C.c_void_p(o.data_ptr()), len(lst), face,
                                                  C.c_void_p(buf.data_ptr())))
        torch.cuda.synchronize()

    lin_full = (keys_full[:, 2].astype(np.int64) * cc + keys_full[:, 1]) * cc + keys_full[:, 0]
    pos = {int(l): i for i, l in enumerate(lin_full)}
    covered = 0
    for dev, plan, s, keys in shards:
        u = dev.download(1)
        for i in range(plan.begin, plan.end):
            l = (int(keys[i, 2]) * cc + int(keys[i, 1])) * cc + int(keys[i, 0])
            j = pos[l]
            assert np.array_equal(u[i], u_full[j]) and np.array_equal(u[i].view(np.uint8), u_full[j].view(np.uint8)), (i, keys[i])
            covered += 1
    assert covered == len(keys_full)
    for dev, plan, s, _ in shards:
        lib.pd_stepper_destroy(s)
        dev.close()
    lib.pd_stepper_destroy(s_full)
    full.close()


def test_march_and_tile_kernels_agree(cuda, golden, monkeypatch):
    """The column-march fast path (non-record steps) and the staged-tile
    kernel (record steps / PD_NO_MARCH=1) give identical bits."""
    from cases import CASES, host_case, sha, sim_config
    from paper_2304_11165_b200 import porediff as pd
    name = "contract40"
    spec, gold = CASES[name], golden[name]
    monkeypatch.setenv("PD_NO_MARCH", "1")
    grid = host_case(name)
    pd.run_simulation(grid, sim_config(spec, float.fromhex(gold["dt"])))
    assert sha(grid.channel_data("u")) == gold["sha_outputs"]["u"]


@pytest.mark.parametrize("world,n", [(2, 40), (3, 64)])
def test_overlapped_enqueue_and_exact_diagnostics(world, n, cuda):
    """The multi-GPU step as bench.py runs it (shard.Domain.run): boundary
    layers enqueued first, their new planes exchanged before the swap,
    interior layers after — emulated for `world` shards on one GPU — equals
    the unsharded run bit for bit, and the rank-ordered partials folded by
    pd_reduce_partials give exactly the unsharded step-N diagnostics row."""
    import torch

    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200 import shard
    from paper_2304_11165_b200._lib import lib
    from paper_2304_11165_b200.synthetic import SpherePacking

    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pk = SpherePacking.random((0, 0, 0), (1, 1, 1), 30, 0.07, 0.15, 5)
    centers, radii = pk.arrays()
    cc = (n + 7) // 8
    full = _build(pd, lib, geom, centers, radii, (0, 0, 0), (cc, cc, cc))
    dt = 0.45 * pd.stability_dt(geom, full.max_active(2))
    steps = 9
    s_full = _stepper(pd, lib, full, dt)
    rows = (pd._lib.pd_diag * 1)()
    nr = C.c_int64()
    pd._check(lib.pd_stepper_run(s_full, 0, steps, 1 << 40, None, rows, C.byref(nr)))
    want = pd._lib.pd_diag()
    pd._check(lib.pd_stepper_snapshot_diag(s_full, C.byref(want)))
    u_full = full.download(1)
    keys_full, _ = full.layout()

    shards = []
    for r in range(world):
        z0, z1 = shard.slab_bounds(cc, world, r)
        dev = _build(pd, lib, geom, centers, radii, (0, 0, max(0, z0 - 1)), (cc, cc, min(cc, z1 + 1)))
        keys, _ = dev.layout()
        plan = shard.exchange_plan(keys, z0, z1, r, world)
        s = _stepper(pd, lib, dev, dt, (plan.begin, plan.end))
        shards.append((dev, plan, s, keys, shard.sub_ranges(keys, plan)))

    def ords(a):
        return torch.from_numpy(np.ascontiguousarray(a, np.int32)).cuda()

    for step in range(steps):
        for dev, plan, s, _, ((b0, b1), (t0, t1), _i) in shards:
            pd._check(lib.pd_stepper_enqueue(s, step, b0, b1, 1.0))
            if (t0, t1) != (b0, b1):
                pd._check(lib.pd_stepper_enqueue(s, step, t0, t1, 1.0))
        sent = {}
        for r, (dev, plan, s, _, _rg) in enumerate(shards):
            for lst, face, to in ((plan.send_down, shard.FACE_ZLO, r - 1), (plan.send_up, shard.FACE_ZHI, r + 1)):
                if len(lst):
                    # keep the ordinal tensor alive: the pack runs on the shard
                    # grid's own stream, not torch's
                    buf = torch.empty((len(lst), 64), dtype=torch.float64, device="cuda")
                    o = ords(lst)
                    torch.cuda.synchronize()
                    pd._check(lib.pd_grid_pack_face(dev.h, 3, C.c_void_p(o.data_ptr()), len(lst), face,
                                                    C.c_void_p(buf.data_ptr())))
                    sent[(r, to)] = (buf, o)
        for dev, plan, s, _, (_b, _t, (i0, i1)) in shards:
            pd._check(lib.pd_stepper_enqueue(s, step, i0, i1, 1.0))
        torch.cuda.synchronize()
        for r, (dev, plan, s, _, _rg) in enumerate(shards):
            for lst, face, frm in ((plan.recv_down, shard.FACE_ZHI, r - 1), (plan.recv_up, shard.FACE_ZLO, r + 1)):
                if len(lst):
                    o = ords(lst)
                    torch.cuda.synchronize()
                    pd._check(lib.pd_grid_unpack_face(dev.h, 3, C.c_void_p(o.data_ptr()), len(lst), face,
                                                      C.c_void_p(sent[(frm, r)][0].data_ptr())))
                    torch.cuda.synchronize()
            pd._check(lib.pd_stepper_swap(s))
        torch.cuda.synchronize()
    for dev, plan, s, _, _rg in shards:
        pd._check(lib.pd_stepper_status(s, steps))

    lin_full = (keys_full[:, 2].astype(np.int64) * cc + keys_full[:, 1]) * cc + keys_full[:, 0]
    pos = {int(l): i for i, l in enumerate(lin_full)}
    parts = []
    for dev, plan, s, keys, _rg in shards:
        u = dev.download(1)
        for i in range(plan.begin, plan.end):
            j = pos[(int(keys[i, 2]) * cc + int(keys[i, 1])) * cc + int(keys[i, 0])]
            assert np.array_equal(u[i].view(np.uint64), u_full[j].view(np.uint64)), (i, keys[i])
        k = plan.end - plan.begin
        p = torch.empty((3, max(1, k)), dtype=torch.float64, device="cuda")
        pd._check(lib.pd_stepper_partials(s, C.c_void_p(p[0].data_ptr()), C.c_void_p(p[1].data_ptr()),
                                          C.c_void_p(p[2].data_ptr())))
        parts.append(p[:, :k])
    torch.cuda.synchronize()  # partials were written on the shard grids' own streams
    glob = torch.cat(parts, dim=1).contiguous()
    torch.cuda.synchronize()
    assert glob.shape[1] == len(keys_full)
    row = (C.c_double * 3)()
    pd._check(lib.pd_reduce_partials(shards[0][0].h, C.c_void_p(glob[0].data_ptr()), C.c_void_p(glob[1].data_ptr()),
                                     C.c_void_p(glob[2].data_ptr()), glob.shape[1], row))
    assert (row[0].hex(), row[1].hex(), row[2].hex()) == (want.total_mass.hex(), want.min_u.hex(), want.max_u.hex())
    for dev, plan, s, _, _rg in shards:
        lib.pd_stepper_destroy(s)
        dev.close()
    lib.pd_stepper_destroy(s_full)
    full.close()


def test_domain_overlapped_path_equals_batched_run(cuda):
    """shard.Domain.run's overlapped branch (enqueue boundary layers, switch
    the grid to the communication stream for the exchange, enqueue the
    interior, swap) gives the same bits as one pd_stepper_run; with one rank
    the exchange itself is empty, the stream and ordering logic is not."""
    import torch

    from paper_2304_11165_b200 import shard
    from paper_2304_11165_b200 import synthetic as sy
    pack = sy.pack_for_porosity(0.25, 12 / 96, 7)
    a = shard.build_domain(96, pack, 0, 1, device=0)
    b = shard.build_domain(96, pack, 0, 1, device=0)
    sa, sb = a.stepper(), b.stepper()
    a.run(sa, 0, 7, overlap=False)
    b.run(sb, 0, 7, overlap=True)
    torch.cuda.synchronize()
    ua, ub = a.dev.download(1), b.dev.download(1)
    assert np.array_equal(ua.view(np.uint64), ub.view(np.uint64))
    assert a.diagnostics(sa) == b.diagnostics(sb)


@pytest.mark.parametrize("world,n", [(2, 48), (3, 64)])
def test_fused_peer_push_equals_unsharded(world, n, cuda):
    """The fused exchange (pd_stepper_set_peer): the march kernel stores each
    boundary chunk's new z=0 / z=7 plane straight into the neighbour shard's
    ghost chunk and per-neighbour step counters order the steps — `world`
    shards on one GPU, each on its own stream, all steps enqueued without a
    host sync — equals the unsharded run bit for bit."""
    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200 import shard
    from paper_2304_11165_b200._lib import lib
    from paper_2304_11165_b200.synthetic import SpherePacking

    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pk = SpherePacking.random((0, 0, 0), (1, 1, 1), 36, 0.06, 0.14, 17)
    centers, radii = pk.arrays()
    cc = (n + 7) // 8
    full = _build(pd, lib, geom, centers, radii, (0, 0, 0), (cc, cc, cc))
    dt = 0.45 * pd.stability_dt(geom, full.max_active(2))
    steps = 11
    s_full = _stepper(pd, lib, full, dt)
    rows = (pd._lib.pd_diag * 1)()
    nr = C.c_int64()
    pd._check(lib.pd_stepper_run(s_full, 0, steps, 1 << 40, None, rows, C.byref(nr)))
    u_full = full.download(1)
    keys_full, _ = full.layout()

    shards = []
    for r in range(world):
        z0, z1 = shard.slab_bounds(cc, world, r)
        dev = _build(pd, lib, geom, centers, radii, (0, 0, max(0, z0 - 1)), (cc, cc, min(cc, z1 + 1)))
        keys, _ = dev.layout()
        plan = shard.exchange_plan(keys, z0, z1, r, world)
        s = _stepper(pd, lib, dev, dt, (plan.begin, plan.end))
        cols = (C.c_void_p * 4)()
        pd._check(lib.pd_grid_column_ptrs(dev.h, cols))
        sync = C.c_void_p()
        pd._check(lib.pd_stepper_sync_words(s, C.byref(sync)))
        shards.append((dev, plan, s, keys, cols, sync))
    for r, (dev, plan, s, keys, cols, sync) in enumerate(shards):
        for side, nb, src in ((0, r - 1, plan.send_down), (1, r + 1, plan.send_up)):
            if nb < 0 or nb >= world:
                continue
            o = shards[nb]
            dst = np.ascontiguousarray(o[1].recv_up if side == 0 else o[1].recv_down, np.int32)
            src = np.ascontiguousarray(src, np.int32)
            assert len(dst) == len(src)
            pd._check(lib.pd_stepper_set_peer(s, side, o[4], 4, o[5], src.ctypes.data, dst.ctypes.data, len(src)))
    for sh in shards:
        pd._check(lib.pd_stepper_peer_reset(sh[2]))
    for step in range(steps):
        for dev, plan, s, *_ in shards:
            pd._check(lib.pd_stepper_enqueue(s, step, plan.begin, plan.end, 1.0))
        for sh in shards:
            pd._check(lib.pd_stepper_swap(sh[2]))
    for dev, plan, s, *_ in shards:
        pd._check(lib.pd_stepper_status(s, steps))

    lin_full = (keys_full[:, 2].astype(np.int64) * cc + keys_full[:, 1]) * cc + keys_full[:, 0]
    pos = {int(l): i for i, l in enumerate(lin_full)}
    covered = 0
    for dev, plan, s, keys, *_ in shards:
        u = dev.download(1)
        for i in range(plan.begin, plan.end):
            j = pos[(int(keys[i, 2]) * cc + int(keys[i, 1])) * cc + int(keys[i, 0])]
            assert np.array_equal(u[i].view(np.uint64), u_full[j].view(np.uint64)), (i, keys[i])
            covered += 1
    assert covered == len(keys_full)
    for dev, plan, s, *_ in shards:
        lib.pd_stepper_destroy(s)
        dev.close()
    lib.pd_stepper_destroy(s_full)
    full.close()


def test_layer_work_matches_built_grid_and_balances(cuda):
    """pd_sphere_pack_layer_work (the builder's mask pass, no grid) gives the
    built grid's chunks and active nodes per z layer exactly; work-balanced
    cuts cover every layer once and even out the chunk counts."""
    from paper_2304_11165_b200 import porediff as pd
    from paper_2304_11165_b200 import shard
    from paper_2304_11165_b200 import synthetic as sy
    n = 96
    geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
    pack = sy.SpherePacking.random((0, 0, 0), (1, 1, 1), 50, 0.05, 0.2, 77)
    chunks, active, full = shard.layer_work(geom, pack)
    c, r = pack.arrays()
    dev = pd.DeviceGrid.sphere_pack(geom, c, r)
    keys, masks = dev.layout()
    cc = (n + 7) // 8
    want_c = np.bincount(keys[:, 2], minlength=cc)
    pop = np.unpackbits(masks.view(np.uint8), bitorder="little").reshape(len(masks), -1).sum(axis=1)
    want_a = np.bincount(keys[:, 2], weights=pop, minlength=cc).astype(np.int64)
    assert np.array_equal(chunks, want_c) and np.array_equal(active, want_a)
    want_f = np.bincount(keys[:, 2], weights=(pop == 512), minlength=cc).astype(np.int64)
    assert np.array_equal(full, want_f) and full.sum() > 0
    dev.close()
    for world in (2, 3, 5):
        b = [shard.slab_bounds(cc, world, r, chunks) for r in range(world)]
        assert b[0][0] == 0 and b[-1][1] == cc and all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        per = [int(chunks[z0:z1].sum()) for z0, z1 in b]
        assert max(per) - min(per) <= 2 * int(chunks.max())
