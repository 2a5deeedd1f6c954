"""Multi-GPU z-slab decomposition of the sparse block grid (north_star
subsystem 4).

Chunk ordinals ascend with the chunk linear index, which is z-slowest
(sparse_block_grid.hpp:105-109), so a contiguous range of chunk layers is a
contiguous ordinal range. Rank r owns chunk layers [z0, z1) and additionally
holds one read-only ghost layer on each side (z0-1 and z1). Keys stay global,
so the step kernel's box / neighbour logic is unchanged; the stepper runs on
the owned ordinal range only (pd_stepper_set_range).

Every update reads only step-n state of its 2*Dims face neighbours
(solver.hpp:29-33), and an owned chunk reads only the one-node face plane of
a ghost chunk that touches it. So after each step rank r sends
  * the z=0 plane of its bottom owned layer to rank r-1 (its upper ghost), and
  * the z=7 plane of its top owned layer to rank r+1 (its lower ghost),
64 nodes x 8 B per chunk, over NCCL. D and phi are static and built
identically on both sides, so they are never exchanged.

The plan functions below are pure host logic (tested with gloo on CPU);
``Domain`` binds them to the device grid and torch.distributed NCCL.

Two exchange transports:

* "peer" (default for 3-D FP64 with world > 1): the exchange is fused into
  the step kernel. Each rank maps its neighbours' u / u_next columns and step
  counters through CUDA IPC (NVLink peer memory); the march kernel stores
  every boundary chunk's new z=0 / z=7 plane straight into the neighbour's
  ghost chunk while it computes the slab, and one-word step counters in the
  neighbours' memory order consecutive steps (pd_peer.cu). A step is one
  kernel plus a 1-thread wait and signal; no pack, no NCCL, no host sync.
* "nccl" (PD_EXCHANGE=nccl, and FP32 / 2-D): each step enqueues the two
  boundary chunk layers first (pd_stepper_enqueue, no host sync), then the
  face exchange of their new planes runs on a communication stream (pack ->
  NCCL send/recv -> unpack into the ghost layers) while the interior layers
  are stepped on the compute stream; the next step starts after both.

Record steps reduce exactly across ranks (``Domain.diagnostics``): per-chunk
partials are gathered in rank (= ordinal) order and folded by the
reference's pairwise tree.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

FACE_ZLO = 4  # axis 2, side 0: the chunk's z=0 plane
FACE_ZHI = 5  # axis 2, side 1: the chunk's z=7 plane


def slab_bounds(n_layers: int, world: int, rank: int, weights: Optional[np.ndarray] = None):
    """Chunk layers [z0, z1) owned by `rank`. With per-layer weights (e.g.
    active nodes per layer) the cuts balance work (prefix sums), else layers
    are split evenly."""
    if weights is None:
        z0 = (n_layers * rank) // world
        z1 = (n_layers * (rank + 1)) // world
        return z0, z1
    c = np.concatenate([[0.0], np.cumsum(np.asarray(weights, np.float64))])
    tot = c[-1]
    cuts = [0] + [int(np.searchsorted(c, tot * k / world, side="left")) for k in range(1, world)] + [n_layers]
    cuts = [min(max(x, 0), n_layers) for x in cuts]
    for k in range(1, len(cuts)):
        cuts[k] = max(cuts[k], cuts[k - 1])
    return cuts[rank], cuts[rank + 1]


@dataclass
class ExchangePlan:
    z0: int
    z1: int
    begin: int  # owned ordinal range [begin, end)
    end: int
    send_down: np.ndarray  # ordinals of the bottom owned layer (to rank-1)
    send_up: np.ndarray  # ordinals of the top owned layer (to rank+1)
    recv_down: np.ndarray  # lower ghost layer ordinals (from rank-1)
    recv_up: np.ndarray  # upper ghost layer ordinals (from rank+1)


def exchange_plan(keys: np.ndarray, z0: int, z1: int, rank: int, world: int) -> ExchangePlan:
    """keys: (n, 3) int32 chunk keys of the local grid (owned + ghost layers)
    in ascending linear order."""
    kz = np.asarray(keys)[:, 2]
    owned = np.nonzero((kz >= z0) & (kz < z1))[0]
    begin = int(owned[0]) if owned.size else int(np.searchsorted(kz, z0))
    end = int(owned[-1]) + 1 if owned.size else begin
    assert np.all((kz[begin:end] >= z0) & (kz[begin:end] < z1)), "owned chunks must be contiguous"
    none = np.zeros(0, np.int32)
    send_down = np.nonzero(kz == z0)[0].astype(np.int32) if rank > 0 and z1 > z0 else none
    send_up = np.nonzero(kz == z1 - 1)[0].astype(np.int32) if rank < world - 1 and z1 > z0 else none
    recv_down = np.nonzero(kz == z0 - 1)[0].astype(np.int32) if rank > 0 else none
    recv_up = np.nonzero(kz == z1)[0].astype(np.int32) if rank < world - 1 else none
    return ExchangePlan(z0, z1, begin, end, send_down, send_up, recv_down, recv_up)


def sub_ranges(keys: np.ndarray, plan: ExchangePlan):
    """Owned ordinal range split into (bottom layer, top layer, interior):
    only the boundary layers read ghost chunks or are read by neighbours."""
    kz = np.asarray(keys)[:, 2]
    b1 = int(np.searchsorted(kz, plan.z0 + 1, side="left"))
    t0 = int(np.searchsorted(kz, plan.z1 - 1, side="left"))
    b1 = min(max(b1, plan.begin), plan.end)
    t0 = min(max(t0, b1), plan.end)
    return (plan.begin, b1), (t0, plan.end), (b1, t0)


def exchange_numpy(plan: ExchangePlan, u: np.ndarray, rank: int, world: int, dist) -> None:
    """Host (gloo) version of the per-step halo exchange on (n, 512) slabs;
    the device version is Domain.exchange. Same plan, same planes."""
    import torch

    def plane(ords, zc):
        return np.ascontiguousarray(u[ords][:, zc * 64:(zc + 1) * 64])

    ops = []
    bufs = []
    if rank > 0:
        s = torch.from_numpy(plane(plan.send_down, 0).copy())
        r = torch.empty((len(plan.recv_down), 64), dtype=s.dtype)
        ops += [dist.P2POp(dist.isend, s, rank - 1), dist.P2POp(dist.irecv, r, rank - 1)]
        bufs.append((plan.recv_down, 7, r))
    if rank < world - 1:
        s = torch.from_numpy(plane(plan.send_up, 7).copy())
        r = torch.empty((len(plan.recv_up), 64), dtype=s.dtype)
        ops += [dist.P2POp(dist.isend, s, rank + 1), dist.P2POp(dist.irecv, r, rank + 1)]
        bufs.append((plan.recv_up, 0, r))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for ords, zc, r in bufs:
        u[ords, zc * 64:(zc + 1) * 64] = r.numpy()


class Domain:
    """One rank's shard of a sphere-pack domain on its GPU."""

    def __init__(self, n, pack, rank, world, device, dtype=np.float64, exchange=None, balance=None):
        import torch

        from . import porediff as pd
        from ._lib import lib

        self.pd, self.lib = pd, lib
        self.n, self.rank, self.world, self.device = n, rank, world, device
        self.geom = pd.GridGeometry.cell_centered_box(n, 0.0, 1.0, 3)
        cc = [(n + 7) // 8] * 3
        self.cc = cc
        # cut the z chunk layers at equal prefix sums of work (allocated chunks
        # per layer; the step costs per chunk), not at equal layer counts
        if balance is None:
            # "chunks" measured best at C5 (profiles/r02_slab_balance.txt: 2.3 % / 3.5 %
            # per-shard kernel-time imbalance at 4 / 8 shards; "cost" 2.4 / 3.7 %,
            # even layers 8.2 / 13.4 %)
            balance = os.environ.get("PD_BALANCE", "chunks") if world > 1 else "layers"
        weights = None
        if balance in ("chunks", "active", "cost"):
            ch, ac, fu = layer_work(self.geom, pack, dtype, device)
            weights = {"chunks": ch, "active": ac, "cost": layer_cost(ch, fu)}[balance]
        self.balance = balance
        z0, z1 = slab_bounds(cc[2], world, rank, weights)
        lo = (C.c_int64 * 3)(0, 0, max(0, z0 - 1))
        hi = (C.c_int64 * 3)(cc[0], cc[1], min(cc[2], z1 + 1))
        centers, radii = pack.arrays()
        size = (C.c_int64 * 3)(*self.geom.size)
        spacing = (C.c_double * 3)(*self.geom.spacing)
        origin = (C.c_double * 3)(*self.geom.origin)
        h = C.c_void_p()
        pd._check(lib.pd_build_sphere_pack_region(
            np.dtype(dtype).itemsize, size, spacing, origin, len(radii),
            centers.ctypes.data_as(C.POINTER(C.c_double)), radii.ctypes.data_as(C.POINTER(C.c_double)),
            0.0, math.inf, lo, hi, 4, 0, device, C.byref(h)))
        nch = C.c_int64()
        lib.pd_grid_info(h, C.byref(nch), None)
        self.dev = pd.DeviceGrid(h, self.geom, dtype, int(nch.value), 4)
        # sigmoid D across the interface (geometry.hpp:182-206), u0 hash
        self.dev.populate_diffusion(0, 2, pd.DiffusionProfile(0.0, 1.0, 0.0, 4.0 * n))
        self.dev.fill_hash(1, 1)
        keys, masks = self.dev.layout()
        self.keys = keys
        self.plan = exchange_plan(keys, z0, z1, rank, world)
        self.ranges = sub_ranges(keys, self.plan)
        act = np.unpackbits(masks.view(np.uint8), bitorder="little").reshape(len(masks), -1).sum(axis=1)
        self.owned_active = int(act[self.plan.begin:self.plan.end].sum())
        self.owned_chunks = self.plan.end - self.plan.begin
        self.torch = torch
        self.stream = torch.cuda.current_stream(device)
        self.comm = torch.cuda.Stream(device=device)
        lib.pd_grid_set_stream(self.dev.h, C.c_void_p(self.stream.cuda_stream))
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(f"cuda:{device}")
        self.d_send_down, self.d_send_up = t(self.plan.send_down), t(self.plan.send_up)
        self.d_recv_down, self.d_recv_up = t(self.plan.recv_down), t(self.plan.recv_up)
        tt = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
        mk = lambda k: torch.empty((max(1, k), 64), dtype=tt, device=f"cuda:{device}")
        self.b_send_down, self.b_send_up = mk(len(self.plan.send_down)), mk(len(self.plan.send_up))
        self.b_recv_down, self.b_recv_up = mk(len(self.plan.recv_down)), mk(len(self.plan.recv_up))
        self._kernel_ms = 0.0
        self._steps = 0
        if exchange is None:
            exchange = os.environ.get("PD_EXCHANGE", "peer")
        if np.dtype(dtype) != np.float64:
            exchange = "nccl"  # the fused push lives in the 3-D FP64 march kernel
        self.exchange_mode = exchange if world > 1 else "none"
        self._ipc = []
        # own kernels per step besides the step kernel: peer wait + signal, or
        # two face packs and two unpacks
        self.extra_launches_per_step = {"peer": 2, "nccl": 4}.get(self.exchange_mode, 0)

    def _allreduce(self, v: float, op: str = "sum") -> float:
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return v
        dev = "cpu" if dist.get_backend() == "gloo" else f"cuda:{self.device}"
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return float(t.item())

    def total_chunks(self, world):
        return int(self._allreduce(float(self.owned_chunks)))

    def stepper(self, dt_frac=0.4, sink_rate=1.0, sink_width=1.0):
        pd = self.pd
        dmax = self._allreduce(self.dev.max_active(2), "max")
        cfg = pd.SimulationConfig(dt=dt_frac * pd.stability_dt(self.geom, dmax), n_steps=1 << 40,
                                  record_every=1 << 40)
        cfg.reaction = pd.ReactionSpec.surface_sink(sink_rate, sink_width)
        ccfg = pd._to_c_config(cfg, -1)
        h = C.c_void_p()
        pd._check(self.lib.pd_stepper_create(self.dev.h, C.byref(ccfg), 0, 1, 2, 3, C.byref(h)))
        pd._check(self.lib.pd_stepper_set_range(h, self.plan.begin, self.plan.end))
        self.cfg = cfg
        if self.exchange_mode == "peer":
            self.setup_peer(h)
        return h

    def setup_peer(self, stepper):
        """Map the neighbours' columns and step counters (CUDA IPC) and bind
        the fused push: my bottom layer -> lower neighbour's upper ghost
        layer, my top layer -> upper neighbour's lower ghost layer."""
        import torch.distributed as dist
        lib, pd = self.lib, self.pd
        hs = lib.pd_ipc_handle_size()
        n_cols = 4
        pd._check(lib.pd_grid_make_shareable(self.dev.h))
        cols = C.create_string_buffer(hs * n_cols)
        pd._check(lib.pd_grid_ipc_handles(self.dev.h, cols))
        sy = C.create_string_buffer(hs)
        pd._check(lib.pd_stepper_sync_ipc_handle(stepper, sy))
        mine = {"cols": cols.raw, "sync": sy.raw, "recv_down": self.plan.recv_down.tolist(),
                "recv_up": self.plan.recv_up.tolist()}
        every = [None] * self.world
        dist.all_gather_object(every, mine)

        def opened(handle: bytes) -> int:
            p = C.c_void_p()
            pd._check(lib.pd_ipc_open(handle, self.device, C.byref(p)))
            self._ipc.append(p.value)
            return p.value

        for side, nb, src in ((0, self.rank - 1, self.plan.send_down), (1, self.rank + 1, self.plan.send_up)):
            if nb < 0 or nb >= self.world:
                continue
            o = every[nb]
            dst = np.asarray(o["recv_up"] if side == 0 else o["recv_down"], np.int32)
            src = np.ascontiguousarray(src, np.int32)
            if len(dst) != len(src):
                raise RuntimeError(f"rank {self.rank}: boundary layer has {len(src)} chunks, "
                                   f"neighbour ghost layer {len(dst)}")
            ptrs = (C.c_void_p * n_cols)(*[opened(o["cols"][c * hs:(c + 1) * hs]) for c in range(n_cols)])
            sp = opened(o["sync"])
            pd._check(lib.pd_stepper_set_peer(stepper, side, ptrs, n_cols, C.c_void_p(sp), src.ctypes.data,
                                              dst.ctypes.data, len(src)))
        pd._check(lib.pd_stepper_peer_reset(stepper))
        dist.barrier()

    def close_peer(self):
        for p in self._ipc:
            self.lib.pd_ipc_close(C.c_void_p(p), self.device)
        self._ipc = []

    def exchange(self, prop: int = 1):
        """Device halo exchange of the face planes of logical property `prop`
        (1 = u after a completed step; 3 = u_next before the swap)."""
        import torch.distributed as dist
        lib, pd = self.lib, self.pd
        P = lambda t: C.c_void_p(t.data_ptr())
        ops = []
        if self.rank > 0 and len(self.plan.send_down):
            pd._check(lib.pd_grid_pack_face(self.dev.h, prop, P(self.d_send_down), len(self.plan.send_down),
                                            FACE_ZLO, P(self.b_send_down)))
        if self.rank < self.world - 1 and len(self.plan.send_up):
            pd._check(lib.pd_grid_pack_face(self.dev.h, prop, P(self.d_send_up), len(self.plan.send_up),
                                            FACE_ZHI, P(self.b_send_up)))
        if self.rank > 0:
            if len(self.plan.send_down):
                ops.append(dist.P2POp(dist.isend, self.b_send_down[:len(self.plan.send_down)], self.rank - 1))
            if len(self.plan.recv_down):
                ops.append(dist.P2POp(dist.irecv, self.b_recv_down[:len(self.plan.recv_down)], self.rank - 1))
        if self.rank < self.world - 1:
            if len(self.plan.send_up):
                ops.append(dist.P2POp(dist.isend, self.b_send_up[:len(self.plan.send_up)], self.rank + 1))
            if len(self.plan.recv_up):
                ops.append(dist.P2POp(dist.irecv, self.b_recv_up[:len(self.plan.recv_up)], self.rank + 1))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if self.rank > 0 and len(self.plan.recv_down):
            pd._check(lib.pd_grid_unpack_face(self.dev.h, prop, P(self.d_recv_down), len(self.plan.recv_down),
                                              FACE_ZHI, P(self.b_recv_down)))
        if self.rank < self.world - 1 and len(self.plan.recv_up):
            pd._check(lib.pd_grid_unpack_face(self.dev.h, prop, P(self.d_recv_up), len(self.plan.recv_up),
                                              FACE_ZLO, P(self.b_recv_up)))

    def run(self, stepper, step0: int, n: int, overlap: Optional[bool] = None) -> float:
        """Advances n steps; returns the device milliseconds (CUDA events on
        the compute stream) of the whole sequence. world == 1: one
        pd_stepper_run call. world > 1: boundary layers, then the exchange on
        the communication stream overlapped with the interior layers."""
        torch, lib, pd = self.torch, self.lib, self.pd
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        if overlap is None:
            overlap = self.exchange_mode == "nccl"
        if not overlap:  # one device call; with "peer" every step waits, pushes, signals
            rows = (pd._lib.pd_diag * 1)()
            nr = C.c_int64()
            pd._check(lib.pd_stepper_run(stepper, step0, n, 1 << 40, None, rows, C.byref(nr)))
            ms_k = C.c_double()
            lib.pd_stepper_last_ms(stepper, C.byref(ms_k))
            kms = ms_k.value
        else:
            (b0, b1), (t0, t1), (i0, i1) = self.ranges
            cs, comm = self.stream, self.comm
            for s in range(n):
                st = step0 + s
                pd._check(lib.pd_stepper_enqueue(stepper, st, b0, b1, 1.0))
                if (t0, t1) != (b0, b1):
                    pd._check(lib.pd_stepper_enqueue(stepper, st, t0, t1, 1.0))
                ev_b = torch.cuda.Event()
                ev_b.record(cs)
                comm.wait_event(ev_b)
                with torch.cuda.stream(comm):
                    lib.pd_grid_set_stream(self.dev.h, C.c_void_p(comm.cuda_stream))
                    self.exchange(prop=3)  # new boundary planes, before the swap
                    lib.pd_grid_set_stream(self.dev.h, C.c_void_p(cs.cuda_stream))
                ev_c = torch.cuda.Event()
                ev_c.record(comm)
                pd._check(lib.pd_stepper_enqueue(stepper, st, i0, i1, 1.0))
                cs.wait_event(ev_c)
                pd._check(lib.pd_stepper_swap(stepper))
            kms = None
        e1.record(self.stream)
        e1.synchronize()
        if overlap or self.exchange_mode == "peer":
            pd._check(lib.pd_stepper_status(stepper, step0 + n))
        ms = e0.elapsed_time(e1)
        kms = ms if kms is None else kms  # overlapped: whole step (kernels + exchange)
        self.last_kernel_ms = kms
        self._kernel_ms += kms
        self._steps += n
        return ms

    def diagnostics(self, stepper):
        """Exact global (total_mass, min_u, max_u) of the current u: per-chunk
        partials of every rank gathered in ordinal order, then the
        reference's pairwise tree and min/max fold (pd_reduce_partials)."""
        import torch
        import torch.distributed as dist
        lib, pd = self.lib, self.pd
        dev = f"cuda:{self.device}"
        n_own = self.plan.end - self.plan.begin
        parts = torch.empty((3, max(1, n_own)), dtype=torch.float64, device=dev)
        P = lambda t: C.c_void_p(t.data_ptr())
        pd._check(lib.pd_stepper_partials(stepper, P(parts[0]), P(parts[1]), P(parts[2])))
        if self.world > 1:
            cdev = "cpu" if dist.get_backend() == "gloo" else dev
            torch.cuda.synchronize(self.device)
            cnt = torch.tensor([n_own], dtype=torch.int64, device=cdev)
            cnts = [torch.zeros_like(cnt) for _ in range(self.world)]
            dist.all_gather(cnts, cnt)
            cnts = [int(c.item()) for c in cnts]
            m = max(1, max(cnts))
            pad = torch.zeros((3, m), dtype=torch.float64, device=cdev)
            pad[:, :n_own] = parts[:, :n_own].to(cdev)
            allp = [torch.empty_like(pad) for _ in range(self.world)]
            dist.all_gather(allp, pad)
            glob = torch.cat([a[:, :c] for a, c in zip(allp, cnts)], dim=1).to(dev).contiguous()
        else:
            glob = parts[:, :n_own].contiguous()
        row = (C.c_double * 3)()
        pd._check(lib.pd_reduce_partials(self.dev.h, P(glob[0]), P(glob[1]), P(glob[2]), glob.shape[1], row))
        return row[0], row[1], row[2]

    def close(self, stepper=None):
        """Frees the rank's device state (stepper, peer mappings, grid,
        exchange buffers)."""
        self.torch.cuda.synchronize(self.device)
        if stepper is not None:
            self.lib.pd_stepper_destroy(stepper)
        if self._ipc:
            self.close_peer()
        if self.world > 1:  # no rank frees memory a neighbour still maps
            import torch.distributed as dist
            dist.barrier()
        self.dev.close()
        for k in ("d_send_down", "d_send_up", "d_recv_down", "d_recv_up", "b_send_down", "b_send_up",
                  "b_recv_down", "b_recv_up"):
            setattr(self, k, None)
        self.torch.cuda.empty_cache()

    def peer_wait_ns(self, stepper) -> int:
        """Total ns the fused exchange's per-step waits spent blocked on the
        neighbours' step counters (0 without the peer exchange)."""
        if self.exchange_mode != "peer":
            return 0
        ns = C.c_uint64()
        n = C.c_int64()
        self.pd._check(self.lib.pd_stepper_peer_stats(stepper, C.byref(ns), C.byref(n)))
        return int(ns.value)

    def kernel_ms(self, stepper) -> float:
        """Average device time of one step kernel launch so far."""
        return self._kernel_ms / max(1, self._steps)

    def launches(self, stepper) -> int:
        n = C.c_int64()
        self.lib.pd_stepper_launch_count(stepper, C.byref(n))
        return int(n.value)


def layer_work(geom, pack, dtype=np.float64, device: int = 0):
    """(allocated chunks, active nodes, fully active chunks) per z chunk layer
    of the sphere-pack domain, from the builder's mask pass without building
    the grid (pd_sphere_pack_layer_cost)."""
    from . import porediff as pd
    from ._lib import lib
    centers, radii = pack.arrays()
    layers = (geom.size[2] + 7) // 8
    chunks = np.zeros(layers, np.int64)
    active = np.zeros(layers, np.int64)
    full = np.zeros(layers, np.int64)
    pd._check(lib.pd_sphere_pack_layer_cost(
        np.dtype(dtype).itemsize, (C.c_int64 * 3)(*geom.size), (C.c_double * 3)(*geom.spacing),
        (C.c_double * 3)(*geom.origin), len(radii), centers.ctypes.data_as(C.POINTER(C.c_double)),
        radii.ctypes.data_as(C.POINTER(C.c_double)), 0.0, math.inf, device, chunks.ctypes.data, active.ctypes.data,
        full.ctypes.data))
    return chunks, active, full


# Step cost of a fully active chunk relative to a partial one: fully active
# chunks mostly take the march kernels' uniform path (no D_eff traffic, ~40 %
# fewer FP64 operations: 8 KB instead of 12 KB per chunk).
UNIFORM_COST = 2.0 / 3.0


def layer_cost(chunks: np.ndarray, full: np.ndarray) -> np.ndarray:
    """Per-layer step cost model for the slab cuts (PD_BALANCE=cost)."""
    return (chunks - full) + UNIFORM_COST * full


def build_domain(n, pack, rank, world, device=0, dtype=np.float64) -> Domain:
    return Domain(n, pack, rank, world, device, dtype)
