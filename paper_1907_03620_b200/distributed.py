"""Multi-GPU contraction + agglomeration (one process per GPU).

The path shards because counts add (TileAccumulator::merge,
accumulator.hpp:137-154) — but significance is global (a tile whose points
are spread over ranks may reach tau only in total), so there is one real
exchange step:

  1. every rank contracts its own points into a local device table (K1);
  2. local (packed key, count) pairs are routed to an owner rank chosen by a
     hash of the key — one all_to_all of keys and one of counts (NCCL over
     NVLink on GPUs; gloo on CPU tensors in tests);
  3. each owner folds what it received into a fresh table (the counts-add
     half of merge) and prunes with tau (K2): owners hold disjoint
     significant sets;
  4. the significant sets are all-gathered (S x 24 bytes; config 4:
     ~210 MB) and every rank runs K3 on the full set, so all ranks hold the
     identical canonical clustering (and can label their own points with K4
     without a second exchange).

The per-rank engine is the sm_100a library (`GpuEngine`); tests inject a
CPU double through `engine=` to exercise the exchange logic on gloo. There is
no CPU fallback in the product path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .raster import FlatClustering, GridParams, _Context, _flat_from_ctx, _Points


def owner_of(keys, world: int):
    """Owner rank of each packed key: the high 31 bits of the splitmix64
    finaliser, mod world. Works on torch int64 tensors (wrapping arithmetic)
    and numpy uint64 arrays, with identical results."""
    if hasattr(keys, "dtype") and "torch" in type(keys).__module__:
        import torch

        z = keys.to(torch.int64)
        z = (z ^ (z >> 30) & 0x3FFFFFFFF) * -4658895280553007687  # 0xbf58476d1ce4e5b9
        z = (z ^ (z >> 27) & 0x1FFFFFFFFF) * -7723592293110705685  # 0x94d049bb133111eb
        z = z ^ ((z >> 31) & 0x1FFFFFFFF)
        return ((z >> 33) & 0x7FFFFFFF) % world
    z = np.asarray(keys, np.uint64).copy()
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return ((z >> np.uint64(33)) % np.uint64(world)).astype(np.int64)


class GpuEngine:
    """One rank's device side: the local accumulator (K1), the owner table
    that folds the pairs routed to this rank and prunes them (K2), and the
    agglomeration context that runs K3 on the gathered significant set.
    Contexts are created once and reset per run (rg_reset), so repeated runs
    reuse their device buffers."""

    def __init__(self, params: GridParams, device: int, stream: int | None = None):
        import torch

        self.torch = torch
        self.params = params
        self.device = device
        self.dev = torch.device("cuda", device)
        self.local = _Context(params, device)
        self.owner = _Context(params, device)
        self.agg = _Context(params, device)
        for c in (self.local, self.owner, self.agg):
            c.check(c.lib.rg_set_stream(c.h, stream))

    def reset(self) -> None:
        for c in (self.local, self.owner):
            c.check(c.lib.rg_reset(c.h))

    # -- step 1
    def ingest(self, pts) -> None:
        p = _Points(pts)
        self.local.check(self.local.lib.rg_ingest(self.local.h, p.ptr, p.n, p.kind))

    def counters(self):
        c = self.local
        return c.u64(c.lib.rg_total_ingested), c.u64(c.lib.rg_skipped)

    # -- step 2 (device tensors)
    def export(self):
        torch = self.torch
        c = self.local
        d = c.u64(c.lib.rg_entry_count)
        keys = torch.empty(d, dtype=torch.int64, device=self.dev)
        cnts = torch.empty(d, dtype=torch.int64, device=self.dev)
        got = C.c_uint64()
        if d:
            c.check(c.lib.rg_export_entries(c.h, keys.data_ptr(), cnts.data_ptr(), d,
                                            C.byref(got), N.RG_MEM_DEVICE))
        return keys, cnts

    # -- step 3
    def owner_prune(self, keys, cnts):
        o = self.owner
        n = int(keys.numel())
        if n:
            o.check(o.lib.rg_ingest_counts(o.h, keys.data_ptr(), cnts.data_ptr(), n,
                                           N.RG_MEM_DEVICE))
        o.check(o.lib.rg_prune(o.h, None))
        s = o.stats().n_significant
        torch = self.torch
        tx, ty, cnt = (torch.empty(s, dtype=torch.int64, device=self.dev) for _ in range(3))
        if s:
            o.check(o.lib.rg_get_significant(o.h, tx.data_ptr(), ty.data_ptr(), cnt.data_ptr(),
                                             None, s, N.RG_MEM_DEVICE))
        return tx, ty, cnt

    # -- step 4 (result stays resident in self.agg)
    def agglomerate(self, tx, ty, cnt):
        a = self.agg
        n = int(tx.numel())
        tx, ty, cnt = tx.contiguous(), ty.contiguous(), cnt.contiguous()
        a.check(a.lib.rg_load_significant(a.h, tx.data_ptr() if n else None,
                                          ty.data_ptr() if n else None,
                                          cnt.data_ptr() if n else None, n, N.RG_MEM_DEVICE))
        a.check(a.lib.rg_agglomerate(a.h, None))
        s = a.stats()
        return int(s.n_significant), int(s.n_clusters)

    def flat(self) -> FlatClustering:
        return _flat_from_ctx(self.agg)

    def launches(self) -> int:
        return sum(int(c.lib.rg_kernel_launches(c.h)) for c in (self.local, self.owner, self.agg))


def _wire_device(dist, group, t):
    """NCCL moves device tensors over NVLink; other backends (gloo in the CPU
    tests) get host copies."""
    return t.device if dist.get_backend(group) == "nccl" else "cpu"


def _all_to_all(dist, group, send, send_counts, torch):
    world = dist.get_world_size(group)
    home, wire = send.device, _wire_device(dist, group, send)
    send = send.to(wire)
    sc = torch.tensor(send_counts, dtype=torch.int64, device=wire)
    rc = torch.empty(world, dtype=torch.int64, device=wire)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = rc.cpu().tolist()
    out = torch.empty(int(sum(recv_counts)), dtype=send.dtype, device=wire)
    dist.all_to_all_single(out, send, recv_counts, list(send_counts), group=group)
    return out.to(home), recv_counts


def _all_gather_var(dist, group, t, torch):
    """all_gather of a variable-length 1-D tensor (rank order preserved)."""
    world = dist.get_world_size(group)
    home, wire = t.device, _wire_device(dist, group, t)
    t = t.to(wire)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=wire)
    sizes = [torch.empty(1, dtype=torch.int64, device=wire) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    pad = torch.zeros(m, dtype=t.dtype, device=wire)
    pad[: t.numel()] = t
    bufs = [torch.empty(m, dtype=t.dtype, device=wire) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)]).to(home)


@dataclass
class DistributedStats:
    n_points: int = 0          # all ranks
    n_skipped: int = 0         # all ranks
    n_local_entries: int = 0   # this rank's distinct tiles before the exchange
    n_owned: int = 0           # pairs this rank received as owner
    n_significant: int = 0     # global
    n_clusters: int = 0        # global
    bytes_sent: int = 0        # this rank's all_to_all payload (keys + counts)


class DistributedPipeline:
    """cluster_sequential (pipeline.hpp:92-126) over the union of every
    rank's points (one process per GPU); every rank ends with the identical
    canonical clustering resident on its device."""

    def __init__(self, params: GridParams, group=None, engine=None, device: int | None = None,
                 stream: int | None = None):
        import torch
        import torch.distributed as dist

        params.validate()
        self.torch, self.dist = torch, dist
        self.params = params
        self.group = group
        self.world = dist.get_world_size(group)
        if engine is None:
            engine = GpuEngine(params, torch.cuda.current_device() if device is None else device,
                               stream)
        self.engine = engine

    def run(self, points) -> DistributedStats:
        torch, dist, group, eng = self.torch, self.dist, self.group, self.engine
        eng.reset()
        eng.ingest(points)
        keys, cnts = eng.export()
        st = DistributedStats(n_local_entries=int(keys.numel()))
        if self.world > 1:
            owner = owner_of(keys, self.world)
            order = torch.argsort(owner, stable=True)
            keys, cnts = keys[order], cnts[order]
            send_counts = torch.bincount(owner, minlength=self.world).cpu().tolist()
            keys, _ = _all_to_all(dist, group, keys, send_counts, torch)
            cnts, _ = _all_to_all(dist, group, cnts, send_counts, torch)
            st.bytes_sent = 16 * st.n_local_entries
        st.n_owned = int(keys.numel())
        tx, ty, cnt = eng.owner_prune(keys, cnts)
        if self.world > 1:
            tx = _all_gather_var(dist, group, tx, torch)
            ty = _all_gather_var(dist, group, ty, torch)
            cnt = _all_gather_var(dist, group, cnt, torch)
        st.n_significant, st.n_clusters = eng.agglomerate(tx, ty, cnt)
        ing, skp = eng.counters()
        tot = torch.tensor([ing, skp], dtype=torch.int64, device=_wire_device(dist, group, keys))
        if self.world > 1:
            dist.all_reduce(tot, group=group)
        st.n_points = int(tot[0].item() + tot[1].item())
        st.n_skipped = int(tot[1].item())
        self.stats = st
        return st

    def flat(self) -> FlatClustering:
        f = self.engine.flat()
        f.stats.n_points = self.stats.n_points
        f.stats.n_skipped = self.stats.n_skipped
        return f


def cluster_distributed(points, params: GridParams, group=None, engine=None,
                        device: int | None = None) -> FlatClustering:
    """One-shot DistributedPipeline: returns the identical canonical
    clustering of the union of all ranks' points on every rank."""
    pl = DistributedPipeline(params, group, engine, device)
    pl.run(points)
    return pl.flat()
