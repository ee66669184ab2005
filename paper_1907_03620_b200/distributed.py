"""Multi-GPU contraction + agglomeration (one process per GPU).

The path shards because counts add (TileAccumulator::merge,
accumulator.hpp:137-154) and because agglomeration over vertical slices
joins exactly at the slice borders (the reference's P-RASTER,
parallel.hpp:146-352). Significance is global (a tile whose points are
spread over ranks may reach tau only in total), so there are two exchange
steps:

  1. every rank contracts its own points into a local device table (K1);
  2. the ranks agree on column ranges, one per rank, balanced by a global
     histogram of their distinct tiles' columns (one all_reduce of 4096
     counts); local (packed key, count) pairs are routed to the owner of
     their column — one all_to_all of keys and one of counts (NCCL over
     NVLink on GPUs; gloo on CPU tensors in tests);
  3. each owner folds what it received (the counts-add half of merge),
     prunes with tau (K2) and runs K3 with mu = 1 on its own columns: its
     local components, in canonical order, with their tile counts;
  4. border join: the tiles within `distance` columns of a range edge, with
     their local component and its size, are all-gathered (a few hundred
     per rank); every rank runs the same small union-find over the
     components that touch across ranks. A joined component's
     representative is its member in the lowest rank (its smallest tile);
     its size is the sum; the mu filter applies to the joined size;
  5. canonical ids: each rank counts its kept representatives (one
     all_gather of one integer per rank), numbers them after the lower
     ranks' (column ranges are in order, so (rank, local order) is the
     lexicographic order of the smallest tiles, finalize_clusters
     agglomerate.hpp:175-191); joined components take their
     representative's id (one more small all_gather).

Each rank ends with its column range of the canonical result resident on
its device (sorted tiles, counts, global cluster ids); `flat()` gathers the
whole clustering (tests, host materialisation). No rank ever holds or
agglomerates the full significant set, so K3 scales with the ranks.

The per-rank engine is the sm_100a library (`GpuEngine`); tests inject a
CPU double through `engine=` to exercise the exchange logic on gloo. There
is no CPU fallback in the product path.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .raster import (FlatClustering, GridParams, PipelineStats, _Context, _Points,
                     neighbor_offsets, stream_arg)

N_BINS = 4096  # column histogram resolution for the range split


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
    """One rank's device side: the local accumulator (K1) and the owner
    context that folds the pairs routed to this rank, prunes them (K2) and
    finds its local components (K3, mu = 1). Contexts are created once and
    reset per run (rg_reset), so repeated runs reuse their device buffers."""

    def __init__(self, params: GridParams, device: int, stream: int | None = None):
        import torch

        self.torch = torch
        self.params = params
        self.device = device
        self.dev = torch.device("cuda", device)
        self.local = _Context(params, device)
        self.owner = _Context(dataclasses.replace(params, min_cluster_size=1), device)
        self.stream = stream
        for c in (self.local, self.owner):
            c.check(c.lib.rg_set_stream(c.h, stream_arg(stream)))
        ox, oy, by = C.c_int64(), C.c_int64(), C.c_uint32()
        self.local.check(self.local.lib.rg_key_packing(self.local.h, C.byref(ox), C.byref(oy),
                                                       C.byref(by)))
        self.origin_x, self.bits_y = int(ox.value), int(by.value)

    def reset(self) -> None:
        for c in (self.local, self.owner):
            c.check(c.lib.rg_reset(c.h))

    # -- step 1
    def ingest(self, pts) -> None:
        p = _Points(pts, self.stream is None)
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

    def route(self, keys, cnts, cmin: int, width: int, splits):
        """Pairs grouped by owner on the device (rg_route_pairs): (keys,
        counts, pairs per owner)."""
        torch = self.torch
        n, world = int(keys.numel()), len(splits) + 1
        ok = torch.empty_like(keys)
        oc = torch.empty_like(cnts)
        pc = torch.empty(world, dtype=torch.int64, device=self.dev)
        sp = torch.tensor(splits if splits else [0], dtype=torch.int32, device=self.dev)
        c = self.local
        c.check(c.lib.rg_route_pairs(c.h, keys.data_ptr() if n else None,
                                     cnts.data_ptr() if n else None, n, int(cmin), int(width),
                                     sp.data_ptr(), world, ok.data_ptr() if n else None,
                                     oc.data_ptr() if n else None, pc.data_ptr()))
        return ok, oc, pc.cpu().tolist()

    def key_column(self, keys):
        """Canvas column of packed keys (key = col << bits_y | row)."""
        return keys >> self.bits_y

    def column_x(self, col: int) -> int:
        return self.origin_x + int(col)

    # -- step 3: fold, prune, local components (result stays in self.owner)
    def owner_cluster(self, keys, cnts):
        """(tx, ty, count, local component id) of the owned significant
        tiles in lexicographic order, and the tile count of every local
        component (all device int64 tensors)."""
        torch = self.torch
        o = self.owner
        n = int(keys.numel())
        if n:
            o.check(o.lib.rg_ingest_counts(o.h, keys.data_ptr(), cnts.data_ptr(), n,
                                           N.RG_MEM_DEVICE))
        st = N.rg_stats()
        o.check(o.lib.rg_prune_agglomerate(o.h, 0, C.byref(st)))
        s, k = int(st.n_significant), int(st.n_clusters)
        tx, ty, cnt, cid = (torch.empty(s, dtype=torch.int64, device=self.dev) for _ in range(4))
        if s:
            o.check(o.lib.rg_get_significant(o.h, tx.data_ptr(), ty.data_ptr(), cnt.data_ptr(),
                                             cid.data_ptr(), s, N.RG_MEM_DEVICE))
        size = torch.empty(k, dtype=torch.int64, device=self.dev)
        if k:
            o.check(o.lib.rg_get_clusters(o.h, size.data_ptr(), None, None, None, k,
                                          N.RG_MEM_DEVICE))
        return tx, ty, cnt, cid, size

    def launches(self) -> int:
        return sum(int(c.lib.rg_kernel_launches(c.h)) for c in (self.local, self.owner))


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
    out = torch.empty((int(sum(recv_counts)),) + tuple(send.shape[1:]), dtype=send.dtype,
                      device=wire)
    dist.all_to_all_single(out, send, recv_counts, list(send_counts), group=group)
    return out.to(home), recv_counts


def _all_to_all_pairs(dist, group, keys, cnts, send_counts, torch):
    """(key, count) pairs to their owners in ONE exchange of a [m, 2] int64
    tensor (rows split by destination), instead of one per column."""
    kd, cd = keys.dtype, cnts.dtype
    pairs = torch.stack([keys.view(torch.int64), cnts.view(torch.int64)], 1).contiguous()
    out, _ = _all_to_all(dist, group, pairs, send_counts, torch)
    return out[:, 0].contiguous().view(kd), out[:, 1].contiguous().view(cd)


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
    n_owned_significant: int = 0  # significant tiles in this rank's columns
    n_border_tiles: int = 0    # tiles all ranks exchanged for the border join
    bytes_sent: int = 0        # this rank's all_to_all payload (keys + counts)


class _UF:
    def __init__(self):
        self.p = {}

    def find(self, a):
        self.p.setdefault(a, a)
        while self.p[a] != a:
            self.p[a] = self.p[self.p[a]]
            a = self.p[a]
        return a

    def union(self, a, b):
        ra, rb = self.find(a), self.find(b)
        if ra != rb:
            lo, hi = (ra, rb) if ra < rb else (rb, ra)
            self.p[hi] = lo


class DistributedPipeline:
    """cluster_sequential (pipeline.hpp:92-126) over the union of every
    rank's points (one process per GPU). Every rank ends with its column
    range of the canonical clustering resident on its device (`part`);
    `flat()` gathers the whole clustering."""

    def __init__(self, params: GridParams, group=None, engine=None, device: int | None = None,
                 stream: int | None = None):
        import torch
        import torch.distributed as dist

        params.validate()
        self.torch, self.dist = torch, dist
        self.params = params
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if engine is None:
            engine = GpuEngine(params, torch.cuda.current_device() if device is None else device,
                               stream)
        self.engine = engine
        self.offsets = [(int(t.x), int(t.y)) for t in neighbor_offsets(params)]
        self.part = None

    # -- step 2a: column ranges balanced by the global distinct-tile histogram
    def _splits(self, col, wire):
        torch, dist, group, world = self.torch, self.dist, self.group, self.world
        big = 1 << 62
        mm = torch.tensor([int(col.min()) if col.numel() else big,
                           -int(col.max()) if col.numel() else big], dtype=torch.int64,
                          device=wire)
        dist.all_reduce(mm, op=dist.ReduceOp.MIN, group=group)
        cmin, cmax = int(mm[0]), -int(mm[1])
        if cmin == big:  # no tiles anywhere
            return 0, 1, [0] * (world - 1)
        width = cmax - cmin + 1
        bins = ((col - cmin) * N_BINS) // width
        h = torch.bincount(bins, minlength=N_BINS).to(torch.int64).to(wire)
        dist.all_reduce(h, group=group)
        cum = torch.cumsum(h.cpu(), 0)
        tot = int(cum[-1])
        # rank r owns bins [s_r, s_r+1); s_r = first bin whose prefix reaches r/world
        sp = [int(torch.searchsorted(cum, (tot * r + world - 1) // world)) for r in range(1, world)]
        return cmin, width, sp

    def _col_lo(self, cmin, width, s):
        """Smallest column whose bin is >= s."""
        return cmin + (s * width + N_BINS - 1) // N_BINS

    def run(self, points) -> DistributedStats:
        torch, dist, group, eng, world, rank = (self.torch, self.dist, self.group, self.engine,
                                                self.world, self.rank)
        gp = self.params
        eng.reset()
        eng.ingest(points)
        keys, cnts = eng.export()
        st = DistributedStats(n_local_entries=int(keys.numel()))
        wire = _wire_device(dist, group, keys)
        col = eng.key_column(keys)
        cmin, width, sp = self._splits(col, wire)
        if world > 1:
            if hasattr(eng, "route"):  # device kernel (GpuEngine)
                keys, cnts, send_counts = eng.route(keys, cnts, cmin, width, sp)
            else:  # engine doubles in the tests
                bins = ((col - cmin) * N_BINS) // width
                owner = torch.searchsorted(torch.tensor(sp, dtype=torch.int64, device=col.device),
                                           bins, right=True)
                order = torch.argsort(owner, stable=True)
                keys, cnts = keys[order], cnts[order]
                send_counts = torch.bincount(owner, minlength=world).cpu().tolist()
            keys, cnts = _all_to_all_pairs(dist, group, keys, cnts, send_counts, torch)
            st.bytes_sent = 16 * st.n_local_entries
        st.n_owned = int(keys.numel())
        tx, ty, cnt, cid, size = eng.owner_cluster(keys, cnts)
        st.n_owned_significant = int(tx.numel())
        # this rank's columns [lo, hi) in tile x
        edges = [None] + sp + [None]
        lo = eng.column_x(self._col_lo(cmin, width, edges[rank])) if rank > 0 else None
        hi = eng.column_x(self._col_lo(cmin, width, edges[rank + 1])) if rank < world - 1 else None
        gid = self._border_join(tx, ty, cid, size, lo, hi, wire, st)
        self.part = (tx, ty, cnt, gid)
        ing, skp = eng.counters()
        tot = torch.tensor([ing, skp, int(tx.numel())], dtype=torch.int64, device=wire)
        if world > 1:
            dist.all_reduce(tot, group=group)
        st.n_points = int(tot[0].item() + tot[1].item())
        st.n_skipped = int(tot[1].item())
        st.n_significant = int(tot[2].item())
        st.n_clusters = self.stats_n_clusters
        self.stats = st
        return st

    # -- steps 4-5
    def _border_join(self, tx, ty, cid, size, lo, hi, wire, st):
        torch, dist, group, world, rank = (self.torch, self.dist, self.group, self.world,
                                           self.rank)
        mu = int(self.params.min_cluster_size)
        d = int(self.params.distance)
        dev = tx.device
        k = int(size.numel())
        # tiles within d columns of an edge shared with another rank
        near = torch.zeros(tx.numel(), dtype=torch.bool, device=dev)
        if lo is not None:
            near |= tx < lo + d
        if hi is not None:
            near |= tx >= hi - d
        idx = torch.nonzero(near).flatten()
        b_cid = cid[idx]
        border = torch.stack([tx[idx], ty[idx], b_cid, size[b_cid] if k else b_cid,
                              torch.full_like(b_cid, rank)], 1).flatten()
        if world > 1:
            border = _all_gather_var(dist, group, border, torch)
        b = border.view(-1, 5).cpu().numpy()
        st.n_border_tiles = int(b.shape[0])
        # union-find over (rank, local component) nodes joined across ranks
        uf = _UF()
        where = {}
        for x, y, c, _, r in b.tolist():
            where[(x, y)] = (r, c)
        node_size = {}
        for x, y, c, sz, r in b.tolist():
            node_size[(r, c)] = sz
            uf.find((r, c))
            for dx, dy in self.offsets:
                o = where.get((x + dx, y + dy))
                if o is not None and o[0] != r:
                    uf.union((r, c), o)
        sets = {}
        for nd, sz in node_size.items():
            rp = uf.find(nd)
            sets[rp] = sets.get(rp, 0) + sz
        # this rank's components: representative and final size
        final = size.clone()
        own_rep = torch.ones(k, dtype=torch.bool, device=dev)
        mine = [(nd, uf.find(nd)) for nd in node_size if nd[0] == rank]
        if mine:
            cs = torch.tensor([nd[1] for nd, _ in mine], dtype=torch.int64, device=dev)
            final[cs] = torch.tensor([sets[rp] for _, rp in mine], dtype=torch.int64, device=dev)
            own_rep[cs] = torch.tensor([rp == nd for nd, rp in mine], dtype=torch.bool,
                                       device=dev)
        kept = own_rep & (final >= mu)
        n_kept = torch.tensor([int(kept.sum())], dtype=torch.int64, device=wire)
        counts = [n_kept.clone() for _ in range(world)]
        if world > 1:
            dist.all_gather(counts, n_kept, group=group)
        counts = [int(c.item()) for c in counts]
        base = sum(counts[:rank])
        self.stats_n_clusters = sum(counts)
        gid_c = torch.where(kept, base + torch.cumsum(kept.to(torch.int64), 0) - 1,
                            torch.full_like(final, -1))
        # ids of joined components' representatives, published by their rank
        reps = sorted(rp for rp in sets if rp[0] == rank)
        pub = torch.tensor([[rp[1], int(gid_c[rp[1]])] for rp in reps] or
                           np.zeros((0, 2), np.int64), dtype=torch.int64,
                           device=wire).flatten()
        if world > 1:
            pub = _all_gather_var(dist, group, pub, torch)
            rank_of = _all_gather_var(dist, group, torch.full((len(reps),), rank,
                                                               dtype=torch.int64, device=wire),
                                      torch)
        else:
            rank_of = torch.full((len(reps),), rank, dtype=torch.int64)
        pub = pub.view(-1, 2).cpu().tolist()
        rep_gid = {(int(r), c): g for r, (c, g) in zip(rank_of.cpu().tolist(), pub)}
        joined = [(nd, rp) for nd, rp in mine if rp != nd]
        if joined:
            cs = torch.tensor([nd[1] for nd, _ in joined], dtype=torch.int64, device=dev)
            gid_c[cs] = torch.tensor([rep_gid[rp] for _, rp in joined], dtype=torch.int64,
                                     device=dev)
        return gid_c[cid] if k else cid

    def flat(self) -> FlatClustering:
        """The whole canonical clustering (every rank's columns, in order)."""
        torch, dist, group = self.torch, self.dist, self.group
        parts = list(self.part)
        if self.world > 1:
            parts = [_all_gather_var(dist, group, t, torch) for t in parts]
        tx, ty, cnt, gid = (t.cpu().numpy() for t in parts)
        stats = PipelineStats()
        stats.n_points = self.stats.n_points
        stats.n_skipped = self.stats.n_skipped
        stats.n_significant = int(tx.shape[0])
        stats.n_clusters = self.stats_n_clusters
        return FlatClustering(tx.astype(np.int64), ty.astype(np.int64),
                              cnt.astype(np.uint64), gid.astype(np.int64),
                              self.stats_n_clusters, stats)


def cluster_distributed(points, params: GridParams, group=None, engine=None,
                        device: int | None = None) -> FlatClustering:
    """One-shot DistributedPipeline: returns the identical canonical
    clustering of the union of all ranks' points on every rank."""
    pl = DistributedPipeline(params, group, engine, device)
    pl.run(points)
    return pl.flat()
