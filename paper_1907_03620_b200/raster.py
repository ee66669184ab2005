"""Python mirror of the reference's public API for the clustering path.

Same names, argument meaning and error behaviour as the reference C++ API in
/root/reference/proj/include/raster (cited per class/function), so parity
tests read like the reference's own tests. Every computation runs in the
sm_100a library through the C-ABI (include/raster_gpu.h); this module only
marshals buffers. The C++ drop-in for reference users is
include/raster_b200/gpu.hpp.

Points are float64 (x, y) pairs: a numpy array of shape (N, 2) (host memory;
pinned or pageable) or a CUDA torch tensor of shape (N, 2) (device memory,
zero-copy).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Iterable

import numpy as np

from . import _native as N


# --------------------------------------------------------------- errors.hpp
class Error(RuntimeError):
    """raster::Error errors.hpp:9-12"""


class ConfigError(Error):
    """raster::ConfigError errors.hpp:15-18"""


class OutOfBoundsError(Error):
    """raster::OutOfBoundsError errors.hpp:39-42"""


_STATUS_TO_EXC = {
    N.RG_ERR_CONFIG: ConfigError,
    N.RG_ERR_OOB: OutOfBoundsError,
    N.RG_ERR_UNSUPPORTED: ConfigError,
}


def _check(status: int, handle=None) -> None:
    if status == N.RG_OK:
        return
    msg = N.gpu().rg_last_error(handle).decode()
    raise _STATUS_TO_EXC.get(status, Error)(msg)


# ----------------------------------------------------------------- core.hpp
@dataclass(frozen=True, order=True)
class Tile:
    """raster::Tile core.hpp:48-54 — lexicographic (x, then y) order."""
    x: int
    y: int


@dataclass
class Bounds:
    """raster::Bounds core.hpp:27-42 (closed canvas)."""
    x_min: float = -180.0
    x_max: float = 180.0
    y_min: float = -90.0
    y_max: float = 90.0

    def contains(self, x: float, y: float) -> bool:
        return self.x_min <= x <= self.x_max and self.y_min <= y <= self.y_max

    @staticmethod
    def gps() -> "Bounds":
        return Bounds()


class Metric(IntEnum):
    chebyshev = 0
    manhattan = 1


class Mode(IntEnum):
    count_only = 0
    retain_points = 1


class OobPolicy(IntEnum):
    skip = 0
    strict = 1


@dataclass
class GridParams:
    """raster::GridParams core.hpp:84-132 (+ capacity_hint for the device table)."""
    precision: float = 3.5
    bounds: Bounds = field(default_factory=Bounds)
    threshold: int = 5
    distance: int = 1
    metric: Metric = Metric.chebyshev
    min_cluster_size: int = 4
    mode: Mode = Mode.count_only
    oob_policy: OobPolicy = OobPolicy.skip
    dedupe_points: bool = False
    capacity_hint: int = 0

    def _c(self) -> N.rg_params:
        p = N.rg_params()
        p.precision = float(self.precision)
        p.x_min, p.x_max = float(self.bounds.x_min), float(self.bounds.x_max)
        p.y_min, p.y_max = float(self.bounds.y_min), float(self.bounds.y_max)
        p.threshold = max(int(self.threshold), 0)
        p.distance = int(self.distance)
        p.metric = int(self.metric)
        p.min_cluster_size = max(int(self.min_cluster_size), 0)
        p.mode = int(self.mode)
        p.oob_policy = int(self.oob_policy)
        p.dedupe_points = int(bool(self.dedupe_points))
        p.capacity_hint = int(self.capacity_hint)
        return p

    def scale(self) -> float:
        """core.hpp:95 — pow(10, p) by the host libm (the device never calls pow)."""
        return N.gpu().rg_params_scale(C.byref(self._c()))

    def validate(self) -> None:
        """core.hpp:98-115 — raises ConfigError."""
        if self.threshold < 1:
            raise ConfigError("threshold must be >= 1")
        if self.min_cluster_size < 1:
            raise ConfigError("min cluster size must be >= 1")
        buf = C.create_string_buffer(512)
        st = N.gpu().rg_params_validate(C.byref(self._c()), buf, 512)
        if st != N.RG_OK:
            raise _STATUS_TO_EXC.get(st, Error)(buf.value.decode())

    def min_column(self) -> int:
        return N.gpu().rg_params_min_column(C.byref(self._c()))

    def max_column(self) -> int:
        return N.gpu().rg_params_max_column(C.byref(self._c()))

    def tile_bound(self) -> float:
        return N.gpu().rg_params_tile_bound(C.byref(self._c()))


@dataclass
class PipelineStats:
    """raster::PipelineStats pipeline.hpp:64-72, plus device-side detail."""
    t_total: float = 0.0
    t_projection: float = 0.0
    t_clustering: float = 0.0
    n_points: int = 0
    n_skipped: int = 0
    peak_accumulator_entries: int = 0
    n_significant: int = 0
    n_clusters: int = 0
    table_capacity: int = 0
    table_grows: int = 0
    ms_contract: float = 0.0
    ms_prune: float = 0.0
    ms_agglomerate: float = 0.0
    ms_label: float = 0.0

    def _fill(self, s: N.rg_stats) -> None:
        self.n_points = s.n_points
        self.n_skipped = s.n_skipped
        self.peak_accumulator_entries = s.peak_accumulator_entries
        self.n_significant = s.n_significant
        self.n_clusters = s.n_clusters
        self.table_capacity = s.table_capacity
        self.table_grows = s.table_grows
        self.ms_contract, self.ms_prune = s.ms_contract, s.ms_prune
        self.ms_agglomerate, self.ms_label = s.ms_agglomerate, s.ms_label
        self.t_projection = (s.ms_contract + s.ms_prune) / 1e3
        self.t_clustering = s.ms_agglomerate / 1e3
        self.t_total = self.t_projection + self.t_clustering


# ---------------------------------------------------------- buffer helpers
def stream_arg(stream_ptr: int | None):
    """rg_set_stream argument for a cudaStream_t handle: None = the
    context's private stream; 0 (the legacy default stream, which is what
    torch.cuda.current_stream() reports by default) = cudaStreamLegacy."""
    if stream_ptr is None:
        return None
    return 1 if int(stream_ptr) == 0 else int(stream_ptr)


class _Points:
    """(pointer, n, memkind) view of a point buffer, keeping it alive."""

    def __init__(self, pts, settle: bool = True):
        """settle: a CUDA tensor may still be being written by torch's
        current stream; unless the context runs on that stream
        (set_stream), wait for it first."""
        self.keep = pts
        if hasattr(pts, "data_ptr") and hasattr(pts, "is_cuda"):
            import torch

            if pts.dtype != torch.float64:
                raise Error("points must be float64")
            if pts.numel() and (pts.dim() != 2 or pts.shape[1] != 2 or not pts.is_contiguous()):
                raise Error("points must be a contiguous (N, 2) tensor")
            self.n = pts.shape[0] if pts.numel() else 0
            self.ptr = pts.data_ptr() if self.n else None
            self.kind = N.RG_MEM_DEVICE if pts.is_cuda else N.RG_MEM_HOST
            if settle and pts.is_cuda and self.n:
                torch.cuda.current_stream(pts.device).synchronize()
            return
        arr = np.asarray(pts, dtype=np.float64)
        if arr.size == 0:
            arr = np.zeros((0, 2), dtype=np.float64)
        arr = np.ascontiguousarray(arr.reshape(-1, 2))
        self.keep = arr
        self.n = arr.shape[0]
        self.ptr = arr.ctypes.data if self.n else None
        self.kind = N.RG_MEM_HOST


class _Context:
    """One device accumulator (rg_ctx*)."""

    def __init__(self, params: GridParams, device: int = -1):
        lib = N.gpu()
        h = C.c_void_p()
        st = lib.rg_create(C.byref(params._c()), int(device), C.byref(h))
        if st != N.RG_OK:
            raise _STATUS_TO_EXC.get(st, Error)(lib.rg_last_error(None).decode())
        self.h = h
        self.lib = lib
        self.params = params

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.rg_destroy(h)
            self.h = None

    def check(self, st: int) -> None:
        _check(st, self.h)

    def u64(self, fn) -> int:
        v = C.c_uint64()
        self.check(fn(self.h, C.byref(v)))
        return v.value

    def stats(self) -> N.rg_stats:
        s = N.rg_stats()
        self.check(self.lib.rg_get_stats(self.h, C.byref(s)))
        return s

    def significant_arrays(self, with_cid: bool):
        n = self.stats().n_significant
        tx = np.empty(n, np.int64)
        ty = np.empty(n, np.int64)
        cnt = np.empty(n, np.uint64)
        cid = np.empty(n, np.int64) if with_cid else None
        if n:
            self.check(self.lib.rg_get_significant(
                self.h, tx.ctypes.data, ty.ctypes.data, cnt.ctypes.data,
                cid.ctypes.data if with_cid else None, n, N.RG_MEM_HOST))
        return tx, ty, cnt, cid


# ----------------------------------------------------------- accumulator.hpp
class SignificantTiles:
    """raster::SignificantTiles accumulator.hpp:21 — tile -> TileStats.

    Backed by sorted flat arrays; keeps the device context that produced it
    so agglomerate() runs on the already-resident set.
    """

    @dataclass
    class TileStats:
        count: int
        points: list = field(default_factory=list)

    def __init__(self, tx, ty, count, ctx: _Context | None = None):
        self.tx = np.asarray(tx, np.int64)
        self.ty = np.asarray(ty, np.int64)
        self.count = np.asarray(count, np.uint64)
        self._ctx = ctx

    @classmethod
    def from_dict(cls, d: dict) -> "SignificantTiles":
        items = sorted(d.items())
        tx = [t.x for t, _ in items]
        ty = [t.y for t, _ in items]
        cnt = [(s.count if hasattr(s, "count") else int(s)) for _, s in items]
        return cls(tx, ty, cnt)

    def __len__(self) -> int:
        return int(self.tx.shape[0])

    def size(self) -> int:
        return len(self)

    def empty(self) -> bool:
        return len(self) == 0

    def _find(self, t: Tile) -> int:
        i = np.searchsorted(self.tx, t.x, side="left")
        j = np.searchsorted(self.tx, t.x, side="right")
        k = i + np.searchsorted(self.ty[i:j], t.y)
        return int(k) if k < j and self.ty[k] == t.y else -1

    def __contains__(self, t: Tile) -> bool:
        return self._find(t) >= 0

    contains = __contains__

    def at(self, t: Tile) -> "SignificantTiles.TileStats":
        k = self._find(t)
        if k < 0:
            raise KeyError(t)
        return SignificantTiles.TileStats(int(self.count[k]))

    def items(self):
        for x, y, c in zip(self.tx.tolist(), self.ty.tolist(), self.count.tolist()):
            yield Tile(x, y), SignificantTiles.TileStats(c)

    def tiles(self) -> list[Tile]:
        return [Tile(x, y) for x, y in zip(self.tx.tolist(), self.ty.tolist())]


class TileAccumulator:
    """raster::TileAccumulator accumulator.hpp:109-214, on the device."""

    def __init__(self, params: GridParams, device: int = -1):
        params.validate()  # accumulator.hpp:112
        self._params = params
        self._ctx = _Context(params, device)

    def params(self) -> GridParams:
        return self._params

    def ingest(self, pts) -> None:
        """accumulator.hpp:117-134 — any chunking, any order."""
        p = _Points(pts, getattr(self, "_settle", True))
        self._ctx.check(self._ctx.lib.rg_ingest(self._ctx.h, p.ptr, p.n, p.kind))

    def ingest_source(self, read, chunk_points: int = 1 << 22) -> int:
        """ingest_all io.hpp:226-241 over a PointSource-like callable:
        read(out) fills the (k, 2) float64 array `out` (a pinned staging
        buffer) with up to k points and returns how many it wrote (0: the
        source is exhausted). Each chunk's copy and contraction run while the
        next read fills the other buffer. Returns the points read."""
        lib, h = self._ctx.lib, self._ctx.h
        self._ctx.check(lib.rg_stream_begin(h, int(chunk_points)))
        total = 0
        try:
            while True:
                buf, cap = C.c_void_p(), C.c_uint64()
                self._ctx.check(lib.rg_stream_buffer(h, C.byref(buf), C.byref(cap)))
                out = np.ctypeslib.as_array((C.c_double * (2 * cap.value)).from_address(buf.value))
                k = int(read(out.reshape(-1, 2)))
                if k <= 0:
                    break
                self._ctx.check(lib.rg_stream_submit(h, k))
                total += k
        finally:
            self._ctx.check(lib.rg_stream_end(h))
        return total

    def merge(self, other: "TileAccumulator") -> None:
        """accumulator.hpp:137-154"""
        self._ctx.check(self._ctx.lib.rg_merge(self._ctx.h, other._ctx.h))

    def prune(self) -> SignificantTiles:
        """accumulator.hpp:156-174 — consumes the accumulator."""
        self._ctx.check(self._ctx.lib.rg_prune(self._ctx.h, None))
        tx, ty, cnt, _ = self._ctx.significant_arrays(False)
        return SignificantTiles(tx, ty, cnt, self._ctx)

    def copy(self) -> "TileAccumulator":
        """The reference's TileAccumulator copy (test_agglomerate.cpp:268)."""
        out = TileAccumulator.__new__(TileAccumulator)
        out._params = self._params
        h = C.c_void_p()
        self._ctx.check(self._ctx.lib.rg_clone(self._ctx.h, C.byref(h)))
        ctx = _Context.__new__(_Context)
        ctx.h, ctx.lib, ctx.params = h, self._ctx.lib, self._params
        out._ctx = ctx
        return out

    __copy__ = copy

    def entry_count(self) -> int:
        return self._ctx.u64(self._ctx.lib.rg_entry_count)

    def count_of(self, t: Tile) -> int:
        v = C.c_uint64()
        self._ctx.check(self._ctx.lib.rg_count_of(self._ctx.h, int(t.x), int(t.y), C.byref(v)))
        return v.value

    def counts(self) -> dict:
        """Snapshot of for_each_count accumulator.hpp:188-191 as {Tile: count}."""
        tx, ty, cnt = self.count_arrays()
        return {Tile(x, y): c for x, y, c in zip(tx.tolist(), ty.tolist(), cnt.tolist())}

    def count_arrays(self):
        n = self.entry_count()
        tx = np.empty(n, np.int64)
        ty = np.empty(n, np.int64)
        cnt = np.empty(n, np.uint64)
        got = C.c_uint64()
        if n:
            self._ctx.check(self._ctx.lib.rg_export_counts(
                self._ctx.h, tx.ctypes.data, ty.ctypes.data, cnt.ctypes.data, n, C.byref(got)))
        return tx, ty, cnt

    def for_each_count(self, fn) -> None:
        for t, c in self.counts().items():
            fn(t, c)

    def total_ingested(self) -> int:
        return self._ctx.u64(self._ctx.lib.rg_total_ingested)

    def skipped(self) -> int:
        return self._ctx.u64(self._ctx.lib.rg_skipped)


def window_fix(acc: TileAccumulator, params: GridParams) -> SignificantTiles:
    """window_fix agglomerate.hpp:212-246 on the device: occupied tiles with
    a 2x2 window of >= threshold points. Like the reference it leaves `acc`
    untouched (it runs on a device copy)."""
    work = acc.copy()
    work._ctx.check(work._ctx.lib.rg_window_fix(work._ctx.h, None))
    tx, ty, cnt, _ = work._ctx.significant_arrays(False)
    return SignificantTiles(tx, ty, cnt, work._ctx)


# ----------------------------------------------------------- agglomerate.hpp
@dataclass
class Cluster:
    """raster::Cluster agglomerate.hpp:18-24"""
    id: int
    tiles: list
    points: list = field(default_factory=list)


@dataclass
class ClusterSet:
    """raster::ClusterSet agglomerate.hpp:28-32"""
    clusters: list = field(default_factory=list)


def neighbor_offsets(params: GridParams) -> list[Tile]:
    """agglomerate.hpp:38-50"""
    d = params.distance
    out = []
    for dx in range(-d, d + 1):
        for dy in range(-d, d + 1):
            if dx == 0 and dy == 0:
                continue
            if params.metric == Metric.manhattan and abs(dx) + abs(dy) > d:
                continue
            out.append(Tile(dx, dy))
    return out


@dataclass
class FlatClustering:
    """Device result in flat canonical form: significant tiles sorted
    lexicographically with counts and cluster ids (-1 = dropped)."""
    tx: np.ndarray
    ty: np.ndarray
    count: np.ndarray
    cluster_id: np.ndarray
    n_clusters: int
    stats: PipelineStats

    def cluster_set(self) -> ClusterSet:
        """finalize_clusters agglomerate.hpp:175-191 form (host materialisation)."""
        keep = self.cluster_id >= 0
        cid = self.cluster_id[keep]
        order = np.argsort(cid, kind="stable")  # tiles already sorted within a cluster
        tx, ty, cid = self.tx[keep][order], self.ty[keep][order], cid[order]
        clusters = []
        if cid.size:
            bounds = np.flatnonzero(np.diff(cid)) + 1
            starts = np.concatenate(([0], bounds))
            ends = np.concatenate((bounds, [cid.size]))
            for s, e in zip(starts.tolist(), ends.tolist()):
                clusters.append(Cluster(int(cid[s]), [Tile(x, y) for x, y in
                                                      zip(tx[s:e].tolist(), ty[s:e].tolist())]))
        return ClusterSet(clusters)


def _flat_from_ctx(ctx: _Context) -> FlatClustering:
    tx, ty, cnt, cid = ctx.significant_arrays(True)
    s = ctx.stats()
    st = PipelineStats()
    st._fill(s)
    return FlatClustering(tx, ty, cnt, cid, int(s.n_clusters), st)


def agglomerate_flat(sig, params: GridParams, device: int = -1) -> FlatClustering:
    """agglomerate agglomerate.hpp:196-201 in flat form."""
    if isinstance(sig, dict):
        sig = SignificantTiles.from_dict(sig)
    ctx = sig._ctx
    if ctx is None or ctx.params is not params:
        ctx = _Context(params, device)
        n = len(sig)
        tx = np.ascontiguousarray(sig.tx)
        ty = np.ascontiguousarray(sig.ty)
        cnt = np.ascontiguousarray(sig.count)
        ctx.check(ctx.lib.rg_load_significant(ctx.h, tx.ctypes.data if n else None,
                                              ty.ctypes.data if n else None,
                                              cnt.ctypes.data if n else None, n, N.RG_MEM_HOST))
    ctx.check(ctx.lib.rg_agglomerate(ctx.h, None))
    return _flat_from_ctx(ctx)


def agglomerate(sig, params: GridParams) -> ClusterSet:
    """agglomerate agglomerate.hpp:196-201 — connected components, the mu
    filter and canonical ids, on the device."""
    params.validate()
    return agglomerate_flat(sig, params).cluster_set()


# -------------------------------------------------------------- pipeline.hpp
class Pipeline:
    """A reusable device context for repeated cluster_sequential calls
    (benchmarks, serving): one accumulator, one stream."""

    def __init__(self, params: GridParams, device: int = -1):
        params.validate()
        self.params = params
        self.ctx = _Context(params, device)

    def set_stream(self, stream_ptr: int | None) -> None:
        """Run on a caller stream, e.g. torch.cuda.current_stream().cuda_stream
        (handle 0, torch's legacy default stream, is passed as
        cudaStreamLegacy so the work stays ordered with it); None restores
        the context's private stream."""
        self.ctx.check(self.ctx.lib.rg_set_stream(self.ctx.h, stream_arg(stream_ptr)))
        self._settle = stream_ptr is None

    def run(self, pts, use_window_fix: bool = False) -> N.rg_stats:
        """cluster_sequential pipeline.hpp:92-126 on the device; results stay
        resident (device_view / flat / labels)."""
        p = _Points(pts, getattr(self, "_settle", True))
        s = N.rg_stats()
        flags = N.RG_CLUSTER_WINDOW_FIX if use_window_fix else 0
        self.ctx.check(self.ctx.lib.rg_cluster_ex(self.ctx.h, p.ptr, p.n, p.kind, flags,
                                                  C.byref(s)))
        return s

    def device_view(self) -> N.rg_device_view:
        v = N.rg_device_view()
        self.ctx.check(self.ctx.lib.rg_device_result(self.ctx.h, C.byref(v)))
        return v

    def flat(self) -> FlatClustering:
        return _flat_from_ctx(self.ctx)

    def label_points(self, pts, out=None):
        """Per-point cluster ids (point-retaining variant). For device points
        `out` may be a preallocated int32 CUDA tensor."""
        p = _Points(pts, getattr(self, "_settle", True))
        if p.kind == N.RG_MEM_DEVICE:
            import torch
            if out is None:
                out = torch.empty(p.n, dtype=torch.int32, device=pts.device)
            ptr = out.data_ptr() if p.n else None
        else:
            if out is None:
                out = np.empty(p.n, np.int32)
            ptr = out.ctypes.data if p.n else None
        self.ctx.check(self.ctx.lib.rg_label_points(self.ctx.h, p.ptr, p.n, ptr, p.kind))
        return out

    def cluster_points(self, pts, device_out: bool = False):
        """RASTER' output on the device (take_points agglomerate.hpp:70-76,
        finalize_clusters :183): (points (M, 2) float64 grouped by cluster id
        and point_less-sorted within a cluster, offsets (C + 1,) uint64)."""
        p = _Points(pts, getattr(self, "_settle", True))
        m, c = C.c_uint64(), C.c_uint64()
        self.ctx.check(self.ctx.lib.rg_cluster_points(self.ctx.h, p.ptr, p.n, p.kind,
                                                      C.byref(m), C.byref(c)))
        if device_out:
            import torch

            xy = torch.empty((m.value, 2), dtype=torch.float64, device="cuda")
            off = torch.empty(c.value + 1, dtype=torch.int64, device="cuda")
            self.ctx.check(self.ctx.lib.rg_get_cluster_points(
                self.ctx.h, xy.data_ptr() if m.value else None, m.value, off.data_ptr(),
                N.RG_MEM_DEVICE))
            return xy, off
        xy = np.empty((m.value, 2), np.float64)
        off = np.empty(c.value + 1, np.uint64)
        self.ctx.check(self.ctx.lib.rg_get_cluster_points(
            self.ctx.h, xy.ctypes.data if m.value else None, m.value, off.ctypes.data,
            N.RG_MEM_HOST))
        return xy, off

    def cluster_facts(self):
        """Per cluster k (canonical id order): (tiles, points, first tile x,
        first tile y) as numpy arrays — the sizes finalize_clusters orders by
        (agglomerate.hpp:175-191) plus the cluster's point total."""
        n = int(self.ctx.stats().n_clusters)
        nt = np.empty(n, np.uint64)
        npnt = np.empty(n, np.uint64)
        fx = np.empty(n, np.int64)
        fy = np.empty(n, np.int64)
        if n:
            self.ctx.check(self.ctx.lib.rg_get_clusters(
                self.ctx.h, nt.ctypes.data, npnt.ctypes.data, fx.ctypes.data, fy.ctypes.data, n,
                N.RG_MEM_HOST))
        return nt, npnt, fx, fy

    def launches(self) -> int:
        return int(self.ctx.lib.rg_kernel_launches(self.ctx.h))


def cluster_flat(pts, params: GridParams, device: int = -1,
                 use_window_fix: bool = False) -> FlatClustering:
    pl = Pipeline(params, device)
    pl.run(pts, use_window_fix)
    return pl.flat()


def cluster_sequential(pts, params: GridParams, use_window_fix: bool = False,
                       stats: PipelineStats | None = None) -> ClusterSet:
    """cluster_sequential pipeline.hpp:92-126 on the device. In
    retain_points mode every cluster's points are attached, grouped and
    point_less-sorted on the device (rg_cluster_points)."""
    params.validate()
    pl = Pipeline(params)
    p = _Points(pts)
    pl.run(pts, use_window_fix)
    flat = pl.flat()
    if stats is not None:
        st = pl.ctx.stats()
        stats._fill(st)
    cs = flat.cluster_set()
    if params.mode == Mode.retain_points and cs.clusters:
        xy, off = pl.cluster_points(p.keep)
        for k, c in enumerate(cs.clusters):
            s, e = int(off[k]), int(off[k + 1])
            c.points = list(zip(xy[s:e, 0].tolist(), xy[s:e, 1].tolist()))
    return cs


def device_count() -> int:
    return int(N.gpu().rg_device_count())
