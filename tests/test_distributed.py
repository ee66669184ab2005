"""The N>1 exchange (paper_1907_03620_b200/distributed.py) on CPU: two gloo
ranks, each holding a shard of the points, must produce exactly the oracle's
single-process clustering of the union — including tiles that reach tau only
when both ranks' counts are added. The per-rank engine is a numpy double
(test-only) so the exchange logic is what is under test here; the GPU engine
runs the same code in test_gpu_distributed.py."""
from __future__ import annotations

import dataclasses
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as O
from paper_1907_03620_b200.distributed import cluster_distributed, owner_of
from paper_1907_03620_b200.raster import FlatClustering, GridParams, PipelineStats

from .gpu_util import numpy_tile_counts

_OFF = 1 << 30


class NumpyEngine:
    """Test double for GpuEngine: dict tallies, the oracle's agglomeration."""

    def __init__(self, gp: GridParams):
        self.gp = gp
        self.tally: dict = {}
        self.ing = self.skp = 0

    def reset(self):
        self.tally, self.ing, self.skp = {}, 0, 0

    def ingest(self, pts):
        pts = np.asarray(pts, np.float64).reshape(-1, 2)
        c = numpy_tile_counts(pts, self.gp)
        for k, v in c.items():
            self.tally[k] = self.tally.get(k, 0) + v
        n_in = sum(c.values())
        self.ing += n_in
        self.skp += len(pts) - n_in

    def counters(self):
        return self.ing, self.skp

    def export(self):
        items = sorted(self.tally.items())
        keys = [((x + _OFF) << 32) | (y + _OFF) for (x, y), _ in items]
        return (torch.tensor(keys, dtype=torch.int64),
                torch.tensor([c for _, c in items], dtype=torch.int64))

    def key_column(self, keys):
        return keys >> 32

    def column_x(self, col):
        return int(col) - _OFF

    def owner_cluster(self, keys, cnts):
        k, inv = np.unique(keys.numpy(), return_inverse=True)
        tot = np.bincount(inv, weights=cnts.numpy().astype(np.float64), minlength=k.size)
        keep = tot >= self.gp.threshold
        k, tot = k[keep], tot[keep].astype(np.int64)
        tx, ty = (k >> 32) - _OFF, (k & 0xFFFFFFFF) - _OFF
        g1 = dataclasses.replace(self.gp, min_cluster_size=1)
        r = O.port_agglomerate(tx, ty, tot.astype(np.uint64), g1)
        size = np.bincount(r.cluster_id, minlength=r.n_clusters) if len(r.tx) else np.zeros(0)
        return (torch.from_numpy(r.tx.astype(np.int64)), torch.from_numpy(r.ty.astype(np.int64)),
                torch.from_numpy(r.count.astype(np.int64)),
                torch.from_numpy(r.cluster_id.astype(np.int64)),
                torch.from_numpy(size.astype(np.int64)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, shards, gp, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        flat = cluster_distributed(shards[rank], gp, engine=NumpyEngine(gp))
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), tx=flat.tx, ty=flat.ty,
                 count=flat.count.astype(np.uint64), cid=flat.cluster_id,
                 n=np.array([flat.n_clusters, flat.stats.n_points, flat.stats.n_skipped]))
    finally:
        dist.destroy_process_group()


def _run(shards, gp, tmp_path, world=2):
    mp.start_processes(_worker, args=(world, _free_port(), shards, gp, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    return [np.load(tmp_path / f"r{r}.npz") for r in range(world)]


def _check(outs, pts, gp):
    ref = O.port_cluster(pts, gp)
    for o in outs:
        assert np.array_equal(o["tx"], ref.tx) and np.array_equal(o["ty"], ref.ty)
        assert np.array_equal(o["count"], ref.count.astype(np.uint64))
        assert np.array_equal(o["cid"], ref.cluster_id)
        n_clusters, n_points, _ = o["n"].tolist()
        assert n_clusters == ref.n_clusters and n_points == len(pts)


def test_owner_hash_torch_matches_numpy():
    rng = np.random.default_rng(3)
    k = rng.integers(0, 2**63 - 1, 10000, dtype=np.int64)
    for world in (2, 3, 8):
        a = owner_of(torch.from_numpy(k), world).numpy()
        b = owner_of(k.astype(np.uint64), world)
        assert np.array_equal(a, b) and a.min() >= 0 and a.max() < world
        assert np.bincount(a, minlength=world).min() > 10000 / world * 0.8


def test_two_ranks_match_single_process(tmp_path):
    rng = np.random.default_rng(11)
    gp = GridParams(precision=2.0, threshold=4, distance=1, min_cluster_size=3)
    blobs = np.concatenate([rng.normal(c, 0.05, size=(3000, 2)) for c in
                            ([0.0, 0.0], [0.4, 0.1], [-1.0, 2.0], [3.0, -3.0])])
    noise = rng.uniform(-5, 5, size=(4000, 2))
    pts = np.concatenate([blobs, noise, [[500.0, 0.0], [np.nan, 1.0]]])
    rng.shuffle(pts)
    half = len(pts) // 2
    _check(_run([pts[:half], pts[half:]], gp, tmp_path), pts, gp)


def test_significance_only_in_total(tmp_path):
    """Each tile gets tau-1 points on one rank and 1 on the other: neither
    rank alone sees a significant tile."""
    gp = GridParams(precision=1.0, threshold=5, distance=1, min_cluster_size=2)
    tiles = np.array([[0, 0], [1, 0], [2, 1], [7, 7], [9, 9], [10, 10]])
    centre = (tiles + 0.5) / 10.0
    a = np.repeat(centre, 4, axis=0)
    b = centre.copy()
    pts = np.concatenate([a, b])
    _check(_run([a, b], gp, tmp_path), pts, gp)


def test_empty_rank(tmp_path):
    gp = GridParams(precision=1.0, threshold=2, min_cluster_size=1)
    pts = np.repeat(np.array([[0.05, 0.05], [0.15, 0.05]]), 3, axis=0)
    _check(_run([pts, np.zeros((0, 2))], gp, tmp_path), pts, gp)


def test_components_across_ranks_three_ranks(tmp_path):
    """Column-partitioned agglomeration: a chain spanning every rank's
    columns, and dominoes placed so that every possible range boundary cuts
    one of them in two — those reach mu = 2 only when joined across ranks
    (P-RASTER's border join, parallel.hpp:146-352)."""
    gp = GridParams(precision=0.0, threshold=1, distance=1, min_cluster_size=2)
    tiles = [(x, 0) for x in range(-150, 150)]
    for row, off in ((20, 0), (40, 1), (60, 2)):
        for x in range(-150 + off, 148, 3):
            tiles += [(x, row), (x + 1, row)]
    tiles += [(-100, -50), (100, -50)]  # singletons: dropped by mu
    pts = np.array(tiles, np.float64) + 0.5
    rng = np.random.default_rng(2)
    rng.shuffle(pts)
    shards = [pts[0::3], pts[1::3], pts[2::3]]
    _check(_run(shards, gp, tmp_path, world=3), pts, gp)


def test_manhattan_delta2_across_ranks(tmp_path):
    """Border strips are `distance` columns wide: Manhattan delta 2 joins
    (x, y) with (x+2, y) and (x+1, y+1) across a range edge."""
    gp = GridParams(precision=0.0, threshold=1, distance=2, metric=1, min_cluster_size=3)
    rng = np.random.default_rng(9)
    tiles = {(int(x), int(y)) for x, y in rng.integers([-120, -60], [120, 60], size=(2500, 2))}
    pts = np.array(sorted(tiles), np.float64) + 0.5
    rng.shuffle(pts)
    _check(_run([pts[0::2], pts[1::2]], gp, tmp_path), pts, gp)
