"""The exchange primitives (rg_export_entries / rg_ingest_counts) and the
N-rank path with the real device engine. Two gloo ranks share cuda:0 here —
their kernels never wait on each other (the exchange goes through host
copies), so this is a correctness check of the GPU engine under the
exchange, not a stand-in for multi-GPU timing. Needs a B200."""
from __future__ import annotations

import ctypes as C
import dataclasses
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1907_03620_b200 import _native as N
from paper_1907_03620_b200 import datagen as D
from paper_1907_03620_b200.distributed import DistributedPipeline, GpuEngine, cluster_distributed
from paper_1907_03620_b200.raster import GridParams, TileAccumulator

from .gpu_util import assert_same, oracle
from .test_distributed import _free_port

pytestmark = pytest.mark.gpu


def test_export_then_ingest_counts_roundtrip():
    pts = D.generate(D.spec(2, 0.2), shuffle_seed=3)
    gp = D.params(2)
    eng = GpuEngine(gp, 0)
    eng.ingest(pts[: len(pts) // 3])
    eng2 = GpuEngine(gp, 0)
    eng2.ingest(pts[len(pts) // 3:])
    k1, c1 = eng.export()
    k2, c2 = eng2.export()
    assert int(c1.sum() + c2.sum()) == eng.counters()[0] + eng2.counters()[0]
    tx, ty, cnt, cid, size = eng.owner_cluster(torch.cat([k1, k2]), torch.cat([c1, c2]))
    ref = oracle(pts, gp)
    assert np.array_equal(tx.cpu().numpy(), ref.tx)
    assert np.array_equal(ty.cpu().numpy(), ref.ty)
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint64), ref.count.astype(np.uint64))
    # the owner's components are found with mu = 1 (the filter is global)
    ref1 = oracle(pts, dataclasses.replace(gp, min_cluster_size=1))
    assert np.array_equal(cid.cpu().numpy(), ref1.cluster_id)
    assert np.array_equal(size.cpu().numpy(), np.bincount(ref1.cluster_id))


def test_export_host_and_ingest_counts_host():
    gp = GridParams(precision=2.0, threshold=1, min_cluster_size=1)
    rng = np.random.default_rng(4)
    pts = rng.normal(0, 0.3, size=(50000, 2))
    a = TileAccumulator(gp)
    a.ingest(pts)
    ctx = a._ctx
    d = a.entry_count()
    keys = np.empty(d, np.uint64)
    cnts = np.empty(d, np.uint64)
    got = C.c_uint64()
    ctx.check(ctx.lib.rg_export_entries(ctx.h, keys.ctypes.data, cnts.ctypes.data, d,
                                        C.byref(got), N.RG_MEM_HOST))
    assert got.value == d and int(cnts.sum()) == len(pts)
    assert np.unique(keys).size == d
    b = TileAccumulator(gp)
    # fold twice: counts must double, entries must not
    for _ in range(2):
        b._ctx.check(b._ctx.lib.rg_ingest_counts(b._ctx.h, keys.ctypes.data, cnts.ctypes.data,
                                                 d, N.RG_MEM_HOST))
    assert b.entry_count() == d and b.total_ingested() == 2 * len(pts)
    ca, cb = a.counts(), b.counts()
    assert ca.keys() == cb.keys() and all(cb[t] == 2 * ca[t] for t in ca)
    # keys that are not packed keys of this context are rejected before any
    # of them reaches the table (EMPTY would alias free slots)
    before = b.counts()
    for badkey in (np.uint64(0xFFFFFFFFFFFFFFFF), np.uint64(1) << np.uint64(62)):
        bk = keys.copy()
        bk[d // 2] = badkey
        with pytest.raises(Exception, match="not packed keys"):
            b._ctx.check(b._ctx.lib.rg_ingest_counts(b._ctx.h, bk.ctypes.data, cnts.ctypes.data,
                                                     d, N.RG_MEM_HOST))
    assert b.counts() == before and b.total_ingested() == 2 * len(pts)
    # a too-small export buffer is an argument error, not a partial write
    with pytest.raises(Exception):
        ctx.check(ctx.lib.rg_export_entries(ctx.h, keys.ctypes.data, cnts.ctypes.data, d - 1,
                                            C.byref(got), N.RG_MEM_HOST))


def test_pipeline_reuse_single_rank(tmp_path):
    """DistributedPipeline at world 1 (gloo, one process) run twice on
    different inputs: rg_reset must leave nothing behind."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        pl = DistributedPipeline(D.params(1), device=0)
        for seed in (1, 2):
            s = D.spec(1, 0.2)
            s.seed += seed
            pts = D.generate(s)
            st = pl.run(torch.from_numpy(pts).cuda())
            ref = oracle(pts, D.params(1))
            assert (st.n_points, st.n_clusters) == (len(pts), ref.n_clusters)
            assert_same(pl.flat(), ref)
    finally:
        dist.destroy_process_group()


def _nccl_worker(rank, world, port, path, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda:0"))
    try:
        pts = np.load(path)
        gp = D.params(3)
        flat = cluster_distributed(torch.from_numpy(pts).cuda(), gp, device=0)
        np.savez(os.path.join(out_dir, "nccl.npz"), tx=flat.tx, ty=flat.ty,
                 count=flat.count.astype(np.uint64), cid=flat.cluster_id,
                 n=np.array([flat.n_clusters, flat.stats.n_points]),
                 backend=np.array([dist.get_backend() == "nccl"]))
    finally:
        dist.destroy_process_group()


def test_nccl_branch_single_rank(tmp_path):
    """The NCCL branch of the exchanges (device tensors on the wire:
    all_reduce of the column histogram, all_to_all_single of the [m, 2]
    pairs, the all_gathers of the border join) on a one-rank NCCL group -
    one GPU is all this box has; the two-rank runs above go over gloo."""
    pts = D.generate(D.spec(3, 0.05), shuffle_seed=6)
    path = tmp_path / "pts.npy"
    np.save(path, pts)
    mp.start_processes(_nccl_worker, args=(1, _free_port(), str(path), str(tmp_path)), nprocs=1,
                       join=True, start_method="spawn")
    ref = oracle(pts, D.params(3))
    o = np.load(tmp_path / "nccl.npz")
    assert bool(o["backend"][0])
    assert np.array_equal(o["tx"], ref.tx) and np.array_equal(o["ty"], ref.ty)
    assert np.array_equal(o["count"], ref.count.astype(np.uint64))
    assert np.array_equal(o["cid"], ref.cluster_id)
    assert o["n"].tolist() == [ref.n_clusters, len(pts)]


def _worker(rank, world, port, path, cfg, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pts = np.load(path)
        shard = pts[rank::world]
        gp = D.params(cfg)
        flat = cluster_distributed(torch.from_numpy(np.ascontiguousarray(shard)).cuda(), gp,
                                   device=0)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), tx=flat.tx, ty=flat.ty,
                 count=flat.count.astype(np.uint64), cid=flat.cluster_id,
                 n=np.array([flat.n_clusters, flat.stats.n_points]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [1, 3])
def test_two_ranks_gpu_engine_match_oracle(cfg, tmp_path):
    pts = D.generate(D.spec(cfg, 0.1), shuffle_seed=5)
    path = tmp_path / "pts.npy"
    np.save(path, pts)
    mp.start_processes(_worker, args=(2, _free_port(), str(path), cfg, str(tmp_path)), nprocs=2,
                       join=True, start_method="spawn")
    ref = oracle(pts, D.params(cfg))
    for r in range(2):
        o = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(o["tx"], ref.tx) and np.array_equal(o["ty"], ref.ty)
        assert np.array_equal(o["count"], ref.count.astype(np.uint64))
        assert np.array_equal(o["cid"], ref.cluster_id)
        assert o["n"].tolist() == [ref.n_clusters, len(pts)]


def test_route_pairs_matches_host_routing():
    """rg_route_pairs groups exported pairs by the owner of their column bin,
    exactly as the host formula the engine doubles use."""
    pts = D.generate(D.spec(3, 0.05), shuffle_seed=3)
    gp = D.params(3)
    eng = GpuEngine(gp, 0)
    eng.ingest(pts)
    keys, cnts = eng.export()
    col = eng.key_column(keys)
    cmin, width = int(col.min()), int(col.max() - col.min() + 1)
    splits = [700, 1500, 1501, 3000]
    ok, oc, pc = eng.route(keys, cnts, cmin, width, splits)
    bins = ((col - cmin) * 4096) // width
    owner = torch.searchsorted(torch.tensor(splits, device=keys.device), bins, right=True)
    assert pc == torch.bincount(owner, minlength=5).cpu().tolist()
    at = 0
    for p in range(5):
        want = keys[owner == p]
        got = ok[at: at + pc[p]]
        assert torch.equal(torch.sort(got).values, torch.sort(want).values)
        at += pc[p]
    ref = dict(zip(keys.cpu().tolist(), cnts.cpu().tolist()))
    assert all(ref[k] == c for k, c in zip(ok.cpu().tolist(), oc.cpu().tolist()))
