"""GPU edge cases the reference tests or the domain has: empty and ragged
inputs, out-of-bounds/NaN points, closed canvas edges, strict policy,
unaligned buffers, table growth, chunk and permutation invariance, merge,
random tile sets against the union-find oracle. Needs a B200."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1907_03620_b200 import datagen as D
from paper_1907_03620_b200.raster import (Bounds, GridParams, Metric, OobPolicy,
                                          OutOfBoundsError, Pipeline, Tile, TileAccumulator,
                                          agglomerate_flat, cluster_flat)

from .gpu_util import assert_same, numpy_tile_counts, oracle

pytestmark = pytest.mark.gpu


def torch_mod():
    import torch

    assert torch.cuda.is_available()
    return torch


def test_empty_input():
    gp = GridParams()
    flat = cluster_flat(np.zeros((0, 2)), gp)
    assert flat.tx.size == 0 and flat.n_clusters == 0
    acc = TileAccumulator(gp)
    acc.ingest(np.array([[1.0, 1.0]]))
    before = acc.counts()
    acc.ingest(np.zeros((0, 2)))  # test_accumulator.cpp:47-54
    assert acc.counts() == before and acc.total_ingested() == 1


def test_all_out_of_bounds_and_nan():
    pts = np.array([[500.0, 0.0], [0.0, -91.0], [np.nan, 0.0], [0.0, np.nan], [np.inf, 1.0],
                    [-np.inf, -1.0], [180.0000001, 0.0]])
    pl = Pipeline(GridParams())
    st = pl.run(pts)
    assert (st.n_ingested, st.n_skipped, st.n_clusters) == (0, len(pts), 0)
    assert np.all(pl.label_points(pts) == -1)


def test_closed_canvas_corners_and_edges():
    gp = GridParams(precision=3.0, threshold=1, min_cluster_size=1)
    corners = np.array([[180.0, 90.0], [-180.0, -90.0], [180.0, -90.0], [-180.0, 90.0],
                        [0.0, 90.0], [180.0, 0.0]])
    pts = np.repeat(corners, 3, axis=0)
    flat = cluster_flat(pts, gp)
    assert_same(flat, oracle(pts, gp))
    assert flat.stats.n_skipped == 0


def test_random_mixed_vs_oracle_many_params():
    rng = np.random.default_rng(2024)
    for trial in range(12):
        gp = GridParams(precision=float(rng.choice([0.5, 1.0, 2.0, 2.5, 3.0, 3.5])),
                        threshold=int(rng.integers(1, 8)), distance=int(rng.integers(1, 4)),
                        metric=Metric(int(rng.integers(0, 2))),
                        min_cluster_size=int(rng.integers(1, 6)),
                        bounds=Bounds(-3.0, 4.0, -2.0, 2.5))
        n = int(rng.integers(1, 60000))
        pts = rng.normal(0.3, 1.2, size=(n, 2))
        pts[rng.random(n) < 0.01] = np.nan
        snap = rng.random(n) < 0.3  # grid-line points
        s = 10.0 ** gp.precision
        pts[snap] = np.round(pts[snap] * s) / s
        assert_same(cluster_flat(pts, gp), oracle(pts, gp), f"trial {trial}")


def test_strict_policy_reports_first_oob_and_keeps_prefix():
    gp = GridParams(precision=2, oob_policy=OobPolicy.strict)
    pts = np.array([[0.5, 0.5], [0.51, 0.5], [500.0, 0.0], [0.6, 0.6], [900.0, 1.0]])
    acc = TileAccumulator(gp)
    with pytest.raises(OutOfBoundsError) as e:
        acc.ingest(pts)
    assert str(e.value) == "point (500.000000, 0.000000) outside canvas bounds"
    assert acc.total_ingested() == 2  # the reference's loop threw at index 2
    if O.ref() is not None:
        thrown, msg, ing = O.ref_strict(pts, gp)
        assert thrown and msg == str(e.value) and ing == acc.total_ingested()


def test_strict_policy_device_buffer():
    torch = torch_mod()
    gp = GridParams(precision=2, oob_policy=OobPolicy.strict)
    pts = torch.tensor([[0.5, 0.5], [1.0, 1.0], [0.0, -95.5]], dtype=torch.float64, device="cuda")
    acc = TileAccumulator(gp)
    with pytest.raises(OutOfBoundsError, match=r"point \(0.000000, -95.500000\)"):
        acc.ingest(pts)
    assert acc.total_ingested() == 2


def test_unaligned_device_pointer():
    torch = torch_mod()
    pts = D.generate(D.spec(1, 0.05))
    gp = D.params(1)
    buf = torch.zeros(pts.size + 1, dtype=torch.float64, device="cuda")
    buf[1:] = torch.from_numpy(pts.reshape(-1)).cuda()
    view = buf[1:].view(-1, 2)  # 8-byte aligned only
    assert view.data_ptr() % 16 == 8
    pl = Pipeline(gp)
    pl.run(view)
    assert_same(pl.flat(), oracle(pts, gp))
    labels = pl.label_points(view).cpu().numpy()
    assert np.array_equal(labels, O.port_labels(pts, gp, oracle(pts, gp)))


@pytest.mark.parametrize("hint", [1, 1000])
def test_tiny_table_grows_exactly(hint):
    s = D.spec(2, 0.3)
    s.n_noise = 4_000_000  # ~4M distinct tiles at p=3: far above the initial table
    pts = D.generate(s, shuffle_seed=1)
    gp = D.params(3)
    gp.threshold = 1
    gp.capacity_hint = hint
    pl = Pipeline(gp)
    st = pl.run(pts)
    ref = oracle(pts, gp)
    assert_same(pl.flat(), ref)
    assert st.peak_accumulator_entries == ref.n_distinct
    assert st.table_grows >= 1


def test_chunk_partition_and_order_invariance():
    """acceptance.cpp:227-258 (criterion 6): random cuts, chunks in random order."""
    pts = D.generate(D.spec(1, 0.1))
    gp = D.params(1)
    ref = oracle(pts, gp)
    rng = np.random.default_rng(0xC4AA)
    n = len(pts)
    for rnd in range(10):
        cuts = sorted({0, n, *rng.integers(0, n, 1 + int(rng.integers(0, 40))).tolist()})
        chunks = [pts[a:b] for a, b in zip(cuts[:-1], cuts[1:])]
        rng.shuffle(chunks)
        acc = TileAccumulator(gp)
        for c in chunks:
            acc.ingest(c)
        sig = acc.prune()
        assert np.array_equal(sig.tx, ref.tx) and np.array_equal(sig.count, ref.count), rnd
        flat = agglomerate_flat(sig, gp)
        assert np.array_equal(flat.cluster_id, ref.cluster_id), rnd


def test_permutation_invariance_and_counts():
    rng = np.random.default_rng(9)
    pts = np.stack([rng.uniform(-10, 10, 5000), rng.uniform(-5, 5, 5000)], 1)
    gp = GridParams(precision=2)
    a = TileAccumulator(gp)
    a.ingest(pts)
    b = TileAccumulator(gp)
    b.ingest(pts[rng.permutation(len(pts))])
    ca = a.counts()
    assert ca == b.counts()
    assert sum(ca.values()) == a.total_ingested() == len(pts)
    assert {(t.x, t.y): c for t, c in ca.items()} == numpy_tile_counts(pts, gp)


def test_entry_bound():
    """test_accumulator.cpp:101-115: entries never exceed the tile bound."""
    gp = GridParams(precision=1.0, bounds=Bounds(0.0, 1.0, 0.0, 1.0))
    rng = np.random.default_rng(5)
    acc = TileAccumulator(gp)
    acc.ingest(rng.uniform(0, 1, size=(20000, 2)))
    assert acc.entry_count() <= gp.tile_bound()


def test_merge_adds_counts_large():
    pts = D.generate(D.spec(2, 0.2))
    gp = D.params(2)
    half = len(pts) // 2
    a, b = TileAccumulator(gp), TileAccumulator(gp)
    a.ingest(pts[:half])
    b.ingest(pts[half:])
    a.merge(b)
    sig = a.prune()
    ref = oracle(pts, gp)
    assert np.array_equal(sig.tx, ref.tx) and np.array_equal(sig.count, ref.count)


def test_random_tile_sets_vs_union_find():
    """acceptance.cpp:97-121 (criterion 2) at GPU scale: random tile sets,
    both metrics, delta 1 and 2."""
    rng = np.random.default_rng(0x02AC1E)
    for rnd in range(60):
        gp = GridParams(metric=Metric(rnd % 2), distance=1 + (rnd // 2) % 2, min_cluster_size=1)
        n = 100 + int(rng.integers(0, 4901))
        ext = int(np.sqrt(n * 2.0))
        t = np.unique(rng.integers(-ext, ext + 1, size=(n * 2, 2)), axis=0)[:n]
        rng.shuffle(t)
        flat = agglomerate_flat({Tile(int(x), int(y)): 5 for x, y in t}, gp)
        ref = O.port_agglomerate(t[:, 0], t[:, 1], np.full(len(t), 5, np.uint64), gp)
        assert np.array_equal(flat.cluster_id, ref.cluster_id), rnd


def test_tiles_off_canvas_agglomerate():
    gp = GridParams(precision=2, min_cluster_size=1)
    tiles = {Tile(10**12, 5): 5, Tile(10**12 + 1, 6): 5, Tile(-(10**12), 0): 5}
    flat = agglomerate_flat(tiles, gp)
    assert flat.n_clusters == 2
    assert flat.cluster_id.tolist() == [0, 1, 1]


def test_long_chain_component():
    """A single 200,000-tile snake: union-find must not depend on diameter."""
    gp = GridParams(precision=3, threshold=1, min_cluster_size=4)
    k = np.arange(200_000)
    tx = (k // 1000) * 2
    ty = np.where((k // 1000) % 2 == 0, k % 1000, 999 - k % 1000)
    # connect column pairs with a bridge tile
    bridges_x = tx[999::1000][:-1] + 1
    bridges_y = ty[999::1000][:-1]
    allx = np.concatenate([tx, bridges_x])
    ally = np.concatenate([ty, bridges_y])
    flat = agglomerate_flat({Tile(int(x), int(y)): 1 for x, y in zip(allx, ally)}, gp)
    assert flat.n_clusters == 1 and np.all(flat.cluster_id == 0)


def test_hot_spot_single_tile():
    """All points in one tile: counts beyond 2^32 are not reachable in a test,
    but a 50M-point single-tile hot spot exercises the aggregation path."""
    torch = torch_mod()
    n = 50_000_000
    pts = torch.full((n, 2), 0.123456, dtype=torch.float64, device="cuda")
    gp = GridParams(precision=3, threshold=3)
    pl = Pipeline(gp)
    st = pl.run(pts)
    flat = pl.flat()
    assert flat.tx.tolist() == [123] and flat.count.tolist() == [n]
    assert st.n_clusters == 0  # one tile < mu


def test_lattice_same_block_position():
    """Every tile at the same position inside its 4x4 (and 8x8) table block:
    a probe scheme that stayed at the home position would overflow."""
    gp = GridParams(precision=3.0, threshold=1, min_cluster_size=1)
    i, j = np.meshgrid(np.arange(400), np.arange(400), indexing="ij")
    tx, ty = (8 * i).ravel(), (8 * j).ravel()
    pts = np.stack([(tx + 0.5) / 1000.0, (ty + 0.5) / 1000.0], 1)
    gp.capacity_hint = 1
    flat = cluster_flat(pts, gp)
    assert_same(flat, oracle(pts, gp))
    assert flat.n_clusters == 160_000


@pytest.mark.parametrize("metric,delta", [(Metric.chebyshev, 1), (Metric.manhattan, 1),
                                          (Metric.chebyshev, 2), (Metric.manhattan, 2),
                                          (Metric.chebyshev, 3)])
def test_adjacency_per_offset(metric, delta):
    """neighbor_offsets agglomerate.hpp:38-50 as the device sees it: two tiles
    form one cluster exactly when their offset is in the neighbourhood
    (test_agglomerate.cpp:30-62)."""
    gp = GridParams(metric=metric, distance=delta, min_cluster_size=1)
    for dx in range(-4, 5):
        for dy in range(-4, 5):
            if dx == 0 and dy == 0:
                continue
            flat = agglomerate_flat({Tile(100, 100): 5, Tile(100 + dx, 100 + dy): 5}, gp)
            near = (max(abs(dx), abs(dy)) if metric == Metric.chebyshev else abs(dx) + abs(dy)) <= delta
            assert flat.n_clusters == (1 if near else 2), (metric, delta, dx, dy)


def test_threshold_one_keeps_every_occupied_tile():
    """test_accumulator.cpp:135-143"""
    rng = np.random.default_rng(11)
    gp = GridParams(precision=2, threshold=1)
    acc = TileAccumulator(gp)
    acc.ingest(rng.uniform(-10, 10, size=(300, 2)))
    occupied = acc.entry_count()
    assert len(acc.prune()) == occupied


def test_dense_cluster_yields_a_significant_tile():
    """test_accumulator.cpp:145-165 (500 points in a square of half-side
    ~2.5 tile sides at p=3.5, tau=5)."""
    rng = np.random.default_rng(2024)
    r = 2.5e-3 / 3.1622776601683795
    pts = 1.0 + rng.uniform(-r, r, size=(500, 2))
    gp = GridParams(precision=3.5, threshold=5)
    assert max(numpy_tile_counts(pts, gp).values()) >= 5
    acc = TileAccumulator(gp)
    acc.ingest(pts)
    assert len(acc.prune()) >= 1


@pytest.mark.parametrize("k3", ["bucket", "seg", "radix"])
def test_top_row_key_wrap_is_not_adjacency(monkeypatch, k3):
    """With a row range of exactly 2^bits_y rows, the packed key of (x, top
    row) + 1 is the key of (x+1, bottom row): consecutive in sorted order but
    not adjacent (agglomerate.hpp:38-50 offsets are geometric). Off-canvas
    tile sets get a key packing sized to their own extent, so 4 rows -> 2
    row bits; every sort path of the sorted K3 must keep them apart."""
    import os
    import subprocess
    import sys

    code = (
        "from paper_1907_03620_b200.raster import GridParams, Tile, agglomerate_flat\n"
        "gp = GridParams(precision=2, min_cluster_size=1)\n"
        "b = 10**12\n"
        "t = {Tile(b, 0): 5, Tile(b, 3): 5, Tile(b + 1, 0): 5, Tile(b + 2, 3): 5, Tile(b + 3, 0): 5}\n"
        "f = agglomerate_flat(t, gp)\n"
        "print(f.n_clusters, f.cluster_id.tolist())\n")
    env = dict(os.environ, RG_K3_SORT=k3[0])
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         check=True).stdout.split("\n")[0]
    # (b,0)-(b+1,0) adjacent; (b,3) alone; (b+2,3) alone; (b+3,0) alone
    assert out == "4 [0, 1, 0, 2, 3]", out


def test_stream_ordering_with_torch_default_stream():
    """Points produced by a torch kernel on the default stream and clustered
    right away (no synchronize) on that stream: set_stream(0) must order
    the work after it (0 is torch's legacy default stream, passed as
    cudaStreamLegacy), so the result equals that of settled data."""
    torch = torch_mod()
    pts = D.generate(D.spec(3, 0.3), shuffle_seed=2)  # 30M points, 480 MB
    src = torch.from_numpy(pts).cuda()
    torch.cuda.synchronize()
    gp = D.params(3)
    ref = Pipeline(gp)
    ref.run(src)
    want = ref.flat()
    pl = Pipeline(gp)
    pl.set_stream(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        dst = torch.empty_like(src)
        dst.copy_(src.flip(0))  # still running when the next call is enqueued
        pl.run(dst)
        assert_same(pl.flat(), want)


@pytest.mark.parametrize("chunk", [65536, 1 << 20])
def test_streaming_ingest_matches_single_span(chunk):
    """rg_stream_* (a PointSource drained chunk by chunk with the next read
    overlapping the previous chunk's copy and K1, io.hpp:226-241): counts,
    counters and table identical to one rg_ingest of the whole span, for
    ordered and shuffled sources; strict policy stops at the first
    out-of-bounds point."""
    import numpy as np

    from paper_1907_03620_b200 import datagen as D
    from paper_1907_03620_b200.raster import TileAccumulator

    gp = D.params(3)
    for shuffle in (None, 3):
        pts = D.generate(D.spec(3, 0.05), shuffle_seed=shuffle)
        pts[::7919] = [1000.0, 0.0]
        one = TileAccumulator(gp)
        one.ingest(pts)
        st = TileAccumulator(gp)
        pos = [0]

        def read(out):
            k = min(len(out), len(pts) - pos[0])
            out[:k] = pts[pos[0]:pos[0] + k]
            pos[0] += k
            return k

        assert st.ingest_source(read, chunk) == len(pts)
        assert st.counts() == one.counts()
        assert (st.total_ingested(), st.skipped()) == (one.total_ingested(), one.skipped())
