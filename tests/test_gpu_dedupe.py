"""dedupe_points in the point-retaining mode (accumulator.hpp:160-174,
199-204) on the device: thresholds, reported counts and cluster points on
unique coordinates; raw counts for count_of and window_fix decisions.
Needs a B200."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1907_03620_b200 import datagen as D
from paper_1907_03620_b200.raster import (GridParams, Mode, Pipeline, Tile, TileAccumulator,
                                          cluster_flat, window_fix)

from .gpu_util import assert_same

pytestmark = pytest.mark.gpu


def dd_params(**kw) -> GridParams:
    gp = GridParams(**kw)
    gp.mode = Mode.retain_points
    gp.dedupe_points = True
    return gp


def test_dedupe_kat(kat):
    for c in kat["dedupe"]:
        gp = GridParams(precision=c["precision"], threshold=c["threshold"], min_cluster_size=1)
        gp.mode = Mode.retain_points
        gp.dedupe_points = c["dedupe"]
        acc = TileAccumulator(gp)
        acc.ingest(np.array(c["points"]))
        assert acc.count_of(Tile(*c["tile"])) == 3  # raw count before prune
        sig = acc.prune()
        assert sig.tx.tolist() == [c["tile"][0]] and sig.count.tolist() == [c["count"]], c["cite"]


@pytest.mark.parametrize("wf", [False, True])
def test_dedupe_random_chunks_vs_oracle(wf):
    rng = np.random.default_rng(21)
    for trial in range(5):
        gp = dd_params(precision=2.0, threshold=int(rng.integers(2, 6)),
                       min_cluster_size=int(rng.integers(1, 4)))
        base = np.round(rng.normal(0, 0.05, size=(20000, 2)), 3)
        pts = base[rng.integers(0, len(base), 60000)]
        pts[:100] *= -0.0
        ref = O.port_cluster(pts, gp, window_fix=wf, dedupe=True)
        pl = Pipeline(gp)
        pl.run(pts, use_window_fix=wf)
        assert_same(pl.flat(), ref, f"trial {trial}")
        # chunked ingest + merge of two accumulators
        a, b = TileAccumulator(gp), TileAccumulator(gp)
        cuts = np.sort(rng.integers(0, len(pts), 6))
        for k, chunk in enumerate(np.split(pts, cuts)):
            (a if k % 2 else b).ingest(chunk)
        a.merge(b)
        sig = window_fix(a, gp) if wf else a.prune()
        assert np.array_equal(sig.tx, ref.tx) and np.array_equal(sig.count, ref.count)


def test_dedupe_cluster_points_vs_reference():
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    gp = dd_params(precision=2.0, threshold=3, min_cluster_size=2)
    base = np.round(rng.normal(0, 0.05, size=(5000, 2)), 3)
    pts = base[rng.integers(0, len(base), 20000)]
    pl = Pipeline(gp)
    pl.run(pts)
    xy, off = pl.cluster_points(pts)
    cid, px, py = O.ref_prime_points(pts, gp, dedupe=True)
    assert np.array_equal(xy[:, 0], px) and np.array_equal(xy[:, 1], py)
    assert np.array_equal(np.repeat(np.arange(len(off) - 1), np.diff(off).astype(np.int64)), cid)


def test_dedupe_doubled_config_equals_plain():
    """Config 3 (100M distinct points) ingested twice with dedupe clusters
    exactly like a single copy without it (200M points through the set)."""
    import torch

    pts = torch.from_numpy(D.generate(D.spec(3))).cuda()
    gp = D.params(3)
    plain = cluster_flat(pts, gp)
    gd = D.params(3)
    gd.mode = Mode.retain_points
    gd.dedupe_points = True
    acc = TileAccumulator(gd)
    acc.ingest(pts)
    acc.ingest(pts.flip(0).contiguous())
    assert acc.total_ingested() == 2 * plain.stats.n_points - 2 * plain.stats.n_skipped
    sig = acc.prune()
    assert np.array_equal(sig.tx, plain.tx) and np.array_equal(sig.count, plain.count)
