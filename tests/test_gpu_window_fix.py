"""window_fix (agglomerate.hpp:212-246) and cluster_sequential with
use_window_fix (pipeline.hpp:103) on the device, against the reference's
known answers and the oracle. Needs a B200."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1907_03620_b200 import datagen as D
from paper_1907_03620_b200.raster import GridParams, Pipeline, TileAccumulator, cluster_flat, window_fix

from .gpu_util import assert_same
from .test_oracle import centre_points

pytestmark = pytest.mark.gpu


def test_window_fix_kats(kat):
    for c in kat["window_fix"]:
        gp = GridParams(precision=c["precision"], threshold=c["threshold"], min_cluster_size=1)
        pts = centre_points(c["tile_copies"], c["precision"])
        acc = TileAccumulator(gp)
        acc.ingest(pts)
        kept = window_fix(acc, gp)
        assert [[int(x), int(y)] for x, y in zip(kept.tx, kept.ty)] == c["window_kept"], c["cite"]
        # the accumulator is untouched: plain pruning still sees every tile
        assert acc.entry_count() == len(c["tile_copies"])
        plain = acc.prune()
        assert [[int(x), int(y)] for x, y in zip(plain.tx, plain.ty)] == c["plain_kept"], c["cite"]


@pytest.mark.parametrize("seed", range(8))
def test_window_fix_random_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    gp = GridParams(precision=float(rng.choice([1.0, 2.0, 3.0])), threshold=int(rng.integers(2, 9)),
                    distance=int(rng.integers(1, 3)), min_cluster_size=int(rng.integers(1, 5)))
    n = int(rng.integers(1000, 200000))
    pts = rng.normal(0, 0.05, size=(n, 2)) * (10 ** (3 - gp.precision))
    pts[rng.random(n) < 0.01] = np.nan
    assert_same(cluster_flat(pts, gp, use_window_fix=True), O.port_cluster(pts, gp, window_fix=True),
                f"seed {seed}")


def test_window_fix_canvas_corners():
    """Windows at the canvas edge reach past the last column/row."""
    gp = GridParams(precision=2.0, threshold=3, min_cluster_size=1)
    pts = np.array([[180.0, 90.0], [179.995, 90.0], [180.0, 89.995], [-180.0, -90.0],
                    [-179.995, -90.0], [-180.0, -89.995], [0.0, 90.0], [0.01, 90.0]])
    assert_same(cluster_flat(pts, gp, use_window_fix=True), O.port_cluster(pts, gp, window_fix=True))


@pytest.mark.parametrize("cfg", [1, 2])
def test_window_fix_configs_vs_oracle(cfg):
    pts = D.generate(D.spec(cfg))
    gp = D.params(cfg)
    assert_same(cluster_flat(pts, gp, use_window_fix=True), O.port_cluster(pts, gp, window_fix=True),
                f"config {cfg}")


def test_window_fix_superset_at_scale():
    """Config 3 (100M points): the window-fixed set contains every plainly
    significant tile with its count (test_agglomerate.cpp:255-277)."""
    import torch

    pts = torch.from_numpy(D.generate(D.spec(3))).cuda()
    gp = D.params(3)
    plain = Pipeline(gp)
    plain.run(pts)
    a = plain.flat()
    fixed = Pipeline(gp)
    fixed.run(pts, use_window_fix=True)
    b = fixed.flat()
    assert b.tx.size >= a.tx.size
    ka = a.tx * (1 << 32) + a.ty
    kb = b.tx * (1 << 32) + b.ty
    pos = np.searchsorted(kb, ka)
    assert np.array_equal(kb[pos], ka)
    assert np.array_equal(b.count[pos], a.count)
