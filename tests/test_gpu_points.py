"""RASTER' cluster points on the device (rg_cluster_points): every in-bounds
point of a kept cluster, grouped by cluster id, point_less-sorted inside a
cluster (agglomerate.hpp:70-76,183; core.hpp:22-24). Checked against the
oracle's labels + a host sort, and against the reference's own
Mode::retain_points output (oracle/_ref) where it was built. Needs a B200."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1907_03620_b200 import datagen as D
from paper_1907_03620_b200.raster import GridParams, Mode, Pipeline, cluster_sequential

from .gpu_util import oracle

pytestmark = pytest.mark.gpu


def expected_points(pts, gp):
    ref = oracle(pts, gp)
    lab = O.port_labels(pts, gp, ref)
    sel = lab >= 0
    lab, xs, ys = lab[sel], pts[sel, 0], pts[sel, 1]
    order = np.lexsort((ys, xs, lab))
    off = np.searchsorted(lab[order], np.arange(ref.n_clusters + 1)).astype(np.uint64)
    return np.stack([xs[order], ys[order]], 1), off


def run_points(pts, gp, dev=False):
    pl = Pipeline(gp)
    if dev:
        import torch

        pts = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
    pl.run(pts)
    return pl.cluster_points(pts)


@pytest.mark.parametrize("dev", [False, True])
def test_points_small_random_with_duplicates(dev):
    rng = np.random.default_rng(17)
    gp = GridParams(precision=2.0, threshold=3, min_cluster_size=2)
    base = rng.normal(0, 0.05, size=(20000, 2))
    pts = np.concatenate([base, base[:5000], [[0.0, -0.0], [-0.0, 0.0], [np.nan, 0.0],
                                             [500.0, 1.0]]])
    rng.shuffle(pts)
    xy, off = run_points(pts, gp, dev)
    exy, eoff = expected_points(pts, gp)
    assert np.array_equal(off, eoff)
    assert np.array_equal(xy, exy)


def test_points_match_reference_prime_mode():
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    pts = D.generate(D.spec(1, 0.3), shuffle_seed=4)
    gp = D.params(1)
    gp.mode = Mode.retain_points
    cs = cluster_sequential(pts, gp)
    cid, px, py = O.ref_prime_points(pts, gp)
    got_cid = np.concatenate([np.full(len(c.points), c.id) for c in cs.clusters])
    got = np.array([p for c in cs.clusters for p in c.points])
    assert np.array_equal(got_cid, cid)
    assert np.array_equal(got[:, 0], px) and np.array_equal(got[:, 1], py)


def test_points_config2_exact():
    pts = D.generate(D.spec(2), shuffle_seed=9)
    gp = D.params(2)
    xy, off = run_points(pts, gp, dev=True)
    exy, eoff = expected_points(pts, gp)
    assert np.array_equal(off, eoff)
    assert np.array_equal(xy, exy)


def test_points_config3_properties():
    """100M points: M = sum of kept tile counts, per-cluster sizes, and
    point_less order inside every cluster."""
    import torch

    pts = torch.from_numpy(D.generate(D.spec(3))).cuda()
    gp = D.params(3)
    pl = Pipeline(gp)
    pl.run(pts)
    flat = pl.flat()
    xy, off = pl.cluster_points(pts, device_out=True)
    kept = flat.cluster_id >= 0
    sizes = np.bincount(flat.cluster_id[kept], weights=flat.count[kept].astype(np.float64),
                        minlength=flat.n_clusters).astype(np.int64)
    off_h = off.cpu().numpy()
    assert off_h[0] == 0 and off_h[-1] == xy.shape[0] == int(flat.count[kept].sum())
    assert np.array_equal(np.diff(off_h), sizes)
    x, y = xy[:, 0], xy[:, 1]
    le = (x[:-1] < x[1:]) | ((x[:-1] == x[1:]) & (y[:-1] <= y[1:]))
    boundary = torch.zeros(xy.shape[0] - 1, dtype=torch.bool, device="cuda")
    inner = torch.from_numpy(off_h[1:-1] - 1).cuda()
    boundary[inner[(inner >= 0) & (inner < boundary.numel())]] = True
    assert bool(torch.all(le | boundary))


def test_points_of_an_unordered_device_input():
    """10M points of config 4 in a random order on the device: the
    partitioned contraction with K2 on its pairs, then the point lists
    (labels through the cell table) against the oracle + host sort."""
    gp = D.params(4)
    pts = D.generate(D.spec(4, 0.02), shuffle_seed=21)
    xy, off = run_points(pts, gp, dev=True)
    exy, eoff = expected_points(pts, gp)
    assert np.array_equal(off, eoff)
    assert np.array_equal(xy, exy)


def test_points_no_clusters_and_empty():
    gp = GridParams(precision=2.0, threshold=100, min_cluster_size=1)
    xy, off = run_points(np.random.default_rng(1).normal(0, 1, size=(1000, 2)), gp)
    assert xy.shape == (0, 2) and off.tolist() == [0]
    pl = Pipeline(GridParams(precision=2.0, threshold=1, min_cluster_size=1))
    pts = np.array([[0.5, 0.5], [0.5, 0.5], [0.51, 0.5]])
    pl.run(pts)
    xy, off = pl.cluster_points(np.zeros((0, 2)))
    assert xy.shape == (0, 2) and off.tolist() == [0, 0]
    xy, off = pl.cluster_points(pts)
    assert xy.tolist() == [[0.5, 0.5], [0.5, 0.5], [0.51, 0.5]] and off.tolist() == [0, 3]


@pytest.mark.parametrize("dedupe", [False, True])
def test_points_many_small_clusters_shared_memory_sort(dedupe):
    """Clusters of a few hundred points (the per-cluster shared-memory sort,
    not the radix fallback), with exact duplicates and signed zeros."""
    rng = np.random.default_rng(23)
    gp = GridParams(precision=2.0, threshold=3, min_cluster_size=2)
    c = rng.uniform([-150, -70], [150, 70], size=(3000, 2))
    pts = c[rng.integers(0, 3000, 600_000)] + rng.normal(0, 0.004, size=(600_000, 2))
    pts = np.concatenate([pts, pts[:50_000], [[0.0, -0.0], [-0.0, 0.0], [0.005, 0.005]] * 4])
    rng.shuffle(pts)
    gp.dedupe_points = dedupe
    gp.mode = Mode.retain_points if dedupe else Mode.count_only
    import torch

    pl = Pipeline(gp)
    dev = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
    pl.run(dev)
    xy, off = pl.cluster_points(dev)
    if dedupe:  # the reference's own Mode::retain_points + dedupe_points output
        if O.ref() is None:
            pytest.skip("oracle/_ref not built")
        cid, px, py = O.ref_prime_points(pts, gp, dedupe=True)
        assert np.array_equal(xy[:, 0], px) and np.array_equal(xy[:, 1], py)
        assert np.array_equal(np.repeat(np.arange(len(off) - 1), np.diff(off).astype(np.int64)),
                              cid)
        assert len(off) - 1 > 2000  # many clusters: the shared-memory sort
    else:
        exy, eoff = expected_points(pts, gp)
        assert np.array_equal(off, eoff)
        assert np.array_equal(xy, exy)


def test_points_unaligned_device_buffer():
    """An 8-byte aligned point buffer takes the radix path (16-byte loads
    elsewhere) with the same output."""
    import torch

    rng = np.random.default_rng(5)
    gp = GridParams(precision=2.0, threshold=3, min_cluster_size=2)
    c = rng.uniform([-150, -70], [150, 70], size=(500, 2))
    pts = c[rng.integers(0, 500, 100_000)] + rng.normal(0, 0.004, size=(100_000, 2))
    buf = torch.zeros(pts.size + 1, dtype=torch.float64, device="cuda")
    buf[1:] = torch.from_numpy(pts.reshape(-1)).cuda()
    view = buf[1:].view(-1, 2)
    pl = Pipeline(gp)
    pl.run(view)
    xy, off = pl.cluster_points(view)
    exy, eoff = expected_points(pts, gp)
    assert np.array_equal(off, eoff) and np.array_equal(xy, exy)
