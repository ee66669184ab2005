"""Pins the CPU oracle (oracle/raster_oracle.c) before it is trusted: against
the reference's own known-answer tests, against fixtures produced by the
reference itself (tests/golden/make_golden.py), and — when oracle/_ref was
built from /root/reference — against the live reference. CPU only."""
from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1907_03620_b200 import datagen as D
from paper_1907_03620_b200.raster import Bounds, GridParams, Metric


def centre_points(tile_copies, precision):
    """oracle::add_tile_points tests/support/oracles.hpp:128-134."""
    side = 10.0 ** -precision
    pts = []
    for (tx, ty), copies in tile_copies:
        pts += [((tx + 0.5) * side, (ty + 0.5) * side)] * copies
    return np.array(pts, np.float64).reshape(-1, 2)


def test_projection_kats(kat):
    for case in kat["projection"]:
        s = math.pow(10.0, case["precision"])
        for (x, y), want in zip(case["points"], case["tiles"]):
            assert O.port_project(x, y, s) == tuple(want), case["cite"]


def test_same_tile_kat(kat):
    c = kat["same_tile"]
    s = 10.0 ** c["precision"]
    a, b = c["same"]
    assert O.port_project(*a, s) == O.port_project(*b, s)
    a, b = c["different"]
    assert O.port_project(*a, s) != O.port_project(*b, s)


def test_scale_kat(kat):
    assert math.pow(10.0, kat["scale"]["precision"]) == kat["scale"]["value"]


def test_three_point_and_prune_kats(kat):
    c = kat["three_point"]
    gp = GridParams(precision=c["precision"], threshold=1, min_cluster_size=1)
    r = O.port_cluster(np.array(c["points"]), gp)
    assert r.n_distinct == c["entries"]
    assert (int(r.tx[0]), int(r.ty[0]), int(r.count[0])) == (*c["tile"], c["count"])

    c = kat["prune"]
    gp = GridParams(precision=c["precision"], threshold=c["threshold"], min_cluster_size=1)
    r = O.port_cluster(centre_points(c["tile_copies"], c["precision"]), gp)
    got = [((int(x), int(y)), int(n)) for x, y, n in zip(r.tx, r.ty, r.count)]
    assert got == [(tuple(t), n) for t, n in c["kept"]]


def test_oob_skip_kat(kat):
    c = kat["oob_skip"]
    r = O.port_cluster(np.array(c["points"]), GridParams(precision=c["precision"]))
    assert (r.n_ingested, r.n_skipped) == (c["ingested"], c["skipped"])


@pytest.mark.parametrize("name", ["group_and_drop", "ids_by_smallest", "singleton", "cluster_csv"])
def test_agglomerate_kats(kat, name):
    c = kat[name]
    t = np.array(c["tiles"], np.int64)
    gp = GridParams(min_cluster_size=c["min_cluster_size"])
    r = O.port_agglomerate(t[:, 0], t[:, 1], np.full(len(t), 5, np.uint64), gp)
    clusters = {}
    for x, y, k in zip(r.tx.tolist(), r.ty.tolist(), r.cluster_id.tolist()):
        if k >= 0:
            clusters.setdefault(k, []).append([x, y])
    if "clusters" in c:
        assert [clusters[k] for k in sorted(clusters)] == c["clusters"], c["cite"]
    if "csv" in c:
        csv = "".join(f"{k},{x},{y}\n" for k in sorted(clusters) for x, y in clusters[k])
        assert csv == c["csv"], c["cite"]


def test_prime_accounting_kat(kat):
    c = kat["prime_accounting"]
    pts = centre_points(c["tile_copies"], c["precision"])
    gp = GridParams(precision=c["precision"], threshold=c["threshold"],
                    min_cluster_size=c["min_cluster_size"])
    r = O.port_cluster(pts, gp)
    labels = O.port_labels(pts, gp, r)
    assert int((labels >= 0).sum()) == c["clustered_points"]


def test_port_matches_reference_fixtures(golden):
    z, meta = golden
    for tag, m in meta["configs"].items():
        cfg = int(tag[3])
        s = D.spec(cfg, 1.0)
        for k, v in m["spec"].items():
            setattr(s, k, v)
        pts = D.generate(s)
        if m["shuffle_seed"] is not None:
            pts = D.shuffle(pts, m["shuffle_seed"])
        assert hashlib.sha256(pts.tobytes()).hexdigest() == m["input_sha256"], tag
        gp = D.params(cfg)
        r = O.port_cluster(pts, gp)
        assert np.array_equal(r.tx, z[f"{tag}_tx"]), tag
        assert np.array_equal(r.ty, z[f"{tag}_ty"]), tag
        assert np.array_equal(r.count, z[f"{tag}_count"]), tag
        assert np.array_equal(r.cluster_id, z[f"{tag}_cid"]), tag
        assert (r.n_ingested, r.n_skipped, r.n_distinct, r.n_clusters) == (
            m["n_ingested"], m["n_skipped"], m["n_distinct"], m["n_clusters"]), tag
        assert np.array_equal(O.port_labels(pts, gp, r), z[f"{tag}_labels"]), tag


def test_port_matches_reference_tile_sets(golden):
    z, meta = golden
    for i, m in enumerate(meta["tiles"]):
        t = z[f"tiles{i}_in"]
        gp = GridParams(distance=m["distance"], metric=Metric(m["metric"]),
                        min_cluster_size=m["min_cluster_size"])
        r = O.port_agglomerate(t[:, 0], t[:, 1], np.full(len(t), 5, np.uint64), gp)
        assert np.array_equal(r.cluster_id, z[f"tiles{i}_cid"]), i
        assert r.n_clusters == m["n_clusters"]


def test_port_gridline_projection(golden):
    z, _ = golden
    for (p, x, y), want in zip(z["gridline_in"], z["gridline_tiles"]):
        assert O.port_project(x, y, math.pow(10.0, p)) == tuple(want)


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref (reference build) not present")
def test_port_matches_live_reference_random():
    rng = np.random.default_rng(99)
    for trial in range(6):
        gp = GridParams(precision=float(rng.choice([1.0, 2.0, 2.5, 3.0])),
                        threshold=int(rng.integers(1, 6)), distance=int(rng.integers(1, 3)),
                        metric=Metric(int(rng.integers(0, 2))),
                        min_cluster_size=int(rng.integers(1, 5)),
                        bounds=Bounds(-5.0, 5.0, -3.0, 3.0))
        n = 20000
        pts = rng.normal(0, 1.5, size=(n, 2))
        pts[::97] = [5.0, 3.0]  # closed upper corner
        pts[::101, 0] = np.nan
        a = O.port_cluster(pts, gp)
        b, _, _ = O.ref_cluster(pts, gp)
        for k in ("tx", "ty", "count", "cluster_id"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), (trial, k)
        assert (a.n_ingested, a.n_skipped, a.n_distinct) == (b.n_ingested, b.n_skipped, b.n_distinct)


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref (reference build) not present")
def test_reference_strict_message_format():
    thrown, msg, ing = O.ref_strict(np.array([[0.5, 0.5], [500.0, 0.0], [0.6, 0.6]]),
                                    GridParams(precision=2))
    assert thrown and msg == "point (500.000000, 0.000000) outside canvas bounds" and ing == 1


def test_window_fix_kats(kat):
    """window_fix agglomerate.hpp:212-246 KATs, on the port and (when built)
    the reference itself."""
    for c in kat["window_fix"]:
        gp = GridParams(precision=c["precision"], threshold=c["threshold"], min_cluster_size=1)
        pts = centre_points(c["tile_copies"], c["precision"])
        plain = O.port_cluster(pts, gp)
        fixed = O.port_cluster(pts, gp, window_fix=True)
        assert [[int(x), int(y)] for x, y in zip(plain.tx, plain.ty)] == c["plain_kept"], c["cite"]
        assert [[int(x), int(y)] for x, y in zip(fixed.tx, fixed.ty)] == c["window_kept"], c["cite"]
        if O.ref() is not None:
            r = O.ref_cluster_window_fix(pts, gp)
            assert np.array_equal(r.tx, fixed.tx) and np.array_equal(r.ty, fixed.ty)
            assert np.array_equal(r.cluster_id, fixed.cluster_id)


def test_window_fix_superset_and_live_reference():
    """test_agglomerate.cpp:255-277 (superset of plain pruning, counts equal)
    plus random inputs against the live reference."""
    rng = np.random.default_rng(99)
    for trial in range(6):
        gp = GridParams(precision=2, threshold=int(rng.integers(2, 7)),
                        min_cluster_size=int(rng.integers(1, 4)))
        tiles = rng.integers(0, 31, size=(120, 2))
        copies = rng.integers(1, 8, size=120)
        pts = centre_points([((int(a), int(b)), int(k)) for (a, b), k in zip(tiles, copies)], 2)
        pts = np.concatenate([pts, rng.uniform(0, 0.31, size=(300, 2))])
        plain = O.port_cluster(pts, gp)
        fixed = O.port_cluster(pts, gp, window_fix=True)
        fx = {(int(x), int(y)): int(n) for x, y, n in zip(fixed.tx, fixed.ty, fixed.count)}
        for x, y, n in zip(plain.tx, plain.ty, plain.count):
            assert fx[(int(x), int(y))] == int(n)
        if O.ref() is not None:
            r = O.ref_cluster_window_fix(pts, gp)
            assert np.array_equal(r.tx, fixed.tx) and np.array_equal(r.ty, fixed.ty), trial
            assert np.array_equal(r.count, fixed.count), trial
            assert np.array_equal(r.cluster_id, fixed.cluster_id), trial


def test_dedupe_kats(kat):
    """test_accumulator.cpp:184-212 (raw multiset vs dedupe_points)."""
    for c in kat["dedupe"]:
        gp = GridParams(precision=c["precision"], threshold=c["threshold"], min_cluster_size=1)
        r = O.port_cluster(np.array(c["points"]), gp, dedupe=c["dedupe"])
        assert r.tx.tolist() == [c["tile"][0]] and r.ty.tolist() == [c["tile"][1]], c["cite"]
        assert r.count.tolist() == [c["count"]], c["cite"]
        if O.ref() is not None:
            cid, px, py = O.ref_prime_points(np.array(c["points"]), gp, dedupe=c["dedupe"])
            assert len(px) == c["n_points"], c["cite"]


def test_dedupe_vs_live_reference():
    """Random inputs with heavy duplication, signed zeros and both
    significance paths, against the reference compiled here."""
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(7)
    for trial in range(8):
        gp = GridParams(precision=2, threshold=int(rng.integers(2, 6)),
                        min_cluster_size=int(rng.integers(1, 4)))
        base = np.round(rng.normal(0, 0.05, size=(3000, 2)), 3)
        pts = base[rng.integers(0, len(base), 9000)]
        pts[:50] *= -0.0  # signed zeros: (-0.0, -0.0) == (0.0, 0.0)
        wf = bool(trial % 2)
        mine = O.port_cluster(pts, gp, window_fix=wf, dedupe=True)
        ref = O.ref_cluster_flags(pts, gp, window_fix=wf, dedupe=True)
        assert np.array_equal(mine.tx, ref.tx) and np.array_equal(mine.ty, ref.ty), trial
        assert np.array_equal(mine.count, ref.count), trial
        assert np.array_equal(mine.cluster_id, ref.cluster_id), trial
        plain = O.port_cluster(pts, gp, window_fix=wf)
        assert mine.tx.size <= plain.tx.size


def test_neighbor_offsets_kats():
    """test_agglomerate.cpp:30-62 on the Python mirror's neighbor_offsets."""
    from paper_1907_03620_b200.raster import Tile, neighbor_offsets

    cheb1 = {(t.x, t.y) for t in neighbor_offsets(GridParams())}
    assert cheb1 == {(-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1)}
    man1 = {(t.x, t.y) for t in neighbor_offsets(GridParams(metric=Metric.manhattan))}
    assert man1 == {(-1, 0), (1, 0), (0, -1), (0, 1)}
    assert len(neighbor_offsets(GridParams(distance=2))) == 24
    man2 = neighbor_offsets(GridParams(metric=Metric.manhattan, distance=2))
    assert len(man2) == 12 and all(abs(t.x) + abs(t.y) <= 2 for t in man2)
    assert Tile(0, 0) not in set(man2)
