"""Generates the committed golden fixtures from the REFERENCE ITSELF.

Run in the build container (where /root/reference exists and oracle/_ref is
built from its headers):

    python tests/golden/make_golden.py

Writes tests/golden/ref_fixtures.npz. Every expected value in it was produced
by the reference's own code through oracle/ref_shim.cpp:
  - cfg{k}_{order}: config-shaped seeded inputs (the generator spec is stored,
    plus a sha256 of the input bytes) -> cluster_sequential canonical output
    (significant tiles sorted, counts, cluster ids) and counters; per-point
    labels cross-checked against the reference's prime-mode output
    (cluster_sequential with Mode::retain_points) before being stored;
  - tiles{i}: random tile sets -> agglomerate() partitions (acceptance.cpp
    criterion 2 style, both metrics, delta 1 and 2);
  - gridline: points on and next to grid lines -> project_unchecked tiles.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import pyoracle as O  # noqa: E402
from paper_1907_03620_b200 import datagen as D  # noqa: E402
from paper_1907_03620_b200.raster import GridParams, Metric  # noqa: E402

FIXTURE_SCALES = {1: 0.01, 2: 0.01, 3: 0.0001, 4: 0.00002, 5: 0.0001}
SHUFFLE_SEED = 0xC0FFEE


def spec_dict(s) -> dict:
    return {name: getattr(s, name) for name, _ in s._fields_}


def labels_from_prime(points: np.ndarray, gp, res) -> np.ndarray:
    """Per-point labels of the port, verified against the reference's
    RASTER' output: for every cluster id k the point_less-sorted multiset of
    points labelled k must equal Cluster::points of cluster k."""
    labels = O.port_labels(points, gp, res)
    cid, px, py = O.ref_prime_points(points, gp)
    sel = labels >= 0
    lab, xs, ys = labels[sel], points[sel, 0], points[sel, 1]
    order = np.lexsort((ys, xs, lab))
    assert np.array_equal(lab[order].astype(np.int64), cid), "labels disagree with prime mode"
    assert np.array_equal(xs[order], px) and np.array_equal(ys[order], py)
    return labels


def main() -> None:
    if O.ref() is None:
        raise SystemExit("oracle/_ref/libraster_ref.so missing: run oracle/build_ref.sh here")
    out: dict[str, np.ndarray] = {}
    meta: dict = {"configs": {}}
    for cfg, scale in FIXTURE_SCALES.items():
        s = D.spec(cfg, scale)
        gp = D.params(cfg)
        base = D.generate(s)
        for order in ("gen", "shuf"):
            pts = base if order == "gen" else D.shuffle(base, SHUFFLE_SEED)
            res, _, _ = O.ref_cluster(pts, gp)
            port = O.port_cluster(pts, gp)
            for k in ("tx", "ty", "count", "cluster_id"):
                assert np.array_equal(getattr(res, k), getattr(port, k)), (cfg, order, k)
            labels = labels_from_prime(pts, gp, res)
            tag = f"cfg{cfg}_{order}"
            out[f"{tag}_tx"] = res.tx
            out[f"{tag}_ty"] = res.ty
            out[f"{tag}_count"] = res.count
            out[f"{tag}_cid"] = res.cluster_id
            out[f"{tag}_labels"] = labels
            meta["configs"][tag] = {
                "spec": spec_dict(s),
                "shuffle_seed": SHUFFLE_SEED if order == "shuf" else None,
                "params": {"precision": gp.precision, "threshold": gp.threshold,
                           "distance": gp.distance, "min_cluster_size": gp.min_cluster_size},
                "n_points": int(pts.shape[0]),
                "input_sha256": hashlib.sha256(pts.tobytes()).hexdigest(),
                "n_ingested": res.n_ingested, "n_skipped": res.n_skipped,
                "n_distinct": res.n_distinct, "n_clusters": res.n_clusters,
            }
    # random tile sets (acceptance.cpp:97-121 style)
    rng = np.random.default_rng(0x02AC1E)
    meta["tiles"] = []
    for i in range(24):
        metric = Metric.manhattan if i % 2 else Metric.chebyshev
        distance = 1 + (i // 2) % 2
        n = int(rng.integers(50, 800))
        extent = int(np.sqrt(n * 2.0))
        pairs = set()
        while len(pairs) < n:
            pairs.add((int(rng.integers(-extent, extent + 1)), int(rng.integers(-extent, extent + 1))))
        arr = np.array(sorted(pairs), np.int64)
        rng.shuffle(arr)
        gp = GridParams(distance=distance, metric=metric, min_cluster_size=1 + (i % 3))
        res = O.ref_agglomerate(arr[:, 0], arr[:, 1], np.full(n, 5, np.uint64), gp)
        out[f"tiles{i}_in"] = arr
        out[f"tiles{i}_cid"] = res.cluster_id
        meta["tiles"].append({"metric": int(metric), "distance": distance,
                              "min_cluster_size": gp.min_cluster_size, "n_clusters": res.n_clusters})
    # grid-line projection vectors
    gl = []
    for p in (1.0, 2.0, 3.0, 3.5):
        s = 10.0 ** p
        for k in range(-2000, 2001, 7):
            v = k / s
            for w in (v, np.nextafter(v, -np.inf), np.nextafter(v, np.inf), k * 10.0 ** -p):
                gl.append((p, w, -w / 2))
    gl = np.array(gl, np.float64)
    tiles = np.array([O.ref_project(x, y, p) for p, x, y in gl], np.int64)
    out["gridline_in"] = gl
    out["gridline_tiles"] = tiles
    dst = Path(__file__).with_name("ref_fixtures.npz")
    np.savez_compressed(dst, meta=np.frombuffer(json.dumps(meta).encode(), np.uint8), **out)
    print(f"wrote {dst} ({dst.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
