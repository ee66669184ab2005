"""Helpers shared by the GPU parity tests."""
from __future__ import annotations

import numpy as np

from oracle import pyoracle as O


def assert_same(flat, ref, what=""):
    """Bit-exact equality of the canonical flat form."""
    assert flat.tx.shape == ref.tx.shape, (what, flat.tx.shape, ref.tx.shape)
    assert np.array_equal(flat.tx, ref.tx), what
    assert np.array_equal(flat.ty, ref.ty), what
    assert np.array_equal(flat.count.astype(np.uint64), ref.count.astype(np.uint64)), what
    assert np.array_equal(flat.cluster_id, ref.cluster_id), what
    assert flat.n_clusters == ref.n_clusters, what


def oracle(points, gp):
    return O.port_cluster(points, gp)


def numpy_tile_counts(points, gp):
    """Brute-force tile tally (tests/support/oracles.hpp:39-47 style) using the
    reference's projection formula: floor(x * 10^p) in IEEE double."""
    pts = np.asarray(points, np.float64).reshape(-1, 2)
    b = gp.bounds
    s = 10.0 ** gp.precision
    inb = (pts[:, 0] >= b.x_min) & (pts[:, 0] <= b.x_max) & (pts[:, 1] >= b.y_min) & (pts[:, 1] <= b.y_max)
    q = pts[inb]
    tx = np.floor(q[:, 0] * s).astype(np.int64)
    ty = np.floor(q[:, 1] * s).astype(np.int64)
    keys, counts = np.unique(np.stack([tx, ty], 1), axis=0, return_counts=True)
    return {(int(a), int(b_)): int(c) for (a, b_), c in zip(keys, counts)}
