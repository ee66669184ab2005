"""GPU parity: the sm_100a path (through the C-ABI) against the reference's
fixtures, the reference's known-answer tests and the CPU oracle, bit-exact.
Needs a B200."""
from __future__ import annotations

import hashlib
import math
from collections import Counter

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1907_03620_b200 import datagen as D
from paper_1907_03620_b200.raster import (Bounds, GridParams, Metric, Pipeline, Tile,
                                          TileAccumulator, agglomerate, agglomerate_flat,
                                          cluster_flat, cluster_sequential)

from .gpu_util import assert_same, numpy_tile_counts, oracle

pytestmark = pytest.mark.gpu


def torch_cuda():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def centre_points(tile_copies, precision):
    side = 10.0 ** -precision
    pts = []
    for (tx, ty), copies in tile_copies:
        pts += [((tx + 0.5) * side, (ty + 0.5) * side)] * copies
    return np.array(pts, np.float64).reshape(-1, 2)


# ------------------------------------------------------------ fixtures


def fixture_points(meta, tag):
    m = meta["configs"][tag]
    s = D.spec(int(tag[3]), 1.0)
    for k, v in m["spec"].items():
        setattr(s, k, v)
    pts = D.generate(s)
    if m["shuffle_seed"] is not None:
        pts = D.shuffle(pts, m["shuffle_seed"])
    assert hashlib.sha256(pts.tobytes()).hexdigest() == m["input_sha256"]
    return pts


@pytest.mark.parametrize("memory", ["host", "device"])
def test_reference_fixtures(golden, memory):
    torch = torch_cuda()
    z, meta = golden
    for tag, m in meta["configs"].items():
        cfg = int(tag[3])
        gp = D.params(cfg)
        pts = fixture_points(meta, tag)
        src = torch.from_numpy(pts).cuda() if memory == "device" else pts
        pl = Pipeline(gp)
        st = pl.run(src)
        flat = pl.flat()
        assert np.array_equal(flat.tx, z[f"{tag}_tx"]), tag
        assert np.array_equal(flat.ty, z[f"{tag}_ty"]), tag
        assert np.array_equal(flat.count, z[f"{tag}_count"]), tag
        assert np.array_equal(flat.cluster_id, z[f"{tag}_cid"]), tag
        assert (st.n_ingested, st.n_skipped, st.peak_accumulator_entries, st.n_clusters) == (
            m["n_ingested"], m["n_skipped"], m["n_distinct"], m["n_clusters"]), tag
        labels = pl.label_points(src)
        labels = labels if isinstance(labels, np.ndarray) else labels.cpu().numpy()
        assert np.array_equal(labels, z[f"{tag}_labels"]), tag


def test_reference_tile_sets(golden):
    z, meta = golden
    for i, m in enumerate(meta["tiles"]):
        t = z[f"tiles{i}_in"]
        gp = GridParams(distance=m["distance"], metric=Metric(m["metric"]),
                        min_cluster_size=m["min_cluster_size"])
        sig = {Tile(int(x), int(y)): 5 for x, y in t}
        flat = agglomerate_flat(sig, gp)
        assert np.array_equal(flat.cluster_id, z[f"tiles{i}_cid"]), i
        assert flat.n_clusters == m["n_clusters"]


def test_gridline_projection(golden):
    z, _ = golden
    gl, want = z["gridline_in"], z["gridline_tiles"]
    inb = (np.abs(gl[:, 1]) <= 180.0) & (np.abs(gl[:, 2]) <= 90.0)  # the fixture projects unchecked
    for p in np.unique(gl[:, 0]):
        sel = (gl[:, 0] == p) & inb
        gp = GridParams(precision=float(p))
        acc = TileAccumulator(gp)
        acc.ingest(gl[sel, 1:])
        got = acc.counts()
        exp = Counter((int(a), int(b)) for a, b in want[sel])
        assert {(t.x, t.y): c for t, c in got.items()} == dict(exp), p


# ------------------------------------------------------------ KATs (reference unit tests)


def test_kat_projection(kat):
    for case in kat["projection"]:
        gp = GridParams(precision=case["precision"], threshold=1, min_cluster_size=1)
        for (x, y), want in zip(case["points"], case["tiles"]):
            acc = TileAccumulator(gp)
            acc.ingest(np.array([[x, y]]))
            assert acc.counts() == {Tile(*want): 1}, case["cite"]


def test_kat_bounds(kat):
    c = kat["bounds"]
    acc = TileAccumulator(GridParams())
    acc.ingest(np.array(c["outside"] + c["inside"]))
    assert acc.skipped() == len(c["outside"])
    assert acc.total_ingested() == len(c["inside"])


def test_kat_three_point(kat):
    c = kat["three_point"]
    acc = TileAccumulator(GridParams(precision=c["precision"]))
    acc.ingest(np.array(c["points"]))
    assert acc.entry_count() == c["entries"]
    assert acc.count_of(Tile(*c["tile"])) == c["count"]


def test_kat_prune(kat):
    c = kat["prune"]
    acc = TileAccumulator(GridParams(precision=c["precision"], threshold=c["threshold"]))
    acc.ingest(centre_points(c["tile_copies"], c["precision"]))
    sig = acc.prune()
    assert len(sig) == len(c["kept"])
    for t, n in c["kept"]:
        assert sig.at(Tile(*t)).count == n
    assert acc.entry_count() == 0  # consumed


def test_kat_threshold_one_keeps_everything():
    rng = np.random.default_rng(11)
    pts = np.stack([rng.uniform(-10, 10, 300), rng.uniform(-5, 5, 300)], 1)
    acc = TileAccumulator(GridParams(precision=2, threshold=1))
    acc.ingest(pts)
    occupied = acc.entry_count()
    assert len(acc.prune()) == occupied


def test_kat_oob_skip(kat):
    c = kat["oob_skip"]
    acc = TileAccumulator(GridParams(precision=c["precision"]))
    acc.ingest(np.array(c["points"]))
    assert (acc.total_ingested(), acc.skipped()) == (c["ingested"], c["skipped"])


def test_kat_merge(kat):
    c = kat["merge"]
    gp = GridParams(precision=c["precision"])
    a, b = TileAccumulator(gp), TileAccumulator(gp)
    a.ingest(centre_points(c["a"], c["precision"]))
    b.ingest(centre_points(c["b"], c["precision"]))
    a.merge(b)
    for t, n in c["counts"]:
        assert a.count_of(Tile(*t)) == n
    assert a.total_ingested() == c["ingested"]
    assert b.entry_count() == 0 and b.total_ingested() == 0


@pytest.mark.parametrize("name", ["group_and_drop", "ids_by_smallest", "singleton", "cluster_csv"])
def test_kat_agglomerate(kat, name):
    c = kat[name]
    gp = GridParams(min_cluster_size=c["min_cluster_size"])
    cs = agglomerate({Tile(*t): 5 for t in c["tiles"]}, gp)
    if "clusters" in c:
        assert [[[t.x, t.y] for t in cl.tiles] for cl in cs.clusters] == c["clusters"]
        assert [cl.id for cl in cs.clusters] == list(range(len(cs.clusters)))
    if "csv" in c:
        csv = "".join(f"{cl.id},{t.x},{t.y}\n" for cl in cs.clusters for t in cl.tiles)
        assert csv == c["csv"]


def test_kat_empty_agglomerate():
    assert agglomerate({}, GridParams()).clusters == []


def test_kat_prime_accounting(kat):
    c = kat["prime_accounting"]
    pts = centre_points(c["tile_copies"], c["precision"])
    gp = GridParams(precision=c["precision"], threshold=c["threshold"],
                    min_cluster_size=c["min_cluster_size"], mode=1)
    cs = cluster_sequential(pts, gp)
    assert sum(len(cl.points) for cl in cs.clusters) == c["clustered_points"]


# ------------------------------------------------------------ full-size configs vs oracle


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_config_full_size_vs_oracle(cfg):
    torch = torch_cuda()
    pts = D.generate(D.spec(cfg))
    gp = D.params(cfg)
    ref = oracle(pts, gp)
    dev = torch.from_numpy(pts).cuda()
    pl = Pipeline(gp)
    st = pl.run(dev)
    assert_same(pl.flat(), ref, f"cfg{cfg}")
    assert (st.n_ingested, st.n_skipped, st.peak_accumulator_entries) == (
        ref.n_ingested, ref.n_skipped, ref.n_distinct)
    labels = pl.label_points(dev).cpu().numpy()
    assert np.array_equal(labels, O.port_labels(pts, gp, ref))


@pytest.mark.parametrize("cfg", [1, 2, 3, 5])
def test_config_shuffled_vs_oracle(cfg):
    torch = torch_cuda()
    scale = {1: 1.0, 2: 1.0, 3: 0.2, 5: 0.05}[cfg]
    pts = D.generate(D.spec(cfg, scale), shuffle_seed=7)
    gp = D.params(cfg)
    ref = oracle(pts, gp)
    pl = Pipeline(gp)
    st = pl.run(torch.from_numpy(pts).cuda())
    assert_same(pl.flat(), ref, f"cfg{cfg} shuffled")
    assert st.peak_accumulator_entries == ref.n_distinct


def test_config5_scaled_vs_oracle():
    torch = torch_cuda()
    pts = D.generate(D.spec(5, 0.1))  # 10M blob, 100 walks, 4M noise
    gp = D.params(5)
    ref = oracle(pts, gp)
    pl = Pipeline(gp)
    pl.run(torch.from_numpy(pts).cuda())
    assert_same(pl.flat(), ref, "cfg5 x0.1")


@pytest.mark.parametrize("cfg", [4, 5])
def test_config_full_size_vs_oracle_and_properties(cfg):
    """Full BASELINE sizes (500M / 200M points) against the CPU oracle
    (the C restatement of cluster_sequential, pipeline.hpp:92-126, and of
    labeled_points, metrics.hpp:78-83): significant tiles, counts, canonical
    ids and counters bit-exact; config 4 also per point (int32 labels).
    Then the same bytes in a seeded random order (config 4 takes the
    partitioned contraction K1' there) and in 7 out-of-order chunks must give
    bit-identical results, and the shuffled labels must be the permuted
    generation-order labels."""
    torch = torch_cuda()
    s = D.spec(cfg)
    n = D.count(s)
    host = np.empty((n, 2), np.float64)
    D.generate_into(s, host.ctypes.data)
    gp = D.params(cfg)
    dev = torch.from_numpy(host).cuda()
    pl = Pipeline(gp)
    st = pl.run(dev)
    a = pl.flat()
    ref = oracle(host, gp)
    assert_same(a, ref, f"cfg{cfg} full size vs oracle")
    assert (st.n_ingested, st.n_skipped, st.peak_accumulator_entries) == (
        ref.n_ingested, ref.n_skipped, ref.n_distinct)
    assert st.n_ingested + st.n_skipped == n
    labels = pl.label_points(dev)
    if cfg == 4:
        want_labels = O.port_labels(host, gp, ref)
        assert np.array_equal(labels.cpu().numpy(), want_labels), "cfg4 per-point labels"
        del want_labels
    else:
        # labels: count per cluster == sum of its tile counts
        hist = torch.bincount(labels[labels >= 0].long(), minlength=a.n_clusters).cpu().numpy()
        keep = a.cluster_id >= 0
        want = np.bincount(a.cluster_id[keep], weights=a.count[keep].astype(np.float64),
                           minlength=a.n_clusters)
        assert np.array_equal(hist.astype(np.float64), want)
    del ref, host
    # chunked ingestion (7 uneven chunks, out of order) == single pass
    acc = TileAccumulator(gp)
    cuts = sorted({0, n, *[int(v) for v in np.random.default_rng(3).integers(0, n, 6)]})
    chunks = list(zip(cuts[:-1], cuts[1:]))
    for lo, hi in reversed(chunks):
        acc.ingest(dev[lo:hi])
    sig = acc.prune()
    assert np.array_equal(sig.tx, a.tx) and np.array_equal(sig.ty, a.ty)
    assert np.array_equal(sig.count, a.count)
    del acc, sig
    # shuffled order (device-side permutation) == generation order
    perm = torch.randperm(n, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    shuf = dev[perm]
    pl2 = Pipeline(gp)
    pl2.run(shuf)
    assert_same(pl2.flat(), a, f"cfg{cfg} order invariance")
    assert torch.equal(pl2.label_points(shuf), labels[perm]), f"cfg{cfg} shuffled labels"


def test_context_reuse_across_growth_and_partitioned_ingest():
    """One Pipeline (one C-ABI context) reused: a shuffled run, a larger run
    whose table grows, then a shuffled run of >= 4 Mi points (the partitioned
    contraction's scratch must survive the table resize), each against the
    oracle."""
    torch = torch_cuda()
    gp = D.params(3)
    pl = Pipeline(gp)
    noise = np.random.default_rng(12).uniform([-180, -90], [180, 90], size=(8_000_000, 2))
    cases = (
        ("shuffled 5M", D.generate(D.spec(3, 0.05), shuffle_seed=7)),
        ("10M + 8M distinct noise tiles (table grows)",
         np.concatenate([D.generate(D.spec(3, 0.1)), noise])),
        ("shuffled 6M after the resize", D.generate(D.spec(3, 0.06), shuffle_seed=9)),
    )
    caps = []
    for what, pts in cases:
        st = pl.run(torch.from_numpy(pts).cuda())
        caps.append(st.table_capacity)
        assert_same(pl.flat(), oracle(pts, gp), what)
    assert caps[1] > caps[0], caps  # the second step really grew the table


@pytest.mark.parametrize("k3", ["bucket", "seg", "hash"])
def test_cluster_facts_vs_oracle(k3):
    """rg_get_clusters: tiles, points and smallest tile of every cluster,
    against the oracle's flat clustering (every K3 path, incl. the bucketed
    one whose point totals are summed on demand)."""
    import os
    import subprocess
    import sys

    code = (
        "import numpy as np\n"
        "from oracle import pyoracle as O\n"
        "from paper_1907_03620_b200 import datagen as D\n"
        "from paper_1907_03620_b200.raster import Pipeline\n"
        "gp = D.params(2)\n"
        "pts = D.generate(D.spec(2, 0.3), shuffle_seed=5)\n"
        "pl = Pipeline(gp)\n"
        "pl.run(pts)\n"
        "nt, npnt, fx, fy = pl.cluster_facts()\n"
        "ref = O.port_cluster(pts, gp)\n"
        "k = ref.cluster_id >= 0\n"
        "c = ref.cluster_id[k]\n"
        "assert len(nt) == ref.n_clusters > 100\n"
        "assert np.array_equal(nt, np.bincount(c, minlength=ref.n_clusters).astype(np.uint64))\n"
        "assert np.array_equal(npnt, np.bincount(c, weights=ref.count[k].astype(np.float64),"
        " minlength=ref.n_clusters).astype(np.uint64))\n"
        "first = np.full(ref.n_clusters, len(k))\n"
        "np.minimum.at(first, c, np.nonzero(k)[0])\n"
        "assert np.array_equal(fx, ref.tx[first]) and np.array_equal(fy, ref.ty[first])\n"
        "print('ok')\n")
    env = dict(os.environ)
    if k3 == "hash":
        env["RG_K3"] = "hash"
    else:
        env["RG_K3_SORT"] = k3[0]
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr[-2000:]


@pytest.mark.parametrize("metric,delta,wf", [(Metric.chebyshev, 1, False), (Metric.chebyshev, 1, True),
                                             (Metric.manhattan, 2, False), (Metric.chebyshev, 3, False)])
def test_labels_every_k3_path_vs_oracle(metric, delta, wf):
    """Per-point labels after the sorted K3 (table SIG marks written lazily,
    carrying cluster ids) and after the hash-probe K3 (delta 3: SIG | dense
    index written by K2); labelling twice gives the same answer."""
    rng = np.random.default_rng(17 + delta)
    gp = GridParams(precision=2, threshold=3, min_cluster_size=2, metric=metric, distance=delta)
    c = rng.uniform([-170, -80], [170, 80], size=(300, 2))
    pts = (c[rng.integers(0, 300, 200_000)] + rng.normal(0, 0.02, size=(200_000, 2))).astype(np.float64)
    pl = Pipeline(gp)
    pl.run(pts, use_window_fix=wf)
    ref = O.port_cluster(pts, gp, window_fix=wf) if wf else O.port_cluster(pts, gp)
    assert_same(pl.flat(), ref)
    want = O.port_labels(pts, gp, ref)
    assert np.array_equal(pl.label_points(pts), want)
    assert np.array_equal(pl.label_points(pts), want)
