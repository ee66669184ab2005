"""Diagnostic: config-2 shuffled parity under different table sizings."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import pyoracle as O
from paper_1907_03620_b200 import datagen as D
from paper_1907_03620_b200.raster import Pipeline, TileAccumulator

pts = D.generate(D.spec(2), shuffle_seed=7)
gp = D.params(2)
ref = O.port_cluster(pts, gp)
refd = {(a, b): c for a, b, c in zip(ref.tx.tolist(), ref.ty.tolist(), ref.count.tolist())}
dev = torch.from_numpy(pts).cuda()
for hint in (0, 20_000_000, 1):
    gp.capacity_hint = hint
    acc = TileAccumulator(gp)
    acc.ingest(dev)
    print('hint', hint, 'ingested', acc.total_ingested(), 'skipped', acc.skipped(), 'entries', acc.entry_count(), 'ref', ref.n_ingested, ref.n_skipped, ref.n_distinct)
    cnt = acc.counts()
    got = {(t.x, t.y): c for t, c in cnt.items()}
    diff = [(k, got.get(k, 0), v) for k, v in refd.items() if got.get(k, 0) != v]
    print('  sig tiles with count diff:', len(diff), diff[:5], 'total gpu', sum(got.values()))
    st = Pipeline(gp).run(dev)
    print('  pipeline ingested', st.n_ingested, 'grows', st.table_grows, 'cap', st.table_capacity)
