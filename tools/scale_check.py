import sys, hashlib, numpy as np, torch
sys.path.insert(0, '.')
from paper_1907_03620_b200 import datagen as D
from paper_1907_03620_b200.raster import Pipeline
for cfg, sc in ((4, 0.25), (3, 0.37), (2, 1.0), (4, 0.013)):
    pts = D.generate(D.spec(cfg, sc), shuffle_seed=5)
    pts[::1013] = [1e9, 0.0]
    dev = torch.from_numpy(pts).cuda()
    pl = Pipeline(D.params(cfg)); st = pl.run(dev); f = pl.flat()
    h = hashlib.sha256()
    for a in (f.tx, f.ty, f.count, f.cluster_id): h.update(np.ascontiguousarray(a).tobytes())
    print(cfg, sc, len(pts), st.n_points, st.n_skipped, len(f.tx), h.hexdigest()[:12])
