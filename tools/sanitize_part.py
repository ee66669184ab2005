"""Small partitioned-contraction run checked against the oracle (also usable under
compute-sanitizer where that is available):
    RG_INGEST=part RG_PART=stream compute-sanitizer --tool memcheck python tools/sanitize_part.py
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from oracle import pyoracle as O  # noqa: E402  (checker)
from paper_1907_03620_b200 import datagen as D  # noqa: E402
from paper_1907_03620_b200.raster import Pipeline  # noqa: E402

gp = D.params(4)
pts = D.generate(D.spec(4, 0.004), shuffle_seed=3)  # 2M points
pts[::997] = [400.0, 0.0]
dev = torch.from_numpy(pts).cuda()
pl = Pipeline(gp)
pl.run(dev)
f = pl.flat()
ref = O.port_cluster(pts, gp)
assert np.array_equal(f.tx, ref.tx) and np.array_equal(f.count, ref.count) and np.array_equal(f.cluster_id, ref.cluster_id)
lab = pl.label_points(dev).cpu().numpy()
assert np.array_equal(lab, O.port_labels(pts, gp, ref))
print("ok", len(pts), len(f.tx))
