"""A/B of K1 variants on one B200: device time of the contraction phase
(ms_contract, CUDA events around K1) and of the whole rg_cluster call, plus a
digest of the canonical result so variants can be compared bit for bit.

    RG_K1=v7 python tools/k1_ab.py [config ...]
"""
import hashlib
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1907_03620_b200 import datagen as D  # noqa: E402
from paper_1907_03620_b200.raster import Pipeline  # noqa: E402

steps = int(os.environ.get("AB_STEPS", "10"))
out = {"variant": os.environ.get("RG_K1", "default")}
for cfg in [int(a) for a in sys.argv[1:]] or [4]:
    dev = torch.from_numpy(D.generate(D.spec(cfg))).cuda()
    pl = Pipeline(D.params(cfg))
    stream = torch.cuda.current_stream()
    pl.set_stream(stream.cuda_stream)
    for _ in range(3):
        pl.run(dev)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    k1, k2, k3 = [], [], []
    a.record(stream)
    for _ in range(steps):
        st_ = pl.run(dev)
        k1.append(st_.ms_contract)
        k2.append(getattr(st_, "ms_prune", 0.0))
        k3.append(getattr(st_, "ms_agglomerate", 0.0))
    b.record(stream)
    torch.cuda.synchronize()
    f = pl.flat()
    h = hashlib.sha256()
    for arr in (f.tx, f.ty, f.count, f.cluster_id):
        h.update(np.ascontiguousarray(arr).tobytes())
    n = dev.shape[0]
    out[f"config{cfg}"] = {"k1_ms": statistics.median(k1), "k1_min_ms": min(k1),
                           "step_ms": a.elapsed_time(b) / steps, "k2_ms": statistics.median(k2), "k3_ms": statistics.median(k3),
                           "k1_frac": 16 * n / (statistics.median(k1) / 1e3) / 6537.6e9,
                           "digest": h.hexdigest()[:16]}
    del dev, pl
print(json.dumps(out))
