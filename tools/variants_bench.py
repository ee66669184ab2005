"""Device timings of the path's variants on one B200 (reported in DESIGN.md):
window_fix, dedupe mode, RASTER' point lists, per-point labels in both input
orders. Points resident in HBM; CUDA events on the pipeline's stream; the
first call of each variant is untimed.

    python tools/variants_bench.py [config] [steps]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1907_03620_b200 import datagen as D  # noqa: E402
from paper_1907_03620_b200.raster import Pipeline  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
s = D.spec(cfg)
n = D.count(s)
host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
D.generate_into(s, host.data_ptr())
dev = host.cuda()
g = torch.Generator(device="cuda")
g.manual_seed(11)
shuf = dev[torch.randperm(n, device="cuda", generator=g)]
stream = torch.cuda.current_stream()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


out = {"config": cfg, "points": n, "steps": steps}
gp = D.params(cfg)
pl = Pipeline(gp)
pl.set_stream(stream.cuda_stream)
labels = torch.empty(n, dtype=torch.int32, device="cuda")
out["cluster_ms"] = timed(lambda: pl.run(dev))
out["cluster_window_fix_ms"] = timed(lambda: pl.run(dev, use_window_fix=True))
out["cluster_shuffled_ms"] = timed(lambda: pl.run(shuf))


def run_label(src):
    pl.run(src)
    pl.label_points(src, labels)


out["cluster_and_labels_ms"] = timed(lambda: run_label(dev))
out["cluster_and_labels_shuffled_ms"] = timed(lambda: run_label(shuf))


def run_points(src):
    pl.run(src)
    pl.cluster_points(src, device_out=True)


out["cluster_and_point_lists_ms"] = timed(lambda: run_points(dev))
gd = D.params(cfg)
gd.mode = 1  # Mode.retain_points
gd.dedupe_points = True
pd = Pipeline(gd)
pd.set_stream(stream.cuda_stream)
out["cluster_dedupe_ms"] = timed(lambda: pd.run(dev))
for k in list(out):
    if k.endswith("_ms"):
        out[k.replace("_ms", "_gpts")] = n / (out[k] / 1e3) / 1e9
print(json.dumps(out))
