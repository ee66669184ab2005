"""Config 4 in a seeded random order: device time of rg_cluster (K1' path)."""
import json, os, statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_1907_03620_b200 import datagen as D  # noqa: E402
from paper_1907_03620_b200.raster import Pipeline  # noqa: E402
import hashlib, numpy as np  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dev = torch.from_numpy(D.generate(D.spec(cfg))).cuda()
g = torch.Generator(device="cuda"); g.manual_seed(11)
shuf = dev[torch.randperm(dev.shape[0], device="cuda", generator=g)]
del dev
pl = Pipeline(D.params(cfg)); st = torch.cuda.current_stream(); pl.set_stream(st.cuda_stream)
for _ in range(3):
    pl.run(shuf)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
k1 = []
a.record(st)
for _ in range(5):
    k1.append(pl.run(shuf).ms_contract)
b.record(st); torch.cuda.synchronize()
f = pl.flat(); h = hashlib.sha256()
for arr in (f.tx, f.ty, f.count, f.cluster_id):
    h.update(np.ascontiguousarray(arr).tobytes())
print(json.dumps({"variant": os.environ.get("V", "default"), "step_ms": a.elapsed_time(b) / 5,
                  "contract_ms": statistics.median(k1), "digest": h.hexdigest()[:12]}))
