"""Labels of config 4 in a seeded random order: device time of rg_label_points
alone (the clustering is done once, untimed)."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_1907_03620_b200 import datagen as D  # noqa: E402
from paper_1907_03620_b200.raster import Pipeline  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dev = torch.from_numpy(D.generate(D.spec(cfg))).cuda()
g = torch.Generator(device="cuda"); g.manual_seed(11)
shuf = dev[torch.randperm(dev.shape[0], device="cuda", generator=g)]
pl = Pipeline(D.params(cfg)); st = torch.cuda.current_stream(); pl.set_stream(st.cuda_stream)
lab = torch.empty(dev.shape[0], dtype=torch.int32, device="cuda")
out = {"variant": os.environ.get("RG_K4", "default")}
for name, x in ((("gen", dev), ("shuffled", shuf)) if len(sys.argv) < 3 else (("shuffled", shuf),)):
    pl.run(x)
    pl.label_points(x, lab)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(5):
        pl.label_points(x, lab)
    b.record(st); torch.cuda.synchronize()
    out[name + "_label_ms"] = a.elapsed_time(b) / 5
print(json.dumps(out))
