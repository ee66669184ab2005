import sys, time
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[1]))
import torch
from paper_1907_03620_b200 import datagen as D
from paper_1907_03620_b200.raster import Pipeline
s = D.spec(4); n = D.count(s)
host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True); D.generate_into(s, host.data_ptr())
dev = host.cuda(); gp = D.params(4); pl = Pipeline(gp)
pl.run(dev); pl.cluster_points(dev, device_out=True); torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter(); pl.run(dev); torch.cuda.synchronize(); t1 = time.perf_counter()
    pl.cluster_points(dev, device_out=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print('run %.2f ms  cluster_points %.2f ms' % ((t1 - t0) * 1e3, (t2 - t1) * 1e3))
