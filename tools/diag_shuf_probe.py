"""Which contraction path does each call take? (RG_DEBUG=1 prints the order
probe's verdicts.) Mirrors bench.py's sequence: device run, host run,
labelled runs, then the shuffled copy."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1907_03620_b200 import datagen as D  # noqa: E402
from paper_1907_03620_b200.raster import Pipeline  # noqa: E402

s = D.spec(4)
n = D.count(s)
host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
D.generate_into(s, host.data_ptr())
dev = host.cuda()
stream = torch.cuda.current_stream()
pl = Pipeline(D.params(4))
pl.set_stream(stream.cuda_stream)
print("device run", file=sys.stderr)
pl.run(dev)
print("host run", file=sys.stderr)
pl.run(host)
g = torch.Generator(device="cuda")
g.manual_seed(11)
shuf = dev[torch.randperm(n, device="cuda", generator=g)]
print("shuffled run", shuf.data_ptr(), dev.data_ptr(), file=sys.stderr)
pl.run(shuf)
torch.cuda.synchronize()
