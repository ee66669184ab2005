import torch, sys
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[1]))
from paper_1907_03620_b200 import datagen as D
s = D.spec(4); n = D.count(s)
host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True); D.generate_into(s, host.data_ptr())
dev = host.cuda()
g = torch.Generator(device="cuda"); g.manual_seed(11)
perm = torch.randperm(n, device="cuda", generator=g)
print("perm min/max", int(perm.min()), int(perm.max()), "unique?", int(torch.bincount(perm[:10_000_000] % 1000).min()))
print("perm sorted equals arange:", bool((torch.sort(perm).values == torch.arange(n, device='cuda')).all()))
shuf = dev[perm]
print("sums dev", float(dev[:,0].sum()), float(dev[:,1].sum()))
print("sums shuf", float(shuf[:,0].sum()), float(shuf[:,1].sum()))
shuf2 = torch.index_select(dev, 0, perm)
print("sums shuf2", float(shuf2[:,0].sum()), float(shuf2[:,1].sum()))
