"""Diagnostic: where does the end-to-end (host-buffer) time go?"""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1907_03620_b200 import datagen as D, _native as N
from paper_1907_03620_b200.raster import Pipeline

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
s = D.spec(cfg); n = D.count(s); gp = D.params(cfg)
host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
D.generate_into(s, host.data_ptr())
dev = host.cuda()
pl = Pipeline(gp)
for _ in range(2):
    pl.run(dev)
torch.cuda.synchronize()
def t(f, k=3):
    out = []
    for _ in range(k):
        torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); out.append(time.perf_counter() - a)
    return min(out) * 1e3
print('device run ms', t(lambda: pl.run(dev)))
print('host run ms', t(lambda: pl.run(host)))
st = pl.ctx.stats()
S = st.n_significant
tx = np.empty(S, np.int64); ty = np.empty(S, np.int64); cnt = np.empty(S, np.uint64); cid = np.empty(S, np.int64)
print('get_significant ms', t(lambda: pl.ctx.lib.rg_get_significant(pl.ctx.h, tx.ctypes.data, ty.ctypes.data, cnt.ctypes.data, cid.ctypes.data, S, N.RG_MEM_HOST)))
print('torch h2d 8GB ms', t(lambda: dev.copy_(host, non_blocking=True)))
ptx = torch.empty(S, dtype=torch.int64, pin_memory=True); pty = torch.empty(S, dtype=torch.int64, pin_memory=True)
pcnt = torch.empty(S, dtype=torch.int64, pin_memory=True); pcid = torch.empty(S, dtype=torch.int64, pin_memory=True)
print('get_significant pinned ms', t(lambda: pl.ctx.lib.rg_get_significant(pl.ctx.h, ptx.data_ptr(), pty.data_ptr(), pcnt.data_ptr(), pcid.data_ptr(), S, N.RG_MEM_HOST)))
for k in range(3):
    print('repeat', k, 'host run ms', t(lambda: pl.run(host), 1), 'torch h2d ms', t(lambda: dev.copy_(host, non_blocking=True), 1))
import subprocess
print(subprocess.run(['nvidia-smi', 'topo', '-m'], capture_output=True, text=True).stdout)
print(subprocess.run(['bash', '-c', 'numactl -H 2>/dev/null | head -5; nproc; lscpu | grep -i "numa\\|model name"'], capture_output=True, text=True).stdout)
