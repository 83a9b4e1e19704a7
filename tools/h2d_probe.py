import time, numpy as np, torch
x = np.random.default_rng(0).normal(size=(100000,128)).astype(np.float32)
pinned = torch.from_numpy(x.copy()).pin_memory()
hv = pinned.numpy()
dev = torch.empty((100000,128), dtype=torch.float32, device='cuda')
def t(f, name):
    for _ in range(2): f()
    torch.cuda.synchronize(); a=time.perf_counter()
    for _ in range(5): f()
    torch.cuda.synchronize(); print(name, (time.perf_counter()-a)/5*1e3, 'ms')
t(lambda: dev.copy_(torch.from_numpy(hv)), 'from_numpy(pinned view)')
t(lambda: dev.copy_(pinned), 'pinned tensor')
t(lambda: dev.copy_(pinned, non_blocking=True), 'pinned nb')
t(lambda: dev.copy_(torch.from_numpy(hv), non_blocking=True), 'from_numpy nb')
t(lambda: dev.copy_(torch.from_numpy(x)), 'pageable')
print(torch.from_numpy(hv).is_pinned())
ro = hv.view()
ro.flags.writeable = False
import warnings
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    t(lambda: dev.copy_(torch.from_numpy(ro)), 'read-only view of pinned')
    t(lambda: dev.copy_(torch.from_numpy(np.ascontiguousarray(ro, dtype=np.float32))), 'ascontiguous(ro)')
import sys
sys.path.insert(0, '/root/repo')
import paper_2312_03940_b200 as pk
p = pk.PointSet(hv)
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    t(lambda: dev.copy_(torch.from_numpy(p.data)), 'PointSet.data')
print(p.data.ctypes.data == hv.ctypes.data, hv.flags.writeable)
import time as _t
for gap in (0.0, 0.005, 0.04):
    ts = []
    for _ in range(5):
        _t.sleep(gap)
        torch.cuda.synchronize(); a = _t.perf_counter(); dev.copy_(pinned); torch.cuda.synchronize(); ts.append((_t.perf_counter() - a) * 1e3)
    print('gap', gap, [round(x, 2) for x in ts])
big = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
ts = []
for _ in range(5):
    big.fill_(1); torch.cuda.synchronize(); a = _t.perf_counter(); dev.copy_(pinned); torch.cuda.synchronize(); ts.append((_t.perf_counter() - a) * 1e3)
print('after flush', [round(x, 2) for x in ts])
stage = torch.empty(29 * (1 << 20), dtype=torch.uint8, pin_memory=True)
src = torch.empty(29 * (1 << 20), dtype=torch.uint8, device='cuda')
ts = []
for _ in range(5):
    stage.copy_(src, non_blocking=True); torch.cuda.synchronize()
    a = _t.perf_counter(); dev.copy_(pinned); torch.cuda.synchronize(); ts.append((_t.perf_counter() - a) * 1e3)
print('after d2h', [round(x, 2) for x in ts])
ts = []
for _ in range(5):
    big.fill_(1); x = torch.randn(4096, 4096, device='cuda'); y = x @ x; torch.cuda.synchronize()
    a = _t.perf_counter(); dev.copy_(pinned); torch.cuda.synchronize(); ts.append((_t.perf_counter() - a) * 1e3)
print('after compute', [round(x, 2) for x in ts])
ts = []
for _ in range(5):
    nb = np.isfinite(hv).all()
    a = _t.perf_counter(); dev.copy_(pinned); torch.cuda.synchronize(); ts.append((_t.perf_counter() - a) * 1e3)
print('after cpu read', [round(x, 2) for x in ts])
from paper_2312_03940_b200 import core as _core
ts = []
for _ in range(5):
    _core._first_nonfinite(hv)
    a = _t.perf_counter(); dev.copy_(pinned); torch.cuda.synchronize(); ts.append((_t.perf_counter() - a) * 1e3)
print('after threaded scan', [round(x, 2) for x in ts])
ts = []
for _ in range(5):
    _t.sleep(0.03)
    a = _t.perf_counter(); dev.copy_(pinned); torch.cuda.synchronize(); ts.append((_t.perf_counter() - a) * 1e3)
print('after sleep', [round(x, 2) for x in ts])
