"""Where the end-to-end (host arrays in, numpy out) time goes at C2: the bench's
e2e loop with timers around each part (instrumented wrappers)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import cluster, core, workloads  # noqa: E402

data, _ = workloads.generate("C2")
kw = workloads.pipeline_args("C2", pk)
pinned = torch.from_numpy(np.array(data, dtype=np.float32, copy=True)).pin_memory()
hv = pinned.numpy()
T = {}


def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + time.perf_counter() - t
        return r
    return w


def upload_split(data):
    import warnings
    arr = np.ascontiguousarray(data, dtype=np.float32)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        host = torch.from_numpy(arr)
    torch.cuda.synchronize()
    t = time.perf_counter()
    dev = torch.empty(arr.shape, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dev.copy_(host)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return dev


core.upload_points = timed("upload", upload_split)
cluster.run_pipeline_device = timed("pipeline", cluster.run_pipeline_device)
cluster._to_host_many = timed("d2h", cluster._to_host_many)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(5):
    T.clear()
    flush.fill_(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = pk.PointSet(hv)
    t1 = time.perf_counter()
    res = pk.run_pipeline(p, **kw)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    del p, res
    print(f"total {1e3 * (t2 - t0):.2f} pointset {1e3 * (t1 - t0):.2f} "
          + " ".join(f"{k} {1e3 * v:.2f}" for k, v in T.items()))
