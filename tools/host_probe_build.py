"""Host time of the build at C2: the start sampling + PCG64 permutation before
the first kernel, the pk_build_vamana call (enqueue + its final sync), and the
remaining device time after it returns.

    python tools/host_probe_build.py
"""
import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2312_03940_b200 as pk
from paper_2312_03940_b200 import workloads, vamana, _lib
data, _ = workloads.generate("C2")
p = pk.PointSet(data)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    starts, order = vamana.sample_starts(p.n, None, 0, False, p)
    t1 = time.perf_counter()
    res = vamana.build_graph_device(p, 64, 128, 1.1, starts, order, seed_cache=True)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"sample_starts {1e3*(t1-t0):.3f} ms, build call {1e3*(t2-t1):.3f} ms, after-sync {1e3*(t3-t2):.3f} ms")
