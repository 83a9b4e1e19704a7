"""A first and a warm pipeline pass of a configuration on the GPU, with stage timings.

    python tools/run_config.py C4 [N] [brute]
"""
import ctypes
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, index, workloads  # noqa: E402
from paper_2312_03940_b200.cluster import run_pipeline_device  # noqa: E402

name = sys.argv[1]
w = workloads.WORKLOADS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else w.n
brute = len(sys.argv) > 3 and sys.argv[3] == "brute"
comps = max(1, int(round(w.components * n / w.n)))
t = time.time()
data, truth = workloads.generate(name, n=n, components=comps)
print(f"{name} n={n} d={w.d} comps={comps} brute={brute}: generated in {time.time() - t:.1f}s", flush=True)
kw = workloads.pipeline_args(name, pk, n_centers=min(w.n_centers, comps), brute=brute)
p = pk.PointSet(data)
print("mode", p.mode, flush=True)
_lib.prof_collect(reset=True)
_lib.prof_enable(True)
trace = []
t = time.time()
out = run_pipeline_device(p, **kw, trace=trace)
torch.cuda.synchronize()
el = time.time() - t
_lib.prof_enable(False)
prof = _lib.prof_collect(reset=True)
print(f"total {el:.3f}s stages { {k: round(v, 3) for k, v in out['timings'].items()} } rounds {trace}")
print("kernels", [(k, round(v[1], 1)) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:8]])
_cs = (ctypes.c_int64 * 2)()
_lib.lib().pk_tc_count_stats(_cs, 1)
print("tc", index.TC_STATS, "count decisions (rows, left open):", tuple(_cs))
labels = _lib.to_host(out["labels"])
print("ARI vs generator", pk.ari(labels, truth))
# second pass in the same process: one-time set-up (module loading, pool growth) excluded
del out
t = time.time()
out = run_pipeline_device(p, **kw)
torch.cuda.synchronize()
print(f"warm total {time.time() - t:.3f}s stages { {k: round(v, 3) for k, v in out['timings'].items()} }")
