"""Tensor-core screening throughput: knn of m queries over n points (d=1024, C5 generator)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, index, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else n
x, _ = workloads.generate("C5", n=n, components=max(1, n // 1281))
p = pk.PointSet(x)
q = torch.arange(m, dtype=torch.int64, device="cuda")
index.brute_device(p, q[:4096], 16)
torch.cuda.synchronize()
_lib.prof_collect(reset=True)
_lib.prof_enable(True)
t = time.time()
ids, sqd = index.brute_device(p, q, 16)
torch.cuda.synchronize()
el = time.time() - t
_lib.prof_enable(False)
prof = _lib.prof_collect(reset=True)
flop = 2.0 * m * n * 1024
scr = prof["tc_screen_kernel"][1]
print(f"n={n} m={m}: total {el:.3f}s  screen {scr:.1f} ms -> {flop / scr / 1e9:.1f} TFLOP/s; "
      f"kernels {[(k, round(v[1], 2)) for k, v in prof.items()]} stats={index.TC_STATS}")
