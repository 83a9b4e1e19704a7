"""Cost of the doubling rounds' wide beam searches (L = k up to 2048) on a
C5-shaped graph: beam_knn time for m queries at each k."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, vamana, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
cfg = sys.argv[2] if len(sys.argv) > 2 else "C5"
w = workloads.WORKLOADS[cfg]
data, _ = workloads.generate(cfg, n=n, components=max(1, int(round(w.components * n / w.n))))
p = pk.PointSet(data)
g = pk.build_vamana(p, R=w.R, L_build=w.L, alpha=w.alpha, seed=0, query_beam=w.L)
rng = np.random.default_rng(0)
plan = [(3000, 32), (1000, 256), (800, 512), (700, 1024), (700, 2048)] if cfg != "C3" else \
    [(30000, 64), (15000, 128), (7600, 256), (3800, 512), (1900, 1024), (970, 2048), (466, 4096)]
for m, k in plan:
    q = torch.from_numpy(np.sort(rng.choice(n, m, replace=False))).cuda()
    for rep in range(2):
        _lib.prof_collect(reset=True)
        _lib.prof_only(["beam_knn_kernel"])
        _lib.prof_enable(True)
        ids, sqd, cnt = vamana.beam_knn_raw(g.graph, q, max(w.L, k), k)
        torch.cuda.synchronize()
        _lib.prof_enable(False)
        ms = _lib.prof_collect(reset=True)["beam_knn_kernel"][1]
    short = int((cnt < min(k, n - 1)).sum())
    print(f"m={m} k={k}: {ms:.1f} ms, {m / ms * 1e3:.0f} queries/s, short {short}", flush=True)
