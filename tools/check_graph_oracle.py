"""Full-size graph parity: the GPU Vamana build of a BASELINE configuration
against the CPU oracle's build (oracle/, the reference restated in C) on the
same points and seed -- adjacency and degrees must be identical.

    python tools/check_graph_oracle.py C2 [n]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = workloads.WORKLOADS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else w.n
data, _ = workloads.generate(name, n=n, components=max(1, int(round(w.components * n / w.n))))
t = time.perf_counter()
g = pk.build_vamana(pk.PointSet(data), R=w.R, L_build=w.L, alpha=w.alpha, seed=0)
adj_g, deg_g = g.graph.adjacency, g.graph.degrees
tg = time.perf_counter() - t
oracle.build()
oracle.set_num_threads(os.cpu_count() or 1)
t = time.perf_counter()
adj_o, deg_o, _ = oracle.build_vamana(data, R=w.R, L_build=w.L, alpha=w.alpha, seed=0)
to = time.perf_counter() - t
print(f"{name} n={n}: GPU build {tg:.2f} s, oracle build {to:.1f} s ({os.cpu_count()} threads); "
      f"degrees identical {np.array_equal(deg_g, deg_o)}, adjacency identical {np.array_equal(adj_g, adj_o)}; "
      f"max degree {int(deg_o.max())}")
