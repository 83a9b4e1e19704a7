"""Large-L beam kNN vs the oracle on a C3-shaped instance (doubling-round widths)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, vamana, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
data, _ = workloads.generate("C3", n=n, components=max(1, n // 1000))
p = pk.PointSet(data)
idx = pk.build_vamana(p, R=64, L_build=128, alpha=1.1, seed=0, query_beam=128)
g = idx.graph
adj, deg, st = g.adjacency, g.degrees, g.start_points
rng = np.random.default_rng(1)
q = np.sort(rng.choice(n, 64, replace=False)).astype(np.int64)
for L in (256, 512, 1024, 2048, 4096):
    t = time.time()
    ids, sqd, cnt = vamana.beam_knn_raw(g, _lib.to_dev(q), L, L)
    ids, sqd, cnt = _lib.to_host(ids), _lib.to_host(sqd), _lib.to_host(cnt)
    tg = time.time() - t
    t = time.time()
    oi, od, oc = oracle.beam_knn_batch(data, adj, deg, st, q, L, L)
    to = time.time() - t
    print(f"L={L}: gpu {tg:.2f}s oracle {to:.2f}s  short gpu={int((cnt < min(L, n - 1)).sum())} "
          f"short oracle={int((oc < min(L, n - 1)).sum())}  ids equal={np.array_equal(ids, oi)} "
          f"sqd equal={np.array_equal(sqd, od)} counts equal={np.array_equal(cnt, oc)}", flush=True)
