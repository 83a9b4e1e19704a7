"""Seeding share of a beam kNN pass (PK_SEED_ONLY=1 stops each query after
seeding): C2 knn_all, k=16, L=128."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, vamana, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = workloads.WORKLOADS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else w.n
data, _ = workloads.generate(name, n=n, components=max(1, int(w.components * n / w.n)))
p = pk.PointSet(data)
g = pk.build_vamana(p, R=w.R, L_build=w.L, alpha=w.alpha, seed=0, query_beam=w.L)
q = torch.arange(n, dtype=torch.int64, device="cuda")
for flag in ("0", "1", "0", "1"):
    os.environ["PK_SEED_ONLY"] = flag
    _lib.prof_collect(reset=True)
    _lib.prof_only(["beam_knn_kernel"])
    _lib.prof_enable(True)
    vamana.beam_knn_raw(g.graph, q, w.L, w.k)
    torch.cuda.synchronize()
    _lib.prof_enable(False)
    print(name, "seed_only" if flag == "1" else "full", round(_lib.prof_collect(reset=True)["beam_knn_kernel"][1], 3), "ms")
