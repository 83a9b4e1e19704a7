"""Scale check of the float-data kernels added this round: the full pipeline
with lazy beam keys + tensor-core RobustPrune (default) against the eager
float64 searches + warp prune (PK_LAZY=0 PK_TC_PRUNE=0) on a BASELINE
generator sample; every output must be bit-identical.  Also reports the ANN
kNN recall@k against exact rows for a sample of queries (identical rows imply
the reference's recall).

    python tools/check_float_paths.py C5 200000
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, index, workloads  # noqa: E402
from paper_2312_03940_b200.cluster import run_pipeline_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
w = workloads.WORKLOADS[name]
comps = max(1, int(round(w.components * n / w.n)))
data, truth = workloads.generate(name, n=n, components=comps)
kw = workloads.pipeline_args(name, pk, n_centers=min(w.n_centers, comps))
p = pk.PointSet(data)
outs = {}
for tag, env in (("fast", {"PK_LAZY": "1", "PK_TC_PRUNE": "1"}), ("eager", {"PK_LAZY": "0", "PK_TC_PRUNE": "0"})):
    os.environ.update(env)
    run_pipeline_device(p, **kw)  # warm-up
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = run_pipeline_device(p, **kw)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    outs[tag] = {k: _lib.to_host(out[k]) for k in ("ids", "dists", "rho", "lam", "delta", "labels")}
    print(f"{name} n={n} {tag}: {el:.3f} s, stages { {k: round(v, 3) for k, v in out['timings'].items()} }",
          flush=True)
same = {k: bool(np.array_equal(outs["fast"][k], outs["eager"][k])) for k in outs["fast"]}
print("bit-identical:", same)
# recall@k of the ANN rows against exact rows (tensor-core exact kNN) on 2,000 queries
rng = np.random.default_rng(0)
q = np.sort(rng.choice(n, 2000, replace=False)).astype(np.int64)
ids_e, _ = index.brute_device(p, _lib.to_dev(q), w.k)
ids_e = _lib.to_host(ids_e)
ids_a = outs["fast"]["ids"][q]
rec = np.mean([len(np.intersect1d(a, b)) / w.k for a, b in zip(ids_a, ids_e)])
print(f"recall@{w.k} of knn_all (2,000 sampled queries): {rec:.4f}; ARI vs generator {pk.ari(outs['fast']['labels'], truth):.5f}")
