"""Full-size C4 / C5 (or any config) checked against the CPU oracle on samples
and on the parts the oracle can afford at full scale:

  1. beam kNN rows of 500 sampled queries: oracle.beam_knn_batch (+ its exact
     fallback for short rows) on the GPU-built graph == the GPU's rows;
  2. exact rows of 256 sampled queries (oracle.brute_knn_batch): recall@k of
     the GPU rows and of the oracle's beam rows against them (north_star:
     ANN recall >= the reference's);
  3. the whole dependent stage replayed by the oracle (oracle.dependents:
     phase 1, every doubling round with beam searches on the GPU graph, the
     exact dp scan of the stragglers) from the GPU's rho and kNN rows == the
     GPU's lam / delta for all n points;
  4. oracle.apply_policies on the GPU's rho / lam / delta == the GPU's labels,
     centers and noise; ARI of both against the generator labels;
  5. with `brute`: the exact (BruteForceIndex) kNN of 256 sampled queries on
     the GPU's tensor-core path == oracle.brute_knn_batch.

    python tools/check_full_sampled.py C5 [brute]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, index, workloads  # noqa: E402
from paper_2312_03940_b200.cluster import run_pipeline_device  # noqa: E402


def say(*a):
    print(*a, flush=True)


name = sys.argv[1]
brute = len(sys.argv) > 2 and sys.argv[2] == "brute"
w = workloads.WORKLOADS[name]
oracle.build()
oracle.set_num_threads(os.cpu_count() or 1)
t = time.time()
data, truth = workloads.generate(name)
n = data.shape[0]
say(f"{name}: n={n} d={w.d} generated in {time.time() - t:.1f}s; oracle threads {oracle.num_threads()}")
kw = workloads.pipeline_args(name, pk)
p = pk.PointSet(data)
t = time.time()
out = run_pipeline_device(p, **kw)
torch.cuda.synchronize()
say(f"GPU pipeline {time.time() - t:.2f}s stages {{{', '.join(f'{k}: {v:.3f}' for k, v in out['timings'].items())}}}")
g = out["index"].graph
adj, deg, starts = g.adjacency, g.degrees, g.start_points
ids, dists = _lib.to_host(out["ids"]), _lib.to_host(out["dists"])
rho, lam, delta = _lib.to_host(out["rho"]), _lib.to_host(out["lam"]), _lib.to_host(out["delta"])
labels = _lib.to_host(out["labels"])
rng = np.random.default_rng(2026)
ok = True

# 1. beam rows of sampled queries on the GPU graph
q = np.sort(rng.choice(n, 500, replace=False)).astype(np.int64)
t = time.time()
oi, od = oracle.GraphIndexOracle(data, adj, deg, starts, w.L).knn_batch(q, w.k)
same_ids, same_d = np.array_equal(oi, ids[q]), np.array_equal(od, dists[q])
ok &= same_ids and same_d
say(f"[1] beam rows of 500 sampled queries (L={w.L}, k={w.k}) on the GPU graph: ids equal {same_ids}, "
    f"dists equal {same_d} ({time.time() - t:.1f}s)")

# 2. recall against exact rows
qe = q[:256]
t = time.time()
ei, _ = oracle.brute_knn_batch(data, qe, w.k)
rec_gpu = np.mean([len(set(ids[x]) & set(ei[j])) / w.k for j, x in enumerate(qe)])
rec_orc = np.mean([len(set(oi[j]) & set(ei[j])) / w.k for j in range(len(qe))])
say(f"[2] recall@{w.k} vs exact rows of 256 sampled queries: GPU {rec_gpu:.4f}, oracle {rec_orc:.4f} "
    f"({time.time() - t:.1f}s)")

# 3. dependent stage replayed by the oracle from the GPU's rho and rows
t = time.time()
trace = []
dp = kw["doubling_params"]
idx = oracle.GraphIndexOracle(data, adj, deg, starts, w.L)
olam, odelta = oracle.dependents(idx, data, rho, ids, dists, dp.initial_k, dp.threshold, trace)
eq_l, eq_d = np.array_equal(olam, lam), np.array_equal(odelta, delta)
ok &= eq_l and eq_d
say(f"[3] oracle dependents from the GPU rho / rows (rounds {trace}): lam equal {eq_l}, delta equal {eq_d} "
    f"for all {n} points ({time.time() - t:.1f}s)")

# 4. policies + labels
t = time.time()
olab, ocen, onoi = oracle.apply_policies(rho, olam, odelta, ids, ("product", w.n_centers), 0.0)
eq_lab = np.array_equal(olab, labels)
ok &= eq_lab
say(f"[4] oracle apply_policies: labels equal {eq_lab}; centers {ocen.shape[0]}, noise {onoi.shape[0]}; "
    f"ARI vs generator: GPU {pk.ari(labels, truth):.6f}, oracle {pk.ari(olab, truth):.6f} ({time.time() - t:.1f}s)")

if brute:
    t = time.time()
    qt = _lib.to_dev(qe)
    bi, bs = index.brute_device(p, qt, w.k)
    bi, bs = _lib.to_host(bi), _lib.to_host(bs)
    ebi, ebs = oracle.brute_knn_batch(data, qe, w.k)
    eq = np.array_equal(bi, ebi) and np.array_equal(bs, ebs)
    ok &= eq
    say(f"[5] exact kNN (BruteForceIndex, tensor-core path) of 256 sampled queries == oracle brute rows: {eq} "
        f"({time.time() - t:.1f}s)")
say("ALL EQUAL" if ok else "MISMATCH")
