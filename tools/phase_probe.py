"""Per-phase cycle split of the beam walk on a configuration (needs a library
built with -DPK_PHASE_TIMERS, e.g.
    tools/variant.sh Makefile 's/-Xptxas -v$/-Xptxas -v -DPK_PHASE_TIMERS/' python tools/phase_probe.py C5
).  Prints the build searches' and the knn_all searches' split."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, workloads  # noqa: E402

NAMES = ["expand", "prefetch", "screens", "resolve", "merge", "emit", "seeding", "-"]


def read(reset=True, fn="pk_phase_timers"):
    buf = (ctypes.c_ulonglong * 8)()
    getattr(_lib.lib(), fn)(buf, 1 if reset else 0)
    return np.array(list(buf), dtype=np.float64)


def show(tag, v):
    spec = int(v[7])
    v = v.copy()
    v[7] = 0
    if spec:
        print(tag, f"speculative row requests: {spec & 0xffffffff} predictions, {spec >> 32} hits")
    tot = v.sum()
    if tot == 0:
        print(tag, "no timers (library built without -DPK_PHASE_TIMERS)")
        return
    print(tag, "  ".join(f"{n} {100 * x / tot:.1f}%" for n, x in zip(NAMES, v) if x), f"(total {tot:.3e} warp-cycles)")


name = sys.argv[1] if len(sys.argv) > 1 else "C5"
w = workloads.WORKLOADS[name]
data, _ = workloads.generate(name)
p = pk.PointSet(data)
for rep in range(2):
    read()
    read(fn="pk_phase_timers_build")
    read(fn="pk_phase_timers_prune")
    idx = pk.build_vamana(p, R=w.R, L_build=w.L, alpha=w.alpha, seed=0, query_beam=w.L)
    torch.cuda.synchronize()
    b = read(fn="pk_phase_timers_build")
    idx.knn_batch_device(torch.arange(p.n, dtype=torch.int64, device="cuda"), w.k)
    torch.cuda.synchronize()
    q = read()
pr = read(fn="pk_phase_timers_prune")
if pr.sum():
    names = ["cand+sort", "norms", "gram", "epilogue", "greedy", "output"]
    tot = pr[:6].sum()
    print("tc build prune:", "  ".join(f"{n} {100 * x / tot:.1f}%" for n, x in zip(names, pr[:6])),
          f"(total {tot:.3e} block-cycles, {int(pr[7])} items, {pr[6] / max(1, pr[7]):.2f} exact pair decisions per item,"
          f" {tot / max(1, pr[7]) / 1.965e3:.1f} us per item)")
show("build searches:", b)
show("knn_all:", q)
