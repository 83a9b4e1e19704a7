"""Tensor-core exact kNN vs the float64 SIMT path (both on device)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, index, workloads  # noqa: E402


def run(name, data, k=16, m=None):
    p = pk.PointSet(data)
    n = p.n
    q = torch.arange(n if m is None else m, dtype=torch.int64, device="cuda")
    os.environ["PEAKANN_B200_TC"] = "0"
    torch.cuda.synchronize(); t = time.time()
    ids0, sqd0 = index.brute_device(p, q, k)
    torch.cuda.synchronize(); t0 = time.time() - t
    os.environ["PEAKANN_B200_TC"] = "1"
    index.TC_STATS.update(rows=0, uncertified=0)
    torch.cuda.synchronize(); t = time.time()
    ids1, sqd1 = index.brute_device(p, q, k)
    torch.cuda.synchronize(); t1 = time.time() - t
    same_i = torch.equal(ids0, ids1)
    same_d = torch.equal(sqd0, sqd1)
    bad = (ids0 != ids1).any(dim=1).sum().item()
    print(f"{name}: n={n} d={data.shape[1]} simt {t0:.3f}s tc {t1:.3f}s  ids equal={same_i} sqd equal={same_d} "
          f"rows differing={bad} stats={index.TC_STATS}", flush=True)


x, _ = workloads.generate("C1", n=4000, components=10)
run("C1-4k", x)
x, _ = workloads.generate("C2", n=20000, components=20)
run("C2-20k", x)
x, _ = workloads.generate("C5", n=20000, components=16)
run("C5-20k", x)
x, _ = workloads.generate("C5", n=100000, components=80)
run("C5-100k(1k queries)", x, m=2048)
