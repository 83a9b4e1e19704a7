"""A/B timing of an environment switch on a configuration sample: per-kernel
times of one pipeline pass with VAR=a and VAR=b (second pass of each).

    python tools/ab_env.py C5 200000 PK_PREFETCH_ROWS 0 1
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, workloads  # noqa: E402
from paper_2312_03940_b200.cluster import run_pipeline_device  # noqa: E402

name, n, var, vals = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4:]
w = workloads.WORKLOADS[name]
comps = max(1, int(round(w.components * n / w.n)))
data, _ = workloads.generate(name, n=n, components=comps)
kw = workloads.pipeline_args(name, pk, n_centers=min(w.n_centers, comps))
p = pk.PointSet(data)
for v in vals * 2:
    os.environ[var] = v
    _lib.prof_collect(reset=True)
    _lib.prof_only([])
    _lib.prof_enable(True)
    out = run_pipeline_device(p, **kw)
    torch.cuda.synchronize()
    _lib.prof_enable(False)
    prof = _lib.prof_collect(reset=True)
    top = sorted(prof.items(), key=lambda kv: -kv[1][1])[:5]
    print(f"{var}={v}: stages { {k: round(x * 1e3, 1) for k, x in out['timings'].items()} } "
          f"{[(k, round(t[1], 1)) for k, t in top]}", flush=True)
