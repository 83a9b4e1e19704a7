"""Pipeline passes of a configuration for ncu captures (the last pass is the
one to capture; earlier passes warm up).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/profile_step.py C2
    ncu --set full -k regex:build_search -s 33 -c 1 python tools/profile_step.py C2   # largest batch, 2nd run
    python tools/profile_step.py C5 1      # one pass only
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import workloads  # noqa: E402
from paper_2312_03940_b200.cluster import run_pipeline_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 2
data, _ = workloads.generate(name)
kw = workloads.pipeline_args(name, pk)
p = pk.PointSet(data)
for _ in range(passes):
    out = run_pipeline_device(p, **kw)
torch.cuda.synchronize()
print({k: round(v * 1e3, 2) for k, v in out["timings"].items()})
