"""GPU-idle time per pipeline stage at C2: stage wall time (synchronised)
minus the event-timed kernels launched in that stage."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, cluster, workloads  # noqa: E402
from paper_2312_03940_b200.cluster import run_pipeline_device  # noqa: E402

data, _ = workloads.generate("C2")
kw = workloads.pipeline_args("C2", pk)
p = pk.PointSet(data)
for _ in range(3):
    run_pipeline_device(p, **kw)
torch.cuda.synchronize()
_lib.prof_only([])
for rep in range(3):
    _lib.prof_collect(reset=True)
    _lib.prof_enable(True)
    out = run_pipeline_device(p, **kw)
    torch.cuda.synchronize()
    _lib.prof_enable(False)
    prof = _lib.prof_collect(reset=True)
    tot = sum(v[1] for v in prof.values())
    launches = sum(v[0] for v in prof.values())
    st = {k: round(v * 1e3, 2) for k, v in out["timings"].items()}
    print(f"stages {st} sum {sum(st.values()):.2f} ms; kernels {tot:.2f} ms over {launches} launches")
    print(sorted(((k, v[0], round(v[1], 3)) for k, v in prof.items()), key=lambda x: -x[2])[:40])
