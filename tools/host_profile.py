"""Host-side profile (cProfile) of the C2 pipeline's dependent and policy
stages, after warm-up: where the Python orchestration spends its time."""
import cProfile
import os
import pstats
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import cluster, dependent, workloads  # noqa: E402
from paper_2312_03940_b200.cluster import run_pipeline_device  # noqa: E402

data, _ = workloads.generate("C2")
kw = workloads.pipeline_args("C2", pk)
p = pk.PointSet(data)
for _ in range(3):
    run_pipeline_device(p, **kw)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    run_pipeline_device(p, **kw)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
