"""Diagnose per-step variance of the C2 timed loop: device-event step time,
sum of event-timed kernels, host wall time, per step."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, workloads  # noqa: E402
from paper_2312_03940_b200.cluster import run_pipeline_device  # noqa: E402
from paper_2312_03940_b200.core import upload_points  # noqa: E402

data, _ = workloads.generate("C2")
kw = workloads.pipeline_args("C2", pk)
p = pk.PointSet(data).attach_device(upload_points(data))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    run_pipeline_device(p, **kw)
torch.cuda.synchronize()
if os.environ.get("PROBE_SLEEP"):
    time.sleep(float(os.environ["PROBE_SLEEP"]))
if os.environ.get("PROBE_EXTRA"):
    for _ in range(int(os.environ["PROBE_EXTRA"])):
        run_pipeline_device(p, **kw)
    torch.cuda.synchronize()
_lib.prof_collect(reset=True)
_lib.prof_only([])
_lib.prof_enable(True)
st = torch.cuda.current_stream()
for i in range(8):
    flush.fill_(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record(st)
    out = run_pipeline_device(p, **kw)
    e1.record(st)
    torch.cuda.synchronize()
    h1 = time.perf_counter()
    prof = _lib.prof_collect(reset=True)
    ksum = sum(v[1] for v in prof.values())
    top = sorted(prof.items(), key=lambda kv: -kv[1][1])[:3]
    print(f"step {i}: events {e0.elapsed_time(e1):.2f} ms host {1e3 * (h1 - h0):.2f} kernels {ksum:.2f} "
          f"{[(k, round(v[1], 2)) for k, v in top]}", flush=True)
