"""Distinct vs total distance evaluations of one pipeline pass (the kernels'
counting mode, as bench.py's untimed pass) under environment settings:

    python tools/count_probe.py C5 PK_START_SKIP=0 PK_START_SKIP=1
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import workloads  # noqa: E402

name = sys.argv[1]
data, _ = workloads.generate(name)
kw = workloads.pipeline_args(name, pk)
p = pk.PointSet(data)
for setting in sys.argv[2:] or ["-"]:
    if "=" in setting:
        k, v = setting.split("=", 1)
        os.environ[k] = v
    c, _ = bench.counting_pass(p, kw, None)
    bx = c["build_evals"] / max(1, c["build_unique"]) - 1
    qx = c["beam_evals"] / max(1, c["beam_unique"]) - 1
    print(setting, c, f"build redundant {100 * bx:.2f}%  beam redundant {100 * qx:.2f}%", flush=True)
