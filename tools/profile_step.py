"""One C2 pipeline pass for profilers (ncu): no warm-up, no CPU baseline.

    python tools/profile_step.py [--config C2] [--n N] [--runs R]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--runs", type=int, default=1)
    a = ap.parse_args()
    import torch

    import paper_2312_03940_b200 as pk
    from paper_2312_03940_b200 import workloads
    from paper_2312_03940_b200.cluster import run_pipeline_device
    from paper_2312_03940_b200.core import upload_points

    w = workloads.WORKLOADS[a.config]
    n = a.n or w.n
    comps = w.components if a.n is None else max(1, int(round(w.components * n / w.n)))
    data, _ = workloads.generate(a.config, n=n, components=comps)
    p = pk.PointSet(data).attach_device(upload_points(data))
    kw = workloads.pipeline_args(a.config, pk, n_centers=min(w.n_centers, comps))
    for _ in range(a.runs):
        out = run_pipeline_device(p, **kw)
    torch.cuda.synchronize()
    print({k: round(v * 1e3, 2) for k, v in out["timings"].items()})


if __name__ == "__main__":
    main()
