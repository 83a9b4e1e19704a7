"""C3 pipeline with the u8 tensor-core count scan vs the CUDA-core scan
(PK_U8_TC_SCAN=0): lambda / delta / labels must be identical."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, workloads  # noqa: E402
from paper_2312_03940_b200.cluster import run_pipeline_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
w = workloads.WORKLOADS["C3"]
data, _ = workloads.generate("C3", n=n, components=max(1, int(round(w.components * n / w.n))))
kw = workloads.pipeline_args("C3", pk)
p = pk.PointSet(data)
res = {}
for flag in ("1", "0", "1"):
    os.environ["PK_U8_TC_SCAN"] = flag
    _lib.prof_collect(reset=True)
    _lib.prof_only([])
    _lib.prof_enable(True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = run_pipeline_device(p, **kw)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    _lib.prof_enable(False)
    prof = _lib.prof_collect(reset=True)
    res[flag] = [_lib.to_host(out[k]) for k in ("lam", "delta", "labels")]
    sc = {k: round(v[1], 1) for k, v in prof.items() if "count" in k or "scan" in k}
    print(f"PK_U8_TC_SCAN={flag}: {el:.3f} s, dependent {out['timings']['dependent']:.3f} s, {sc}", flush=True)
print("identical:", all(np.array_equal(a, b) for a, b in zip(res["0"], res["1"])))
