"""Tensor-core RobustPrune vs the warp prune on the golden graph cases
(first differing row per case)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_03940_b200 as pk  # noqa: E402

z = np.load(os.path.join(ROOT, "tests/golden/graphs.npz"))
tags = sorted({k.split("__")[0] for k in z.files if k.endswith("__adj")})
for tag in tags:
    data = z[f"{tag}__data"]
    R, L, seed, ns, medoid = (int(v) for v in z[f"{tag}__params"])
    alpha = float(z[f"{tag}__alpha"][0])
    res = {}
    for flag in ("0", os.environ.get("TCF", "1")):
        os.environ["PK_TC_PRUNE"] = flag
        p = pk.PointSet(data)
        g = pk.build_vamana(p, R=R, L_build=L, alpha=alpha, num_starts=None if ns < 0 else ns, seed=seed,
                            medoid_start=bool(medoid))
        res[flag] = (g.graph.adjacency.copy(), g.graph.degrees.copy())
    ref = (z[f"{tag}__adj"], z[f"{tag}__deg"])
    print(tag, data.shape, "warp==ref", np.array_equal(res["0"][0], ref[0]), "tc==ref", np.array_equal(res[flag][0], ref[0]))
    bad = np.nonzero((res[flag][0] != ref[0]).any(axis=1))[0]
    if len(bad):
        i = bad[0]
        print("  rows differing:", len(bad), "first", i, "deg tc", res[flag][1][i], "ref", ref[1][i])
        print("  tc ", res[flag][0][i][:20])
        print("  ref", ref[0][i][:20])
