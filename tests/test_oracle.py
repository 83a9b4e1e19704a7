"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import hashlib
import warnings

import numpy as np
import pytest

from conftest import FIG_COORDS, golden

import oracle
from paper_2312_03940_b200 import workloads


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256(f"{a.dtype.str}{a.shape}".encode())
    h.update(a.tobytes())
    return h.hexdigest()


def _tags(z, suffix):
    return sorted({k.split("__")[0] for k in z.files if k.endswith(suffix)})


def test_brute_knn_matches_reference():
    z = golden("brute")
    for tag in _tags(z, "__data"):
        data = z[f"{tag}__data"]
        n = data.shape[0]
        for key in z.files:
            if key.startswith(f"{tag}__k") and key.endswith("__ids"):
                k = int(key.split("__")[1][1:])
                ids, sqd = oracle.brute_knn_batch(data, np.arange(n), k)
                assert np.array_equal(ids, z[key]), (tag, k)
                assert np.array_equal(sqd, z[key.replace("__ids", "__sqd")]), (tag, k)
        ids, sqd = oracle.brute_knn_vector(data, z[f"{tag}__vec__q"], 7)
        assert np.array_equal(ids, z[f"{tag}__vec__ids"])
        assert np.array_equal(sqd, z[f"{tag}__vec__sqd"])


def test_build_and_beam_match_reference():
    z = golden("graphs")
    for tag in _tags(z, "__adj"):
        data = z[f"{tag}__data"]
        R, L, seed, ns, medoid = (int(v) for v in z[f"{tag}__params"])
        alpha = float(z[f"{tag}__alpha"][0])
        adj, deg, starts = oracle.build_vamana(data, R, L, alpha, None if ns < 0 else ns, seed, bool(medoid))
        assert np.array_equal(starts, z[f"{tag}__starts"]), tag
        assert np.array_equal(deg, z[f"{tag}__deg"]), tag
        assert np.array_equal(adj, z[f"{tag}__adj"]), tag
        qids = z[f"{tag}__qids"]
        for key in z.files:
            if key.startswith(f"{tag}__beam_") and key.endswith("__ids"):
                _, spec, _ = key.split("__")
                Lq, k = (int(x[1:]) for x in spec.split("_")[1:])
                ids, sqd, counts = oracle.beam_knn_batch(data, adj, deg, starts, qids, Lq, k)
                pre = key[: -len("__ids")]
                assert np.array_equal(ids, z[pre + "__ids"]), key
                assert np.array_equal(sqd, z[pre + "__sqd"]), key
                assert np.array_equal(counts, z[pre + "__counts"]), key
        gi = oracle.GraphIndexOracle(data, adj, deg, starts, L)
        ids, dists = gi.knn_batch(qids, 5)
        assert np.array_equal(ids, z[f"{tag}__knn5__ids"])
        assert np.array_equal(dists, z[f"{tag}__knn5__dists"])
        ci, cd, vi, vd = oracle.beam_search_single(data, adj, deg, starts, z[f"{tag}__single__q"], L)
        assert np.array_equal(ci, z[f"{tag}__single__cand_ids"])
        assert np.array_equal(cd, z[f"{tag}__single__cand_sqd"])
        assert np.array_equal(vi, z[f"{tag}__single__vis_ids"])
        assert np.array_equal(vd, z[f"{tag}__single__vis_sqd"])


def test_prune_matches_reference():
    z = golden("prune")
    data = z["data"]
    for c in range(4):
        p, R, _ = (int(v) for v in z[f"c{c}__args"])
        out = oracle.robust_prune(data, p, z[f"c{c}__cand"], z[f"c{c}__cand_sqd"], z[f"c{c}__cur"],
                                  float(z[f"c{c}__alpha"][0]), R)
        assert np.array_equal(out, z[f"c{c}__out"]), c
    assert oracle.nearest_to_centroid(z["line"]) == int(z["line_centroid"][0])


KINDS = ["kth", "kth_normalized", "exp_sum", "sum_exp", "sum"]


def _policy(meta, fmeta):
    code, arg = int(meta[4]), int(meta[5])
    return [("threshold", float(fmeta[0])), ("product", arg), ("local", None)][code]


def test_small_pipelines_match_reference():
    z = golden("pipelines")
    fig = oracle.pipeline(FIG_COORDS, index="brute", k=1, density_kind="kth",
        center_policy=("threshold", 2.5), rho_min=1 / np.sqrt(2.0), initial_k=2, threshold=0)
    for key in ("rho", "lam", "delta", "labels", "centers", "noise"):
        assert np.array_equal(fig[key], z[f"fig__{key}"]), key
    for t in range(15):
        meta = z[f"t{t}__meta"]
        k, vam, thr, kind = int(meta[0]), int(meta[1]), int(meta[2]), KINDS[int(meta[3])]
        with np.errstate(all="ignore"), warnings.catch_warnings():
            warnings.simplefilter("ignore")
            out = oracle.pipeline(z[f"t{t}__data"], index="vamana" if vam else "brute", R=8, L_build=12, L=12,
                                  alpha=1.1, seed=t, k=k, density_kind=kind,
                                  center_policy=_policy(meta, z[f"t{t}__fmeta"]), rho_min=0.0,
                                  initial_k=2 * k, threshold=thr)
        assert np.array_equal(out["nbr_ids"], z[f"t{t}__nbr_ids"]), t
        assert np.array_equal(out["nbr_dists"], z[f"t{t}__nbr_dists"]), t
        assert np.array_equal(out["rho"], z[f"t{t}__rho"]), t
        assert np.array_equal(out["lam"], z[f"t{t}__lam"]), t
        assert np.array_equal(out["delta"], z[f"t{t}__delta"]), t
        assert np.array_equal(out["labels"], z[f"t{t}__labels"]), t


@pytest.mark.parametrize("tag,name,n,comps,brute", [
    ("c1", "C1", 10_000, 10, False),
    ("c1brute", "C1", 4_000, 10, True),
    ("c2s", "C2", 20_000, 20, False),
    ("c3s", "C3", 30_000, 300, False),
])
def test_config_pipelines_match_reference(tag, name, n, comps, brute):
    z = golden(tag)
    data, _ = workloads.generate(name, n=n, components=comps)
    w = workloads.WORKLOADS[name]
    out = oracle.pipeline(data, index="brute" if brute else "vamana", R=w.R, L_build=w.L, L=w.L, alpha=w.alpha,
                          seed=0, k=w.k, density_kind=w.density, center_policy=("product", comps), rho_min=0.0,
                          initial_k=2 * w.k, threshold=0 if brute else 300)
    if not brute:
        assert digest(out["adjacency"]) == str(z["digest__adj"]), "graph differs"
        assert np.array_equal(out["degrees"], z["deg"])
        assert np.array_equal(out["starts"], z["starts"])
    for key in ("nbr_ids", "nbr_dists", "rho", "lam", "delta", "labels", "centers", "noise"):
        assert digest(out[key]) == str(z[f"digest__{key}"]), key
