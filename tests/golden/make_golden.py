"""Generate golden vectors by running the REFERENCE implementation itself.

    python tests/golden/make_golden.py          (build container only)

Loads /root/reference/pkg/src/peakann as `peakann_ref` and records its
outputs on seeded inputs into tests/golden/*.npz.  The fixtures pin both the
CPU oracle (tests/test_oracle.py) and the CUDA path (tests/test_parity_gpu.py)
on the GPU box, where /root/reference does not exist.  Inputs are either
stored inline (small cases) or regenerated from a seed by
paper_2312_03940_b200.workloads / numpy default_rng.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

from refload import load_reference  # noqa: E402

from paper_2312_03940_b200 import workloads  # noqa: E402

FIG_COORDS = np.array([[5, 1], [4, 3], [4, 2], [1, 2], [1, 0], [0, 3]], dtype=np.float32)


def digest(a) -> str:
    """sha256 of an array's canonical little-endian bytes (dtype + shape included)."""
    a = np.ascontiguousarray(a)
    h = hashlib.sha256(f"{a.dtype.str}{a.shape}".encode())
    h.update(a.tobytes())
    return h.hexdigest()


def save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}: {os.path.getsize(path) / 1024:.1f} KiB")


def random_sets():
    """(tag, data) small inputs shared by the brute / graph cases."""
    out = []
    for seed, n, d in [(0, 50, 8), (1, 120, 2), (2, 300, 32), (3, 500, 4)]:
        out.append((f"normal_{seed}", np.random.default_rng(seed).standard_normal((n, d)).astype(np.float32)))
    out.append(("grid", np.random.default_rng(37).integers(0, 6, size=(200, 3)).astype(np.float32)))
    dup = np.random.default_rng(77).standard_normal((300, 16)).astype(np.float32)
    dup[13] = dup[40]
    out.append(("dup", dup))
    out.append(("zeros", np.zeros((5, 3), np.float32)))
    return out


def gen_brute(pk, K):
    arrays = {}
    for tag, data in random_sets():
        n = data.shape[0]
        arrays[f"{tag}__data"] = data
        for k in (1, 5, 16, n + 3) if n <= 120 else (1, 5, 16):
            ids, sqd = K.brute_knn_batch(data, np.arange(n, dtype=np.int64), k)
            arrays[f"{tag}__k{k}__ids"] = ids
            arrays[f"{tag}__k{k}__sqd"] = sqd
        q = np.linspace(-1, 1, data.shape[1]).astype(np.float64)
        ids, sqd = K.brute_knn_vector(data, q, 7)
        arrays[f"{tag}__vec__q"] = q
        arrays[f"{tag}__vec__ids"] = ids
        arrays[f"{tag}__vec__sqd"] = sqd
    save("brute", **arrays)


GRAPH_CASES = [
    # tag, generator, R, L_build, alpha, seed, num_starts, medoid
    ("g300", lambda: np.random.default_rng(4).standard_normal((300, 6)).astype(np.float32), 8, 12, 1.1, 7, None, False),
    ("g500a1", lambda: np.random.default_rng(21).standard_normal((500, 8)).astype(np.float32), 10, 16, 1.0, 0, None, False),
    ("gauss2k", lambda: workloads.generate("C1", n=2000, components=5)[0][:, :32].copy(), 32, 32, 1.1, 3, None, False),
    ("sift3k", lambda: workloads.generate("C2", n=3000, components=10)[0][:, :16].copy(), 16, 24, 1.1, 5, None, False),
    ("medoid", lambda: np.random.default_rng(9).standard_normal((80, 4)).astype(np.float32), 6, 10, 1.1, 1, None, True),
    ("onestart", lambda: np.random.default_rng(55).standard_normal((40, 3)).astype(np.float32), 4, 6, 1.05, 11, 1, False),
    ("tiny", lambda: np.arange(10, dtype=np.float32).reshape(5, 2), 8, 8, 1.0, 0, 2, False),
]


def gen_graphs(pk, K):
    arrays = {}
    for tag, make, R, L, alpha, seed, ns, medoid in GRAPH_CASES:
        data = make()
        p = pk.PointSet(data)
        t = time.perf_counter()
        idx = pk.build_vamana(p, R=R, L_build=L, alpha=alpha, num_starts=ns, seed=seed, medoid_start=medoid)
        g = idx.graph
        arrays[f"{tag}__data"] = data
        arrays[f"{tag}__params"] = np.array([R, L, seed, -1 if ns is None else ns, int(medoid)], np.int64)
        arrays[f"{tag}__alpha"] = np.array([alpha])
        arrays[f"{tag}__adj"] = g.adjacency
        arrays[f"{tag}__deg"] = g.degrees
        arrays[f"{tag}__starts"] = g.start_points
        n = p.n
        qids = np.arange(0, n, 1 if n <= 500 else 7, dtype=np.int64)
        arrays[f"{tag}__qids"] = qids
        for Lq, k in [(L, min(8, n)), (max(L, 16), 16), (64, 64)]:
            ids, sqd, counts = K.beam_knn_batch(data, g.adjacency, g.degrees, g.start_points, qids, Lq, k)
            arrays[f"{tag}__beam_L{Lq}_k{k}__ids"] = ids
            arrays[f"{tag}__beam_L{Lq}_k{k}__sqd"] = sqd
            arrays[f"{tag}__beam_L{Lq}_k{k}__counts"] = counts
        nb = idx.knn_batch(qids, 5)
        arrays[f"{tag}__knn5__ids"] = nb.ids
        arrays[f"{tag}__knn5__dists"] = nb.dists
        q = data[n // 2].astype(np.float64) + 0.25
        ci, cd, vi, vd = K.beam_search_single(data, g.adjacency, g.degrees, g.start_points, q, L)
        arrays[f"{tag}__single__q"] = q
        arrays[f"{tag}__single__cand_ids"] = ci
        arrays[f"{tag}__single__cand_sqd"] = cd
        arrays[f"{tag}__single__vis_ids"] = vi
        arrays[f"{tag}__single__vis_sqd"] = vd
        print(f"  graph {tag} n={n} built in {time.perf_counter() - t:.2f}s")
    save("graphs", **arrays)


def gen_prune(pk, K):
    arrays = {}
    rng = np.random.default_rng(0)
    data = rng.standard_normal((40, 4)).astype(np.float32)
    arrays["data"] = data
    for case, (p, alpha, R, ncur) in enumerate([(0, 1.1, 6, 0), (3, 1.0, 3, 2), (7, 2.0, 10, 3), (11, 1.3, 40, 5)]):
        cand = np.array([j for j in range(40) if j != p][::2], np.int64)
        sqd = np.array([K.point_sqdist(data, p, int(j)) for j in cand])
        sqd_from_dist = np.sqrt(sqd) ** 2  # what robust_prune passes (vamana.py:101)
        cur = np.arange(1, 1 + 3 * ncur, 3, dtype=np.int64)[:ncur]
        out = K.robust_prune_standalone(data, p, cand, sqd_from_dist, cur, alpha, R)
        arrays[f"c{case}__args"] = np.array([p, R, ncur], np.int64)
        arrays[f"c{case}__alpha"] = np.array([alpha])
        arrays[f"c{case}__cand"] = cand
        arrays[f"c{case}__cand_sqd"] = sqd_from_dist
        arrays[f"c{case}__cur"] = cur
        arrays[f"c{case}__out"] = out
    line = np.array([[0.0], [1.0], [2.0], [4.0]], np.float32)
    arrays["line"] = line
    arrays["line_centroid"] = np.array([K.nearest_to_centroid(line)])
    save("prune", **arrays)


def _run(pk, data, **kw):
    t = time.perf_counter()
    res = pk.run_pipeline(pk.PointSet(data), **kw)
    return res, time.perf_counter() - t


def _pack_digest(res, arrays, sample=1000):
    """Large configurations: full digests + the first `sample` rows in clear."""
    st = res.state
    full = dict(rho=st.rho, lam=st.lam, delta=st.delta, nbr_ids=st.neighbors.ids, nbr_dists=st.neighbors.dists,
                labels=res.clustering.labels, centers=res.clustering.centers, noise=res.clustering.noise)
    for key, val in full.items():
        arrays[f"digest__{key}"] = np.array(digest(val))
        arrays[f"head__{key}"] = val[:sample]
    arrays["labels"] = res.clustering.labels
    arrays["lam"] = st.lam


def _pack(prefix, res, arrays):
    st = res.state
    arrays[f"{prefix}__rho"] = st.rho
    arrays[f"{prefix}__lam"] = st.lam
    arrays[f"{prefix}__delta"] = st.delta
    arrays[f"{prefix}__nbr_ids"] = st.neighbors.ids
    arrays[f"{prefix}__nbr_dists"] = st.neighbors.dists
    arrays[f"{prefix}__labels"] = res.clustering.labels
    arrays[f"{prefix}__centers"] = res.clustering.centers
    arrays[f"{prefix}__noise"] = res.clustering.noise


def gen_pipelines(pk, K):
    arrays = {}
    # the paper's running example (test_acceptance.py:35-54)
    res, _ = _run(pk, FIG_COORDS, index_config=pk.BruteForceConfig(), k=1, density_kind="kth",
                  center_policy=pk.ThresholdCenter(2.5), noise_policy=pk.NoisePolicy(1 / np.sqrt(2.0)),
                  doubling_params=pk.DoublingParams(initial_k=2, threshold=0))
    _pack("fig", res, arrays)
    kinds = ["kth", "kth_normalized", "exp_sum", "sum_exp", "sum"]
    policies = ["threshold", "product", "local"]
    for trial in range(15):
        rng = np.random.default_rng(9000 + trial)
        d = [2, 8, 32][trial % 3]
        n = int(rng.integers(30, 400))
        kind = kinds[trial % 5]
        pol = policies[trial % 3]
        data = rng.standard_normal((n, d)).astype(np.float32) * (1 + (trial % 4))
        if trial % 4 == 0:
            data[n // 2] = data[n // 3]
        k = int(rng.choice([1, 2, 5, 16]))
        if pol == "threshold":
            cp = pk.ThresholdCenter(float(rng.uniform(0.5, 2.0)))
            pol_arr = np.array([0, 0]), float(cp.delta_min)
        elif pol == "product":
            cp = pk.ProductCenter(int(rng.integers(1, 7)))
            pol_arr = np.array([1, cp.n_clusters]), 0.0
        else:
            cp = pk.LocalCenter()
            pol_arr = np.array([2, 0]), 0.0
        vam = trial % 2 == 1
        icfg = pk.VamanaConfig(R=8, L_build=12, L=12, alpha=1.1, seed=trial) if vam else pk.BruteForceConfig()
        thr = int(rng.choice([0, 10, 300]))
        res, _ = _run(pk, data, index_config=icfg, k=k, density_kind=kind, center_policy=cp,
                      noise_policy=pk.NoisePolicy(0.0), doubling_params=pk.DoublingParams(initial_k=2 * k, threshold=thr))
        pre = f"t{trial}"
        arrays[f"{pre}__data"] = data
        arrays[f"{pre}__meta"] = np.array([k, int(vam), thr, kinds.index(kind), pol_arr[0][0], pol_arr[0][1]], np.int64)
        arrays[f"{pre}__fmeta"] = np.array([pol_arr[1]])
        _pack(pre, res, arrays)
    save("pipelines", **arrays)


def gen_config(pk, name, n, comps, tag, brute=False):
    data, truth = workloads.generate(name, n=n, components=comps)
    kw = workloads.pipeline_args(name, pk, n_centers=comps, brute=brute)
    res, secs = _run(pk, data, **kw)
    arrays = {"meta": np.array([n, comps], np.int64), "seconds": np.array([secs])}
    _pack_digest(res, arrays)
    if not brute:
        # rebuild to capture the graph (same seed -> identical graph)
        w = workloads.WORKLOADS[name]
        idx = pk.build_vamana(pk.PointSet(data), R=w.R, L_build=w.L, alpha=w.alpha, seed=0, query_beam=w.L)
        g = idx.graph
        arrays["digest__adj"] = np.array(digest(g.adjacency))
        arrays["digest__deg"] = np.array(digest(g.degrees))
        arrays["head__adj"] = g.adjacency[:1000]
        arrays["deg"] = g.degrees
        arrays["starts"] = g.start_points
    arrays["ari_truth"] = np.array([pk.ari(res.clustering.labels, truth)])
    print(f"  {tag}: reference run_pipeline {secs:.1f}s timings={res.timings}")
    save(tag, **arrays)


def main():
    pk = load_reference()
    from peakann_ref import _kernels as K

    which = sys.argv[1:] or ["brute", "graphs", "prune", "pipelines", "c1", "c1brute", "c2s", "c3s"]
    if "brute" in which:
        gen_brute(pk, K)
    if "graphs" in which:
        gen_graphs(pk, K)
    if "prune" in which:
        gen_prune(pk, K)
    if "pipelines" in which:
        gen_pipelines(pk, K)
    if "c1" in which:
        gen_config(pk, "C1", 10_000, 10, "c1")
    if "c1brute" in which:
        gen_config(pk, "C1", 4_000, 10, "c1brute", brute=True)
    if "c2s" in which:
        gen_config(pk, "C2", 20_000, 20, "c2s")
    if "c3s" in which:
        gen_config(pk, "C3", 30_000, 300, "c3s")


if __name__ == "__main__":
    main()
