"""CUDA path vs the reference's golden vectors and the CPU oracle (GPU only).

Bit-exact comparisons everywhere except exp-based densities (exp_sum,
sum_exp), which are compared within 1e-12 relative (CUDA exp vs host libm)."""

import hashlib
import os
import warnings

import numpy as np
import pytest

from conftest import FIG_COORDS, golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, vamana, workloads  # noqa: E402

KINDS = ["kth", "kth_normalized", "exp_sum", "sum_exp", "sum"]


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256(f"{a.dtype.str}{a.shape}".encode())
    h.update(a.tobytes())
    return h.hexdigest()


def _tags(z, suffix):
    return sorted({k.split("__")[0] for k in z.files if k.endswith(suffix)})


def points(data, mode=None):
    p = pk.PointSet(data)
    if mode == "seq64":
        p._mode = _lib.MODE_SEQ64
    elif mode == "exact32" and p.mode == _lib.MODE_EXACT_U8:
        p._mode = _lib.MODE_EXACT32
    return p


@pytest.mark.parametrize("mode", [None, "exact32", "seq64"])
def test_brute_knn_golden(mode):
    z = golden("brute")
    for tag in _tags(z, "__data"):
        data = z[f"{tag}__data"]
        p = points(data, mode)
        idx = pk.build_bruteforce(p)
        for key in z.files:
            if key.startswith(f"{tag}__k") and key.endswith("__ids"):
                k = int(key.split("__")[1][1:])
                nb = idx.knn_batch(np.arange(p.n), k)
                assert np.array_equal(nb.ids, z[key]), (tag, k)
                assert np.array_equal(nb.dists, np.sqrt(z[key.replace("__ids", "__sqd")])), (tag, k)
        nl = idx.find_knn(z[f"{tag}__vec__q"], 7)
        assert np.array_equal(nl.ids, z[f"{tag}__vec__ids"]), tag
        assert np.array_equal(nl.dists, np.sqrt(z[f"{tag}__vec__sqd"])), tag


@pytest.mark.parametrize("mode", [None, "exact32", "seq64"])
def test_build_matches_reference_graph(mode):
    z = golden("graphs")
    for tag in _tags(z, "__adj"):
        data = z[f"{tag}__data"]
        R, L, seed, ns, medoid = (int(v) for v in z[f"{tag}__params"])
        alpha = float(z[f"{tag}__alpha"][0])
        p = points(data, mode)
        idx = pk.build_vamana(p, R=R, L_build=L, alpha=alpha, num_starts=None if ns < 0 else ns, seed=seed,
                              medoid_start=bool(medoid))
        g = idx.graph
        assert np.array_equal(g.start_points, z[f"{tag}__starts"]), tag
        assert np.array_equal(g.degrees, z[f"{tag}__deg"]), tag
        assert np.array_equal(g.adjacency, z[f"{tag}__adj"]), tag


@pytest.mark.parametrize("mode", [None, "exact32", "seq64"])
def test_beam_knn_on_reference_graphs(mode):
    z = golden("graphs")
    for tag in _tags(z, "__adj"):
        data = z[f"{tag}__data"]
        p = points(data, mode)
        g = pk.GraphIndex(p, z[f"{tag}__adj"], z[f"{tag}__deg"], int(z[f"{tag}__params"][0]), z[f"{tag}__starts"], 1.0)
        qids = z[f"{tag}__qids"]
        qt = _lib.to_dev(qids)
        for key in z.files:
            if key.startswith(f"{tag}__beam_") and key.endswith("__ids"):
                _, spec, _ = key.split("__")
                Lq, k = (int(x[1:]) for x in spec.split("_")[1:])
                if Lq < min(k, p.n - 1):
                    # the public API always searches with L = max(L, k) (vamana.py:218);
                    # the kernel only supports L >= kk and rejects the rest loudly
                    with pytest.raises(RuntimeError, match="L must be >= k"):
                        vamana.beam_knn_raw(g, qt, Lq, k)
                    continue
                ids, sqd, counts = vamana.beam_knn_raw(g, qt, Lq, k)
                pre = key[: -len("__ids")]
                assert np.array_equal(_lib.to_host(ids), z[pre + "__ids"]), key
                assert np.array_equal(_lib.to_host(sqd), z[pre + "__sqd"]), key
                assert np.array_equal(_lib.to_host(counts), z[pre + "__counts"]), key
        vi = pk.VamanaIndex(g, int(z[f"{tag}__params"][1]))
        nb = vi.knn_batch(qids, 5)
        assert np.array_equal(nb.ids, z[f"{tag}__knn5__ids"]), tag
        assert np.array_equal(nb.dists, z[f"{tag}__knn5__dists"]), tag
        # single vector-query search: first L candidates + visit log
        L = int(z[f"{tag}__params"][1])
        cand = z[f"{tag}__single__cand_ids"]
        kk = min(L, cand.shape[0])
        nl, visited = pk.beam_search(g, z[f"{tag}__single__q"], g.start_points, L, kk)
        assert np.array_equal(nl.ids, cand[:kk]), tag
        assert np.array_equal(nl.dists, np.sqrt(z[f"{tag}__single__cand_sqd"][:kk])), tag
        assert [v.id for v in visited] == list(z[f"{tag}__single__vis_ids"]), tag
        assert np.array_equal(np.array([v.dist for v in visited]), np.sqrt(z[f"{tag}__single__vis_sqd"])), tag


def test_robust_prune_golden():
    z = golden("prune")
    data = z["data"]
    p = pk.PointSet(data)
    for c in range(4):
        pp, R, ncur = (int(v) for v in z[f"c{c}__args"])
        adj = np.full((40, max(R, 8)), -1, np.int32)
        deg = np.zeros(40, np.int32)
        cur = z[f"c{c}__cur"]
        adj[pp, : cur.shape[0]] = cur
        deg[pp] = cur.shape[0]
        g = pk.GraphIndex(p, adj, deg, adj.shape[1], np.array([0]), 1.0)
        cands = [pk.Neighbor(int(i), float(np.sqrt(d))) for i, d in zip(z[f"c{c}__cand"], z[f"c{c}__cand_sqd"])]
        out = pk.robust_prune(g, pp, cands, float(z[f"c{c}__alpha"][0]), R)
        assert np.array_equal(out, z[f"c{c}__out"]), c
    idx = pk.build_vamana(pk.PointSet(z["line"]), R=3, L_build=4, medoid_start=True, seed=0)
    assert idx.graph.start_points[0] == int(z["line_centroid"][0])


def _policy(meta, fmeta):
    code, arg = int(meta[4]), int(meta[5])
    return [pk.ThresholdCenter(float(fmeta[0])), pk.ProductCenter(arg), pk.LocalCenter()][code]


def test_small_pipelines_golden():
    z = golden("pipelines")
    res = pk.run_pipeline(pk.PointSet(FIG_COORDS), pk.BruteForceConfig(), k=1, density_kind="kth",
                          center_policy=pk.ThresholdCenter(2.5), noise_policy=pk.NoisePolicy(1 / np.sqrt(2.0)),
                          doubling_params=pk.DoublingParams(initial_k=2, threshold=0))
    assert np.array_equal(res.state.rho, z["fig__rho"])
    assert np.array_equal(res.state.lam, z["fig__lam"])
    assert np.array_equal(res.clustering.labels, z["fig__labels"])
    assert np.array_equal(res.clustering.centers, z["fig__centers"])
    assert np.array_equal(res.clustering.noise, z["fig__noise"])
    for t in range(15):
        meta = z[f"t{t}__meta"]
        k, vam, thr, kind = int(meta[0]), int(meta[1]), int(meta[2]), KINDS[int(meta[3])]
        icfg = pk.VamanaConfig(R=8, L_build=12, L=12, alpha=1.1, seed=t) if vam else pk.BruteForceConfig()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = pk.run_pipeline(pk.PointSet(z[f"t{t}__data"]), icfg, k=k, density_kind=kind,
                                  center_policy=_policy(meta, z[f"t{t}__fmeta"]), noise_policy=pk.NoisePolicy(0.0),
                                  doubling_params=pk.DoublingParams(initial_k=2 * k, threshold=thr))
        st = res.state
        assert np.array_equal(st.neighbors.ids, z[f"t{t}__nbr_ids"]), t
        assert np.array_equal(st.neighbors.dists, z[f"t{t}__nbr_dists"]), t
        if kind in ("exp_sum", "sum_exp"):
            np.testing.assert_allclose(st.rho, z[f"t{t}__rho"], rtol=1e-12, atol=0)
        else:
            assert np.array_equal(st.rho, z[f"t{t}__rho"]), t
        assert np.array_equal(st.lam, z[f"t{t}__lam"]), t
        assert np.array_equal(st.delta, z[f"t{t}__delta"]), t
        assert np.array_equal(res.clustering.labels, z[f"t{t}__labels"]), t
        assert np.array_equal(res.clustering.centers, z[f"t{t}__centers"]), t


@pytest.mark.parametrize("tag,name,n,comps,brute", [
    ("c1", "C1", 10_000, 10, False),
    ("c1brute", "C1", 4_000, 10, True),
    ("c2s", "C2", 20_000, 20, False),
    ("c3s", "C3", 30_000, 300, False),
])
def test_config_pipelines_golden(tag, name, n, comps, brute):
    z = golden(tag)
    data, _ = workloads.generate(name, n=n, components=comps)
    kw = workloads.pipeline_args(name, pk, n_centers=comps, brute=brute)
    res = pk.run_pipeline(pk.PointSet(data), **kw)
    st = res.state
    got = dict(rho=st.rho, lam=st.lam, delta=st.delta, nbr_ids=st.neighbors.ids, nbr_dists=st.neighbors.dists,
               labels=res.clustering.labels, centers=res.clustering.centers, noise=res.clustering.noise)
    bad = [key for key, val in got.items() if digest(val) != str(z[f"digest__{key}"])]
    if bad:
        head = {key: np.flatnonzero(got[key][:1000] != z[f"head__{key}"])[:5].tolist() for key in bad
                if got[key][:1000].shape == z[f"head__{key}"].shape}
        raise AssertionError(f"{tag}: digests differ for {bad}; first mismatching rows in head: {head}")
    if not brute:
        w = workloads.WORKLOADS[name]
        idx = pk.build_vamana(pk.PointSet(data), R=w.R, L_build=w.L, alpha=w.alpha, seed=0, query_beam=w.L)
        assert digest(idx.graph.adjacency) == str(z["digest__adj"])


def _tc_cases():
    rng = np.random.default_rng(11)
    grid = rng.integers(0, 3, size=(2_000, 8)).astype(np.float32)  # heavy exact ties + duplicates
    gauss = rng.normal(size=(3_000, 40)).astype(np.float32)
    c5, _ = workloads.generate("C5", n=4_096, components=4)
    return {"grid": grid, "gauss": gauss, "c5": c5}


@pytest.mark.parametrize("case", ["grid", "gauss", "c5"])
def test_tensor_core_knn_equals_float64_path(case, monkeypatch):
    """pk_brute_knn_tc (fp16 tcgen05 screening + float64 rescoring + certificate,
    uncertified rows recomputed) returns exactly the float64 path's rows."""
    from paper_2312_03940_b200 import index

    data = _tc_cases()[case]
    p = pk.PointSet(data)
    q = torch.arange(p.n, dtype=torch.int64, device="cuda")
    for k in (1, 16, 32):
        monkeypatch.setenv("PEAKANN_B200_TC", "0")
        i0, s0 = index.brute_device(p, q, k)
        monkeypatch.setenv("PEAKANN_B200_TC", "1")
        before = index.TC_STATS["rows"]
        i1, s1 = index.brute_device(p, q, k)
        assert index.TC_STATS["rows"] == before + p.n, "tensor-core path not taken"
        assert torch.equal(i0, i1), (case, k, int((i0 != i1).any(dim=1).sum()))
        assert torch.equal(s0, s1), (case, k)


def test_c1brute_golden_without_tensor_cores(monkeypatch):
    monkeypatch.setenv("PEAKANN_B200_TC", "0")
    test_config_pipelines_golden("c1brute", "C1", 4_000, 10, True)


def test_fp32_screened_prune_equals_float64_prune(monkeypatch):
    """Float data: the screened RobustPrune (build prune, reverse re-prune,
    hub groups) builds exactly the graph of the all-float64 prune."""
    rng = np.random.default_rng(5)
    hubs = rng.normal(size=(12, 384)).astype(np.float32)
    lab = rng.integers(0, 12, 6_000)
    x = (hubs[lab] + 0.05 * rng.normal(size=(6_000, 384))).astype(np.float32)
    x[:40] = hubs[lab[:40]]  # exact duplicates of cluster centres: ties and zero distances
    p = pk.PointSet(x)
    assert p.mode == _lib.MODE_SEQ64
    starts, order = vamana.sample_starts(p.n, None, 0, False, p)
    monkeypatch.setenv("PK_SCREEN", "0")
    a0, d0 = vamana.build_graph_device(p, 24, 48, 1.2, starts, order)
    monkeypatch.setenv("PK_SCREEN", "1")
    a1, d1 = vamana.build_graph_device(p, 24, 48, 1.2, starts, order)
    assert torch.equal(d0, d1)
    assert torch.equal(a0, a1)


def test_fp32_screened_beam_search_equals_float64(monkeypatch):
    """Float data with d >= 256: the beam searches' fp32 pre-screen against a
    full beam changes nothing -- same graph, same kNN rows and counts."""
    from paper_2312_03940_b200 import index as _idx  # noqa: F401

    data, _ = workloads.generate("C4", n=8_000, components=40)
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("PK_SCREEN", flag)
        p = pk.PointSet(data)
        g = pk.build_vamana(p, R=32, L_build=64, alpha=1.1, seed=0, query_beam=64)
        nb = g.knn_all(16)
        out[flag] = (g.graph.adjacency.copy(), nb.ids.copy(), nb.dists.copy())
    for a, b in zip(out["0"], out["1"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("case", ["c5", "dup128"])
def test_lazy_keys_equal_eager(monkeypatch, case):
    """Float data: beam searches holding fp32 screen values as lazy keys
    (exact float64 only where an ordering decision or an output needs it)
    build the same graph and return the same kNN rows, distances and labels
    as the eager float64 searches (PK_LAZY=0)."""
    if case == "c5":
        data, _ = workloads.generate("C5", n=6_000, components=8)
    else:
        rng = np.random.default_rng(3)
        hubs = rng.normal(size=(12, 128))
        lab = rng.integers(0, 12, 5_000)
        data = (hubs[lab] + 0.1 * rng.normal(size=(5_000, 128))).astype(np.float32)
        data[:60] = hubs[lab[:60]]  # exact duplicates: zero distances and tied keys
        data[60:90] = data[100:130]
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("PK_LAZY", flag)
        p = pk.PointSet(data)
        assert p.mode == _lib.MODE_SEQ64
        res = pk.run_pipeline(p, pk.VamanaConfig(R=24, L_build=64, L=64, alpha=1.1, seed=0), k=16,
                              density_kind="kth", center_policy=pk.ProductCenter(8), noise_policy=pk.NoisePolicy(0.0),
                              doubling_params=pk.DoublingParams(initial_k=32, threshold=50))
        st = res.state
        g = pk.build_vamana(p, R=32, L_build=96, alpha=1.2, seed=1, query_beam=128)
        nb = g.knn_all(40)
        out[flag] = [st.neighbors.ids, st.neighbors.dists, st.rho, st.lam, st.delta, res.clustering.labels,
                     g.graph.adjacency, nb.ids, nb.dists]
    for a, b in zip(out["0"], out["1"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("case", ["c5", "c4", "dup128", "wide", "huge", "tiny", "mixed"])
def test_tensor_core_prune_equals_warp_prune(monkeypatch, case):
    """Float data: RobustPrune decided from tcgen05 Gram tiles (fp16 copy of the
    rows; PK_PRUNE_F16=0: tf32) with a rigorous error bound (uncertain pairs
    decided exactly) builds the same graph as the warp-per-item screened prune
    (PK_TC_PRUNE=0) -- also where the fp16 bound does not hold or is loose:
    coordinates past the fp16 range (non-finite accumulators), subnormal fp16
    coordinates, rows of very different norms."""
    if case in ("huge", "tiny", "mixed"):
        rng = np.random.default_rng(21)
        hubs = rng.normal(size=(12, 96))
        lab = rng.integers(0, 12, 5_000)
        data = hubs[lab] + 0.15 * rng.normal(size=(5_000, 96))
        data[:40] = hubs[lab[:40]]
        if case == "huge":
            data[::7] *= 2.0e5   # fp16 overflow on every 7th row
        elif case == "tiny":
            data *= 1.0e-6       # fp16 subnormals
        else:
            data[::5] *= 300.0   # norms 300x apart: the bound |t||u| dwarfs the small rows' distances
            data[1::5] *= 1.0e-3
        data = data.astype(np.float32)
        out = {}
        for flag in ("0", "1"):
            monkeypatch.setenv("PK_TC_PRUNE", flag)
            g = pk.build_vamana(pk.PointSet(data), R=32, L_build=96, alpha=1.2, seed=2, query_beam=96)
            out[flag] = (g.graph.adjacency.copy(), g.graph.degrees.copy())
        assert np.array_equal(out["0"][1], out["1"][1])
        assert np.array_equal(out["0"][0], out["1"][0])
        return
    if case == "c5":
        data, _ = workloads.generate("C5", n=6_000, components=8)
    elif case == "c4":
        data, _ = workloads.generate("C4", n=8_000, components=40)
    elif case == "wide":
        # long candidate lists (up to ~400) and R = 160: several 128-row bit blocks
        rng = np.random.default_rng(8)
        data = (rng.normal(size=(5_000, 48)) + 2.0 * rng.normal(size=(6, 48))[rng.integers(0, 6, 5_000)])
        data = data.astype(np.float32)
        out = {}
        for flag in ("0", "1"):
            monkeypatch.setenv("PK_TC_PRUNE", flag)
            g = pk.build_vamana(pk.PointSet(data), R=160, L_build=320, alpha=1.05, seed=3, query_beam=64)
            out[flag] = (g.graph.adjacency.copy(), g.graph.degrees.copy())
        assert np.array_equal(out["0"][1], out["1"][1])
        assert np.array_equal(out["0"][0], out["1"][0])
        return
    else:
        rng = np.random.default_rng(5)
        hubs = rng.normal(size=(10, 128)) * 3.0
        lab = rng.integers(0, 10, 6_000)
        data = (hubs[lab] + 0.2 * rng.normal(size=(6_000, 128))).astype(np.float32)
        data[:50] = hubs[lab[:50]]
        data[50:80] = data[200:230]
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("PK_TC_PRUNE", flag)
        p = pk.PointSet(data)
        g = pk.build_vamana(p, R=32, L_build=96, alpha=1.2, seed=2, query_beam=96)
        out[flag] = (g.graph.adjacency.copy(), g.graph.degrees.copy())
    assert np.array_equal(out["0"][1], out["1"][1])
    assert np.array_equal(out["0"][0], out["1"][0])


@pytest.mark.parametrize("case", ["c5", "dup128", "huge", "tiny"])
def test_tensor_core_seeding_equals_fp32_seeding(monkeypatch, case):
    """Float builds with >= 256 starts: the tcgen05 screens of every point
    against the start set (fp16 operands, certified bound) only decide which
    starts get an fp32 screen; the graph and the kNN rows equal the ones of the
    plain fp32-screened seeding (PK_SEED_TC=0), also where the fp16 bound does
    not hold (coordinates past the fp16 range, subnormal fp16 coordinates)."""
    rng = np.random.default_rng(11)
    if case == "c5":
        data, _ = workloads.generate("C5", n=6_000, components=8)
    else:
        hubs = rng.normal(size=(12, 96))
        lab = rng.integers(0, 12, 5_000)
        data = hubs[lab] + 0.15 * rng.normal(size=(5_000, 96))
        data[:40] = hubs[lab[:40]]  # duplicates: tied start distances
        data[40:70] = data[300:330]
        if case == "huge":
            data[::7] *= 2.0e5  # fp16 overflow on every 7th row (queries and starts)
        elif case == "tiny":
            data *= 1.0e-6  # fp16 subnormals
        data = data.astype(np.float32)
    out = {}
    # several screening chunks of 1,300 rows on the C5 sample
    monkeypatch.setenv("PK_SEED_CHUNK", "1300" if case == "c5" else "0")
    for flag in ("0", "1"):
        monkeypatch.setenv("PK_SEED_TC", flag)
        p = pk.PointSet(data)
        assert p.mode == _lib.MODE_SEQ64
        _lib.prof_collect(reset=True)
        _lib.prof_only([])
        _lib.prof_enable(True)
        g = pk.build_vamana(p, R=32, L_build=128, alpha=1.2, num_starts=400, seed=4, query_beam=128)
        _lib.prof_enable(False)
        ran = "tc_seed_screen_kernel" in _lib.prof_collect(reset=True)
        assert ran == (flag == "1")
        nb = g.knn_all(16)
        out[flag] = (g.graph.adjacency.copy(), g.graph.degrees.copy(), nb.ids.copy(), nb.dists.copy())
    for a, b in zip(out["0"], out["1"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("case", ["c5", "dup128", "huge"])
def test_tensor_core_count_decision_equals_exact_count(monkeypatch, case):
    """Float data, doubling rounds: the short rows' "fewer than kk points closer
    than the nearest denser point" decision taken from tcgen05 bounds (exact count
    scan only for the rows the bounds leave open) gives the same lambda, delta and
    labels as the exact count scan (PK_TC_COUNT=0)."""
    import ctypes

    rng = np.random.default_rng(21)
    if case == "c5":
        data, _ = workloads.generate("C5", n=8_000, components=12)
    else:
        hubs = rng.normal(size=(12, 96))
        lab = rng.integers(0, 12, 6_000)
        data = hubs[lab] + 0.2 * rng.normal(size=(6_000, 96))
        data[:50] = hubs[lab[:50]]  # duplicates: ties at the key distance
        data[50:90] = data[400:440]
        if case == "huge":
            data[::9] *= 3.0e5  # fp16 overflow: those rows stay undecided
        data = data.astype(np.float32)
    monkeypatch.setenv("PK_TC_COUNT_MIN", "1")
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("PK_TC_COUNT", flag)
        st = (ctypes.c_int64 * 2)()
        _lib.lib().pk_tc_count_stats(st, 1)
        res = pk.run_pipeline(pk.PointSet(data), pk.VamanaConfig(R=16, L_build=32, L=32, alpha=1.1, seed=0), k=16,
                              density_kind="kth", center_policy=pk.ProductCenter(10), noise_policy=pk.NoisePolicy(0.0),
                              doubling_params=pk.DoublingParams(initial_k=32, threshold=0))
        _lib.lib().pk_tc_count_stats(st, 1)
        assert (st[0] > 0) == (flag == "1")
        s = res.state
        out[flag] = [s.rho, s.lam, s.delta, res.clustering.labels]
    for a, b in zip(out["0"], out["1"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("case", ["c2", "c3", "dup"])
def test_u8_seed_table_equals_warp_seeding(monkeypatch, case):
    """u8 rows of d = 128: the build's start distances precomputed on the integer
    tensor cores (exact) give the same graph and kNN rows as the warp-evaluated
    seeding (PK_SEED_TAB=0)."""
    if case in ("c2", "c3"):
        data, _ = workloads.generate(case.upper(), n=20_000, components=20)
    else:
        rng = np.random.default_rng(31)
        data = rng.integers(0, 4, size=(12_000, 128)).astype(np.float32)  # heavy ties
        data[:100] = data[100:200]
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("PK_SEED_TAB", flag)
        p = pk.PointSet(data)
        assert p.mode == _lib.MODE_EXACT_U8
        _lib.prof_collect(reset=True)
        _lib.prof_only([])
        _lib.prof_enable(True)
        g = pk.build_vamana(p, R=32, L_build=128, alpha=1.1, seed=5, query_beam=128)
        _lib.prof_enable(False)
        assert ("seed_u8_tc_kernel" in _lib.prof_collect(reset=True)) == (flag == "1")
        nb = g.knn_all(16)
        out[flag] = (g.graph.adjacency.copy(), g.graph.degrees.copy(), nb.ids.copy(), nb.dists.copy())
    for a, b in zip(out["0"], out["1"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", ["u8", "float"])
def test_build_with_short_candidate_lists_matches_oracle(kind):
    """L_build < R: many items have at most R candidates, and the build still
    runs RobustPrune on them (_kernels.py:370) -- in the block kernels too."""
    rng = np.random.default_rng(11)
    if kind == "u8":
        mu = rng.uniform(0, 255, (20, 128))
        data = np.clip(np.round(mu[rng.integers(0, 20, 2_500)] + rng.normal(0, 20, (2_500, 128))), 0, 255)
        data = data.astype(np.float32)
    else:
        data = (rng.normal(size=(2_500, 64)) + 3.0 * rng.normal(size=(12, 64))[rng.integers(0, 12, 2_500)])
        data = data.astype(np.float32)
    p = pk.PointSet(data)
    g = pk.build_vamana(p, R=32, L_build=12, alpha=1.2, seed=4)
    adj, deg, starts = oracle.build_vamana(data, R=32, L_build=12, alpha=1.2, seed=4)[:3]
    assert np.array_equal(g.graph.degrees, deg)
    assert np.array_equal(g.graph.adjacency, adj)


@pytest.mark.parametrize("d", [48, 384, 1024, "u8"])
def test_count_below_matches_exact_rows(d):
    """pk_count_below (float data: fp32-screened count scan, exact float64 inside
    the band; u8 rows: register-blocked exact integer scan) == the position of
    the key in the exact brute-force row (oracle)."""
    import torch

    rng = np.random.default_rng(7 if d == "u8" else d)
    n = 3_000
    if d == "u8":
        mu = rng.uniform(0, 255, (8, 128))
        data = np.clip(np.round(mu[rng.integers(0, 8, n)] + rng.normal(0, 20, (n, 128))), 0, 255).astype(np.float32)
    else:
        data = (rng.normal(size=(n, d)) + rng.normal(size=(8, d))[rng.integers(0, 8, n)]).astype(np.float32)
    data[:20] = data[20:40]  # duplicates: zero distances and tied keys
    p = pk.PointSet(data)
    if d == "u8":
        assert p.mode == _lib.MODE_EXACT_U8
    qids = np.sort(rng.choice(n, 40, replace=False)).astype(np.int64)
    ids, sqd = oracle.brute_knn_batch(data, qids, n - 1)
    pos = rng.integers(0, n - 1, qids.shape[0])
    pos[:5] = 0
    key_i = ids[np.arange(len(qids)), pos].astype(np.int64)
    key_d = sqd[np.arange(len(qids)), pos]
    cnt = torch.zeros(len(qids), dtype=torch.int64, device="cuda")
    _lib.call("pk_count_below", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, _lib.to_dev(qids), len(qids),
              _lib.to_dev(key_d), _lib.to_dev(key_i), cnt, _lib.stream())
    assert np.array_equal(_lib.to_host(cnt), pos)


def test_pointset_device_validation_reports_first_nonfinite():
    """With a GPU the PointSet check runs on the device (pk_scan_points); the
    error names the same first (point, dimension) as numpy's argwhere."""
    x = np.random.default_rng(0).normal(size=(5_000, 37)).astype(np.float32)
    x[4_000, 36] = np.inf
    x[1_234, 5] = np.nan
    x[1_234, 9] = -np.inf
    with pytest.raises(ValueError, match="point 1234, dimension 5"):
        pk.PointSet(x.copy())
    assert pk.PointSet(np.ones((3, 5), np.float32)).mode in (_lib.MODE_EXACT_U8, _lib.MODE_EXACT32)


@pytest.mark.parametrize("case", ["gauss", "c5", "grid"])
def test_tensor_core_dp_scan_equals_exact_scan(case):
    """pk_dp_scan_tc (denser-only tensor-core screen + float64 rescoring +
    certificate, uncertified rows rescanned) == pk_dp_scan."""
    from paper_2312_03940_b200 import density, dependent

    data = _tc_cases()[case]
    p = pk.PointSet(data)
    p._mode = _lib.MODE_SEQ64  # the scan the tensor cores replace (float data)
    rng = np.random.default_rng(2)
    rho = torch.from_numpy(rng.integers(0, 50, p.n).astype(np.float64)).cuda()  # many density ties
    rank = density.rank_order_device(rho)
    q = torch.from_numpy(rng.choice(p.n, 700, replace=False).astype(np.int64)).cuda()
    top = int(torch.argmax(rank).item())
    q = q[q != top].contiguous()
    m = q.shape[0]
    i0 = torch.empty(m, dtype=torch.int64, device="cuda")
    s0 = torch.empty(m, dtype=torch.float64, device="cuda")
    _lib.call("pk_dp_scan", p.device(), p.n, p.dp, None, 0, p.mode, rank, q, m, i0, s0, _lib.stream())
    i1 = torch.empty_like(i0)
    s1 = torch.empty_like(s0)
    dependent._dp_scan_tc(p, rank, q, m, i1, s1)
    assert torch.equal(i0, i1)
    assert torch.equal(s0, s1)


def test_u8_tensor_core_dp_scan_equals_cuda_core_scan(monkeypatch):
    """u8 rows (d = 128): the integer tensor-core nearest-denser scan (packed
    (d, id) keys, atomicMin) == the CUDA-core scan, with density ties and
    duplicate points."""
    rng = np.random.default_rng(4)
    mu = rng.uniform(0, 255, (6, 128))
    data = np.clip(np.round(mu[rng.integers(0, 6, 5_000)] + rng.normal(0, 20, (5_000, 128))), 0, 255)
    data[:30] = data[30:60]
    p = pk.PointSet(data.astype(np.float32))
    assert p.mode == _lib.MODE_EXACT_U8
    from paper_2312_03940_b200 import density

    rho = torch.from_numpy(rng.integers(0, 40, p.n).astype(np.float64)).cuda()
    rank = density.rank_order_device(rho)
    q = torch.from_numpy(np.sort(rng.choice(p.n, 900, replace=False)).astype(np.int64)).cuda()
    m = q.shape[0]
    out = []
    for flag in ("0", "1"):
        monkeypatch.setenv("PK_U8_TC_SCAN", flag)
        i = torch.empty(m, dtype=torch.int64, device="cuda")
        d = torch.empty(m, dtype=torch.float64, device="cuda")
        _lib.call("pk_dp_scan", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, rank, q, m, i, d, _lib.stream())
        out.append((i, d))
    assert torch.equal(out[0][0], out[1][0])
    assert torch.equal(out[0][1], out[1][1])


def test_device_contingency_equals_host():
    from paper_2312_03940_b200 import metrics

    rng = np.random.default_rng(9)
    a = rng.integers(-50, 900, 300_000)
    b = rng.integers(0, 1_000, 300_000)
    dev = metrics._contingency_device(a, b)
    metrics_min, metrics.DEVICE_MIN = metrics.DEVICE_MIN, 10**12
    try:
        host = metrics.contingency(a, b)
        h_ari = pk.ari(a, b)
    finally:
        metrics.DEVICE_MIN = metrics_min
    for f in ("rows", "cols", "counts", "row_sums", "col_sums"):
        assert np.array_equal(getattr(dev, f), getattr(host, f)), f
    assert pk.ari(a, b) == h_ari  # device path (n >= DEVICE_MIN)


def _pipeline_vs_oracle(data, R, L, k, nc, alpha=1.2, threshold=50, density="kth", seed=0):
    res = pk.run_pipeline(pk.PointSet(data), pk.VamanaConfig(R=R, L_build=L, L=L, alpha=alpha, seed=seed), k=k,
                          density_kind=density, center_policy=pk.ProductCenter(nc), noise_policy=pk.NoisePolicy(0.0),
                          doubling_params=pk.DoublingParams(initial_k=2 * k, threshold=threshold))
    ref = oracle.pipeline(data, index="vamana", R=R, L_build=L, L=L, alpha=alpha, seed=seed, k=k, density_kind=density,
                          center_policy=("product", nc), rho_min=0.0, initial_k=2 * k, threshold=threshold)
    st = res.state
    assert np.array_equal(st.neighbors.ids, ref["nbr_ids"])
    assert np.array_equal(st.neighbors.dists, ref["nbr_dists"])
    assert np.array_equal(st.rho, ref["rho"])
    assert np.array_equal(st.lam, ref["lam"])
    assert np.array_equal(st.delta, ref["delta"])
    assert np.array_equal(res.clustering.labels, ref["labels"])


@pytest.mark.parametrize("case", ["identical1024", "few_distinct256", "huge_scale", "tiny_scale", "d1", "n3", "n2",
                                  "identical_u8", "grid_u8_ties", "wide_beam"])
def test_degenerate_float_data_matches_oracle(case):
    """Float data the lazy keys / tensor-core prune / fp32 screens find hardest:
    all points identical (every key tied, zero distances, cancellation in the
    Gram epilogue), a handful of distinct rows, coordinates near the fp32 range
    limits (screens overflow / underflow and fall back), d = 1, and n = 3."""
    rng = np.random.default_rng(17)
    if case == "identical1024":
        data = np.tile(rng.normal(size=(1, 1024)).astype(np.float32), (400, 1))
    elif case == "few_distinct256":
        data = rng.normal(size=(5, 256)).astype(np.float32)[rng.integers(0, 5, 600)]
    elif case == "huge_scale":
        data = (rng.normal(size=(700, 300)) * 3e18).astype(np.float32)
    elif case == "tiny_scale":
        data = (rng.normal(size=(700, 300)) * 1e-19).astype(np.float32)
    elif case == "d1":
        data = rng.normal(size=(900, 1)).astype(np.float32)
    elif case == "n3":
        data = rng.normal(size=(3, 40)).astype(np.float32)
    elif case == "n2":
        data = rng.normal(size=(2, 7)).astype(np.float32)
    elif case == "identical_u8":
        data = np.full((500, 128), 7.0, np.float32)
    elif case == "grid_u8_ties":
        # integer grid: many exactly equal distances (ties broken by id)
        data = np.stack(np.meshgrid(np.arange(30), np.arange(30), indexing="ij"), -1).reshape(-1, 2)
        data = np.concatenate([data, data[:100]]).astype(np.float32)
    else:  # beam wider than n, every point a start
        data = rng.normal(size=(120, 16)).astype(np.float32)
        res = pk.run_pipeline(pk.PointSet(data), pk.VamanaConfig(R=8, L_build=200, L=200, alpha=1.0, seed=1,
                                                                 num_starts=120), k=12, density_kind="sum",
                              center_policy=pk.ProductCenter(4), noise_policy=pk.NoisePolicy(0.0),
                              doubling_params=pk.DoublingParams(initial_k=24, threshold=5))
        ref = oracle.pipeline(data, index="vamana", R=8, L_build=200, L=200, alpha=1.0, seed=1, num_starts=120, k=12,
                              density_kind="sum", center_policy=("product", 4), rho_min=0.0, initial_k=24,
                              threshold=5)
        assert np.array_equal(res.state.neighbors.ids, ref["nbr_ids"])
        assert np.array_equal(res.state.lam, ref["lam"])
        assert np.array_equal(res.clustering.labels, ref["labels"])
        return
    n = data.shape[0]
    k = min(8, n - 1)
    _pipeline_vs_oracle(data, R=16, L=max(24, k), k=k, nc=min(3, n))


@pytest.mark.parametrize("mode", [None, "exact32"])
def test_wide_beam_integer_modes_match_oracle(mode):
    """Integer data with L = 128 (seeding by selection, packed beam keys) in the
    u8 and the exact-fp32 policies: graph, kNN rows and labels == the oracle."""
    rng = np.random.default_rng(21)
    mu = rng.uniform(0, 255, (12, 64))
    data = np.clip(np.round(mu[rng.integers(0, 12, 3_000)] + rng.normal(0, 25, (3_000, 64))), 0, 255)
    data = data.astype(np.float32)
    data[:20] = data[20:40]
    p = points(data, mode)
    assert p.mode == (_lib.MODE_EXACT32 if mode == "exact32" else _lib.MODE_EXACT_U8)
    g = pk.build_vamana(p, R=24, L_build=128, alpha=1.2, seed=5, query_beam=128)
    adj, deg, _ = oracle.build_vamana(data, R=24, L_build=128, alpha=1.2, seed=5)
    assert np.array_equal(g.graph.degrees, deg)
    assert np.array_equal(g.graph.adjacency, adj)
    nb = g.knn_all(20)
    ids, sqd = oracle.GraphIndexOracle(data, adj, deg, g.graph.start_points, 128).knn_batch(
        np.arange(3_000, dtype=np.int64), 20)
    assert np.array_equal(nb.ids, ids)
    assert np.array_equal(nb.dists, sqd)


@pytest.mark.parametrize("case", ["u8", "float"])
def test_seeded_beam_cache_equals_fresh_seeding(monkeypatch, case):
    """Member queries with L == L_build start from the beams the build saved
    (pk_build_vamana_seeds / pk_beam_knn_seeded): same kNN rows, densities,
    dependent points and labels as seeding afresh (PK_SEED_CACHE=0)."""
    if case == "u8":
        data, _ = workloads.generate("C2", n=20_000, components=20)
    else:
        data, _ = workloads.generate("C5", n=6_000, components=8)
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("PK_SEED_CACHE", flag)
        res = pk.run_pipeline(pk.PointSet(data), pk.VamanaConfig(R=32, L_build=128, L=128, alpha=1.1, seed=3), k=16,
                              density_kind="kth", center_policy=pk.ProductCenter(10),
                              noise_policy=pk.NoisePolicy(0.0), doubling_params=pk.DoublingParams(initial_k=32,
                                                                                                 threshold=40))
        st = res.state
        out[flag] = [st.neighbors.ids, st.neighbors.dists, st.rho, st.lam, st.delta, res.clustering.labels]
    for a, b in zip(out["0"], out["1"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("switch,values", [("PK_TICKETS", ("0", "1")), ("PK_RING", ("0", "2")),
                                           ("PK_PRUNE_F16", ("0", "1")), ("PK_PREFETCH", ("0", "1")),
                                           ("PK_PREFETCH_ROWS", ("0", "1"))])
def test_round2_switches_are_output_neutral(monkeypatch, switch, values):
    """Round-2 scheduling / staging switches change how the work is
    done, never its result: ticket assignment vs the static stride, the row ring of the
    float kNN searches, the fp16 vs tf32 Gram of the tensor-core prune, the two prefetches.
    A C5-shaped instance wide enough for the ring (d = 1024) with s >= 256 starts; the
    graph, kNN rows, densities, dependent points and labels must be identical (the default
    settings are compared with the oracle in test_parity_scale_gpu.py)."""
    data, _ = workloads.generate("C5", n=70_000, components=55)
    out = {}
    for v in values:
        monkeypatch.setenv(switch, v)
        ps = pk.PointSet(data)
        idx = pk.build_vamana(ps, R=32, L_build=128, alpha=1.1, seed=5, query_beam=128)
        res = pk.run_pipeline(ps, pk.VamanaConfig(R=32, L_build=128, L=128, alpha=1.1, seed=5), k=16,
                              density_kind="kth", center_policy=pk.ProductCenter(55),
                              noise_policy=pk.NoisePolicy(0.0),
                              doubling_params=pk.DoublingParams(initial_k=32, threshold=100))
        st = res.state
        out[v] = [idx.graph.adjacency, idx.graph.degrees, st.neighbors.ids, st.neighbors.dists, st.rho, st.lam, st.delta,
                  res.clustering.labels]
    for a, b in zip(out[values[0]], out[values[1]]):
        assert np.array_equal(np.asarray(a), np.asarray(b))
