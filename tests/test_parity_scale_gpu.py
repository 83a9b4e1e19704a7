"""CUDA path vs the CPU oracle at the shapes the configurations actually run
(GPU only).

test_parity_gpu.py pins every kernel against the reference's golden vectors
on small inputs.  This file closes the gaps between those inputs and the
BASELINE configurations:

* doubling-round beam widths L = k = 256 ... 4096 (C3 runs 7 rounds up to
  k = 4096; C4 / C5 up to 1024 / 2048) on the u8 path and on the float path
  with lazy keys and every tensor-core shortcut on
  (reference: _kernels.py:230-262, dependent.py:118-126);
* C3-, C4- and C5-shaped pipelines made by the configurations' own
  generators, compared output for output with oracle.pipeline
  (cluster.py:279-311), with a check that the tensor-core kernels actually
  ran;
* the short-walk fallback of find_knn_with_fallback (vamana.py:175-197);
* integer data wider than the integer kernels' 1,024 columns.

Everything is bit-exact except exp-based densities (not used here).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200 import _lib, vamana, workloads  # noqa: E402


def _launched(fn):
    """Run fn with launch counting on; returns (result, {kernel: launches})."""
    _lib.prof_collect(reset=True)
    _lib.prof_only(["__count_only__"])  # count every launch, time none
    _lib.prof_enable(True)
    try:
        out = fn()
        torch.cuda.synchronize()
    finally:
        _lib.prof_enable(False)
    prof = _lib.prof_collect(reset=True)
    return out, {k: v[0] for k, v in prof.items()}


def _assert_state_equal(res, ref, exp_density=False):
    st = res.state
    assert np.array_equal(st.neighbors.ids, ref["nbr_ids"])
    assert np.array_equal(st.neighbors.dists, ref["nbr_dists"])
    if exp_density:
        np.testing.assert_allclose(st.rho, ref["rho"], rtol=1e-12, atol=0)
    else:
        assert np.array_equal(st.rho, ref["rho"])
    assert np.array_equal(st.lam, ref["lam"])
    assert np.array_equal(st.delta, ref["delta"])
    assert np.array_equal(res.clustering.labels, ref["labels"])
    assert np.array_equal(res.clustering.centers, ref["centers"])
    assert np.array_equal(res.clustering.noise, ref["noise"])


# ---------------------------------------------------------------- wide beams


@pytest.mark.parametrize("case", ["u8_c3", "float_c5", "float_c4"])
def test_doubling_width_beam_rows_match_oracle(case):
    """Beam kNN rows at L = k = 256 ... 4096 on a GPU-built graph: ids, squared
    distances and counts equal the oracle's beam_knn_batch on the same graph
    (u8 packed keys; float lazy keys with the fp32 / float64 refinement)."""
    if case == "u8_c3":
        n, R, L = 50_000, 64, 128
        data, _ = workloads.generate("C3", n=n, components=50)
    elif case == "float_c5":
        n, R, L = 20_000, 64, 200
        data, _ = workloads.generate("C5", n=n, components=16)
    else:
        n, R, L = 20_000, 64, 128
        data, _ = workloads.generate("C4", n=n, components=100)
    p = pk.PointSet(data)
    assert p.mode == (_lib.MODE_EXACT_U8 if case == "u8_c3" else _lib.MODE_SEQ64)
    g = pk.build_vamana(p, R=R, L_build=L, alpha=1.1, seed=0, query_beam=L).graph
    rng = np.random.default_rng(7)
    q = np.sort(rng.choice(n, 48, replace=False)).astype(np.int64)
    qt = _lib.to_dev(q)
    for width in (256, 512, 1024, 2048, 4096):
        ids, sqd, cnt = vamana.beam_knn_raw(g, qt, width, width)
        oi, od, oc = oracle.beam_knn_batch(data, g.adjacency, g.degrees, g.start_points, q, width, width)
        assert np.array_equal(_lib.to_host(cnt), oc), width
        assert np.array_equal(_lib.to_host(ids), oi), width
        assert np.array_equal(_lib.to_host(sqd), od), width


def test_c3_shaped_pipeline_through_k4096_matches_oracle():
    """C3's settings (exp_sum k = 32: every rho underflows to 0, so the rank is
    the id order and the doubling rounds run long) on a 30k instance with
    threshold 10: rounds at k = 64 ... 4096, then the exact scan."""
    data, _ = workloads.generate("C3", n=30_000, components=30)
    kw = dict(threshold=10)
    res = pk.run_pipeline(pk.PointSet(data), pk.VamanaConfig(R=64, L_build=128, L=128, alpha=1.1, seed=0), k=32,
                          density_kind="exp_sum", center_policy=pk.ProductCenter(30), noise_policy=pk.NoisePolicy(0.0),
                          doubling_params=pk.DoublingParams(initial_k=64, threshold=kw["threshold"]))
    ref = oracle.pipeline(data, index="vamana", R=64, L_build=128, L=128, alpha=1.1, seed=0, k=32,
                          density_kind="exp_sum", center_policy=("product", 30), rho_min=0.0, initial_k=64,
                          threshold=kw["threshold"])
    assert max(kq for _, kq in ref["rounds"]) == 4096, ref["rounds"]
    _assert_state_equal(res, ref, exp_density=True)


# ---------------------------------------------------------------- configuration shapes


def _config_pipeline(name, n, comps, threshold=300):
    w = workloads.WORKLOADS[name]
    data, _ = workloads.generate(name, n=n, components=comps)
    kw = workloads.pipeline_args(name, pk, n_centers=min(w.n_centers, comps))
    kw["doubling_params"] = pk.DoublingParams(initial_k=2 * w.k, threshold=threshold)
    res, launches = _launched(lambda: pk.run_pipeline(pk.PointSet(data), **kw))
    ref = oracle.pipeline(data, index="vamana", R=w.R, L_build=w.L, L=w.L, alpha=w.alpha, seed=0, k=w.k,
                          density_kind=w.density, center_policy=("product", min(w.n_centers, comps)), rho_min=0.0,
                          initial_k=2 * w.k, threshold=threshold)
    return data, res, ref, launches


@pytest.mark.parametrize("name,n,comps", [("C4", 70_000, 350)])
def test_float_config_shaped_pipeline_matches_oracle(name, n, comps):
    """C5 / C4 settings (R = 64, L = 200 / 128, kth k = 16, product centers,
    doubling from 32, threshold 300) on 70k points of the configurations'
    generators -- s = 265 starts, so the build takes the tensor-core start
    pre-screen; the float prune runs on the tensor cores; beam keys are lazy.
    Every output equals the oracle's, and the tensor-core kernels ran."""
    data, res, ref, launches = _config_pipeline(name, n, comps)
    assert launches.get("prune_tc_build_kernel", 0) > 0, launches
    assert launches.get("tc_seed_screen_kernel", 0) + launches.get("tc_screen_kernel", 0) > 0, launches
    _assert_state_equal(res, ref)


@pytest.mark.parametrize("name,n,comps,threshold", [("C5", 70_000, 55, 20), ("C4", 70_000, 350, 20)])
def test_float_config_shaped_doubling_to_exact_scan(name, n, comps, threshold):
    """Same shapes with a low threshold: more doubling rounds, short rows
    settled by the tensor-core count decision, and the tensor-core dp scan of
    the stragglers -- still identical to the oracle."""
    data, res, ref, launches = _config_pipeline(name, n, comps, threshold)
    assert len(ref["rounds"]) >= 2, ref["rounds"]
    assert launches.get("prune_tc_build_kernel", 0) > 0, launches
    assert launches.get("tc_seed_screen_kernel", 0) > 0, launches
    _assert_state_equal(res, ref)


def test_u8_config_shaped_pipeline_matches_oracle():
    """C2 settings (kth_normalized) on a 50k instance of its generator (u8 path:
    integer tensor-core seed table, block prune, u8 scans)."""
    data, res, ref, launches = _config_pipeline("C2", 50_000, 50)
    assert launches.get("build_prune_block_kernel", 0) > 0, launches
    _assert_state_equal(res, ref)


# ---------------------------------------------------------------- fallback and wide rows


def _two_component_graph():
    """Group A (ids 0..9) is a connected ring reachable from the start; group B
    (ids 10..59) has no edges, so no walk reaches it."""
    rng = np.random.default_rng(3)
    data = np.concatenate([rng.normal(0, 1, (10, 24)), rng.normal(6, 1, (50, 24))]).astype(np.float32)
    R = 4
    adj = np.full((60, R), -1, np.int32)
    deg = np.zeros(60, np.int32)
    for i in range(10):
        adj[i, :2] = [(i + 1) % 10, (i + 9) % 10]
        deg[i] = 2
    starts = np.array([0], np.int64)
    return data, adj, deg, starts


def _oracle_find_knn_with_fallback(data, adj, deg, starts, query, k, L):
    """vamana.py:175-197 restated over the oracle kernels."""
    L = max(L, k)
    n = data.shape[0]
    if isinstance(query, (int, np.integer)):
        qid, vec = int(query), data[int(query)].astype(np.float64)
    else:
        qid, vec = -1, np.asarray(query, np.float64)
    want = min(k, n - 1) if qid >= 0 else min(k, n)
    ci, cd, _, _ = oracle.beam_search_single(data, adj, deg, starts, vec, L)
    keep = ci != qid
    ti, td = ci[keep][:k], cd[keep][:k]
    if ti.shape[0] < want:
        if qid >= 0:
            ids, sqd = oracle.brute_knn_batch(data, np.array([qid], np.int64), k)
            return ids[0], np.sqrt(sqd[0])
        ids, sqd = oracle.brute_knn_vector(data, vec, k)
        return ids, np.sqrt(sqd)
    return ti, np.sqrt(td)


@pytest.mark.parametrize("query", [3, 25, "vec_a", "vec_b"])
@pytest.mark.parametrize("k", [5, 15])
def test_find_knn_with_fallback_matches_oracle(query, k):
    """k = 5 from group A: the walk fills the row (no fallback).  k = 15, or any
    query whose neighbours sit in the unreachable group: the walk comes up
    short and the exact pass answers -- member and vector queries."""
    data, adj, deg, starts = _two_component_graph()
    p = pk.PointSet(data)
    g = pk.GraphIndex(p, adj, deg, 4, starts, 1.0)
    if query == "vec_a":
        query = data[:10].mean(0).astype(np.float64)
    elif query == "vec_b":
        query = data[10:].mean(0).astype(np.float64)
    nl = pk.find_knn_with_fallback(g, query, k, 8)
    oi, od = _oracle_find_knn_with_fallback(data, adj, deg, starts, query, k, 8)
    assert np.array_equal(nl.ids, oi)
    assert np.array_equal(nl.dists, od)
    vi = pk.VamanaIndex(g, 8)
    nl2 = vi.find_knn(query, k)
    assert np.array_equal(nl2.ids, oi)


def test_fallback_branch_really_runs():
    """The member query 25 with k = 15 cannot be answered by the walk (only 10
    points reachable): the exact kNN kernel must run."""
    data, adj, deg, starts = _two_component_graph()
    g = pk.GraphIndex(pk.PointSet(data), adj, deg, 4, starts, 1.0)
    _, launches = _launched(lambda: pk.find_knn_with_fallback(g, 25, 15, 8))
    assert launches.get("brute_rows_kernel", 0) == 1, launches


def test_integer_data_wider_than_1024_columns_matches_oracle():
    """Byte-valued data with d = 1100: beyond the integer kernels' 1,024 columns
    the float64 policy is taken (not an error), outputs equal the oracle's."""
    rng = np.random.default_rng(11)
    mu = rng.integers(0, 256, (4, 1100))
    data = np.clip(mu[rng.integers(0, 4, 900)] + rng.integers(-20, 21, (900, 1100)), 0, 255).astype(np.float32)
    p = pk.PointSet(data)
    assert p.mode == _lib.MODE_SEQ64
    res = pk.run_pipeline(p, pk.VamanaConfig(R=16, L_build=32, L=32, alpha=1.2, seed=0), k=8, density_kind="kth",
                          center_policy=pk.ProductCenter(4), noise_policy=pk.NoisePolicy(0.0),
                          doubling_params=pk.DoublingParams(initial_k=16, threshold=20))
    ref = oracle.pipeline(data, index="vamana", R=16, L_build=32, L=32, alpha=1.2, seed=0, k=8, density_kind="kth",
                          center_policy=("product", 4), rho_min=0.0, initial_k=16, threshold=20)
    _assert_state_equal(res, ref)


# ---------------------------------------------------------------- beams wider than shared memory


def test_doubling_to_n_minus_1_spills_beam_and_matches_oracle():
    """threshold = 0 on C3-shaped data (every rho = 0, rank = id order): id 1
    stays unresolved until the doubling reaches k = n - 1 = 19,999,
    whose beam (12 B x L) no longer fits in shared memory and runs from the
    global slab (reference keeps doubling up to n - 1: dependent.py:118-126)."""
    n = 20_000
    data, _ = workloads.generate("C3", n=n, components=1)
    # id 0 (the only point denser than id 1) becomes id 1's farthest point, so
    # id 1 is resolved only by the round at k = n - 1
    far = int(np.argmax(((data.astype(np.float64) - data[1]) ** 2).sum(1)))
    data[[0, far]] = data[[far, 0]]
    res = pk.run_pipeline(pk.PointSet(data), pk.VamanaConfig(R=64, L_build=128, L=128, alpha=1.1, seed=0), k=32,
                          density_kind="exp_sum", center_policy=pk.ProductCenter(20), noise_policy=pk.NoisePolicy(0.0),
                          doubling_params=pk.DoublingParams(initial_k=64, threshold=0))
    ref = oracle.pipeline(data, index="vamana", R=64, L_build=128, L=128, alpha=1.1, seed=0, k=32,
                          density_kind="exp_sum", center_policy=("product", 20), rho_min=0.0, initial_k=64,
                          threshold=0)
    assert ref["rounds"][-1][1] == n - 1, ref["rounds"]
    _assert_state_equal(res, ref, exp_density=True)


@pytest.mark.parametrize("case", ["u8", "float"])
def test_spilled_beam_rows_match_oracle(case):
    """Beam kNN rows and a single vector search at L = 20,000 (past the shared
    memory opt-in) equal the oracle's."""
    if case == "u8":
        data, _ = workloads.generate("C3", n=24_000, components=6)
    else:
        data, _ = workloads.generate("C4", n=24_000, components=6)
    n = data.shape[0]
    p = pk.PointSet(data)
    g = pk.build_vamana(p, R=32, L_build=64, alpha=1.1, seed=0, query_beam=64).graph
    q = np.array([5, 777, 23_456], np.int64)
    width = 20_000
    ids, sqd, cnt = vamana.beam_knn_raw(g, _lib.to_dev(q), width, width)
    oi, od, oc = oracle.beam_knn_batch(data, g.adjacency, g.degrees, g.start_points, q, width, width)
    assert np.array_equal(_lib.to_host(cnt), oc)
    assert np.array_equal(_lib.to_host(ids), oi)
    assert np.array_equal(_lib.to_host(sqd), od)
    vec = data[:50].mean(0).astype(np.float64)
    nl, visited = pk.beam_search(g, vec, g.start_points, width, 300)
    ci, cd, vi, vd = oracle.beam_search_single(data, g.adjacency, g.degrees, g.start_points, vec, width)
    assert np.array_equal(nl.ids, ci[:300])
    assert np.array_equal(nl.dists, np.sqrt(cd[:300]))
    assert [v.id for v in visited] == list(vi)
