"""Host-side logic that needs no GPU: API surface, validation errors, the PCG64
start stream, the PECG format, metrics, and the no-CPU-fallback rule."""

import numpy as np
import pytest

from conftest import FIG_COORDS, golden, has_gpu

import paper_2312_03940_b200 as pk
from paper_2312_03940_b200 import vamana, workloads

REFERENCE_EXPORTS = {
    "PointSet", "distance", "squared_distance", "Neighbor", "NeighborList", "Neighborhoods", "KnnIndex",
    "BruteForceIndex", "build_bruteforce", "find_knn", "knn_all", "GraphIndex", "VamanaIndex", "beam_search",
    "robust_prune", "build_vamana", "find_knn_with_fallback", "save_graph", "load_graph", "compute_densities",
    "rank_order", "DoublingParams", "Dependents", "dp_brute_force", "compute_dependent_points", "NoisePolicy",
    "ThresholdCenter", "ProductCenter", "LocalCenter", "BruteForceConfig", "VamanaConfig", "Clustering",
    "DpcState", "PipelineResult", "find_noise", "find_centers_threshold", "find_centers_product",
    "find_centers_local", "assign_clusters", "run_pipeline", "reapply_policies",
}


def test_hot_path_api_names_present():
    missing = [n for n in REFERENCE_EXPORTS if not hasattr(pk, n)]
    assert not missing


def test_pointset_validation():
    with pytest.raises(ValueError):
        pk.PointSet(np.zeros(3, np.float32))
    with pytest.raises(ValueError):
        pk.PointSet(np.zeros((0, 2), np.float32))
    with pytest.raises(ValueError, match="non-finite"):
        pk.PointSet(np.array([[0.0, np.nan]], np.float32))
    p = pk.PointSet(FIG_COORDS)
    assert (p.n, p.d, p.dp) == (6, 2, 4)
    with pytest.raises(IndexError):
        p.check_id(6)
    assert not p.data.flags.writeable


def test_scalar_distance_matches_reference_order():
    p = pk.PointSet(FIG_COORDS)
    assert pk.squared_distance(p, 3, 2) == 9.0
    assert pk.distance(p, 0, 2) == np.sqrt(2.0)


def test_doubling_params_validation():
    with pytest.raises(ValueError):
        pk.DoublingParams(initial_k=1).validated_against(1)
    with pytest.raises(ValueError):
        pk.DoublingParams(initial_k=4, threshold=-1).validated_against(2)
    assert pk.DoublingParams(initial_k=4).validated_against(2).threshold == 300


def test_start_stream_matches_reference_graphs():
    """Starts and insertion order come from one PCG64 stream in the reference's
    draw order (vamana.py:132-143): the sampled starts equal the golden ones."""
    z = golden("graphs")
    for tag in {k.split("__")[0] for k in z.files if k.endswith("__adj")}:
        R, L, seed, ns, medoid = (int(v) for v in z[f"{tag}__params"])
        if medoid:
            continue
        n = z[f"{tag}__data"].shape[0]
        starts, order = vamana.sample_starts(n, None if ns < 0 else ns, seed, False)
        assert np.array_equal(starts, z[f"{tag}__starts"]), tag
        assert sorted(order.tolist()) == list(range(n))


def test_num_starts_validation():
    with pytest.raises(ValueError):
        vamana.sample_starts(6, 0, 0, False)
    with pytest.raises(ValueError):
        vamana.sample_starts(6, 7, 0, False)


def test_build_parameter_validation_before_any_device_work():
    p = pk.PointSet(FIG_COORDS)
    with pytest.raises(ValueError):
        pk.build_vamana(p, R=1)
    with pytest.raises(ValueError):
        pk.build_vamana(p, alpha=0.9)
    with pytest.raises(ValueError):
        pk.build_vamana(p, L_build=0)


def _fig_graph():
    p = pk.PointSet(FIG_COORDS)
    adj = np.full((6, 4), -1, np.int32)
    deg = np.zeros(6, np.int32)
    for u, v in [(5, 3), (3, 4), (5, 2), (2, 1), (0, 1)]:
        adj[u, deg[u]] = v
        deg[u] += 1
        adj[v, deg[v]] = u
        deg[v] += 1
    return pk.GraphIndex(p, adj, deg, 4, np.array([0], np.int64), 1.0)


def test_pecg_round_trip(tmp_path):
    g = _fig_graph()
    path = tmp_path / "g.bin"
    pk.save_graph(g, path)
    blob = path.read_bytes()
    assert blob[:4] == b"PECG"
    assert tuple(np.frombuffer(blob, "<u4", 3, 4)) == (6, 4, 1)
    back = pk.load_graph(path, g.points, alpha=1.0)
    assert back.R == 4
    assert np.array_equal(back.adjacency, g.adjacency)
    assert np.array_equal(back.degrees, g.degrees)
    assert np.array_equal(back.start_points, g.start_points)


def test_pecg_errors(tmp_path):
    g = _fig_graph()
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOPE" + b"\x00" * 16)
    with pytest.raises(ValueError, match="magic"):
        pk.load_graph(bad, g.points)
    path = tmp_path / "g.bin"
    pk.save_graph(g, path)
    with pytest.raises(ValueError, match="vertices"):
        pk.load_graph(path, pk.PointSet(np.zeros((2, 2), np.float32)))
    good = path.read_bytes()
    path.write_bytes(good + b"\x00\x00\x00\x00")
    with pytest.raises(ValueError, match="trailing"):
        pk.load_graph(path, g.points)
    path.write_bytes(good + b"\x00\x00")
    with pytest.raises(ValueError, match="2 trailing bytes"):
        pk.load_graph(path, g.points)
    path.write_bytes(good[:-4])
    with pytest.raises(ValueError, match="truncated"):
        pk.load_graph(path, g.points)
    # vertex 0's degree word (after the 16-byte header and one start id) set past R
    blob = bytearray(good)
    blob[20:24] = (9).to_bytes(4, "little")
    path.write_bytes(bytes(blob))
    with pytest.raises(ValueError, match="vertex 0 degree 9 exceeds bound 4"):
        pk.load_graph(path, g.points)


def test_pecg_parse_matches_python_loop(tmp_path):
    """pk_parse_pecg equals the reference's per-vertex loop (vamana.py:253-264)
    on a random graph with ragged degrees."""
    import struct

    rng = np.random.default_rng(5)
    n, R = 500, 12
    p = pk.PointSet(rng.normal(size=(n, 3)).astype(np.float32))
    deg = rng.integers(0, R + 1, n).astype(np.int32)
    adj = np.full((n, R), -1, np.int32)
    for i in range(n):
        adj[i, : deg[i]] = rng.choice(n, deg[i], replace=False)
    g = pk.GraphIndex(p, adj, deg, R, np.array([3, 9], np.int64), 1.0)
    path = tmp_path / "r.bin"
    pk.save_graph(g, path)
    blob = path.read_bytes()
    off = 16 + 8
    want_adj = np.full((n, R), -1, np.int32)
    want_deg = np.zeros(n, np.int32)
    for i in range(n):
        (d,) = struct.unpack_from("<I", blob, off)
        want_adj[i, :d] = np.frombuffer(blob, "<u4", d, off + 4).astype(np.int32)
        want_deg[i] = d
        off += 4 + 4 * d
    back = pk.load_graph(path, p)
    assert np.array_equal(back.adjacency, want_adj)
    assert np.array_equal(back.degrees, want_deg)


def test_metrics():
    assert pk.ari([0, 0, 1, 1], [0, 1, 0, 1]) == -0.5
    assert pk.ari([1, 1, 2, 2], [5, 5, 7, 7]) == 1.0
    rng = np.random.default_rng(0)
    a, b = rng.integers(0, 4, 60), rng.integers(0, 3, 60)
    # brute pair counting
    n = 60
    sa = sb = sab = 0
    for i in range(n):
        for j in range(i + 1, n):
            x, y = a[i] == a[j], b[i] == b[j]
            sa += x
            sb += y
            sab += x and y
    tot = n * (n - 1) // 2
    exp = sa * sb / tot
    want = (sab - exp) / ((sa + sb) / 2 - exp)
    assert abs(pk.ari(a, b) - want) < 1e-12
    h, c = pk.homogeneity_completeness([0, 0, 1, 1], [0, 0, 1, 1])
    assert h == pytest.approx(1.0) and c == pytest.approx(1.0)


def test_workload_generators_are_deterministic():
    a, la = workloads.generate("C2", n=500, components=5)
    b, lb = workloads.generate("C2", n=500, components=5)
    assert np.array_equal(a, b) and np.array_equal(la, lb)
    assert a.dtype == np.float32 and a.min() >= 0 and a.max() <= 255 and np.all(a == np.round(a))
    x, _ = workloads.generate("C4", n=300, components=7)
    assert np.allclose(np.linalg.norm(x.astype(np.float64), axis=1), 1.0, atol=1e-6)
    kw = workloads.pipeline_args("C2", pk)
    assert kw["k"] == 16 and kw["density_kind"] == "kth_normalized"
    assert kw["doubling_params"].initial_k == 32


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_product_path_fails_loudly_without_gpu():
    with pytest.raises(RuntimeError, match="CUDA"):
        pk.build_bruteforce(pk.PointSet(FIG_COORDS)).knn_all(1)


def test_permutation_matches_numpy_stream():
    """The library's PCG64 shuffle (int32 insertion order) equals numpy's
    Generator.permutation and leaves the generator in the same state."""
    from paper_2312_03940_b200 import vamana

    for seed in (0, 1, 42, 2**40 + 7):
        for n in (1, 2, 3, 17, 1000, 70_001):
            a = np.random.default_rng(seed)
            b = np.random.default_rng(seed)
            a.choice(max(n, 1), size=1, replace=False)  # odd number of 32-bit halves drawn first
            b.choice(max(n, 1), size=1, replace=False)
            got = vamana.permutation_int32(a, n)
            want = b.permutation(n)
            assert got.dtype == np.int32
            assert np.array_equal(got, want), (seed, n)
            assert a.bit_generator.state == b.bit_generator.state
            assert a.integers(0, 2**62) == b.integers(0, 2**62)
