"""Graph index: beam search, RobustPrune and the batch build on the GPU
(mirrors /root/reference/pkg/src/peakann/vamana.py:35-267).

The search and build kernels live in csrc/beam.cuh, csrc/knn.cu and
csrc/build.cu; this module keeps the reference's API (names, parameters,
validation errors, return types) and owns host-side orchestration only:
the PCG64 start/permutation stream (so graphs can be bit-identical to the
reference's), argument checks, and the PECG file format.
"""

from __future__ import annotations

import hashlib
import struct

import numpy as np

from . import _lib
from .core import PointSet
from .index import (
    KnnIndex,
    Neighbor,
    NeighborList,
    Neighborhoods,
    Query,
    _as_query_vector,
    _padded_query,
    brute_device,
    brute_vector,
    sqrt_device,
)

__all__ = [
    "GraphIndex",
    "VamanaIndex",
    "beam_search",
    "robust_prune",
    "build_vamana",
    "find_knn_with_fallback",
    "save_graph",
    "load_graph",
]

GRAPH_MAGIC = b"PECG"

# Optional device counters (set by bench.py): "build" -> int64[4] (search
# evals, prune evals, reverse evals, expansions), "beam" -> int64[2]
# (evals, expansions) accumulated over every pipeline kNN query.
STATS = {"build": None, "beam": None}


def _digest(*arrays) -> bytes:
    h = hashlib.blake2b(digest_size=16)
    for a in arrays:
        h.update(np.ascontiguousarray(a).view(np.uint8).reshape(-1).data)
    return h.digest()


class GraphIndex:
    """Directed out-neighbour lists with degree bound R plus search seeds.

    Fields as in the reference dataclass (vamana.py:35-50).  Host arrays and
    device tensors are kept coherent: a graph built on the GPU exposes its
    numpy arrays lazily; host arrays handed to the caller may be mutated (the
    reference's tests do), so they are re-uploaded whenever their content
    changed since the last upload.
    """

    def __init__(self, points: PointSet, adjacency, degrees, R: int, start_points, alpha: float):
        self.points = points
        self.R = int(R)
        self.alpha = alpha
        self._adj = None if adjacency is None else np.ascontiguousarray(adjacency, dtype=np.int32)
        self._deg = None if degrees is None else np.ascontiguousarray(degrees, dtype=np.int32)
        self.start_points = np.asarray(start_points, dtype=np.int64)
        self._adj_t = None
        self._deg_t = None
        self._uploaded = None

    @classmethod
    def on_device(cls, points, adj_t, deg_t, R, start_points, alpha):
        g = cls(points, None, None, R, start_points, alpha)
        g._adj_t = adj_t
        g._deg_t = deg_t
        return g

    @property
    def adjacency(self) -> np.ndarray:
        if self._adj is None:
            self._adj = _lib.to_host(self._adj_t)
            self._uploaded = None
        return self._adj

    @adjacency.setter
    def adjacency(self, v):
        self._adj = np.ascontiguousarray(v, dtype=np.int32)
        self._adj_t = None

    @property
    def degrees(self) -> np.ndarray:
        if self._deg is None:
            self._deg = _lib.to_host(self._deg_t)
            self._uploaded = None
        return self._deg

    @degrees.setter
    def degrees(self, v):
        self._deg = np.ascontiguousarray(v, dtype=np.int32)
        self._deg_t = None

    def device_arrays(self):
        """(adj (n,R) int32, deg (n,) int32, starts (s,) int32) on device."""
        frozen = (self._uploaded == "read-only" and self._adj_t is not None and self._deg_t is not None
                  and not self._adj.flags.writeable and not self._deg.flags.writeable)
        if (self._adj is not None or self._deg is not None) and not frozen:
            adj, deg = self.adjacency, self.degrees
            dig = _digest(adj, deg)
            if self._adj_t is None or self._deg_t is None or dig != self._uploaded:
                self._adj_t = _lib.to_dev(adj, np.int32)
                self._deg_t = _lib.to_dev(deg, np.int32)
                self._uploaded = dig
        starts = getattr(self, "_starts_t", None)
        if starts is None or getattr(self, "_starts_src", None) is not self.start_points:
            self._starts_t = _lib.to_dev(np.asarray(self.start_points, np.int32))
            self._starts_src = self.start_points
        return self._adj_t, self._deg_t, self._starts_t

    def out_neighbors(self, i: int) -> np.ndarray:
        return self.adjacency[i, : self.degrees[i]].astype(np.int64)

    def max_degree(self) -> int:
        if self._deg is None and self._deg_t is not None:
            return int(self._deg_t.max().item())
        return int(self.degrees.max())

    def __repr__(self) -> str:
        return f"GraphIndex(n={self.points.n}, R={self.R}, starts={self.start_points.shape[0]}, alpha={self.alpha})"


def _normalize_starts(g: GraphIndex, starts) -> np.ndarray:
    arr = np.asarray(list(starts) if not isinstance(starts, np.ndarray) else starts, dtype=np.int64)
    if arr.ndim != 1 or arr.shape[0] == 0:
        raise ValueError("starts must be a non-empty set of point ids")
    for s in arr:
        g.points.check_id(int(s))
    return arr


def _single_search(g: GraphIndex, vec, qid: int, starts: np.ndarray, L: int, k: int):
    """pk_beam_search_single -> (top ids, top sqd, visit ids, visit sqd) on host."""
    import torch

    p = g.points
    adj, deg, _ = g.device_arrays()
    dev = _lib.device()
    st = _lib.to_dev(starts.astype(np.int32))
    top_i = torch.full((k,), -1, dtype=torch.int64, device=dev)
    top_d = torch.full((k,), float("inf"), dtype=torch.float64, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    vcap = p.n
    vis_i = torch.empty(vcap, dtype=torch.int64, device=dev)
    vis_d = torch.empty(vcap, dtype=torch.float64, device=dev)
    qvec = None if qid >= 0 else _padded_query(p, vec)
    _lib.call("pk_beam_search_single", p.device(), p.n, p.dp, adj, g.R, deg, st, starts.shape[0], qid, qvec, L, k,
              top_i, top_d, cnt[0:1], vis_i, vis_d, vcap, cnt[1:2], _lib.stream())
    c = _lib.to_host(cnt)
    got, vl = int(c[0]), min(int(c[1]), vcap)
    return (_lib.to_host(top_i[:got]), _lib.to_host(top_d[:got]), _lib.to_host(vis_i[:vl]), _lib.to_host(vis_d[:vl]))


def beam_search(g: GraphIndex, query: Query, starts, L: int, k: int) -> tuple[NeighborList, list[Neighbor]]:
    """Greedy beam search; the k best of beam-union-visited, and the visited set
    (vamana.py:62-84)."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    if L < k:
        raise ValueError(f"beam width L={L} must be >= k={k}")
    vec, qid = _as_query_vector(g.points, query)
    sarr = _normalize_starts(g, starts)
    ti, td, vi, vd = _single_search(g, vec, qid, sarr, L, k)
    visited = [Neighbor(int(i), float(d)) for i, d in zip(vi, np.sqrt(vd))]
    return NeighborList(ti, np.sqrt(td)), visited


def robust_prune(g: GraphIndex, p: int, candidates, alpha: float, R: int) -> np.ndarray:
    """New out-list for p: nearest-first selection with alpha-slack pruning
    (vamana.py:87-103)."""
    if alpha < 1.0:
        raise ValueError(f"alpha must be >= 1, got {alpha}")
    if R < 1:
        raise ValueError(f"R must be >= 1, got {R}")
    import torch

    p = g.points.check_id(p)
    cand = list(candidates)
    cand_ids = np.array([int(c.id) for c in cand], dtype=np.int64)
    cand_d = np.array([float(c.dist) ** 2 for c in cand], dtype=np.float64)
    adj, deg, _ = g.device_arrays()
    dcount = int(deg[p].item())
    cur = adj[p, :dcount].to(torch.int64).contiguous()
    dev = _lib.device()
    out = torch.empty(R, dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    ci = _lib.to_dev(cand_ids) if cand_ids.size else torch.empty(0, dtype=torch.int64, device=dev)
    cd = _lib.to_dev(cand_d) if cand_d.size else torch.empty(0, dtype=torch.float64, device=dev)
    pts = g.points
    _lib.call("pk_robust_prune", pts.device(), pts.n, pts.dp, p, ci, cd, cand_ids.shape[0], cur, dcount,
              float(alpha), R, out, cnt, _lib.stream())
    return _lib.to_host(out[: int(cnt.item())])


def sample_starts(n: int, num_starts, seed: int, medoid_start: bool, p: PointSet | None = None):
    """Start set and insertion order from one PCG64 stream, in the reference's
    draw order (vamana.py:132-143)."""
    rng = np.random.default_rng(seed)
    if medoid_start:
        import torch

        out = torch.zeros(1, dtype=torch.int64, device=_lib.device())
        _lib.call("pk_nearest_to_centroid", p.device(), p.n, p.dp, out, _lib.stream())
        starts = np.array([int(out.item())], dtype=np.int64)
    else:
        s = int(np.ceil(np.sqrt(n))) if num_starts is None else int(num_starts)
        if not 1 <= s <= n:
            raise ValueError(f"num_starts must be in [1, {n}], got {s}")
        starts = np.sort(rng.choice(n, size=s, replace=False).astype(np.int64))
    order = permutation_int32(rng, n)
    return starts, order


def permutation_int32(rng: np.random.Generator, n: int) -> np.ndarray:
    """rng.permutation(n) as int32 (the build's insertion order), drawn by the
    library's restatement of numpy's shuffle on the same PCG64 stream; the
    generator's state is advanced exactly as numpy would."""
    bg = rng.bit_generator
    st = bg.state
    if st.get("bit_generator") != "PCG64":
        return rng.permutation(n).astype(np.int32)
    mask = (1 << 64) - 1
    s, inc = st["state"]["state"], st["state"]["inc"]
    words = np.array([s >> 64, s & mask, inc >> 64, inc & mask], dtype=np.uint64)
    out = np.empty(n, dtype=np.int32)
    after = np.zeros(4, dtype=np.uint64)
    _lib.call_host("pk_pcg64_permutation", words.ctypes.data, int(st["has_uint32"]), int(st["uinteger"]), n,
                   out.ctypes.data, after.ctypes.data)
    st["state"]["state"] = (int(after[0]) << 64) | int(after[1])
    st["has_uint32"] = int(after[2])
    st["uinteger"] = int(after[3])
    bg.state = st
    return out


# batches smaller than this run replicated on every rank of a sharded build
MIN_SHARD_BATCH = 2048


def build_graph_device(p: PointSet, R: int, L_build: int, alpha: float, starts: np.ndarray, order: np.ndarray,
                       stats=None, order_t=None, starts_t=None, comm=None, seed_cache=False):
    """Run pk_build_vamana (or pk_build_vamana_sharded over `comm`); returns
    (adj_t, deg_t), plus the seeded-beam cache (seed slots, id words, lengths,
    L) with seed_cache=True on a single GPU (pk_build_vamana_seeds)."""
    import torch

    dev = _lib.device()
    adj = torch.empty((p.n, R), dtype=torch.int32, device=dev)
    deg = torch.empty(p.n, dtype=torch.int32, device=dev)
    st = starts_t if starts_t is not None else _lib.to_dev(starts.astype(np.int32))
    od = order_t if order_t is not None else _lib.to_dev(np.asarray(order, dtype=np.int32))
    if stats is None:
        stats = STATS["build"]
    if comm is None or comm.world == 1:
        if seed_cache:
            sbd = torch.empty((p.n, L_build), dtype=torch.float64, device=dev)
            sbi = torch.empty((p.n, L_build), dtype=torch.int32, device=dev)
            sbl = torch.empty(p.n, dtype=torch.int32, device=dev)
            _lib.call("pk_build_vamana_seeds", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, R, L_build,
                      float(alpha), st, st.shape[0], od, adj, deg, stats, 0, sbd, sbi, sbl, _lib.stream())
            return adj, deg, (sbd, sbi, sbl, int(L_build))
        _lib.call("pk_build_vamana", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, R, L_build, float(alpha), st,
                  st.shape[0], od, adj, deg, stats, 0, _lib.stream())
        return adj, deg
    from .shard import BuildExchange

    ex = BuildExchange(comm, p.n, R, dev)
    try:
        _lib.call("pk_build_vamana_sharded", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, R, L_build,
                  float(alpha), st, st.shape[0], od, adj, deg, stats, 0, comm.rank, comm.world, MIN_SHARD_BATCH,
                  *ex.pointers(), _lib.stream())
    except RuntimeError:
        if ex.error is not None:
            raise ex.error from None
        raise
    return adj, deg


def build_vamana(
    p: PointSet,
    R: int = 32,
    L_build: int = 32,
    alpha: float = 1.1,
    num_starts: int | None = None,
    seed: int = 42,
    medoid_start: bool = False,
    query_beam: int | None = None,
    comm=None,
) -> "VamanaIndex":
    """Construct the search graph by batched insertion of doubling size
    (vamana.py:106-172), entirely on the GPU."""
    if R < 2:
        raise ValueError(f"R must be >= 2, got {R}")
    if L_build < 1:
        raise ValueError(f"L_build must be >= 1, got {L_build}")
    if alpha < 1.0:
        raise ValueError(f"alpha must be >= 1, got {alpha}")
    starts, order = sample_starts(p.n, num_starts, seed, medoid_start, p)
    qb = query_beam if query_beam is not None else L_build
    single = comm is None or comm.world == 1
    # the seeded beams of the build are reused by member queries with L == L_build
    res = build_graph_device(p, R, L_build, alpha, starts, order, comm=comm, seed_cache=single and qb == L_build)
    graph = GraphIndex.on_device(p, res[0], res[1], R, starts, float(alpha))
    if len(res) == 3:
        graph._seed_cache = res[2]
        graph._seed_src = graph.start_points
    return VamanaIndex(graph, qb)


def _seed_cache(g: "GraphIndex", L: int):
    """The build's seeded beams when they apply to a search with beam width L
    from the graph's current start list, else None."""
    c = getattr(g, "_seed_cache", None)
    if c is None or c[3] != L or getattr(g, "_seed_src", None) is not g.start_points:
        return None
    return c


def beam_knn_raw(g: GraphIndex, qids_t, L: int, k: int, evals=None, hash_bits: int = 0):
    """_kernels.beam_knn_batch on device, without the exact fallback:
    (ids_t, sqd_t, counts_t)."""
    import torch

    p = g.points
    adj, deg, st = g.device_arrays()
    m = qids_t.shape[0]
    kk = max(0, min(k, p.n - 1))
    dev = qids_t.device
    ids = torch.empty((m, kk), dtype=torch.int64, device=dev)
    sqd = torch.empty((m, kk), dtype=torch.float64, device=dev)
    counts = torch.zeros(m, dtype=torch.int64, device=dev)
    if kk > 0 and m > 0:
        c = _seed_cache(g, L)
        if c is not None:
            _lib.call("pk_beam_knn_seeded", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, adj, g.R, deg, st,
                      st.shape[0], qids_t, m, L, k, ids, sqd, counts, 0, evals, hash_bits, c[0], c[1], c[2],
                      _lib.stream())
        else:
            _lib.call("pk_beam_knn", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, adj, g.R, deg, st, st.shape[0],
                      qids_t, m, L, k, ids, sqd, counts, 0, evals, hash_bits, _lib.stream())
    return ids, sqd, counts


def beam_knn_device(g: GraphIndex, qids_t, k: int, L: int, evals=None):
    """Member-query beam kNN with the exact fallback for short rows
    (_kernels.beam_knn_batch + vamana.py:220-225).  Returns (ids_t, sqd_t)."""
    import torch

    if evals is None:
        evals = STATS["beam"]
    p = g.points
    adj, deg, st = g.device_arrays()
    m = qids_t.shape[0]
    kk = max(0, min(k, p.n - 1))
    dev = qids_t.device
    ids = torch.empty((m, kk), dtype=torch.int64, device=dev)
    sqd = torch.empty((m, kk), dtype=torch.float64, device=dev)
    counts = torch.empty(m, dtype=torch.int64, device=dev)
    if kk > 0 and m > 0:
        c = _seed_cache(g, L)
        if c is not None:
            _lib.call("pk_beam_knn_seeded", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, adj, g.R, deg, st,
                      st.shape[0], qids_t, m, L, k, ids, sqd, counts, 1, evals, 0, c[0], c[1], c[2], _lib.stream())
        else:
            _lib.call("pk_beam_knn", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, adj, g.R, deg, st, st.shape[0],
                      qids_t, m, L, k, ids, sqd, counts, 1, evals, 0, _lib.stream())
    return ids, sqd


def find_knn_with_fallback(g: GraphIndex, query: Query, k: int, L: int) -> NeighborList:
    """Beam-search kNN with L = max(L, k); exact if it comes up short
    (vamana.py:175-197)."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    L = max(L, k)
    vec, qid = _as_query_vector(g.points, query)
    n = g.points.n
    want = min(k, n - 1) if qid >= 0 else min(k, n)
    ti, td, _, _ = _single_search(g, vec, qid, g.start_points, L, k)
    if ti.shape[0] < want:
        if qid >= 0:
            ids, sqd = brute_device(g.points, _lib.to_dev(np.array([qid], np.int64)), k)
            return NeighborList(_lib.to_host(ids[0]), _lib.to_host(sqrt_device(sqd[0])))
        ids, sqd = brute_vector(g.points, vec, k)
        return NeighborList(_lib.to_host(ids), _lib.to_host(sqrt_device(sqd)))
    return NeighborList(ti, np.sqrt(td))


class VamanaIndex(KnnIndex):
    """KnnIndex adapter: beam queries over a built graph, with exact fallback."""

    def __init__(self, graph: GraphIndex, query_beam: int):
        if query_beam < 1:
            raise ValueError(f"query_beam must be >= 1, got {query_beam}")
        self.graph = graph
        self.points = graph.points
        self.query_beam = query_beam

    def find_knn(self, query: Query, k: int) -> NeighborList:
        return find_knn_with_fallback(self.graph, query, k, self.query_beam)

    def knn_batch_device(self, qids_t, k: int, evals=None):
        return beam_knn_device(self.graph, qids_t, k, max(self.query_beam, k), evals)

    def knn_rows_raw(self, qids_t, k: int):
        """Beam rows without the exact fallback: (ids_t, sqd_t, counts_t);
        rows with counts < kk are left for the caller (dependent rounds)."""
        return beam_knn_raw(self.graph, qids_t, max(self.query_beam, k), k, STATS["beam"])

    def knn_batch(self, qids: np.ndarray, k: int) -> Neighborhoods:
        if k < 1:
            raise ValueError(f"k must be >= 1, got {k}")
        ids, sqd = self.knn_batch_device(_lib.to_dev(np.asarray(qids, np.int64)), k)
        return Neighborhoods.on_device(ids, sqrt_device(sqd))


def save_graph(g: GraphIndex, path) -> None:
    """PECG: magic, u32 n/R/num_starts, u32 start ids, then per vertex a u32
    degree followed by its u32 neighbour ids, little-endian (vamana.py:229-240)."""
    n = g.points.n
    adj, deg = g.adjacency, g.degrees.astype(np.int64)
    with open(path, "wb") as f:
        f.write(GRAPH_MAGIC)
        f.write(struct.pack("<III", n, g.R, g.start_points.shape[0]))
        f.write(g.start_points.astype("<u4").tobytes())
        # interleave degree + row prefix per vertex without a Python loop
        width = deg + 1
        off = np.concatenate([[0], np.cumsum(width)])
        buf = np.empty(int(off[-1]), dtype="<u4")
        buf[off[:-1]] = deg
        cols = np.arange(g.R)
        mask = cols[None, :] < deg[:, None]
        pos = (off[:-1, None] + 1 + cols[None, :])[mask]
        buf[pos] = adj[mask].astype("<u4")
        f.write(buf.tobytes())


def load_graph(path, points: PointSet, alpha: float = 1.0) -> GraphIndex:
    """Read a graph written by save_graph (format and errors of vamana.py:243-267).

    The vertex records are parsed by one native pass (pk_parse_pecg) straight
    into pinned host buffers, then uploaded once; the returned host arrays are
    read-only views of those buffers (the device copy stays authoritative)."""
    with open(path, "rb") as f:
        head = f.read(16)
        if head[:4] != GRAPH_MAGIC:
            raise ValueError(f"{path}: bad magic {head[:4]!r}")
        if len(head) < 16:
            raise ValueError(f"{path}: truncated header")
        n, R, ns = struct.unpack_from("<III", head, 4)
        if n != points.n:
            raise ValueError(f"{path}: graph has {n} vertices but points has {points.n}")
        starts_raw = f.read(4 * ns)
        if len(starts_raw) != 4 * ns:
            raise ValueError(f"{path}: truncated start list")
        body = f.read()
    starts = np.frombuffer(starts_raw, "<u4").astype(np.int64)
    words = np.frombuffer(body, "<u4", len(body) // 4)
    odd = len(body) % 4
    pinned = _host_cuda()
    if pinned:
        import torch

        adj_h = torch.empty((n, R), dtype=torch.int32, pin_memory=True)
        deg_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
        adj, deg = adj_h.numpy(), deg_h.numpy()
    else:
        adj = np.empty((n, R), np.int32)
        deg = np.empty(n, np.int32)
    info = np.zeros(2, np.int64)
    rc = _lib.lib().pk_parse_pecg(words.ctypes.data, words.shape[0], n, R, adj.ctypes.data, deg.ctypes.data,
                                  info.ctypes.data)
    if rc == 3:
        raise ValueError(f"{path}: truncated at vertex {info[0]}")
    if rc == 4:
        raise ValueError(f"{path}: vertex {info[0]} degree {info[1]} exceeds bound {R}")
    if rc == 5 or (rc == 0 and odd):
        raise ValueError(f"{path}: {int(info[0]) + odd if rc == 5 else odd} trailing bytes")
    if rc != 0:
        raise RuntimeError(f"pk_parse_pecg failed ({rc})")
    g = GraphIndex(points, adj, deg, R, starts, alpha)
    if pinned:
        g._adj_t = adj_h.to(_lib.device(), non_blocking=True)
        g._deg_t = deg_h.to(_lib.device(), non_blocking=True)
        adj.flags.writeable = False
        deg.flags.writeable = False
        g._uploaded = "read-only"
    return g


def _host_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False
