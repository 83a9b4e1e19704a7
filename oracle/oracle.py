"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the density-peaks hot path.

This module restates the reference `peakann` algorithm on the CPU so the
CUDA path can be checked on machines where `/root/reference` does not exist
(the GPU box).  The compiled part lives in `oracle.c` (a C restatement of
/root/reference/pkg/src/peakann/_kernels.py); the numpy part below restates
the Python-level stages:

  densities        density.py:26-55, 92-113
  rank order       density.py:116-129
  dependents       dependent.py:80-133
  policies         cluster.py:134-180, 223-254
  assignment       cluster.py:183-220 (restated as chain walking, as the
                   reference's own tests/oracles.py:104-134 does)
  pipeline         cluster.py:279-311

Only tests/, __graft_entry__.smoke() and bench.py's CPU baseline leg import
this.  It is pinned against vectors produced by the reference itself
(tests/golden/, made by tests/golden/make_golden.py; checked in
tests/test_oracle.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
import warnings

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_I = ctypes.c_int64


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.or_point_sqdist.argtypes = [_f32p, _I, _I, _I]
        L.or_point_sqdist.restype = ctypes.c_double
        L.or_brute_knn_batch.argtypes = [_f32p, _I, _I, _i64p, _I, _I, _i64p, _f64p]
        L.or_brute_knn_vector.argtypes = [_f32p, _I, _I, _f64p, _I, _i64p, _f64p]
        L.or_beam_search_single.argtypes = [_f32p, _I, _I, _i32p, _I, _i32p, _i64p, _I, _f64p, _I,
                                            _i64p, _f64p, _i64p, _f64p, ctypes.POINTER(_I)]
        L.or_beam_search_single.restype = _I
        L.or_beam_knn_batch.argtypes = [_f32p, _I, _I, _i32p, _I, _i32p, _i64p, _I, _i64p, _I, _I, _I,
                                        _i64p, _f64p, _i64p, ctypes.POINTER(_I)]
        L.or_robust_prune.argtypes = [_f32p, _I, _I, _I, _i64p, _f64p, _I, _i64p, _I, ctypes.c_double, _I, _i64p]
        L.or_robust_prune.restype = _I
        L.or_build_vamana.argtypes = [_f32p, _I, _I, _I, _I, ctypes.c_double, _i64p, _I, _i64p, _i32p, _i32p]
        L.or_nearest_to_centroid.argtypes = [_f32p, _I, _I]
        L.or_nearest_to_centroid.restype = _I
        L.or_dp_scan_all.argtypes = [_f32p, _I, _I, _i64p, _i64p, _I, _i64p, _f64p]
        L.or_num_threads.restype = ctypes.c_int
        L.or_set_num_threads.argtypes = [ctypes.c_int]
        _LIB = L
    return _LIB


def num_threads() -> int:
    return int(lib().or_num_threads())


def set_num_threads(t: int) -> None:
    lib().or_set_num_threads(int(t))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# ---------------------------------------------------------------------------
# compiled kernels (oracle.c)


def point_sqdist(data, i, j) -> float:
    data = _f32(data)
    return float(lib().or_point_sqdist(data, data.shape[1], int(i), int(j)))


def brute_knn_batch(data, qids, k):
    data = _f32(data)
    qids = _i64(qids)
    n, d = data.shape
    kk = max(0, min(k, n - 1))
    ids = np.full((qids.shape[0], kk), -1, np.int64)
    sqd = np.full((qids.shape[0], kk), np.inf, np.float64)
    if kk > 0 and qids.shape[0] > 0:
        lib().or_brute_knn_batch(data, n, d, qids, qids.shape[0], k, ids, sqd)
    return ids, sqd


def brute_knn_vector(data, q, k):
    data = _f32(data)
    n, d = data.shape
    kk = min(k, n)
    ids = np.full(kk, -1, np.int64)
    sqd = np.full(kk, np.inf, np.float64)
    lib().or_brute_knn_vector(data, n, d, np.ascontiguousarray(q, np.float64), k, ids, sqd)
    return ids, sqd


def beam_search_single(data, adj, deg, starts, q, L):
    data = _f32(data)
    n, d = data.shape
    ci = np.empty(n + 1, np.int64)
    cd = np.empty(n + 1, np.float64)
    vi = np.empty(n + 1, np.int64)
    vd = np.empty(n + 1, np.float64)
    vl = _I(0)
    adj = np.ascontiguousarray(adj, np.int32)
    c = lib().or_beam_search_single(data, n, d, adj, adj.shape[1], np.ascontiguousarray(deg, np.int32),
                                    _i64(starts), len(starts), np.ascontiguousarray(q, np.float64), L,
                                    ci, cd, vi, vd, ctypes.byref(vl))
    return ci[:c].copy(), cd[:c].copy(), vi[: vl.value].copy(), vd[: vl.value].copy()


def beam_knn_batch(data, adj, deg, starts, qids, L, k, return_evals=False):
    data = _f32(data)
    qids = _i64(qids)
    n, d = data.shape
    kk = max(0, min(k, n - 1))
    m = qids.shape[0]
    ids = np.full((m, kk), -1, np.int64)
    sqd = np.full((m, kk), np.inf, np.float64)
    counts = np.zeros(m, np.int64)
    ev = _I(0)
    adj = np.ascontiguousarray(adj, np.int32)
    if kk > 0 and m > 0:
        lib().or_beam_knn_batch(data, n, d, adj, adj.shape[1], np.ascontiguousarray(deg, np.int32),
                                _i64(starts), len(starts), qids, m, L, k, ids, sqd, counts, ctypes.byref(ev))
    if return_evals:
        return ids, sqd, counts, int(ev.value)
    return ids, sqd, counts


def robust_prune(data, p, cand_ids, cand_sqd, cur_ids, alpha, R):
    data = _f32(data)
    n, d = data.shape
    out = np.empty(max(R, 1), np.int64)
    sel = lib().or_robust_prune(data, n, d, int(p), _i64(cand_ids), np.ascontiguousarray(cand_sqd, np.float64),
                                len(cand_ids), _i64(cur_ids), len(cur_ids), float(alpha), R, out)
    return out[:sel].copy()


def sample_starts(n, num_starts, seed, medoid_start=False, data=None):
    """Start set and insertion order from one PCG64 stream (vamana.py:132-143)."""
    rng = np.random.default_rng(seed)
    if medoid_start:
        starts = np.array([nearest_to_centroid(data)], np.int64)
    else:
        s = int(np.ceil(np.sqrt(n))) if num_starts is None else int(num_starts)
        if not 1 <= s <= n:
            raise ValueError(f"num_starts must be in [1, {n}], got {s}")
        starts = np.sort(rng.choice(n, size=s, replace=False).astype(np.int64))
    order = rng.permutation(n).astype(np.int64)
    return starts, order


def build_vamana(data, R=32, L_build=32, alpha=1.1, num_starts=None, seed=42, medoid_start=False):
    """(adjacency (n,R) int32, degrees (n,) int32, starts (s,) int64)."""
    data = _f32(data)
    n, d = data.shape
    starts, order = sample_starts(n, num_starts, seed, medoid_start, data)
    adj = np.full((n, R), -1, np.int32)
    deg = np.zeros(n, np.int32)
    lib().or_build_vamana(data, n, d, R, L_build, float(alpha), starts, len(starts), order, adj, deg)
    return adj, deg, starts


def nearest_to_centroid(data) -> int:
    data = _f32(data)
    return int(lib().or_nearest_to_centroid(data, data.shape[0], data.shape[1]))


def dp_scan_all(data, rank, qids):
    data = _f32(data)
    qids = _i64(qids)
    m = qids.shape[0]
    out_id = np.full(m, -1, np.int64)
    out_d = np.full(m, np.inf, np.float64)
    if m:
        lib().or_dp_scan_all(data, data.shape[0], data.shape[1], _i64(rank), qids, m, out_id, out_d)
    return out_id, out_d


# ---------------------------------------------------------------------------
# index adapters (index.py:115-139, vamana.py:200-226)


class BruteIndex:
    def __init__(self, data):
        self.data = _f32(data)

    def knn_batch(self, qids, k):
        ids, sqd = brute_knn_batch(self.data, qids, k)
        return ids, np.sqrt(sqd)


class GraphIndexOracle:
    def __init__(self, data, adj, deg, starts, query_beam):
        self.data = _f32(data)
        self.adj = np.ascontiguousarray(adj, np.int32)
        self.deg = np.ascontiguousarray(deg, np.int32)
        self.starts = _i64(starts)
        self.query_beam = query_beam

    def knn_batch(self, qids, k):
        qids = _i64(qids)
        L = max(self.query_beam, k)
        ids, sqd, counts = beam_knn_batch(self.data, self.adj, self.deg, self.starts, qids, L, k)
        short = np.flatnonzero(counts < ids.shape[1])
        if short.shape[0]:
            bi, bs = brute_knn_batch(self.data, qids[short], k)
            ids[short] = bi
            sqd[short] = bs
        return ids, np.sqrt(sqd)


# ---------------------------------------------------------------------------
# numpy stages


def densities(kind, ids, dists):
    """rho for every point from its kNN row (density.py:29-55, 92-113)."""
    k = dists.shape[1]
    if kind == "kth":
        with np.errstate(divide="ignore"):
            return 1.0 / dists[:, -1]
    if kind == "kth_normalized":
        base = densities("kth", ids, dists)
        s = base[ids].sum(axis=1)
        with np.errstate(divide="ignore", invalid="ignore"):
            r = base * k / s
        r[s == 0.0] = np.inf
        r[np.isnan(r)] = np.inf
        return r
    if kind == "exp_sum":
        return np.exp(-(dists * dists).sum(axis=1) / k)
    if kind == "sum_exp":
        return np.exp(-(dists * dists)).sum(axis=1) / k
    if kind == "sum":
        return -dists.sum(axis=1)
    raise ValueError(kind)


def rank_order(rho):
    n = rho.shape[0]
    order = np.lexsort((np.arange(n), -rho))
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n, 0, -1)
    return rank


def _first_denser(rank, qids, ids, dists, lam, delta):
    if ids.shape[1] == 0:
        return qids
    ok = rank[ids] > rank[qids][:, None]
    any_ok = ok.any(axis=1)
    col = ok.argmax(axis=1)
    hit = qids[any_ok]
    lam[hit] = ids[any_ok, col[any_ok]]
    delta[hit] = dists[any_ok, col[any_ok]]
    return qids[~any_ok]


def dependents(index, data, rho, nbr_ids, nbr_dists, initial_k, threshold, trace=None):
    """(lam, delta) by the three-phase doubling search (dependent.py:96-133)."""
    n = rho.shape[0]
    rank = rank_order(rho)
    lam = np.full(n, -1, np.int64)
    delta = np.full(n, np.inf)
    top = int(np.argmax(rank))
    todo = _first_denser(rank, np.arange(n, dtype=np.int64), nbr_ids, nbr_dists, lam, delta)
    todo = todo[todo != top]
    if n > 1:
        if initial_k <= nbr_ids.shape[1]:
            raise ValueError("initial_k must be > k")
        kd = initial_k
        while todo.shape[0] > threshold:
            kq = min(kd, n - 1)
            if trace is not None:
                trace.append((int(todo.shape[0]), kq))
            ids, dists = index.knn_batch(todo, kq)
            todo = _first_denser(rank, todo, ids, dists, lam, delta)
            if kq >= n - 1:
                break
            kd *= 2
    if todo.shape[0]:
        sid, ssq = dp_scan_all(data, rank, todo)
        lam[todo] = sid
        delta[todo] = np.sqrt(ssq)
    return lam, delta


def _products(rho, delta, ids):
    dl = delta[ids]
    with np.errstate(invalid="ignore"):
        pr = dl * rho[ids]
    pr[np.isinf(dl)] = np.inf
    bad = np.isnan(pr)
    pr[bad] = np.where(dl[bad] == 0.0, 0.0, np.inf)
    return pr


def select_centers(policy, rho, lam, delta, nbr_ids, non_noise):
    """policy = ("threshold", dmin) | ("product", n_c) | ("local", None)."""
    kind, arg = policy
    if kind == "threshold":
        return np.sort(non_noise[delta[non_noise] >= arg])
    if kind == "product":
        if arg < 1:
            raise ValueError("n_c must be >= 1")
        if arg >= non_noise.shape[0]:
            if arg > non_noise.shape[0]:
                warnings.warn("requested more centers than non-noise points", stacklevel=2)
            return np.sort(non_noise)
        pr = _products(rho, delta, non_noise)
        o = np.lexsort((non_noise, -delta[non_noise], -pr))
        return np.sort(non_noise[o[:arg]])
    if kind == "local":
        rank = rank_order(rho)
        best = rank[nbr_ids].max(axis=1)
        return np.sort(non_noise[rank[non_noise] > best[non_noise]])
    raise ValueError(kind)


def label_forest(lam, centers, noise):
    """Canonical labels by walking each dependency chain to its first center
    or noise point (restates cluster.py:183-220's outcome without union-find)."""
    n = lam.shape[0]
    stop = np.zeros(n, bool)
    stop[centers] = True
    stop[noise] = True
    labels = np.where(stop, np.arange(n), -1)
    for i in range(n):
        if labels[i] >= 0:
            continue
        chain = []
        j = i
        while labels[j] < 0:
            chain.append(j)
            j = int(lam[j])
            if j < 0 or len(chain) > n:
                raise RuntimeError(f"point {chain[-1]} has no center on its dependency chain")
        labels[chain] = labels[j]
    return labels


def apply_policies(rho, lam, delta, nbr_ids, center_policy, rho_min):
    n = rho.shape[0]
    noise = np.flatnonzero(rho < rho_min).astype(np.int64)
    is_noise = np.zeros(n, bool)
    is_noise[noise] = True
    non_noise = np.flatnonzero(~is_noise).astype(np.int64)
    centers = select_centers(center_policy, rho, lam, delta, nbr_ids, non_noise)
    orphans = np.flatnonzero(lam < 0)
    extra = orphans[~is_noise[orphans] & ~np.isin(orphans, centers)]
    if extra.shape[0]:
        centers = np.sort(np.concatenate([centers, extra]))
    return label_forest(lam, centers, noise), centers, noise


def pipeline(data, index="vamana", R=32, L_build=32, L=32, alpha=1.1, num_starts=None, seed=42,
             medoid_start=False, k=16, density_kind="kth", center_policy=("product", 10), rho_min=0.0,
             initial_k=None, threshold=300):
    """End-to-end CPU pipeline (cluster.py:279-311). Returns a dict with the
    stage timings under the reference's keys."""
    data = _f32(data)
    n = data.shape[0]
    if initial_k is None:
        initial_k = 2 * k
    t0 = time.perf_counter()
    out = {}
    if index == "vamana":
        adj, deg, starts = build_vamana(data, R, L_build, alpha, num_starts, seed, medoid_start)
        idx = GraphIndexOracle(data, adj, deg, starts, L)
        out.update(adjacency=adj, degrees=deg, starts=starts)
    else:
        idx = BruteIndex(data)
    t1 = time.perf_counter()
    ids, dists = idx.knn_batch(np.arange(n, dtype=np.int64), k)
    rho = densities(density_kind, ids, dists)
    t2 = time.perf_counter()
    trace = []
    lam, delta = dependents(idx, data, rho, ids, dists, initial_k, threshold, trace)
    t3 = time.perf_counter()
    labels, centers, noise = apply_policies(rho, lam, delta, ids, center_policy, rho_min)
    t4 = time.perf_counter()
    out.update(nbr_ids=ids, nbr_dists=dists, rho=rho, lam=lam, delta=delta, labels=labels,
               centers=centers, noise=noise, rounds=trace,
               timings=dict(index=t1 - t0, density=t2 - t1, dependent=t3 - t2, unionfind=t4 - t3))
    return out
