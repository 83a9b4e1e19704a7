"""Dependent points: each point's nearest neighbour of strictly higher density
(mirrors /root/reference/pkg/src/peakann/dependent.py:31-133).

Three phases on the GPU: (1) the first denser entry of each point's own kNN
row (pk_resolve_lists); (2) doubling rounds that re-query the index with
k = initial_k, 2*initial_k, ... for the still-unresolved points while more
than `threshold` remain (the beam kernel with L = max(query L, k), then
pk_resolve_lists); (3) an exact masked scan of all points for the stragglers
(pk_dp_scan).  The only host synchronisation is one int64 per round (the
unresolved count drives the reference's data-dependent loop).

Exact backends: with a BruteForceIndex every round resolves a point to its
exact nearest denser point (the first denser entry of an exact (dist, id)
list is the global minimum), so the rounds are replaced by one dp scan of
all phase-1 stragglers -- the same lam/delta as the reference's rounds, with
one exact pass instead of up to log2(n) brute kNN passes.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple, Optional, Sequence

import numpy as np

from . import _lib
from .core import PointSet
from .density import rank_order_device
from .index import BruteForceIndex, KnnIndex, Neighbor, Neighborhoods, sqrt_device

__all__ = ["DoublingParams", "DependentInfo", "Dependents", "dp_brute_force", "compute_dependent_points"]


@dataclass(frozen=True)
class DoublingParams:
    """initial_k is the first kNN width of the doubling rounds (must exceed
    the density k); once at most `threshold` points remain unresolved they
    are finished by exact full scans instead of further rounds."""

    initial_k: int
    threshold: int = 300

    def validated_against(self, k: int) -> "DoublingParams":
        if self.initial_k <= k:
            raise ValueError(f"initial_k must be > k, got initial_k={self.initial_k}, k={k}")
        if self.threshold < 0:
            raise ValueError(f"threshold must be >= 0, got {self.threshold}")
        return self


class DependentInfo(NamedTuple):
    lam: Optional[int]
    delta: float


class Dependents:
    """Per-point dependent ids (-1 when absent) and dependent distances.

    Host arrays by default; pipeline results may be device-backed and are
    downloaded on first access.
    """

    __slots__ = ("_lam", "_delta", "_lam_t", "_delta_t")

    def __init__(self, lam: np.ndarray, delta: np.ndarray):
        self._lam, self._delta = lam, delta
        self._lam_t = self._delta_t = None

    @classmethod
    def on_device(cls, lam_t, delta_t) -> "Dependents":
        obj = cls(None, None)
        obj._lam_t, obj._delta_t = lam_t, delta_t
        return obj

    @property
    def lam(self) -> np.ndarray:
        if self._lam is None:
            self._lam = _lib.to_host(self._lam_t)
        return self._lam

    @lam.setter
    def lam(self, v):
        self._lam, self._lam_t = v, None

    @property
    def delta(self) -> np.ndarray:
        if self._delta is None:
            self._delta = _lib.to_host(self._delta_t)
        return self._delta

    @delta.setter
    def delta(self, v):
        self._delta, self._delta_t = v, None

    def device_lam(self):
        if self._lam_t is None:
            self._lam_t = _lib.to_dev(np.asarray(self._lam, np.int64))
        return self._lam_t

    def device_delta(self):
        if self._delta_t is None:
            self._delta_t = _lib.to_dev(np.asarray(self._delta, np.float64))
        return self._delta_t

    def __len__(self) -> int:
        return (self._lam_t if self._lam is None else self._lam).shape[0]

    def __getitem__(self, i: int) -> DependentInfo:
        l = int(self.lam[i])
        return DependentInfo(l if l >= 0 else None, float(self.delta[i]))


def dp_brute_force(i: int, candidates: Sequence[Neighbor], rho: np.ndarray) -> Optional[Neighbor]:
    """Closest candidate ranked denser than i, by (dist, id); None if none
    (dependent.py:70-77; a scalar helper over an explicit candidate list)."""
    key_i = (rho[i], -i)
    best: Optional[Neighbor] = None
    for nb in candidates:
        if (rho[nb.id], -nb.id) > key_i and (best is None or (nb.dist, nb.id) < (best.dist, best.id)):
            best = nb
    return best


def _resolve(rank_t, qids_t, ids_t, dists_t, lam_t, delta_t, skip: int, counts_t=None):
    """pk_resolve_lists -> (unresolved qids, count, short qids, short count).
    With counts_t, rows the beam search could not fill are returned as
    "short" instead of being resolved from their partial list."""
    import torch

    m = qids_t.shape[0]
    dev = qids_t.device
    out = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    short = torch.empty(max(m, 1), dtype=torch.int64, device=dev) if counts_t is not None else None
    k = ids_t.shape[1] if ids_t.dim() == 2 else 0
    _lib.call("pk_resolve_lists", rank_t, qids_t, m, ids_t, dists_t, k, lam_t, delta_t, out, cnt[0:1], skip,
              counts_t, short, cnt[1:2] if counts_t is not None else None, _lib.stream())
    c, s = (int(v) for v in _lib.to_host(cnt))
    return out[:c], c, (short[:s] if short is not None else None), s


def _resolve_short(p: PointSet, rank_t, short_t, ms: int, kk: int, lam_t, delta_t):
    """Rows whose beam search came up short: exact resolution by a dp scan +
    count scan (pk_resolve_short) instead of full exact kNN rows."""
    import torch

    out = torch.empty(max(ms, 1), dtype=torch.int64, device=short_t.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=short_t.device)
    if _dp_scan_on_tensor_cores(p, ms):
        # the dp scan on the tensor cores (certificate + exact rescan), then the count scan
        sid = torch.empty(ms, dtype=torch.int64, device=short_t.device)
        ssq = torch.empty(ms, dtype=torch.float64, device=short_t.device)
        _dp_scan_tc(p, rank_t, short_t, ms, sid, ssq)
        _lib.call("pk_resolve_short_scanned", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, short_t, ms, kk, sid,
                  ssq, lam_t, delta_t, out, cnt, _lib.stream())
    else:
        _lib.call("pk_resolve_short", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, rank_t, short_t, ms, kk,
                  lam_t, delta_t, out, cnt, _lib.stream())
    c = int(cnt.item())
    return out[:c], c


def _dp_scan_on_tensor_cores(p: PointSet, m: int) -> bool:
    """Float data, enough work for a tensor-core screen (exact integer modes
    already scan with exact fp32 / u8 arithmetic)."""
    from .index import use_tensor_cores

    return p.mode == _lib.MODE_SEQ64 and m >= 64 and p.n >= 4096 and use_tensor_cores(p, max(m, 256), 1)


def _dp_scan_tc(p: PointSet, rank_t, q, m: int, sid, ssq):
    """pk_dp_scan_tc, then the exact scan for the rows its certificate rejects."""
    import torch

    flags = torch.zeros(m, dtype=torch.uint8, device=q.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=q.device)
    _lib.call("pk_dp_scan_tc", p.device(), p.n, p.dp, rank_t, q, m, sid, ssq, flags, cnt, _lib.stream())
    nbad = int(cnt.item())
    if nbad:
        bad = torch.nonzero(flags, as_tuple=True)[0]
        bq = q[bad].contiguous()
        bi = torch.empty(nbad, dtype=torch.int64, device=q.device)
        bs = torch.empty(nbad, dtype=torch.float64, device=q.device)
        _lib.call("pk_dp_scan", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, rank_t, bq, nbad, bi, bs,
                  _lib.stream())
        sid[bad] = bi
        ssq[bad] = bs


def dependents_device(g: KnnIndex, p: PointSet, rho_t, ids_t, dists_t, params: DoublingParams, trace=None,
                      comm=None, row0: int = 0):
    """(lam_t, delta_t) on device; `trace` collects (unresolved, kq) per round.
    ids_t / dists_t are the kNN rows of points row0, row0 + 1, ... (all n on
    one GPU).  With `comm` each rank resolves its own rows in phase 1, and
    every doubling round and the final scan split the sorted unresolved ids
    across the ranks (shard.py)."""
    import torch

    def mine(t):
        if comm is None:
            return t
        lo, hi = comm.my_range(t.shape[0])
        return t[lo:hi]

    def regroup(t):
        if comm is None:
            return t, t.shape[0]
        t = torch.sort(comm.all_gather_varlen(t)).values
        return t, t.shape[0]

    n = p.n
    dev = rho_t.device
    rank_t = rank_order_device(rho_t)
    lam_t = torch.full((n,), -1, dtype=torch.int64, device=dev)
    delta_t = torch.full((n,), float("inf"), dtype=torch.float64, device=dev)
    top_t = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.call("pk_argmax_rank", rank_t, n, top_t, _lib.stream())
    top = int(top_t.item())
    own_t = torch.arange(row0, row0 + ids_t.shape[0], dtype=torch.int64, device=dev)
    todo, m, _, _ = _resolve(rank_t, own_t, ids_t, dists_t, lam_t, delta_t, top)
    if comm is not None:
        todo, m = regroup(todo)  # every rank's phase-1 leftovers, sorted: the same list on every rank
    if n > 1:
        kdep = params.validated_against(ids_t.shape[1]).initial_k
        if not isinstance(g, BruteForceIndex):
            raw = getattr(g, "knn_rows_raw", None)
            while m > params.threshold:
                kq = min(kdep, n - 1)
                if trace is not None:
                    trace.append((m, kq))
                ms = 0
                q = mine(todo)
                if raw is not None:
                    r_ids, r_sqd, r_cnt = raw(q, kq)
                    todo, m, short, ms = _resolve(rank_t, q, r_ids, sqrt_device(r_sqd), lam_t, delta_t, -1, r_cnt)
                    if ms:
                        left, ml = _resolve_short(p, rank_t, short, ms, min(kq, n - 1), lam_t, delta_t)
                        if ml:
                            todo = torch.cat([todo, left])
                            m += ml
                else:
                    r_ids, r_sqd = g.knn_batch_device(q, kq)
                    todo, m, _, _ = _resolve(rank_t, q, r_ids, sqrt_device(r_sqd), lam_t, delta_t, -1)
                if trace is not None and ms:
                    trace[-1] = trace[-1] + (ms,)  # rows the beam search left short (exact scans)
                if comm is not None:
                    todo, m = regroup(todo)
                if kq >= n - 1:
                    break
                kdep *= 2
    if m > 0:
        if trace is not None:
            trace.append((m, "scan"))
        q = mine(todo)
        mq = q.shape[0]
        if mq:
            sid = torch.empty(mq, dtype=torch.int64, device=dev)
            ssq = torch.empty(mq, dtype=torch.float64, device=dev)
            if _dp_scan_on_tensor_cores(p, mq):
                _dp_scan_tc(p, rank_t, q, mq, sid, ssq)
            else:
                _lib.call("pk_dp_scan", p.device(), n, p.dp, p.packed(), p.dw, p.mode, rank_t, q, mq, sid, ssq,
                          _lib.stream())
            _lib.call("pk_scatter_dependents", q, mq, sid, ssq, lam_t, delta_t, _lib.stream())
    if comm is not None:
        # each point was resolved by exactly one rank; the others hold -1 / +inf
        comm.all_reduce(lam_t, "max")
        comm.all_reduce(delta_t, "min")
    return lam_t, delta_t, rank_t


def compute_dependent_points(
    g: KnnIndex,
    p: PointSet,
    rho: np.ndarray,
    neighbors_all: Neighborhoods,
    params: DoublingParams,
) -> Dependents:
    """Dependent point and distance for every point; the globally densest
    point keeps lam=None, delta=+inf (dependent.py:96-133)."""
    n = p.n
    rho = np.asarray(rho, dtype=np.float64)
    if rho.shape[0] != n or neighbors_all.n != n:
        raise ValueError("rho and neighbors_all must cover the whole point set")
    lam_t, delta_t, _ = dependents_device(g, p, _lib.to_dev(rho), neighbors_all.device_ids(),
                                          neighbors_all.device_dists(), params)
    return Dependents(_lib.to_host(lam_t), _lib.to_host(delta_t))
