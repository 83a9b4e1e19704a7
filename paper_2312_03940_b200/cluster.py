"""Noise filtering, center selection, union-find assignment and the end-to-end
pipeline (mirrors /root/reference/pkg/src/peakann/cluster.py:47-311).

Every stage runs on the GPU and keeps its state in HBM; the numpy arrays of
`PipelineResult` are materialised after the last timed stage.  Assignment
replaces the reference's Python union-find loop with pointer jumping on
parent[i] = (center or noise) ? i : lam[i] (pk_assign_clusters): dependency
edges point strictly up in density rank, so every component is a tree whose
root is its center / noise point and the canonical label is that root.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, field
from typing import Optional, Union

import numpy as np

from . import _lib
from .core import PointSet
from .density import check_neighborhoods, densities_device, rank_order_device
from .dependent import Dependents, DoublingParams, dependents_device
from .index import KnnIndex, Neighborhoods, build_bruteforce, sqrt_device
from .vamana import build_vamana

__all__ = [
    "NoisePolicy",
    "ThresholdCenter",
    "ProductCenter",
    "LocalCenter",
    "CenterPolicy",
    "BruteForceConfig",
    "VamanaConfig",
    "IndexConfig",
    "Clustering",
    "DpcState",
    "PipelineResult",
    "find_noise",
    "find_centers_threshold",
    "find_centers_product",
    "find_centers_local",
    "assign_clusters",
    "run_pipeline",
    "reapply_policies",
]


@dataclass(frozen=True)
class NoisePolicy:
    """Points with density strictly below rho_min become singleton noise."""

    rho_min: float = 0.0


@dataclass(frozen=True)
class ThresholdCenter:
    """Centers are non-noise points with dependent distance >= delta_min."""

    delta_min: float


@dataclass(frozen=True)
class ProductCenter:
    """Centers are the n_clusters non-noise points with the largest
    delta * rho products (an infinite delta beats any finite product)."""

    n_clusters: int


@dataclass(frozen=True)
class LocalCenter:
    """Centers are non-noise points denser than all of their own neighbours."""


CenterPolicy = Union[ThresholdCenter, ProductCenter, LocalCenter]


@dataclass(frozen=True)
class BruteForceConfig:
    """Exact kNN backend."""


@dataclass(frozen=True)
class VamanaConfig:
    R: int = 32
    L_build: int = 32
    L: int = 32
    alpha: float = 1.1
    num_starts: Optional[int] = None
    seed: int = 42
    medoid_start: bool = False


IndexConfig = Union[BruteForceConfig, VamanaConfig]


@dataclass
class Clustering:
    """Canonical labels: every point carries the id of its cluster's center
    (or its own id if it is noise)."""

    labels: np.ndarray
    centers: np.ndarray
    noise: np.ndarray

    @property
    def n_clusters(self) -> int:
        return self.centers.shape[0] + self.noise.shape[0]


@dataclass
class DpcState:
    """Per-point pipeline state sufficient to re-run the policy steps."""

    rho: np.ndarray
    dependents: Dependents
    neighbors: Optional[Neighborhoods] = None

    @property
    def lam(self) -> np.ndarray:
        return self.dependents.lam

    @property
    def delta(self) -> np.ndarray:
        return self.dependents.delta


@dataclass
class PipelineResult:
    clustering: Clustering
    state: DpcState
    timings: dict = field(default_factory=dict)


# ---- device helpers -------------------------------------------------------------------


def _u8(n):
    import torch

    return torch.zeros(n, dtype=torch.uint8, device=_lib.device())


def _ids_of_device(flags_t):
    import torch

    n = flags_t.shape[0]
    out = torch.empty(max(n, 1), dtype=torch.int64, device=flags_t.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=flags_t.device)
    _lib.call("pk_flags_to_ids", flags_t, n, out, cnt, _lib.stream())
    return out[: int(cnt.item())]


def _ids_of(flags_t) -> np.ndarray:
    return _lib.to_host(_ids_of_device(flags_t))


def _to_host_many(tensors):
    """Device tensors -> numpy arrays: async copies into one pinned staging
    buffer (torch's caching host allocator), one stream sync."""
    import torch

    offs, total = [], 0
    for t in tensors:
        offs.append(total)
        total += (t.numel() * t.element_size() + 63) // 64 * 64
    buf = torch.empty(max(total, 64), dtype=torch.uint8, pin_memory=True)
    views = []
    for t, o in zip(tensors, offs):
        v = buf[o:o + t.numel() * t.element_size()].view(t.dtype).view(t.shape)
        v.copy_(t, non_blocking=True)
        views.append(v)
    torch.cuda.current_stream().synchronize()
    return [v.numpy() for v in views]


def _noise_flags(rho_t, rho_min: float):
    import torch

    n = rho_t.shape[0]
    flags = _u8(n)
    cnt = torch.zeros(1, dtype=torch.int64, device=rho_t.device)
    _lib.call("pk_flag_noise", rho_t, n, float(rho_min), flags, cnt, _lib.stream())
    return flags, int(cnt.item())


def _product_flags(rho_t, delta_t, noise_t, n_noise: int, n_c: int):
    n = rho_t.shape[0]
    if n_c < 1:
        raise ValueError(f"n_c must be >= 1, got {n_c}")
    non_noise = n - n_noise
    flags = _u8(n)
    if n_c >= non_noise:
        if n_c > non_noise:
            warnings.warn(f"requested {n_c} centers but only {non_noise} non-noise points; returning all",
                          stacklevel=3)
        flags.copy_(1 - noise_t)
        return flags
    _lib.call("pk_centers_product", rho_t, delta_t, noise_t, n, n_c, flags, _lib.stream())
    return flags


def _threshold_flags(delta_t, noise_t, delta_min: float):
    n = delta_t.shape[0]
    flags = _u8(n)
    _lib.call("pk_centers_threshold", delta_t, noise_t, n, float(delta_min), flags, _lib.stream())
    return flags


def _local_flags(rank_t, nbr_ids_t, noise_t):
    n, k = nbr_ids_t.shape
    flags = _u8(n)
    _lib.call("pk_centers_local", rank_t, nbr_ids_t.contiguous(), k, noise_t, n, flags, _lib.stream())
    return flags


def _assign_device(lam_t, center_t, noise_t):
    import torch

    n = lam_t.shape[0]
    labels = torch.empty(n, dtype=torch.int64, device=lam_t.device)
    status = torch.zeros(3, dtype=torch.int64, device=lam_t.device)
    _lib.call("pk_assign_clusters", lam_t, center_t, noise_t, n, labels, status, _lib.stream())
    st = _lib.to_host(status)
    if st[0] == 1:
        raise RuntimeError(f"point {int(st[1])} has no dependent point but is neither a center nor noise")
    if st[0] == 3:
        raise RuntimeError(f"point {int(st[1])} is in a component with no center or noise point")
    return labels


# ---- public policy API (host arrays in, host arrays out) --------------------------------


def find_noise(rho: np.ndarray, policy: NoisePolicy) -> np.ndarray:
    """Ids with density strictly below rho_min, ascending."""
    flags, _ = _noise_flags(_lib.to_dev(np.asarray(rho, np.float64)), policy.rho_min)
    return _ids_of(flags)


def _noise_of(n: int, non_noise: np.ndarray):
    noise = np.ones(n, np.uint8)
    noise[np.asarray(non_noise, np.int64)] = 0
    return _lib.to_dev(noise)


def find_centers_threshold(dep: Dependents, non_noise: np.ndarray, delta_min: float) -> np.ndarray:
    """Non-noise ids whose dependent distance is at least delta_min."""
    n = len(dep)
    return _ids_of(_threshold_flags(dep.device_delta(), _noise_of(n, non_noise), delta_min))


def find_centers_product(rho: np.ndarray, dep: Dependents, non_noise: np.ndarray, n_c: int) -> np.ndarray:
    """The n_c non-noise ids with the largest delta * rho products; ties by
    larger delta, then smaller id (cluster.py:155-172)."""
    if n_c < 1:
        raise ValueError(f"n_c must be >= 1, got {n_c}")
    ids = np.asarray(non_noise, np.int64)
    if n_c >= ids.shape[0]:
        if n_c > ids.shape[0]:
            warnings.warn(f"requested {n_c} centers but only {ids.shape[0]} non-noise points; returning all",
                          stacklevel=2)
        return np.sort(ids)
    n = len(dep)
    noise_t = _noise_of(n, ids)
    flags = _product_flags(_lib.to_dev(np.asarray(rho, np.float64)), dep.device_delta(), noise_t,
                           n - ids.shape[0], n_c)
    return _ids_of(flags)


def find_centers_local(rho: np.ndarray, neighbors_all: Neighborhoods, non_noise: np.ndarray) -> np.ndarray:
    """Non-noise ids that outrank every point in their own neighbour list."""
    rank_t = rank_order_device(_lib.to_dev(np.asarray(rho, np.float64)))
    n = rank_t.shape[0]
    return _ids_of(_local_flags(rank_t, neighbors_all.device_ids(), _noise_of(n, non_noise)))


def assign_clusters(dep: Dependents, centers: np.ndarray, noise: np.ndarray) -> Clustering:
    """Union every remaining point with its dependent, then canonicalise
    (cluster.py:183-220), on the GPU by pointer jumping."""
    n = len(dep)
    centers = np.sort(np.asarray(centers, np.int64))
    noise = np.sort(np.asarray(noise, np.int64))
    skip = np.zeros(n, dtype=bool)
    skip[centers] = True  # IndexError on out-of-range ids, as the reference
    skip[noise] = True
    lam = dep.lam
    bad = np.flatnonzero(~skip & (lam < 0))
    if bad.shape[0]:
        raise RuntimeError(f"point {int(bad[0])} has no dependent point but is neither a center nor noise")
    # duplicate / overlapping skip sets collapse components in the reference
    seen = {}
    for c in centers.tolist():
        if c in seen:
            raise RuntimeError(f"centers {seen[c]} and {c} collapsed into one component")
        seen[c] = c
    for x in noise.tolist():
        if x in seen:
            raise RuntimeError(f"noise point {x} shares a component with {seen[x]}")
        seen[x] = x
    cflag = np.zeros(n, np.uint8)
    cflag[centers] = 1
    nflag = np.zeros(n, np.uint8)
    nflag[noise] = 1
    labels = _assign_device(dep.device_lam(), _lib.to_dev(cflag), _lib.to_dev(nflag))
    return Clustering(_lib.to_host(labels), centers, noise)


# ---- pipeline ----------------------------------------------------------------------------


def _apply_policies_device(rho_t, lam_t, delta_t, nbr_ids_t, center_policy, noise_policy, rank_t=None):
    """(labels_t, center_flags_t, noise_flags_t) -- cluster.py:241-254 on device."""
    noise_t, n_noise = _noise_flags(rho_t, noise_policy.rho_min)
    if isinstance(center_policy, ThresholdCenter):
        center_t = _threshold_flags(delta_t, noise_t, center_policy.delta_min)
    elif isinstance(center_policy, ProductCenter):
        center_t = _product_flags(rho_t, delta_t, noise_t, n_noise, center_policy.n_clusters)
    elif isinstance(center_policy, LocalCenter):
        if nbr_ids_t is None:
            raise ValueError("local center policy needs the neighbor lists in the state")
        if rank_t is None:
            rank_t = rank_order_device(rho_t)
        center_t = _local_flags(rank_t, nbr_ids_t, noise_t)
    else:
        raise TypeError(f"unknown center policy {center_policy!r}")
    # points without a dependent (the densest) are promoted to centers unless noise
    _lib.call("pk_promote_orphans", lam_t, noise_t, lam_t.shape[0], center_t, _lib.stream())
    labels_t = _assign_device(lam_t, center_t, noise_t)
    return labels_t, center_t, noise_t


def _apply_policies(state: DpcState, center_policy: CenterPolicy, noise_policy: NoisePolicy) -> Clustering:
    rho_t = _lib.to_dev(np.asarray(state.rho, np.float64))
    nbr = state.neighbors.device_ids() if state.neighbors is not None else None
    labels_t, c_t, n_t = _apply_policies_device(rho_t, state.dependents.device_lam(),
                                                state.dependents.device_delta(), nbr, center_policy, noise_policy)
    return Clustering(_lib.to_host(labels_t), _ids_of(c_t), _ids_of(n_t))


def reapply_policies(state: DpcState, center_policy: CenterPolicy, noise_policy: NoisePolicy) -> Clustering:
    """Re-run only the policy steps over previously computed state."""
    return _apply_policies(state, center_policy, noise_policy)


def _build_index(p: PointSet, config: IndexConfig, comm=None) -> KnnIndex:
    if isinstance(config, BruteForceConfig):
        return build_bruteforce(p)
    if isinstance(config, VamanaConfig):
        return build_vamana(
            p,
            R=config.R,
            L_build=config.L_build,
            alpha=config.alpha,
            num_starts=config.num_starts,
            seed=config.seed,
            medoid_start=config.medoid_start,
            query_beam=config.L,
            comm=comm,
        )
    raise TypeError(f"unknown index config {config!r}")


def _sync():
    import torch

    torch.cuda.synchronize()


def _knn_all_device(index: KnnIndex, n: int, k: int, comm=None):
    """knn_all on device -> (ids_t, sqd_t, row0): every row on one GPU; with
    `comm` only this rank's contiguous chunk of the query rows (starting at
    point row0) -- the rows are never all-gathered."""
    import torch

    dev = _lib.device()
    if comm is None or comm.world == 1:
        ids, sqd = index.knn_batch_device(torch.arange(n, dtype=torch.int64, device=dev), k)
        return ids, sqd, 0
    lo, hi = comm.my_range(n)
    ids, sqd = index.knn_batch_device(torch.arange(lo, hi, dtype=torch.int64, device=dev), k)
    return ids, sqd, lo


def _densities_sharded(kind: str, ids_t, dists_t, row0: int, n: int, comm):
    """rho of all n points from each rank's own rows: densities of the local
    rows, then one all-gather of rho (kth_normalized: all-gather the raw kth
    values, normalise the local rows against them, all-gather again)."""
    from .density import densities_device

    if kind == "kth_normalized":
        base = comm.all_gather_rows(densities_device("kth", ids_t, dists_t), n)
        import torch

        m, k = ids_t.shape
        rho = torch.empty(m, dtype=torch.float64, device=ids_t.device)
        _lib.call("pk_normalize_rho_rows", base, ids_t.contiguous(), row0, m, k, rho, _lib.stream())
        return comm.all_gather_rows(rho, n)
    return comm.all_gather_rows(densities_device(kind, ids_t, dists_t), n)


def run_pipeline_device(p: PointSet, index_config: IndexConfig, k: int, density_kind: str,
                        center_policy: CenterPolicy, noise_policy: NoisePolicy = NoisePolicy(),
                        doubling_params: Optional[DoublingParams] = None, trace=None, comm=None):
    """The pipeline with every intermediate left in HBM.  Returns a dict of
    device tensors plus the stage timings (cluster.py:279-311).  With `comm`
    (shard.Comm, one process per GPU) the build, the kNN queries and the
    dependent-point queries are split across the ranks (shard.py); every rank
    returns the full result."""
    import torch

    if doubling_params is None:
        doubling_params = DoublingParams(initial_k=2 * k)
    n = p.n
    timings: dict = {}
    _sync()
    t0 = time.perf_counter()
    index = _build_index(p, index_config, comm)
    _sync()
    t1 = time.perf_counter()
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    ids_t, sqd_t, row0 = _knn_all_device(index, n, k, comm)
    dists_t = sqrt_device(sqd_t)
    sharded = comm is not None and comm.world > 1
    if sharded:
        check_neighborhoods(density_kind, p, _RowsView(n, ids_t.shape[1]))
        rho_t = _densities_sharded(density_kind, ids_t, dists_t, row0, n, comm)
    else:
        check_neighborhoods(density_kind, p, Neighborhoods.on_device(ids_t, dists_t))
        rho_t = densities_device(density_kind, ids_t, dists_t)
    _sync()
    t2 = time.perf_counter()
    lam_t, delta_t, rank_t = dependents_device(index, p, rho_t, ids_t, dists_t, doubling_params, trace, comm,
                                               row0=row0)
    _sync()
    t3 = time.perf_counter()
    # the local-center policy reads every kNN row: the only step that needs them all
    rows_all = comm.all_gather_rows(ids_t, n) if sharded and isinstance(center_policy, LocalCenter) else ids_t
    labels_t, c_t, n_t = _apply_policies_device(rho_t, lam_t, delta_t, rows_all, center_policy, noise_policy, rank_t)
    _sync()
    t4 = time.perf_counter()
    timings["index"] = t1 - t0
    timings["density"] = t2 - t1
    timings["dependent"] = t3 - t2
    timings["unionfind"] = t4 - t3
    return dict(index=index, ids=ids_t, dists=dists_t, rows=(row0, row0 + ids_t.shape[0]), rho=rho_t, lam=lam_t,
                delta=delta_t, labels=labels_t, centers=c_t, noise=n_t, timings=timings)


class _RowsView:
    """Shape-only stand-in for the full Neighborhoods in the argument checks of
    a sharded run (each rank holds only its own rows)."""

    def __init__(self, n, k):
        self.n, self.k = n, k


def run_pipeline(
    p: PointSet,
    index_config: IndexConfig,
    k: int,
    density_kind: str,
    center_policy: CenterPolicy,
    noise_policy: NoisePolicy = NoisePolicy(),
    doubling_params: Optional[DoublingParams] = None,
    comm=None,
) -> PipelineResult:
    """Index build, kNN, densities, dependent points, policies, union-find.
    `comm` (shard.Comm) splits the work across one process per GPU; every rank
    returns the full clustering, rho, lam and delta, and rank 0 also the full
    (n, k) kNN rows (gathered to it alone; the other ranks' state carries
    neighbors=None)."""
    out = run_pipeline_device(p, index_config, k, density_kind, center_policy, noise_policy, doubling_params,
                              comm=comm)
    ids_t, dists_t = out["ids"], out["dists"]
    if comm is not None and comm.world > 1:
        ids_t = comm.gather_rows_to_root(ids_t, p.n)
        dists_t = comm.gather_rows_to_root(dists_t, p.n)
    rows = [ids_t, dists_t] if ids_t is not None else []
    got = _to_host_many([out["rho"], out["lam"], out["delta"], out["labels"], _ids_of_device(out["centers"]),
                         _ids_of_device(out["noise"])] + rows)
    rho, lam, delta, labels, centers, noise = got[:6]
    nbrs = Neighborhoods(got[6], got[7]) if rows else None
    state = DpcState(rho=rho, dependents=Dependents(lam, delta), neighbors=nbrs)
    clustering = Clustering(labels, centers, noise)
    return PipelineResult(clustering=clustering, state=state, timings=out["timings"])
