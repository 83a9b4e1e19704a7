"""Per-point densities from kNN lists and the strict density rank
(mirrors /root/reference/pkg/src/peakann/density.py:26-129).

Computed on the GPU by pk_densities / pk_rank_order.  Row sums replay
numpy's pairwise summation order (8 interleaved accumulators, recursive
halving above 128), so `kth`, `kth_normalized` and `sum` are bit-identical
to the reference; `exp_sum` / `sum_exp` go through CUDA's exp, which may
differ from the host libm by an ulp (tolerance-checked in the tests).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import PointSet
from .index import NeighborList, Neighborhoods

__all__ = [
    "DENSITY_KINDS",
    "density_kth",
    "density_kth_normalized",
    "density_exp_sum",
    "density_sum_exp",
    "density_sum",
    "compute_densities",
    "rank_order",
]

DENSITY_KINDS = ("kth", "kth_normalized", "exp_sum", "sum_exp", "sum")


def densities_device(kind: str, ids_t, dists_t):
    """rho (n,) float64 tensor from device (n,k) ids / true distances."""
    import torch

    n, k = dists_t.shape
    rho = torch.empty(n, dtype=torch.float64, device=dists_t.device)
    _lib.call("pk_densities", _lib.DENSITY_CODES[kind], ids_t.contiguous(), dists_t.contiguous(), n, k, rho,
              _lib.stream())
    return rho


def _row(kind: str, neighbors: NeighborList) -> float:
    if len(neighbors) == 0:
        raise ValueError("density needs at least one neighbor")
    d = _lib.to_dev(neighbors.dists[None, :], np.float64)
    ids = _lib.to_dev(np.zeros((1, len(neighbors)), np.int64))
    return float(_lib.to_host(densities_device(kind, ids, d))[0])


def density_kth(neighbors: NeighborList) -> float:
    """Inverse distance to the furthest (k-th) neighbour; +inf for duplicates."""
    return _row("kth", neighbors)


def density_exp_sum(neighbors: NeighborList) -> float:
    """exp of the negated mean squared neighbour distance."""
    return _row("exp_sum", neighbors)


def density_sum_exp(neighbors: NeighborList) -> float:
    """Mean of exp(-distance^2) over the neighbours."""
    return _row("sum_exp", neighbors)


def density_sum(neighbors: NeighborList) -> float:
    """Negated sum of neighbour distances."""
    return _row("sum", neighbors)


def density_kth_normalized(rho: np.ndarray, neighbors_all: Neighborhoods) -> np.ndarray:
    """Rescale kth densities by k over the summed densities of each point's neighbours."""
    rho = np.asarray(rho, dtype=np.float64)
    if neighbors_all.k == 0:
        raise ValueError("density needs at least one neighbor")
    base = _lib.to_dev(rho)
    return _lib.to_host(_normalize_from_base(base, neighbors_all.device_ids()))


def _normalize_from_base(base_t, ids_t):
    import torch

    n, k = ids_t.shape
    out = torch.empty(n, dtype=torch.float64, device=base_t.device)
    _lib.call("pk_normalize_rho", base_t.contiguous(), ids_t.contiguous(), n, k, out, _lib.stream())
    return out


def check_neighborhoods(kind: str, p: PointSet, neighbors_all: Neighborhoods) -> None:
    if kind not in DENSITY_KINDS:
        raise ValueError(f"unknown density kind {kind!r}; expected one of {DENSITY_KINDS}")
    if neighbors_all.n != p.n:
        raise ValueError(f"neighborhoods cover {neighbors_all.n} points, point set has {p.n}")
    if neighbors_all.k == 0:
        raise ValueError("density needs at least one neighbor per point (is n == 1?)")


def compute_densities(kind: str, p: PointSet, neighbors_all: Neighborhoods) -> np.ndarray:
    """Densities of all points under the chosen variant (density.py:92-113)."""
    check_neighborhoods(kind, p, neighbors_all)
    rho = densities_device(kind, neighbors_all.device_ids(), neighbors_all.device_dists())
    return _lib.to_host(rho)


def rank_order_device(rho_t):
    """rank (n,) int64 tensor: higher = denser, ties to the smaller id."""
    import torch

    n = rho_t.shape[0]
    rank = torch.empty(n, dtype=torch.int64, device=rho_t.device)
    flag = torch.zeros(1, dtype=torch.int32, device=rho_t.device)
    _lib.call("pk_rank_order", rho_t.contiguous(), n, rank, flag, _lib.stream())
    if int(flag.item()):
        raise ValueError("densities must not contain NaN")
    return rank


def rank_order(rho: np.ndarray) -> np.ndarray:
    """Strict density ranks: higher rank is denser, ties go to the smaller id."""
    rho = np.asarray(rho, dtype=np.float64)
    return _lib.to_host(rank_order_device(_lib.to_dev(rho)))
