"""Multi-GPU split of the hot path: one process per GPU.

Every rank holds the full point set; the work is partitioned, and the
exchange steps are the ones the reference algorithm has:

* graph build (vamana.py:146-169): each doubling batch of at least
  `min_shard` points is cut into `world` contiguous chunks; rank r runs
  GreedySearch + RobustPrune for chunk r and the out-lists are all-gathered
  (PK_XCHG_OUTLISTS).  The reverse-edge re-prunes of a batch are split by
  target (u % world) and the re-pruned rows are all-gathered (PK_XCHG_ROWS).
  Every rank ends with the same graph, identical to the single-GPU build.
* kNN densities (cluster.py:299): queries cut into contiguous chunks; each
  rank keeps its own (chunk, k) rows and computes their densities; only rho
  is all-gathered (n x 8 B; kth_normalized all-gathers the raw kth values
  first, then normalises its rows against them, then all-gathers again).
* dependent points (dependent.py:96-133): phase 1 runs on each rank's own
  rows; the unresolved ids are all-gathered (variable length) and every
  doubling round and the final scan split the sorted set again; lam / delta
  are merged with one MAX / MIN all-reduce (each point is resolved by exactly
  one rank; untouched entries hold -1 / +inf).
* policies + union-find: replicated on the identical rho / lam / delta (the
  local-center policy, which reads the kNN rows, all-gathers them first).
* the returned state: the (n, k) rows are gathered to rank 0 only.

`Comm` wraps torch.distributed (NCCL on GPUs; gloo in the CPU tests).  The
collectives are the same calls on both backends (all_gather_into_tensor,
all_reduce, gather); with gloo, device tensors are staged through host
copies (several ranks sharing one device in a functional test).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib

__all__ = ["Comm", "BuildExchange", "largest_batch"]


class Comm:
    """Rank / world view of a process group plus the collectives the split uses."""

    def __init__(self, group=None, rank: int | None = None, world: int | None = None):
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group) if rank is None else rank
            self.world = dist.get_world_size(group) if world is None else world
            self.backend = dist.get_backend(group)
        else:
            self.rank, self.world, self.backend = 0, 1, None

    @classmethod
    def auto(cls):
        """A Comm when a process group with more than one rank is up, else None."""
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            return cls()
        return None

    # ---- partitioning
    def chunk(self, m: int) -> int:
        return (m + self.world - 1) // self.world

    def my_range(self, m: int) -> tuple[int, int]:
        """Contiguous chunk of [0, m) owned by this rank (chunk = ceil(m / world))."""
        c = self.chunk(m)
        lo = min(m, self.rank * c)
        return lo, min(m, lo + c)

    # ---- collectives
    def _host_staged(self, t: torch.Tensor) -> bool:
        """gloo cannot reduce / gather device tensors: stage them through the host."""
        return self.backend != "nccl" and t.device.type != "cpu"

    def _all_gather_tensor(self, out: torch.Tensor, send: torch.Tensor) -> None:
        """dist.all_gather_into_tensor(out, send) on either backend."""
        if self._host_staged(send):
            ho = torch.empty(out.shape, dtype=out.dtype)
            dist.all_gather_into_tensor(ho, send.cpu(), group=self.group)
            out.copy_(ho)
        else:
            dist.all_gather_into_tensor(out, send.contiguous(), group=self.group)

    def all_gather_chunks(self, buf: torch.Tensor, chunk: int) -> None:
        """In-place all-gather of equal chunks: rank r owns buf[r*chunk:(r+1)*chunk]
        (flat first dimension); afterwards every rank holds all world*chunk."""
        if self.world == 1 or chunk == 0:
            return
        full = buf[: self.world * chunk]
        own = full[self.rank * chunk:(self.rank + 1) * chunk].clone()
        self._all_gather_tensor(full, own)

    def all_gather_into(self, out: torch.Tensor, send: torch.Tensor) -> None:
        """out[r*len(send):(r+1)*len(send)] = send of rank r."""
        if self.world == 1:
            out[: send.shape[0]].copy_(send)
            return
        self._all_gather_tensor(out[: self.world * send.shape[0]], send)

    def all_gather_counts(self, count: int, device) -> list[int]:
        dev = device if self.backend == "nccl" else "cpu"
        if self.world == 1:
            return [count]
        out = torch.empty(self.world, dtype=torch.int64, device=dev)
        self._all_gather_tensor(out, torch.tensor([count], dtype=torch.int64, device=dev))
        return [int(x) for x in out.tolist()]

    def all_gather_varlen(self, t: torch.Tensor) -> torch.Tensor:
        """Concatenation over ranks (rank order) of tensors of different lengths."""
        if self.world == 1:
            return t
        counts = self.all_gather_counts(t.shape[0], t.device)
        maxc = max(counts)
        if maxc == 0:
            return t[:0]
        pad = torch.zeros((maxc,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        out = torch.empty((self.world * maxc,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        self.all_gather_into(out, pad)
        return torch.cat([out[r * maxc:r * maxc + counts[r]] for r in range(self.world)])

    def all_gather_rows(self, local: torch.Tensor, n: int) -> torch.Tensor:
        """Rows [lo, hi) of every rank (my_range(n)) -> the full (n, ...) array."""
        if self.world == 1:
            return local
        c = self.chunk(n)
        pad = torch.empty((c,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
        out = torch.empty((self.world * c,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        self._all_gather_tensor(out, pad)
        return out[:n]

    def gather_rows_to_root(self, local: torch.Tensor, n: int, root: int = 0):
        """Rows [lo, hi) of every rank -> the full (n, ...) array on `root`, None elsewhere."""
        if self.world == 1:
            return local
        c = self.chunk(n)
        pad = torch.empty((c,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
        staged = self._host_staged(pad)
        send = pad.cpu() if staged else pad
        parts = [torch.empty_like(send) for _ in range(self.world)] if self.rank == root else None
        dist.gather(send, parts, dst=root, group=self.group)
        if self.rank != root:
            return None
        full = torch.cat(parts)[:n]
        return full.to(local.device) if staged else full

    def all_reduce(self, t: torch.Tensor, op: str) -> None:
        if self.world == 1:
            return
        rop = {"max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN, "sum": dist.ReduceOp.SUM}[op]
        if self._host_staged(t):
            h = t.cpu()
            dist.all_reduce(h, op=rop, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=rop, group=self.group)

    def broadcast(self, t: torch.Tensor, src: int = 0) -> None:
        if self.world == 1:
            return
        if self._host_staged(t):
            h = t.cpu()
            dist.broadcast(h, src=src, group=self.group)
            t.copy_(h)
        else:
            dist.broadcast(t, src=src, group=self.group)

    def max_time(self, ms: float, device) -> float:
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        self.all_reduce(t, "max")
        return float(t.item())


def largest_batch(n: int) -> int:
    """Upper bound of a doubling batch (batches 1, 2, 4, ...; vamana.py:146)."""
    b = 1
    while b < n:
        b <<= 1
    return min(b, n)


class BuildExchange:
    """Buffers and host callback of pk_build_vamana_sharded.

    kind PK_XCHG_OUTLISTS (a = chunk): all-gather xids[0, world*a*R) and
    xlen[0, world*a) in place.  kind PK_XCHG_ROWS (a = own record count):
    gather the counts into xcnt and the records xsend[0, maxc*(R+2)) into
    xrecv; returns maxc.  kind PK_XCHG_ORDER (a = n): broadcast xids[0, n) from
    rank 0.  Errors are kept in `.error` and reported to the C
    side as -1 (the build then fails with a status instead of raising through
    the C frame)."""

    OUTLISTS = 0
    ROWS = 1
    ORDER = 2  # a = n: broadcast xids[0, n) from rank 0 (search order inside the batches)

    def __init__(self, comm: Comm, n: int, R: int, device):
        self.comm = comm
        self.R = R
        w = comm.world
        mb = largest_batch(n)
        U = min(n, mb * R)
        self.xids = torch.empty((mb + w) * R, dtype=torch.int32, device=device)
        self.xlen = torch.empty(mb + w, dtype=torch.int32, device=device)
        self.xsend = torch.empty(U * (R + 2), dtype=torch.int32, device=device)
        self.xrecv = torch.empty(w * U * (R + 2), dtype=torch.int32, device=device)
        self.xcnt = torch.zeros(w, dtype=torch.int32, device=device)
        self.error = None
        self.calls = {self.OUTLISTS: 0, self.ROWS: 0, self.ORDER: 0}
        self.callback = _lib.EXCHANGE_FN(self._exchange)

    def _exchange(self, ctx, kind, a, b):
        try:
            return self.exchange(kind, a)
        except Exception as e:  # noqa: BLE001 -- surfaced after the C call returns
            self.error = e
            return -1

    def exchange(self, kind: int, a: int) -> int:
        if kind not in self.calls:
            raise ValueError(f"unknown exchange kind {kind}")
        self.calls[kind] += 1
        if kind == self.ORDER:
            self.comm.broadcast(self.xids[:a], src=0)
            return 0
        if kind == self.OUTLISTS:
            self.comm.all_gather_chunks(self.xids, a * self.R)
            self.comm.all_gather_chunks(self.xlen, a)
            return 0
        if kind == self.ROWS:
            counts = self.comm.all_gather_counts(a, self.xcnt.device)
            self.xcnt.copy_(torch.tensor(counts, dtype=torch.int32))
            maxc = max(counts)
            if maxc > 0:
                W = self.R + 2
                self.comm.all_gather_into(self.xrecv, self.xsend[: maxc * W])
        return maxc

    def pointers(self):
        return (self.callback, None, self.xids, self.xlen, self.xsend, self.xrecv, self.xcnt)
