"""Multi-GPU split of the hot path: one process per GPU.

Every rank holds the full point set; the work is partitioned, and the
exchange steps are the ones the reference algorithm has:

* graph build (vamana.py:146-169): each doubling batch of at least
  `min_shard` points is cut into `world` contiguous chunks; rank r runs
  GreedySearch + RobustPrune for chunk r and the out-lists are all-gathered
  (PK_XCHG_OUTLISTS).  The reverse-edge re-prunes of a batch are split by
  target (u % world) and the re-pruned rows are all-gathered (PK_XCHG_ROWS).
  Every rank ends with the same graph, identical to the single-GPU build.
* kNN densities (cluster.py:299): queries cut into contiguous chunks, the
  (n, k) rows all-gathered, densities computed replicated.
* dependent points (dependent.py:96-133): phase 1 is replicated (a cheap
  pass over resident lists); each doubling round and the final scan split the
  (sorted) unresolved ids, and the per-round unresolved sets are all-gathered;
  lam / delta are merged with one MAX / MIN all-reduce (each point is resolved
  by exactly one rank; untouched entries hold -1 / +inf).
* policies + union-find: replicated (O(n) passes).

`Comm` wraps torch.distributed (NCCL on GPUs; gloo in the CPU tests).
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
    def all_gather_chunks(self, buf: torch.Tensor, chunk: int) -> None:
        """In-place all-gather of equal chunks: rank r owns buf[r*chunk:(r+1)*chunk]
        (flat first dimension); afterwards every rank holds all world*chunk."""
        if self.world == 1 or chunk == 0:
            return
        full = buf[: self.world * chunk]
        own = full[self.rank * chunk:(self.rank + 1) * chunk]
        if self.backend == "nccl":
            dist.all_gather_into_tensor(full, own, group=self.group)
        else:  # gloo: host copies (CPU tests, or a functional check with several ranks on one device)
            src = own.cpu()
            parts = [torch.empty_like(src) for _ in range(self.world)]
            dist.all_gather(parts, src, group=self.group)
            for r, t in enumerate(parts):
                if r != self.rank:
                    full[r * chunk:(r + 1) * chunk].copy_(t)

    def all_gather_into(self, out: torch.Tensor, send: torch.Tensor) -> None:
        """out[r*len(send):(r+1)*len(send)] = send of rank r."""
        if self.world == 1:
            out[: send.shape[0]].copy_(send)
            return
        if self.backend == "nccl":
            dist.all_gather_into_tensor(out[: self.world * send.shape[0]], send, group=self.group)
        else:
            src = send.cpu()
            parts = [torch.empty_like(src) for _ in range(self.world)]
            dist.all_gather(parts, src, group=self.group)
            out[: self.world * send.shape[0]].copy_(torch.cat(parts))

    def all_gather_counts(self, count: int, device) -> list[int]:
        t = torch.tensor([count], dtype=torch.int64, device=device if self.backend == "nccl" else "cpu")
        if self.world == 1:
            return [count]
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t, group=self.group)
        return [int(x.item()) for x in parts]

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

    def all_reduce(self, t: torch.Tensor, op: str) -> None:
        if self.world == 1:
            return
        rop = {"max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN, "sum": dist.ReduceOp.SUM}[op]
        if self.backend == "nccl" or t.device.type == "cpu":
            dist.all_reduce(t, op=rop, group=self.group)
        else:
            h = t.cpu()
            dist.all_reduce(h, op=rop, group=self.group)
            t.copy_(h)

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
    xrecv; returns maxc.  Errors are kept in `.error` and reported to the C
    side as -1 (the build then fails with a status instead of raising through
    the C frame)."""

    OUTLISTS = 0
    ROWS = 1

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
        self.calls = {self.OUTLISTS: 0, self.ROWS: 0}
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
