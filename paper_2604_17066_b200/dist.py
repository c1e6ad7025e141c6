"""Sample sharding across ranks (one process per GPU, torch.distributed).

The RSR path partitions naturally: rank g owns samples
[start_g, start_g + count_g) of the *same* (seed, generation) stream, so the
union over ranks is bit-identical to the single-device batch (the counter
stream is indexed by flat sample position, sampling.py:45-66).  The only
exchanges are:

* class counts -- one all-reduce(sum) of a few int64 per classified batch;
* Stage-1 iterations -- ONE all-gather per iteration of a byte record per
  rank: its class counts (the sums and the per-rank unclassified counts are
  derived on the host) plus the rows of its first C unclassified samples
  (speculative prefix).  Every rank computes the reference's numpy picks
  identically; when every pick falls inside its owner's prefix (always, once
  few samples stay unclassified) the picked rows are already on every rank.
  Otherwise a second all-gather fetches the picked rows.  Every rank then runs
  the same boundary searches and keeps identical reference sets.

All helpers take a ``Comm``; ``Comm.single()`` is the 1-process identity, and
with the ``gloo`` backend the same code runs on CPU tensors (tests).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

__all__ = ["Comm", "shard_range", "global_pick_owners", "counts_record", "split_records",
           "picks_in_prefix"]


@dataclass
class Comm:
    rank: int = 0
    world: int = 1
    device: torch.device | None = None
    group: object = None

    @classmethod
    def single(cls) -> "Comm":
        return cls(0, 1, None, None)

    @classmethod
    def from_env(cls, backend: str | None = None) -> "Comm":
        """Initialise from torchrun's RANK / WORLD_SIZE (127.0.0.1 rendezvous)."""
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if world == 1:
            return cls.single()
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if backend is None:
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
            dist.init_process_group(backend=backend)
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" \
            else torch.device("cpu")
        return cls(dist.get_rank(), dist.get_world_size(), dev, None)

    @property
    def distributed(self) -> bool:
        return self.world > 1

    def allreduce_sum_i64(self, values) -> np.ndarray:
        arr = np.asarray(values, dtype=np.int64)
        if not self.distributed:
            return arr
        import torch.distributed as dist
        t = torch.as_tensor(arr, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()

    def allreduce_max_u8(self, t: torch.Tensor) -> torch.Tensor:
        """OR of 0/1 flags across ranks (NCCL has no bitwise OR; max on 0/1 is OR)."""
        if not self.distributed:
            return t
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def allreduce_or_hits(self, flags: torch.Tensor) -> torch.Tensor:
        """In-place OR of classifier hit flags (bit0 lower hit, bit1 upper hit) across
        ranks: MAX on the raw bytes would turn lower-on-one-rank + upper-on-another
        (1, 2) into 2 instead of 3, so each bit travels as its own 0/1 plane.  The
        two planes live in one buffer kept across calls (no allocation per call)."""
        if not self.distributed:
            return flags
        n = flags.numel()
        planes = getattr(self, "_planes", None)
        if planes is None or planes.shape[1] < n or planes.device != flags.device:
            planes = self._planes = torch.empty((2, n), dtype=torch.uint8, device=flags.device)
        p = planes[:, :n]
        torch.bitwise_and(flags, 1, out=p[0])
        torch.bitwise_right_shift(flags, 1, out=p[1])
        if self.device is not None and p.device != self.device:  # gloo: CPU transport
            host = p.to(self.device)
            self.allreduce_max_u8(host)
            p.copy_(host)
        else:
            self.allreduce_max_u8(p)
        torch.bitwise_left_shift(p[1], 1, out=p[1])
        torch.bitwise_or(p[0], p[1], out=flags)
        return flags

    def allgather_bytes(self, buf: torch.Tensor) -> torch.Tensor:
        """One all-gather of an equal-size uint8 record per rank -> [world, len] on the
        record's device (the comm device carries it: NCCL in place, gloo via host)."""
        if not self.distributed:
            return buf.reshape(1, -1)
        import torch.distributed as dist
        src = buf if (self.device is None or buf.device == self.device) else buf.to(self.device)
        out = torch.empty((self.world, src.numel()), dtype=torch.uint8, device=src.device)
        dist.all_gather_into_tensor(out.view(-1), src.reshape(-1), group=self.group)
        return out if out.device == buf.device else out.to(buf.device)

    def allgather_i64(self, value: int) -> np.ndarray:
        if not self.distributed:
            return np.array([value], dtype=np.int64)
        import torch.distributed as dist
        t = torch.tensor([value], dtype=torch.int64, device=self.device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return np.array([int(o.item()) for o in out], dtype=np.int64)

    def allgather_i64_vec(self, values) -> np.ndarray:
        """Every rank's int64 vector -> host [world, len] with one all-gather (sums over
        ranks are column sums: no separate all-reduce)."""
        arr = np.asarray(values, dtype=np.int64).reshape(-1)
        if not self.distributed:
            return arr.reshape(1, -1)
        import torch.distributed as dist
        t = torch.as_tensor(arr, device=self.device)
        out = torch.empty((self.world, arr.size), dtype=torch.int64, device=self.device)
        dist.all_gather_into_tensor(out.view(-1), t, group=self.group)
        return out.cpu().numpy()

    def allgather_rows(self, rows: torch.Tensor, counts: np.ndarray) -> torch.Tensor:
        """Concatenate per-rank row blocks (rank order); counts = rows per rank."""
        if not self.distributed:
            return rows
        import torch.distributed as dist
        width = rows.shape[1]
        mx = int(max(1, counts.max()))
        pad = torch.zeros((mx, width), dtype=rows.dtype, device=self.device)
        if rows.shape[0]:
            pad[: rows.shape[0]].copy_(rows.to(self.device))
        out = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(out, pad, group=self.group)
        return torch.cat([o[: int(c)] for o, c in zip(out, counts)], dim=0)

    def grid(self, ref_shards: int) -> tuple["Comm", "Comm", int, int]:
        """2-D process grid for reference-sharded classification:
        G = G_s x G_k ranks, rank r -> sample shard r // G_k, reference shard r % G_k.
        Returns (ref_group, sample_group, sample_shard, ref_shard): hit flags are
        OR-reduced over ref_group (same samples, different references), counts
        summed over sample_group (same reference shard, different samples).
        Every rank must call this collectively (torch.distributed.new_group)."""
        if ref_shards < 1 or self.world % ref_shards:
            raise ValueError(f"ref_shards={ref_shards} must divide world={self.world}")
        gs, gk = self.world // ref_shards, ref_shards
        s_idx, k_idx = divmod(self.rank, gk)
        if not self.distributed:
            return Comm.single(), Comm.single(), 0, 0
        import torch.distributed as dist
        ref_group = sample_group = None
        for s in range(gs):  # every rank creates every group, in the same order
            g = dist.new_group([s * gk + k for k in range(gk)])
            if s == s_idx:
                ref_group = g
        for k in range(gk):
            g = dist.new_group([s * gk + k for s in range(gs)])
            if k == k_idx:
                sample_group = g
        return (Comm(k_idx, gk, self.device, ref_group), Comm(s_idx, gs, self.device, sample_group),
                s_idx, k_idx)

    def barrier(self) -> None:
        if self.distributed:
            import torch.distributed as dist
            dist.barrier(group=self.group)


def shard_range(n_samples: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, near-equal split of [0, n_samples): (start, count) of ``rank``."""
    base, extra = divmod(n_samples, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def counts_record(counts, rows: torch.Tensor | None = None) -> torch.Tensor:
    """Byte record of one rank for `Comm.allgather_bytes`: int64 counts, then the
    rows (uint8 [C, N]) of its first C unclassified samples."""
    c = torch.as_tensor(np.asarray(counts, dtype=np.int64)) if not isinstance(counts, torch.Tensor) \
        else counts.to(torch.int64)
    head = c.reshape(-1).view(torch.uint8)
    if rows is None:
        return head
    return torch.cat([head.to(rows.device), rows.reshape(-1)])


def split_records(recs: torch.Tensor, n_counts: int, c_rows: int, n_cols: int):
    """[world, bytes] records -> (int64 counts [world, n_counts] on the host, row prefix
    view uint8 [world, c_rows, n_cols] on the records' device)."""
    head = recs[:, :8 * n_counts].contiguous()
    counts = head.cpu().view(torch.int64).numpy().reshape(recs.shape[0], n_counts)
    rows = recs[:, 8 * n_counts:8 * n_counts + c_rows * n_cols].reshape(recs.shape[0], c_rows, n_cols)
    return counts, rows


def picks_in_prefix(owner: np.ndarray, local: np.ndarray, prefix: int) -> bool:
    """True when every pick lies within its owner's exchanged prefix of `prefix`
    unclassified rows (then no second exchange is needed)."""
    return bool(np.all(local < prefix)) if len(local) else True


def global_pick_owners(unclassified_per_rank: np.ndarray, positions: np.ndarray):
    """Map global positions in the rank-ordered unclassified list to (rank, local pos).

    The global sorted unclassified index list is the concatenation of the
    ranks' sorted local lists (rank g's samples precede rank g+1's).
    """
    offsets = np.concatenate([[0], np.cumsum(unclassified_per_rank)])
    owner = np.searchsorted(offsets, positions, side="right") - 1
    return owner, positions - offsets[owner]
