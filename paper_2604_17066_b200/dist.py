"""Sample sharding across ranks (one process per GPU, torch.distributed).

The RSR path partitions naturally: rank g owns samples
[start_g, start_g + count_g) of the *same* (seed, generation) stream, so the
union over ranks is bit-identical to the single-device batch (the counter
stream is indexed by flat sample position, sampling.py:45-66).  The only
exchanges are:

* class counts -- one all-reduce(sum) of a few int64 per classified batch;
* Stage-1 picks -- all-gather of per-rank unclassified counts, identical
  numpy picks on every rank, and an all-gather of the picked rows so every
  rank runs the same boundary searches and keeps identical reference sets.

All helpers take a ``Comm``; ``Comm.single()`` is the 1-process identity, and
with the ``gloo`` backend the same code runs on CPU tensors (tests).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

__all__ = ["Comm", "shard_range", "global_pick_owners"]


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
        (1, 2) into 2 instead of 3, so each bit travels as its own 0/1 plane."""
        if not self.distributed:
            return flags
        planes = torch.stack([flags & 1, flags >> 1])
        self.allreduce_max_u8(planes)
        torch.bitwise_or(planes[0], planes[1] << 1, out=flags)
        return flags

    def allgather_i64(self, value: int) -> np.ndarray:
        if not self.distributed:
            return np.array([value], dtype=np.int64)
        import torch.distributed as dist
        t = torch.tensor([value], dtype=torch.int64, device=self.device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return np.array([int(o.item()) for o in out], dtype=np.int64)

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


def global_pick_owners(unclassified_per_rank: np.ndarray, positions: np.ndarray):
    """Map global positions in the rank-ordered unclassified list to (rank, local pos).

    The global sorted unclassified index list is the concatenation of the
    ranks' sorted local lists (rank g's samples precede rank g+1's).
    """
    offsets = np.concatenate([[0], np.cumsum(unclassified_per_rank)])
    owner = np.searchsorted(offsets, positions, side="right") - 1
    return owner, positions - offsets[owner]
