"""World-size-2 gloo run of the sharding/exchange logic (CPU)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2604_17066_b200.dist import Comm, global_pick_owners, shard_range
    import oracle
    comm = Comm.from_env(backend="gloo")
    H, N = 1001, 7
    probs = np.tile([0.3, 0.7], (N, 1))
    start, count = shard_range(H, world, rank)
    # each rank draws its shard of the same stream with the oracle sampler
    xs = oracle.sample_states(probs, count, seed=5, generation_index=2, start=start)
    unc = np.flatnonzero(xs.sum(1) <= 3)  # stand-in "unclassified" predicate
    counts = comm.allreduce_sum_i64([len(unc), count])
    per = comm.allgather_i64(len(unc))
    total = int(per.sum())
    pos = np.random.default_rng([5, 2]).choice(total, size=min(6, total), replace=False)
    owner, local = global_pick_owners(per, pos)
    mine = np.flatnonzero(owner == comm.rank)
    rows = torch.as_tensor(xs[unc[local[mine]]].astype(np.uint8))
    gathered = comm.allgather_rows(rows, np.bincount(owner, minlength=world))
    order = np.argsort(owner, kind="stable")
    inv = np.empty_like(order)
    inv[order] = np.arange(len(order))
    picked = gathered[torch.as_tensor(inv)].numpy()
    flags = torch.tensor([rank % 2, 1 - rank % 2], dtype=torch.uint8)
    orf = comm.allreduce_max_u8(flags).tolist()
    # classifier hit flags (bit0 lower, bit1 upper) OR-reduced across reference shards
    hits = torch.tensor([[1, 0, 2, 0, 3], [2, 0, 0, 1, 1]][rank], dtype=torch.uint8)
    orh = comm.allreduce_or_hits(hits).tolist()
    q.put((rank, counts.tolist(), picked.tolist(), orf, orh))
    import torch.distributed as dist
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_sharding_matches_single_process():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=100) for _ in range(world)]
    for p in procs:
        p.join(timeout=30)
    import oracle
    xs = oracle.sample_states(np.tile([0.3, 0.7], (7, 1)), 1001, seed=5, generation_index=2)
    unc = np.flatnonzero(xs.sum(1) <= 3)
    pos = np.random.default_rng([5, 2]).choice(len(unc), size=min(6, len(unc)), replace=False)
    want = xs[unc[pos]].tolist()
    for rank, counts, picked, orf, orh in out:
        assert orh == [3, 0, 2, 1, 3]
        assert counts == [len(unc), 1001]
        assert picked == want  # every rank sees the picks in single-process order
        assert orf == [1, 1]


def _grid_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2604_17066_b200.dist import Comm
    comm = Comm.from_env(backend="gloo")
    ref_comm, samp_comm, s_idx, k_idx = comm.grid(2)
    # rank (s, k): sample shard s classified against reference shard k; hit bits of
    # sample i on shard k: lower if i % 4 == k, upper if i % 3 == k + s
    flags = torch.tensor([(1 if i % 4 == k_idx else 0) | (2 if i % 3 == k_idx + s_idx else 0)
                          for i in range(12)], dtype=torch.uint8)
    ref_comm.allreduce_or_hits(flags)
    lab = np.where(flags.numpy() & 1, 0, np.where(flags.numpy() & 2, 1, 2))
    counts = samp_comm.allreduce_sum_i64([int((lab == c).sum()) for c in range(3)])
    q.put((rank, s_idx, k_idx, ref_comm.world, samp_comm.world, flags.tolist(), counts.tolist()))
    import torch.distributed as dist
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_four_rank_grid_or_reduce_and_counts():
    """2 x 2 process grid (samples x reference shards): hit flags OR-reduced
    inside each reference group, label counts summed across sample groups."""
    world, port = 4, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_grid_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
    want_counts = np.zeros(3, dtype=np.int64)
    for s in range(2):
        f = [(1 if i % 4 in (0, 1) else 0) | (2 if i % 3 in (s, s + 1) else 0) for i in range(12)]
        lab = np.where(np.array(f) & 1, 0, np.where(np.array(f) & 2, 1, 2))
        want_counts += [int((lab == c).sum()) for c in range(3)]
        for rank, s_idx, k_idx, gk, gs, flags, counts in out:
            if s_idx == s:
                assert flags == f and (gk, gs) == (2, 2)
    for rank, s_idx, k_idx, gk, gs, flags, counts in out:
        assert (s_idx, k_idx) == divmod(rank, 2)
    for rank, *_, counts in out:
        assert counts == want_counts.tolist()
