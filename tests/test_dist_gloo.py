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


def _fused_worker(rank, world, port, q):
    """The Stage-1 iteration exchange of workflow._stage1_loop_async on gloo: one
    all-gather of [counts | first C unclassified rows] per iteration, the picks taken
    from the exchanged prefixes when they all fall inside them, a second all-gather of
    the picked rows otherwise."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from paper_2604_17066_b200.dist import (Comm, counts_record, global_pick_owners,
                                            picks_in_prefix, shard_range, split_records)
    import oracle
    comm = Comm.from_env(backend="gloo")
    calls = {"n": 0}
    for name in ("all_gather_into_tensor", "all_gather", "all_reduce"):
        orig = getattr(dist, name)

        def counted(*a, _orig=orig, **k):
            calls["n"] += 1
            return _orig(*a, **k)
        setattr(dist, name, counted)
    H, N, B = 997, 9, 6
    probs = np.tile([0.35, 0.65], (N, 1))
    start, count = shard_range(H, world, rank)
    results = []
    for it, thr in enumerate((6, 3, 1)):  # many, fewer, few unclassified samples
        xs = oracle.sample_states(probs, count, seed=9, generation_index=it, start=start)
        unc = np.flatnonzero(xs.sum(1) <= thr)
        counts = [7, 11, len(unc), 0]
        C = B
        pref = np.zeros((C, N), dtype=np.uint8)
        pref[:min(C, len(unc))] = xs[unc[:C]]
        before = calls["n"]
        recs = comm.allgather_bytes(counts_record(counts, torch.as_tensor(pref)))
        all_counts, prefix = split_records(recs, 4, C, N)
        per_rank = all_counts[:, 2].copy()
        total = int(per_rank.sum())
        pos = np.random.default_rng([9, it]).choice(total, size=min(B, total), replace=False)
        owner, local = global_pick_owners(per_rank, pos)
        fused = picks_in_prefix(owner, local, C)
        if fused:
            rows = prefix.reshape(-1, N)[torch.as_tensor(owner * C + local)]
        else:
            mine = np.flatnonzero(owner == comm.rank)
            g = comm.allgather_rows(torch.as_tensor(xs[unc[local[mine]]].astype(np.uint8)),
                                    np.bincount(owner, minlength=world))
            order = np.argsort(owner, kind="stable")
            inv = np.empty_like(order)
            inv[order] = np.arange(len(order))
            rows = g[torch.as_tensor(inv)]
        results.append((rows.tolist(), all_counts.sum(0).tolist(), fused, calls["n"] - before))
    # counts matrix of several values in one all-gather
    per = comm.allgather_i64_vec([rank, 10 * rank + 1])
    # in-place OR of hit planes twice (the planes buffer is reused)
    for _ in range(2):
        hits = torch.tensor([[1, 0, 2, 0, 3], [2, 0, 0, 1, 1]][rank], dtype=torch.uint8)
        comm.allreduce_or_hits(hits)
    q.put((rank, results, per.tolist(), hits.tolist()))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_fused_iteration_exchange_two_ranks():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=100) for _ in range(world)]
    for p in procs:
        p.join(timeout=30)
    import oracle
    fused_seen = set()
    for it, thr in enumerate((6, 3, 1)):
        xs = oracle.sample_states(np.tile([0.35, 0.65], (9, 1)), 997, seed=9, generation_index=it)
        unc = np.flatnonzero(xs.sum(1) <= thr)
        pos = np.random.default_rng([9, it]).choice(len(unc), size=min(6, len(unc)), replace=False)
        want = xs[unc[pos]].tolist()
        for rank, results, per, hits in out:
            rows, sums, fused, n_coll = results[it]
            assert rows == want and sums == [14, 22, len(unc), 0]
            assert n_coll == (1 if fused else 2)  # one collective when the prefix covers the picks
            fused_seen.add(fused)
    assert fused_seen == {True, False}
    for rank, results, per, hits in out:
        assert per == [[0, 1], [1, 11]] and hits == [3, 0, 2, 1, 3]
