"""Sharded Stage 1 / Stage 2 over 2 ranks reproduces the single-device results.

gloo: both ranks run on the one visible GPU with host-side collectives; no
kernel waits on another rank, so sharing the device is safe.  nccl: one GPU per
rank (skipped with fewer than 2 GPUs) -- the same code with CUDA tensors in the
collectives (dist.Comm: fused per-iteration all-gather, row all-gather).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from _specs import load_json

pytestmark = pytest.mark.gpu

CASES = ["grid_st_b8", "grid_widest_m3", "cones6"]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, q, sync_loop="0", backend="gloo"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank), RSR_SYNC_LOOP=sync_loop)
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    import torch
    torch.cuda.set_device(rank if backend == "nccl" else 0)
    import paper_2604_17066_b200 as P
    from paper_2604_17066_b200.dist import Comm
    from _specs import device_model, load_json as lj
    rec = next(c for c in lj("workflow.json") if c["spec"]["name"] == case)
    spec = rec["spec"]
    comm = Comm.from_env(backend=backend)
    model = device_model(spec["model"])
    dist = P.ComponentDistribution(np.array(spec["probs"]))
    cfg = P.RunConfig(**spec["config"])
    out = []
    for st in rec["stages"]:
        s1 = P.stage1_find_references(model, dist, cfg, st["threshold"], comm)
        rep = P.stage2_evaluate(model, dist, s1.lower, s1.upper, cfg, st["threshold"], comm)
        out.append({
            "lower": [list(v) for v in s1.lower.members],
            "upper": [list(v) for v in s1.upper.members],
            "trace": [[t.reference_count, t.phi_evaluations, t.p_lower, t.p_upper,
                       t.p_unclassified] for t in s1.trace],
            "iterations": s1.iterations, "redundant": s1.redundant_searches,
            "p_lower": rep.p_lower, "unclassified_resolved": rep.unclassified_resolved,
            "phi_total": model.evaluation_count})
    q.put((rank, out))
    import torch.distributed as dist_
    dist_.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("backend", ["gloo", "nccl"])
@pytest.mark.parametrize("loop", ["async", "sync"])
@pytest.mark.parametrize("case", CASES)
def test_two_rank_workflow_matches_single_device(case, loop, backend):
    # async: device-resident reference sets, rows of the picks exchanged per
    # iteration; sync: the host-resolved insertion path
    import torch
    if backend == "nccl" and torch.cuda.device_count() < 2:
        pytest.skip("NCCL ranks need one GPU each")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, 2, port, case, q, "1" if loop == "sync" else "0", backend))
             for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=280) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    rec = next(c for c in load_json("workflow.json") if c["spec"]["name"] == case)
    for rank in (0, 1):
        for got, st in zip(res[rank], rec["stages"]):
            want = st["stage1"]
            assert got["lower"] == want["lower"] and got["upper"] == want["upper"]
            assert got["trace"] == want["trace"]
            assert got["iterations"] == want["iterations"]
            assert got["redundant"] == want["redundant_searches"]
            assert got["p_lower"] == st["stage2"]["p_lower"]
            assert got["unclassified_resolved"] == st["stage2"]["unclassified_resolved"]
            assert got["phi_total"] == st["stage2"]["phi_total"]


def test_c_abi_comm_single_rank():
    """The C-ABI exchange entry points (include/rsr_b200.h) on a
    one-rank NCCL communicator: counts sum, rows gather and hit-flag OR are the
    identity; bad ranks raise ValueError."""
    import ctypes

    import torch

    from paper_2604_17066_b200 import _abi
    torch.cuda.set_device(0)
    uid = (ctypes.c_uint8 * 128)()
    _abi.call("rsr_comm_unique_id", uid)
    comm = ctypes.c_void_p()
    with pytest.raises(ValueError):
        _abi.call("rsr_comm_init", uid, 2, 2, ctypes.byref(comm))
    _abi.call("rsr_comm_init", uid, 1, 0, ctypes.byref(comm))
    st = _abi.stream_ptr()
    counts = torch.tensor([3, 5, 7], dtype=torch.int64, device="cuda")
    _abi.call("rsr_allreduce_counts", comm, _abi.ptr(counts), 3, st)
    rows = torch.randint(0, 3, (64, 295), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(rows)
    _abi.call("rsr_allgather_refs", comm, _abi.ptr(rows), rows.numel(), _abi.ptr(out), st)
    flags = torch.randint(0, 4, (10_001,), dtype=torch.uint8, device="cuda")
    want = flags.clone()
    scratch = torch.empty(2 * flags.numel(), dtype=torch.uint8, device="cuda")
    _abi.call("rsr_or_reduce_flags", comm, _abi.ptr(flags), flags.numel(), _abi.ptr(scratch), st)
    torch.cuda.synchronize()
    assert counts.tolist() == [3, 5, 7] and torch.equal(out, rows) and torch.equal(flags, want)
    _abi.call("rsr_comm_destroy", comm)


def _cov_worker(rank, world, port, q, rng):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    import torch
    torch.cuda.set_device(0)
    import paper_2604_17066_b200 as P
    from paper_2604_17066_b200 import workloads as W
    from paper_2604_17066_b200.dist import Comm
    from _specs import device_model
    comm = Comm.from_env(backend="gloo")
    g = W.cfg1(0)
    spec = {"kind": "st", "n_nodes": g["n_nodes"], "edges": g["edges"], "s": 0, "t": 24,
            "m": 2, "ms": 2}
    model = device_model(spec)
    dist = P.ComponentDistribution(g["probs"])
    cfg = P.RunConfig(n_samples=3001, eps_u=1e-3, r_max=60, seed=4, parallel_searches=4, rng=rng)
    s1 = P.stage1_find_references(model, dist, cfg, 0, comm)
    rep = P.stage2_until_cov(model, dist, s1.lower, s1.upper, cfg, 0, 0.05, batch_samples=5001,
                             comm=comm)
    q.put((rank, [list(v) for v in s1.lower.members], [list(v) for v in s1.upper.members],
           s1.iterations, rep.n_samples, rep.p_lower, rep.unclassified_resolved,
           model.evaluation_count))
    import torch.distributed as dist_
    dist_.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("rng", ["shared", "device"])
def test_two_rank_run_to_cov_matches_single_device(rng):
    """Stage 1 and the run-to-c.o.v. loop sharded over 2 ranks (odd batch
    sizes: uneven shards) equal the single-device run, on both sample streams."""
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    import paper_2604_17066_b200 as P
    from paper_2604_17066_b200 import workloads as W
    from _specs import device_model
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cov_worker, args=(r, 2, port, q, rng)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=280) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
    g = W.cfg1(0)
    spec = {"kind": "st", "n_nodes": g["n_nodes"], "edges": g["edges"], "s": 0, "t": 24,
            "m": 2, "ms": 2}
    model = device_model(spec)
    dist = P.ComponentDistribution(g["probs"])
    cfg = P.RunConfig(n_samples=3001, eps_u=1e-3, r_max=60, seed=4, parallel_searches=4, rng=rng)
    s1 = P.stage1_find_references(model, dist, cfg, 0)
    rep = P.stage2_until_cov(model, dist, s1.lower, s1.upper, cfg, 0, 0.05, batch_samples=5001)
    want = ([list(v) for v in s1.lower.members], [list(v) for v in s1.upper.members],
            s1.iterations, rep.n_samples, rep.p_lower, rep.unclassified_resolved,
            model.evaluation_count)
    assert rep.n_samples > 5001  # several batches
    for rank in (0, 1):
        assert tuple(res[rank]) == want
