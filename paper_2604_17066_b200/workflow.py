"""Two-stage RSR workflow on the device (mirror of reference ``workflow.py``).

Stage 1 (workflow.py:122-195), per iteration ``i``:
  rsr_sample (gen = i) -> rsr_encode_samples_fp4 -> rsr_classify_fp4 -> rsr_finalize
  -> trace record -> termination test -> picks from
  ``default_rng([seed, i]).choice(U, size, replace=False)`` (the reference's
  own RNG call; positions into the sorted unclassified list, which
  ``rsr_compact`` produces on the device) -> rsr_gather_rows ->
  rsr_boundary_search (all picks in parallel, one warp each) ->
  ReferenceSet.insert_batch (rsr_dominance_scan) in pick order.
Stage 2 (workflow.py:198-245): one generation-0 batch, classify, then
  rsr_phi_eval on the compacted unclassified rows with the <= m' count fused.
The trace, reference sets (ordered), redundant-search count, Phi-evaluation
counts and estimates equal the reference's on the same inputs.

With a multi-rank ``Comm`` the batch is sharded by sample position (same
stream, ``start`` offsets) and only counts / picked rows are exchanged, so
results are identical to one device.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi, _device
from .boundary import ReferenceSet, ReferenceState, Side, boundary_search_batch
from .classify import cov, classify
from .dist import Comm, global_pick_owners, shard_range
from .model import ComponentDistribution, SystemModel
from .sampling import sample_batch

__all__ = ["RunConfig", "TraceRecord", "Stage1Result", "Stage2Report", "PmfReport",
           "stage1_find_references", "stage2_evaluate", "stage2_until_cov", "multistate_pmf",
           "assemble_pmf"]

_STAGE2_GENERATION = 0  # workflow.py:38-40


def _rss_bytes() -> int | None:
    try:
        import resource
        return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss * 1024
    except Exception:  # pragma: no cover
        return None


@dataclass(frozen=True)
class RunConfig:
    """Knobs for both stages (workflow.py:53-75)."""

    n_samples: int = 1_000_000
    eps_u: float = 1e-5
    r_max: int = 10_000
    chunk_size: int = 65536
    seed: int = 0
    parallel_searches: int = 1
    n_workers: int = 1
    stage2_samples: int | None = None
    boundary_search_enabled: bool = True

    def __post_init__(self) -> None:
        if self.n_samples < 1:
            raise ValueError("n_samples must be >= 1")
        if not 0.0 <= self.eps_u <= 1.0:
            raise ValueError("eps_u must lie in [0, 1]")
        if self.r_max < 1:
            raise ValueError("r_max must be >= 1")
        if self.parallel_searches < 1:
            raise ValueError("parallel_searches must be >= 1")


@dataclass(frozen=True)
class TraceRecord:
    reference_count: int
    elapsed_seconds: float
    phi_evaluations: int
    p_lower: float
    p_upper: float
    p_unclassified: float
    resident_memory_bytes: int | None = None


@dataclass
class Stage1Result:
    lower: ReferenceSet
    upper: ReferenceSet
    trace: list
    iterations: int
    redundant_searches: int
    terminated_by: str


@dataclass(frozen=True)
class Stage2Report:
    p_lower: float
    p_upper: float
    cov_lower: float | None
    cov_upper: float | None
    n_samples: int
    unclassified_resolved: int
    threshold: int
    seed: int


@dataclass(frozen=True)
class PmfReport:
    pmf: np.ndarray
    cumulative_lower: np.ndarray
    stage2_reports: tuple
    stage1_results: tuple
    max_chain_discrepancy: float
    renormalization_adjustment: float


def _check_threshold(model: SystemModel, threshold: int) -> None:
    if not 0 <= threshold <= model.n_system_states - 2:
        raise ValueError(f"threshold must lie in [0, {model.n_system_states - 2}]")


class _BatchBuffers:
    """Reused device buffers for the per-iteration sample batch."""

    def __init__(self, count: int, n: int, m: int):
        dev = _device.device()
        self.states = torch.empty((count, n), dtype=torch.uint8, device=dev)
        self.fp4_ok = _abi.fp4_row_bytes(n, m) <= _abi.FP4_MAX_ROW_BYTES
        self.fp4 = (torch.empty((count, 2 * _abi.fp4_row_bytes(n, m)), dtype=torch.uint8, device=dev)
                    if self.fp4_ok else None)


_STREAMS: dict = {}


def _high_priority_stream() -> torch.cuda.Stream:
    """One persistent high-priority stream per device (allocations made on it stay
    in one caching-allocator pool across calls)."""
    key = torch.cuda.current_device()
    st = _STREAMS.get(key)
    if st is None:
        st = _STREAMS[key] = torch.cuda.Stream(priority=-1)
    return st


class _Prefetcher:
    """Double-buffered sampling on a side stream: batch i+1 (generation i+1 does
    not depend on the references) is drawn while iteration i searches and
    inserts on the main stream."""

    def __init__(self, dist_, seed, start, count):
        self.dist, self.seed, self.start, self.count = dist_, seed, start, count
        self.bufs = [_BatchBuffers(max(count, 1), dist_.n_components, dist_.n_states)
                     for _ in range(2)]
        self.stream = torch.cuda.Stream()
        self.free = [None, None]  # main-stream events: slot no longer read

    def launch(self, gen):
        slot = gen & 1
        b = self.bufs[slot]
        with torch.cuda.stream(self.stream):
            if self.free[slot] is not None:
                self.stream.wait_event(self.free[slot])
            batch = sample_batch(self.dist, self.count, self.seed, gen, self.start,
                                 out_states=b.states, out_fp4=b.fp4 if b.fp4_ok else None)
            ready = torch.cuda.Event()
            ready.record(self.stream)
        return batch, ready

    def release(self, gen):
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.free[gen & 1] = ev

    def close(self):
        torch.cuda.current_stream().wait_stream(self.stream)


def _classify_shard(model, pending, lower, upper, comm):
    batch, ready = pending
    torch.cuda.current_stream().wait_event(ready)
    res = classify(batch, lower, upper, n_states=model.n_component_states)
    counts = comm.allreduce_sum_i64(list(res.counts)) if comm.distributed else np.array(res.counts)
    return batch, res, counts


def stage1_find_references(model: SystemModel, dist: ComponentDistribution, config: RunConfig,
                           threshold: int, comm: Comm | None = None) -> Stage1Result:
    """Discover boundary reference sets for one threshold (workflow.py:122-195)."""
    _check_threshold(model, threshold)
    comm = comm or Comm.single()
    phi = model.device_phi()
    lower = ReferenceSet(Side.LOWER, threshold)
    upper = ReferenceSet(Side.UPPER, threshold)
    phi_start = model.evaluation_count
    t_start = time.perf_counter()
    H = config.n_samples
    start, count = shard_range(H, comm.world, comm.rank)
    # the loop's own kernels run on a high-priority stream so the prefetched
    # sampler (low priority, all SMs) does not delay the small search kernels
    caller = torch.cuda.current_stream()
    loop_stream = _high_priority_stream()
    loop_stream.wait_stream(caller)
    with torch.cuda.stream(loop_stream):
        result = _stage1_loop(model, dist, config, threshold, comm, phi, lower, upper, start,
                              count, H, t_start, phi_start)
    caller.wait_stream(loop_stream)
    return result


def _stage1_loop(model, dist, config, threshold, comm, phi, lower, upper, start, count, H,
                 t_start, phi_start) -> Stage1Result:
    trace: list[TraceRecord] = []
    redundant = 0
    terminated_by = "r_max"
    pre = _Prefetcher(dist, config.seed, start, count)
    pending = pre.launch(0)
    N = dist.n_components
    iteration = 0
    while True:
        batch, res, counts = _classify_shard(model, pending, lower, upper, comm)
        pending = pre.launch(iteration + 1)
        n_l, n_u, n_x = (int(c) for c in counts[:3])
        trace.append(TraceRecord(
            reference_count=len(lower) + len(upper),
            elapsed_seconds=time.perf_counter() - t_start,
            phi_evaluations=model.evaluation_count - phi_start,
            p_lower=n_l / H, p_upper=n_u / H, p_unclassified=n_x / H,
            resident_memory_bytes=_rss_bytes()))
        if n_x / H <= config.eps_u:
            terminated_by = "eps_u"
            break
        if len(lower) + len(upper) >= config.r_max:
            break
        rng = np.random.default_rng([config.seed, iteration])
        n_pick = min(config.parallel_searches, n_x)
        positions = rng.choice(n_x, size=n_pick, replace=False)
        x0 = _gather_picks(batch, res, positions, comm, N)
        if config.boundary_search_enabled:
            refs_d, side_d, calls_d = boundary_search_batch(model, x0, threshold)
        else:
            vals = torch.empty(n_pick, dtype=torch.uint8, device=x0.device)
            phi.eval_into(x0, None, n_pick, model.n_component_states, vals)
            refs_d = x0
            side_d = torch.where(vals <= threshold, _abi.SIDE_LOWER, _abi.SIDE_UPPER).to(torch.uint8)
            calls_d = None
        refs_h, side_h, calls_h = _to_host(refs_d, side_d, calls_d)
        model.add_evaluations(int(calls_h.sum()) if calls_h is not None else n_pick)
        for code, target in ((_abi.SIDE_LOWER, lower), (_abi.SIDE_UPPER, upper)):
            sel = np.flatnonzero(side_h == code)
            if sel.size == 0:
                continue
            sel_d = torch.as_tensor(sel, dtype=torch.int64, device=refs_d.device)
            outcome = target.insert_batch(refs_d.index_select(0, sel_d).contiguous(), refs_h[sel])
            redundant += sum(1 for o in outcome if o == "redundant")
        pre.release(iteration)
        iteration += 1
    pre.close()
    return Stage1Result(lower=lower, upper=upper, trace=trace, iterations=iteration + 1,
                        redundant_searches=redundant, terminated_by=terminated_by)


def _to_host(*tensors):
    """Several small device tensors -> numpy with a single stream synchronisation."""
    outs = []
    for t in tensors:
        if t is None:
            outs.append(None)
            continue
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        outs.append(h)
    torch.cuda.current_stream().synchronize()
    return [None if h is None else h.numpy() for h in outs]


def _gather_picks(batch, res, positions: np.ndarray, comm: Comm, N: int) -> torch.Tensor:
    """Rows of the picked unclassified samples, in pick order, on every rank."""
    dev = batch.device_states().device
    if not comm.distributed:
        idx_all = res.indices_device(_abi.LABEL_UNCLASSIFIED)
        sel = idx_all.index_select(0, torch.as_tensor(positions, dtype=torch.int64, device=dev))
        out = torch.empty((len(positions), N), dtype=torch.uint8, device=dev)
        _abi.call("rsr_gather_rows", _abi.ptr(batch.device_states()), N, _abi.ptr(sel),
                  len(positions), _abi.ptr(out), _device.stream())
        return out
    per_rank = comm.allgather_i64(res.counts[2])
    owner, local = global_pick_owners(per_rank, np.asarray(positions, dtype=np.int64))
    mine = np.flatnonzero(owner == comm.rank)
    rows = torch.empty((len(mine), N), dtype=torch.uint8, device=dev)
    if len(mine):
        idx_all = res.indices_device(_abi.LABEL_UNCLASSIFIED)
        sel = idx_all.index_select(0, torch.as_tensor(local[mine], dtype=torch.int64, device=dev))
        _abi.call("rsr_gather_rows", _abi.ptr(batch.device_states()), N, _abi.ptr(sel), len(mine),
                  _abi.ptr(rows), _device.stream())
    counts = np.bincount(owner, minlength=comm.world)
    gathered = comm.allgather_rows(rows, counts).to(dev)
    order = np.argsort(owner, kind="stable")  # rank-major position of each pick
    inv = np.empty_like(order)
    inv[order] = np.arange(len(order))
    return gathered.index_select(0, torch.as_tensor(inv, dtype=torch.int64, device=dev)).contiguous()


def _stage2_counts(model, dist, lower, upper, threshold, seed, start, count, comm):
    """(n_low, n_up, unclassified) of samples [start, start+count) of generation 0."""
    phi = model.device_phi()
    batch = sample_batch(dist, count, seed, _STAGE2_GENERATION, start)
    res = classify(batch, lower, upper, n_states=model.n_component_states)
    n_low, n_up, n_x = res.counts
    leq = 0
    if n_x:
        idx = res.indices_device(_abi.LABEL_UNCLASSIFIED)
        acc = torch.zeros(1, dtype=torch.int64, device=idx.device)
        phi.eval_into(batch.device_states(), idx, n_x, model.n_component_states, None, threshold, acc)
        leq = int(acc.item())
    local = np.array([n_low + leq, n_up + (n_x - leq), n_x], dtype=np.int64)
    return comm.allreduce_sum_i64(local) if comm.distributed else local


def stage2_evaluate(model: SystemModel, dist: ComponentDistribution, lower: ReferenceSet | None,
                    upper: ReferenceSet | None, config: RunConfig, threshold: int,
                    comm: Comm | None = None) -> Stage2Report:
    """Estimate P(S <= m') and P(S >= m'+1) from one classified batch (workflow.py:198-245)."""
    _check_threshold(model, threshold)
    for s in (lower, upper):
        if s is not None and s.threshold != threshold:
            raise ValueError(f"reference set threshold {s.threshold} != requested m'={threshold}")
    comm = comm or Comm.single()
    h = config.stage2_samples or config.n_samples
    start, count = shard_range(h, comm.world, comm.rank)
    n_low, n_up, n_x = (int(v) for v in _stage2_counts(model, dist, lower, upper, threshold,
                                                       config.seed, start, count, comm))
    model.add_evaluations(n_x)
    p_low, p_up = n_low / h, n_up / h
    return Stage2Report(p_lower=p_low, p_upper=p_up, cov_lower=cov(p_low, h),
                        cov_upper=cov(p_up, h), n_samples=h, unclassified_resolved=n_x,
                        threshold=threshold, seed=config.seed)


def stage2_until_cov(model: SystemModel, dist: ComponentDistribution, lower, upper,
                     config: RunConfig, threshold: int, target_cov: float = 0.05,
                     batch_samples: int | None = None, max_batches: int = 1_000_000,
                     side: str = "lower", comm: Comm | None = None) -> Stage2Report:
    """Run-to-c.o.v. loop (not in the reference).

    Batch j is samples [j*H, (j+1)*H) of the generation-0 stream, so batch 0
    is exactly ``stage2_evaluate``; integer counts accumulate until the
    c.o.v. of the chosen side's estimate is <= ``target_cov``.
    """
    _check_threshold(model, threshold)
    comm = comm or Comm.single()
    h = batch_samples or config.stage2_samples or config.n_samples
    tot = np.zeros(3, dtype=np.int64)
    n = 0
    for j in range(max_batches):
        start, count = shard_range(h, comm.world, comm.rank)
        tot += _stage2_counts(model, dist, lower, upper, threshold, config.seed, j * h + start,
                              count, comm)
        n += h
        p = (tot[0] if side == "lower" else tot[1]) / n
        c = cov(p, n)
        if c is not None and c <= target_cov:
            break
    model.add_evaluations(int(tot[2]))
    p_low, p_up = tot[0] / n, tot[1] / n
    return Stage2Report(p_lower=p_low, p_upper=p_up, cov_lower=cov(p_low, n),
                        cov_upper=cov(p_up, n), n_samples=n, unclassified_resolved=int(tot[2]),
                        threshold=threshold, seed=config.seed)


def assemble_pmf(cumulative) -> tuple[np.ndarray, float]:
    """diff / clamp / renormalise (workflow.py:258-271)."""
    cum = np.asarray(cumulative, dtype=np.float64)
    if cum.size and (cum.min() < 0.0 or cum.max() > 1.0):
        raise ValueError("cumulative probabilities must lie in [0, 1]")
    ext = np.concatenate([[0.0], cum, [1.0]])
    pmf = np.diff(ext)
    clipped = np.clip(pmf, 0.0, None)
    adjustment = float(np.abs(clipped - pmf).sum())
    return clipped / clipped.sum(), adjustment


def multistate_pmf(model: SystemModel, dist: ComponentDistribution, config: RunConfig,
                   comm: Comm | None = None) -> PmfReport:
    """Both stages for every threshold, composed into the PMF (workflow.py:274-321)."""
    m_s = model.n_system_states
    s1s, reps = [], []
    for threshold in range(m_s - 1):
        s1 = stage1_find_references(model, dist, config, threshold, comm)
        s2 = stage2_evaluate(model, dist, s1.lower, s1.upper, config, threshold, comm)
        s1s.append(s1)
        reps.append(s2)
    cum = np.array([r.p_lower for r in reps])
    sig = np.array([np.sqrt(r.p_lower * (1.0 - r.p_lower) / r.n_samples) for r in reps])
    for i in range(1, len(cum)):
        tol = 4.0 * (sig[i] + sig[i - 1])
        if cum[i] < cum[i - 1] - tol:
            raise ValueError(
                f"cumulative estimates non-monotone beyond tolerance at m'={i} "
                f"({cum[i]:.3e} < {cum[i - 1]:.3e} - {tol:.1e}); increase n_samples")
    pmf, adjustment = assemble_pmf(cum)
    surv = np.concatenate([[1.0], [r.p_upper for r in reps], [0.0]])
    pmf_upper_n, _ = assemble_pmf(np.cumsum(-np.diff(surv))[:-1])
    return PmfReport(pmf=pmf, cumulative_lower=cum, stage2_reports=tuple(reps),
                     stage1_results=tuple(s1s),
                     max_chain_discrepancy=float(np.max(np.abs(pmf - pmf_upper_n))),
                     renormalization_adjustment=adjustment)
