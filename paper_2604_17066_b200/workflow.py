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

import ctypes
import os
import time
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi, _device
from .boundary import ReferenceSet, Side, boundary_search_batch
from .classify import classify, cov, fp4_exact
from .dist import (Comm, counts_record, global_pick_owners, picks_in_prefix, shard_range,
                   split_records)
from .model import ComponentDistribution, SystemModel
from .sampling import rng_code as _rng_code
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
    # not in the reference: "shared" draws the reference's Philox4x64-10 stream
    # (bit-exact results); "device" the independent Philox4x32-10 device stream
    # (statistically equivalent estimates, north_star "independent device RNG")
    rng: str = "shared"

    def __post_init__(self) -> None:
        if self.n_samples < 1:
            raise ValueError("n_samples must be >= 1")
        if not 0.0 <= self.eps_u <= 1.0:
            raise ValueError("eps_u must lie in [0, 1]")
        if self.r_max < 1:
            raise ValueError("r_max must be >= 1")
        if self.parallel_searches < 1:
            raise ValueError("parallel_searches must be >= 1")
        if self.rng not in ("shared", "device"):
            raise ValueError("rng must be 'shared' or 'device'")


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

    def __init__(self, dist_, seed, start, count, rng="shared"):
        self.dist, self.seed, self.start, self.count = dist_, seed, start, count
        self.rng = rng
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
                                 out_states=b.states, out_fp4=b.fp4 if b.fp4_ok else None,
                                 rng=self.rng)
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
    if not comm.distributed:
        return batch, res, np.array(res.counts), None
    # one all-gather of every rank's counts: sums and per-rank unclassified counts
    per = comm.allgather_i64_vec(list(res.counts))
    return batch, res, per.sum(0), per[:, 2].copy()


def stage1_find_references(model: SystemModel, dist: ComponentDistribution, config: RunConfig,
                           threshold: int, comm: Comm | None = None, *,
                           _batch_cache: "_BatchCache | None" = None) -> Stage1Result:
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
    use_async = (os.environ.get("RSR_SYNC_LOOP") != "1"
                 and _abi.fp4_row_bytes(dist.n_components, dist.n_states) <= _abi.REFSET_MAX_ROW_BYTES
                 and fp4_exact()
                 and dist.n_states == model.n_component_states
                 and config.parallel_searches <= 4096)
    with torch.cuda.stream(loop_stream):
        if use_async:
            result = _stage1_loop_async(model, dist, config, threshold, comm, phi, lower, upper,
                                        start, count, H, t_start, phi_start, _batch_cache)
        else:
            result = _stage1_loop(model, dist, config, threshold, comm, phi, lower, upper, start,
                                  count, H, t_start, phi_start)
    caller.wait_stream(loop_stream)
    return result


def _stage1_loop(model, dist, config, threshold, comm, phi, lower, upper, start, count, H,
                 t_start, phi_start) -> Stage1Result:
    trace: list[TraceRecord] = []
    redundant = 0
    terminated_by = "r_max"
    pre = _Prefetcher(dist, config.seed, start, count, config.rng)
    pending = pre.launch(0)
    N = dist.n_components
    iteration = 0
    while True:
        batch, res, counts, per_rank = _classify_shard(model, pending, lower, upper, comm)
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
        x0 = _gather_picks(batch, res, positions, comm, N, per_rank)
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


class _DeviceRefs:
    """Both sides' members for one Stage-1 run, resident on the device.

    Per side: u8 rows [cap, N], FP4 operand rows [cap, row_bytes] (rows past
    the member count are never-hit pad rows, so the classifier may stream a
    host-side upper bound of the count), alive flags and counters, all updated
    by ``rsr_refset_insert`` (csrc/refset.cu).  The host learns the counts one
    iteration later from the loop's report buffer.
    """

    def __init__(self, n: int, m: int, dev: torch.device):
        self.N, self.M, self.dev = n, m, dev
        self.rb = _abi.fp4_row_bytes(n, m)
        self.ctr = torch.zeros((2, 2), dtype=torch.int64, device=dev)
        self.cap = [0, 0]
        self.rows: list = [None, None]
        self.fp4: list = [None, None]
        self.alive: list = [None, None]
        self.known = [0, 0]   # rows as of the last report read
        self.pending = 0      # candidates inserted since then (bound on new rows per side)
        self.desc = [_abi.RefsetDev(), _abi.RefsetDev()]
        for s in (0, 1):
            self._grow(s, 4 * _abi.FP4_TILE_ROWS)

    def _grow(self, s: int, need: int) -> None:
        tile = _abi.FP4_TILE_ROWS
        cap = max(need, 2 * self.cap[s])
        cap = (cap + tile - 1) // tile * tile
        rows = torch.zeros((cap, self.N), dtype=torch.uint8, device=self.dev)
        fp4 = torch.empty((cap, self.rb), dtype=torch.uint8, device=self.dev)
        alive = torch.zeros(cap, dtype=torch.uint8, device=self.dev)
        # all pad rows (bias column 1): never hit until a member overwrites them
        _abi.call("rsr_encode_refs_fp4", None, 0, cap, self.N, self.M, _side_code_int(s),
                  _abi.ptr(fp4), self.rb, _device.stream())
        old = self.cap[s]
        if old:
            rows[:old].copy_(self.rows[s])
            fp4[:old].copy_(self.fp4[s])
            alive[:old].copy_(self.alive[s])
        self.rows[s], self.fp4[s], self.alive[s], self.cap[s] = rows, fp4, alive, cap
        d = self.desc[s]
        d.rows, d.fp4, d.alive = rows.data_ptr(), fp4.data_ptr(), alive.data_ptr()
        d.ctr = self.ctr[s].data_ptr()
        d.cap = cap

    def bound(self, s: int) -> int:
        return self.known[s] + self.pending

    def prepare_insert(self, b: int, full_grid: bool = False) -> bool:
        """Capacity for b more rows per side; returns True if a buffer moved.
        full_grid sizes the member scan for the whole capacity (blocks past the
        device-side count exit at once), so the call can be replayed from a graph."""
        moved = False
        for s in (0, 1):
            if self.bound(s) + b > self.cap[s]:
                self._grow(s, self.bound(s) + b)
                moved = True
            self.desc[s].n_bound = self.cap[s] if full_grid else self.bound(s)
        return moved

    def to_sets(self, lower: ReferenceSet, upper: ReferenceSet, dropped: bool) -> None:
        """Hand the final members (alive rows in physical order) to the ReferenceSets."""
        for s, target in ((0, lower), (1, upper)):
            n = self.known[s]
            if n == 0:
                continue
            rows_h = self.rows[s][:n].cpu().numpy()
            if dropped:
                alive_h = self.alive[s][:n].cpu().numpy().astype(bool)
                if not alive_h.all():
                    target._set_rows(rows_h[alive_h])
                    continue
            target._append_host(rows_h)
            target._dev_rows, target._dev_n = self.rows[s], n
            target._fp4[self.M] = [self.fp4[s], n]


class _BatchCache:
    """FP4 sample operands by generation, kept in HBM across the thresholds of
    `multistate_pmf`.  Every threshold's Stage 1 walks generations 0, 1, ... of the
    same (seed, start, count) stream, so each threshold after the first reads the
    batches the first one drew instead of drawing them again (identical bits).
    Bounded by a share of the free device memory (B200: 180 GB; config 5 needs
    ~111 GB for 166 generations); generations past the budget are drawn as usual."""

    def __init__(self, count: int, row_bytes: int):
        free, total = torch.cuda.mem_get_info()
        # memory torch's caching allocator holds but does not use (e.g. a previous run's
        # cache slabs) is available too: counting only the driver's free memory left a
        # repeated multistate_pmf in one process with a smaller cache (config 5:
        # 0.37 -> 0.44 s on the second run)
        free += torch.cuda.memory_reserved() - torch.cuda.memory_allocated()
        self.shape = (max(count, 1), 2 * row_bytes)
        self.nbytes = self.shape[0] * self.shape[1]
        self.max_batches = max(0, free - max(16 << 30, total // 8)) // self.nbytes
        cap = os.environ.get("RSR_BATCH_CACHE_MAX")  # tests: force a partial cache
        if cap is not None:
            self.max_batches = min(self.max_batches, int(cap))
        self.batches: dict[int, torch.Tensor] = {}
        self.slabs: list[torch.Tensor] = []
        self.free_in_slab = 0

    def get(self, gen: int):
        return self.batches.get(gen)

    def reserve(self, gen: int):
        if len(self.batches) >= self.max_batches:
            return None
        if self.free_in_slab == 0:
            # slabs doubling from 16 batches: a handful of allocations (each cudaMalloc
            # costs milliseconds regardless of size, one per 671 MB batch would add up)
            n = min(max(16, len(self.batches)), self.max_batches - len(self.batches))
            self.slabs.append(torch.empty((n,) + self.shape, dtype=torch.uint8,
                                          device=_device.device()))
            self.free_in_slab = n
        slab = self.slabs[-1]
        t = slab[slab.shape[0] - self.free_in_slab]
        self.free_in_slab -= 1
        self.batches[gen] = t
        return t


class _LeanPrefetcher:
    """`_Prefetcher` for the one-sync loop: preallocated double buffers and events,
    `rsr_sample_fp4` called directly on the side stream (no per-batch Python objects).
    With a `_BatchCache`, generations already drawn are read from it (their picks are
    decoded from the FP4 rows) and new ones are drawn into it."""

    def __init__(self, dist_, seed, start, count, m, cache: _BatchCache | None = None,
                 rng: str = "shared"):
        dev = _device.device()
        self.rng = _rng_code(rng)
        n = dist_.n_components
        self.n, self.m, self.seed, self.start, self.count = n, m, seed, start, count
        self.rb = _abi.fp4_row_bytes(n, m)
        self.probs = _abi.ptr(dist_.device_probs())
        self.fp4 = [torch.empty((max(count, 1), 2 * self.rb), dtype=torch.uint8, device=dev)
                    for _ in range(2)]
        self.stream = torch.cuda.Stream()
        self.sptr = self.stream.cuda_stream
        self.ready = [torch.cuda.Event(), torch.cuda.Event()]
        self.free = [torch.cuda.Event(), torch.cuda.Event()]
        self.free_used = [False, False]
        self.cache = cache
        self.src = list(self.fp4)        # FP4 operand of the batch in each slot

    def launch(self, gen: int) -> int:
        slot = gen & 1
        if self.free_used[slot]:
            self.stream.wait_event(self.free[slot])
        cached = self.cache.get(gen) if self.cache is not None else None
        if cached is not None:
            self.src[slot] = cached
        else:
            dst = self.cache.reserve(gen) if self.cache is not None else None
            dst = self.fp4[slot] if dst is None else dst
            mask = (1 << 64) - 1
            # FP4 operand only: the picks are decoded from its rows (rsr_gather_picks_fp4),
            # so the u8 state rows are not written at all
            _abi.call("rsr_sample_fp4_ex", self.probs, self.n, self.m, self.seed & mask,
                      gen & mask, self.start, self.count, None, _abi.ptr(dst), self.rb, 0,
                      self.rng, self.sptr)
            self.src[slot] = dst
        self.ready[slot].record(self.stream)
        return slot

    def release(self, gen: int, stream: torch.cuda.Stream) -> None:
        self.free[gen & 1].record(stream)
        self.free_used[gen & 1] = True

    def close(self, stream: torch.cuda.Stream) -> None:
        stream.wait_stream(self.stream)


def _side_code_int(s: int) -> int:
    return _abi.SIDE_UPPER if s == 1 else _abi.SIDE_LOWER


def _stage1_loop_async(model, dist, config, threshold, comm, phi, lower, upper, start, count, H,
                       t_start, phi_start, batch_cache=None) -> Stage1Result:
    """Stage-1 loop with one host synchronisation per iteration.

    Stream order per iteration i: classify(i) -> finalize counts -> report
    copy (also carries iteration i-1's insertion outcome) | host: trace,
    termination tests, the reference's picks (default_rng([seed, i]).choice)
    -> compact + gather picks -> boundary search -> rsr_refset_insert ->
    classify(i+1).  The host's bookkeeping for iteration i+1 overlaps the
    device's search and insertion of iteration i; results (ordered sets, trace,
    redundant searches, Phi counts) are those of workflow.py:122-195.
    """
    dev = _device.device()
    N, M = dist.n_components, model.n_component_states
    B = config.parallel_searches
    st_ptr = _device.stream()
    main = torch.cuda.current_stream()
    refs = _DeviceRefs(N, M, dev)
    rb = refs.rb
    report_d = torch.zeros(16, dtype=torch.int64, device=dev)  # [0:4] counts, [4:12] insert report
    report_h = torch.empty(16, dtype=torch.int64, pin_memory=True)
    rep = report_h.numpy()
    flags = torch.empty(max(count, 1), dtype=torch.uint8, device=dev)
    labels = torch.empty(max(count, 1), dtype=torch.uint8, device=dev)
    # zero-initialised: the speculative prefix gather may read entries past the count
    idx = torch.zeros(max(count, 1), dtype=torch.int64, device=dev)
    cnt = torch.empty(1, dtype=torch.int64, device=dev)
    cscratch = torch.empty(max(1, _abi.call("rsr_compact_scratch", count)), dtype=torch.int64,
                           device=dev)
    # multi-rank: one all-gather per iteration of [counts | rows of the first C
    # unclassified samples] (dist.py); C = B covers every pick of a rank with at most
    # B unclassified samples
    C = B if comm.distributed else 0
    pref_pos = torch.arange(max(C, 1), dtype=torch.int64, device=dev)
    pref_rows = torch.zeros((max(C, 1), N), dtype=torch.uint8, device=dev)
    exch = {}
    pos_h = torch.empty(B, dtype=torch.int64, pin_memory=True)
    pos_d = torch.empty(B, dtype=torch.int64, device=dev)
    x0 = torch.empty((B, N), dtype=torch.uint8, device=dev)
    out_refs = torch.empty((B, N), dtype=torch.uint8, device=dev)
    out_side = torch.empty(B, dtype=torch.uint8, device=dev)
    out_calls = torch.empty(B, dtype=torch.int64, device=dev)
    outcome = torch.empty(B, dtype=torch.uint8, device=dev)
    iscratch = torch.empty(max(1, _abi.call("rsr_refset_scratch", B, rb)), dtype=torch.uint8,
                           device=dev)
    phi_vals = torch.empty(B, dtype=torch.uint8, device=dev)
    desc = phi.descriptor(M)
    ready_ev = torch.cuda.Event()
    lo_p = ctypes.byref(refs.desc[0])
    up_p = ctypes.byref(refs.desc[1])

    pre = _LeanPrefetcher(dist, config.seed, start, count, M, batch_cache, config.rng)

    # Two-pass classification: most samples are dominated by one of the first
    # upper references (tools/first_match_hist.py: after 480 of cfg3's 10^4
    # references 0.4 % remain), so pass 1 runs every lower reference and the
    # first `pass1` upper rows over the whole batch, and pass 2 only the samples
    # still without a hit (compacted and gathered on the device, count never
    # leaves the device) against the remaining upper rows.  Labels are those of
    # a single pass.
    pass1 = int(os.environ.get("RSR_LOOP_PASS1_ROWS", str(2 * _abi.FP4_TILE_ROWS)))
    pass2_min = int(os.environ.get("RSR_LOOP_PASS2_MIN", str(2 * _abi.FP4_TILE_ROWS)))
    two_pass = {}

    def two_pass_buffers():  # allocated up front: a large first allocation costs milliseconds
        if not two_pass:
            two_pass["a2"] = torch.empty((max(count, 1), 2 * rb), dtype=torch.uint8, device=dev)
            two_pass["f2"] = torch.empty(max(count, 1), dtype=torch.uint8, device=dev)
            two_pass["idx"] = torch.empty(max(count, 1), dtype=torch.int64, device=dev)
            two_pass["cnt"] = torch.empty(1, dtype=torch.int64, device=dev)
        return two_pass["a2"], two_pass["f2"], two_pass["idx"], two_pass["cnt"]

    if pass1 > 0:
        two_pass_buffers()

    def launch_classify(slot):
        main.wait_event(pre.ready[slot])
        a = pre.src[slot]
        nl, nu = refs.bound(0), refs.bound(1)
        bl = _abi.ptr(refs.fp4[0]) if nl else None
        # rows past a side's bound are never-hit pad rows up to its capacity
        cl, cu = refs.cap
        if pass1 > 0 and nu > pass1 + pass2_min:
            a2, f2, idx2, cnt2 = two_pass_buffers()
            _abi.call("rsr_classify_fp4_ex", _abi.ptr(a), count, None, bl, nl, cl,
                      _abi.ptr(refs.fp4[1]), pass1, pass1, rb, _abi.ptr(flags), None, None, 0,
                      st_ptr)
            _abi.call("rsr_compact", _abi.ptr(flags), count, 0, _abi.ptr(idx2), _abi.ptr(cnt2),
                      _abi.ptr(cscratch), st_ptr)
            _abi.call("rsr_gather_rows_dev", _abi.ptr(a), 2 * rb, rb, _abi.ptr(idx2), _abi.ptr(cnt2),
                      count, _abi.ptr(a2), 2 * rb, st_ptr)
            _abi.call("rsr_classify_fp4_ex", _abi.ptr(a2), count, _abi.ptr(cnt2), None, 0, 0,
                      _abi.ptr(refs.fp4[1][pass1:]), nu - pass1, cu - pass1, rb, _abi.ptr(f2), None,
                      None, 0, st_ptr)
            _abi.call("rsr_scatter_or_dev", _abi.ptr(f2), _abi.ptr(idx2), _abi.ptr(cnt2), count,
                      _abi.ptr(flags), st_ptr)
        else:
            _abi.call("rsr_classify_fp4_ex", _abi.ptr(a), count, None, bl, nl, cl,
                      _abi.ptr(refs.fp4[1]) if nu else None, nu, cu, rb, _abi.ptr(flags), None,
                      None, 0, st_ptr)
        _abi.call("rsr_finalize", _abi.ptr(flags), count, _abi.ptr(labels), _abi.ptr(report_d),
                  st_ptr)
        if comm.distributed:
            _abi.call("rsr_compact", _abi.ptr(labels), count, _abi.LABEL_UNCLASSIFIED,
                      _abi.ptr(idx), _abi.ptr(cnt), _abi.ptr(cscratch), st_ptr)
            gather_rows_at(slot, pref_pos, C, pref_rows, st_ptr)
            exch["recs"] = comm.allgather_bytes(counts_record(report_d[:4], pref_rows))
        report_h.copy_(report_d, non_blocking=True)
        ready_ev.record(main)
        return slot

    def gather_rows_at(slot, pos_dev, n, out, sp):
        """out[j] = state row of local unclassified position pos_dev[j] (idx compacted)."""
        _abi.call("rsr_gather_picks_fp4", _abi.ptr(pre.src[slot]), rb, N, M, _abi.ptr(idx),
                  _abi.ptr(pos_dev), n, _abi.ptr(out), sp)

    def gather_local(slot, n_local, out):
        """Rows of this rank's picks (local positions in pos_h) -> out[:n_local]."""
        pos_d[:n_local].copy_(pos_h[:n_local], non_blocking=True)
        sp = _device.stream()
        _abi.call("rsr_compact", _abi.ptr(labels), count, _abi.LABEL_UNCLASSIFIED, _abi.ptr(idx),
                  _abi.ptr(cnt), _abi.ptr(cscratch), sp)
        gather_rows_at(slot, pos_d, n_local, out, sp)

    def search_and_insert(slot, n_pick, gather=True):
        """positions -> picked rows -> boundary searches -> device insertion: fixed
        pointers and sizes per (batch slot, number of picks), so after the first
        iteration of each kind the sequence replays as one CUDA graph."""
        if gather:
            gather_local(slot, n_pick, x0)
        sp = _device.stream()
        if config.boundary_search_enabled:
            _abi.call("rsr_boundary_search", ctypes.byref(desc), int(threshold), _abi.ptr(x0),
                      n_pick, _abi.ptr(out_refs), _abi.ptr(out_side), _abi.ptr(out_calls), sp)
            cands, calls_p = out_refs, _abi.ptr(out_calls)
        else:
            phi.eval_into(x0, None, n_pick, M, phi_vals)
            # SIDE_LOWER = 0 when Phi <= m', SIDE_UPPER = 1 otherwise
            torch.gt(phi_vals[:n_pick], threshold, out=out_side[:n_pick])
            cands, calls_p = x0, None
        _abi.call("rsr_refset_insert", _abi.ptr(cands), _abi.ptr(out_side), n_pick, N, M, lo_p,
                  up_p, calls_p, _abi.ptr(outcome), _abi.ptr(report_d[4:]), _abi.ptr(iscratch), sp)

    # graphs only for the boundary-search path (the raw-sample path runs torch ops)
    # on one rank (a multi-rank iteration exchanges picked rows through the host)
    # (and not with a batch cache, whose source buffers change per generation)
    use_graphs = (config.boundary_search_enabled and not comm.distributed
                  and batch_cache is None and os.environ.get("RSR_LOOP_GRAPHS", "1") != "0")
    graphs: dict = {}
    trace: list[TraceRecord] = []
    terminated_by = "r_max"
    slot = launch_classify(pre.launch(0))
    pending = pre.launch(1)
    iteration = 0
    searched = False          # an insertion report is outstanding
    no_search_picks = 0       # Phi calls of the last batch when searches are disabled
    nvtx = torch.cuda.nvtx if os.environ.get("RSR_NVTX") == "1" else None  # profiler ranges
    while True:
        if nvtx is not None:
            if iteration:
                nvtx.range_pop()
            nvtx.range_push(f"rsr.stage1 m'={threshold} it={iteration}")
        ready_ev.synchronize()
        n_l, n_u, n_x = int(rep[0]), int(rep[1]), int(rep[2])
        if comm.distributed:  # shard counts -> batch counts; per-rank unclassified counts
            counts_all, prefix = split_records(exch.pop("recs"), 4, C, N)
            per_rank = counts_all[:, 2].copy()
            n_l, n_u, n_x = (int(v) for v in counts_all[:, :3].sum(0))
        if searched:
            refs.known = [int(rep[4]), int(rep[6])]
            refs.pending = 0
            model.add_evaluations(int(rep[10]) if config.boundary_search_enabled else no_search_picks)
            if rep[11]:
                raise RuntimeError("rsr_refset_insert: reference capacity overflow")
            searched = False
        n_refs = int(rep[5] + rep[7]) if iteration else 0
        trace.append(TraceRecord(
            reference_count=n_refs,
            elapsed_seconds=time.perf_counter() - t_start,
            phi_evaluations=model.evaluation_count - phi_start,
            p_lower=n_l / H, p_upper=n_u / H, p_unclassified=n_x / H,
            resident_memory_bytes=_rss_bytes()))
        if n_x / H <= config.eps_u:
            terminated_by = "eps_u"
            break
        if n_refs >= config.r_max:
            break
        rng = np.random.default_rng([config.seed, iteration])
        n_pick = min(B, n_x)
        positions = rng.choice(n_x, size=n_pick, replace=False)
        if comm.distributed:
            # global positions (rank-ordered unclassified list) -> owners; every rank
            # gathers its own rows, then all picked rows in pick order on every rank
            owner, local = global_pick_owners(per_rank, np.asarray(positions, dtype=np.int64))
            if picks_in_prefix(owner, local, C):
                # every picked row arrived with the counts: no second exchange
                sel = torch.as_tensor(owner * C + local, dtype=torch.int64).to(dev, non_blocking=True)
                torch.index_select(prefix.reshape(-1, N), 0, sel, out=x0[:n_pick])
            else:
                mine = np.flatnonzero(owner == comm.rank)
                pos_h.numpy()[:len(mine)] = local[mine]
                rows = torch.empty((len(mine), N), dtype=torch.uint8, device=dev)
                if len(mine):
                    gather_local(slot, len(mine), rows)
                gathered = comm.allgather_rows(rows, np.bincount(owner, minlength=comm.world)).to(dev)
                order = np.argsort(owner, kind="stable")
                inv = np.empty_like(order)
                inv[order] = np.arange(len(order))
                x0[:n_pick].copy_(gathered.index_select(
                    0, torch.as_tensor(inv, dtype=torch.int64, device=dev)))
        else:
            pos_h.numpy()[:n_pick] = positions
        if refs.prepare_insert(n_pick, full_grid=use_graphs):
            graphs.clear()  # device buffers moved: captured launches are stale
        key = (slot, n_pick)
        g = graphs.get(key)
        # capture only the steady state (a full batch of picks): the tail of a run,
        # where fewer than B samples stay unclassified, changes n_pick every iteration
        if g is None and use_graphs and n_pick == B:
            g = graphs[key] = torch.cuda.CUDAGraph()
            g.capture_begin(capture_error_mode="relaxed")
            search_and_insert(slot, n_pick)
            g.capture_end()
        if g is not None:
            g.replay()
        else:
            search_and_insert(slot, n_pick, gather=not comm.distributed)
            if not config.boundary_search_enabled:
                no_search_picks = n_pick
        pre.release(iteration, main)
        refs.pending = n_pick
        searched = True
        iteration += 1
        slot = launch_classify(pending)
        pending = pre.launch(iteration + 1)
    if nvtx is not None:
        nvtx.range_pop()
    pre.close(main)
    refs.to_sets(lower, upper, dropped=bool(rep[9]))
    return Stage1Result(lower=lower, upper=upper, trace=trace, iterations=iteration + 1,
                        redundant_searches=int(rep[8]), terminated_by=terminated_by)


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


def _gather_picks(batch, res, positions: np.ndarray, comm: Comm, N: int,
                  per_rank: np.ndarray | None = None) -> torch.Tensor:
    """Rows of the picked unclassified samples, in pick order, on every rank."""
    dev = batch.device_states().device
    if not comm.distributed:
        idx_all = res.indices_device(_abi.LABEL_UNCLASSIFIED)
        sel = idx_all.index_select(0, torch.as_tensor(positions, dtype=torch.int64, device=dev))
        out = torch.empty((len(positions), N), dtype=torch.uint8, device=dev)
        _abi.call("rsr_gather_rows", _abi.ptr(batch.device_states()), N, _abi.ptr(sel),
                  len(positions), _abi.ptr(out), _device.stream())
        return out
    if per_rank is None:
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


def _stage2_counts(model, dist, lower, upper, threshold, seed, start, count, comm, rng="shared"):
    """(n_low, n_up, unclassified) of samples [start, start+count) of generation 0."""
    phi = model.device_phi()
    batch = sample_batch(dist, count, seed, _STAGE2_GENERATION, start, rng=rng)
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
                                                       config.seed, start, count, comm,
                                                       config.rng))
    model.add_evaluations(n_x)
    p_low, p_up = n_low / h, n_up / h
    return Stage2Report(p_lower=p_low, p_upper=p_up, cov_lower=cov(p_low, h),
                        cov_upper=cov(p_up, h), n_samples=h, unclassified_resolved=n_x,
                        threshold=threshold, seed=config.seed)


def stage2_until_cov(model: SystemModel, dist: ComponentDistribution, lower, upper,
                     config: RunConfig, threshold: int, target_cov: float = 0.05,
                     batch_samples: int | None = None, max_batches: int = 1_000_000,
                     side: str = "lower", comm: Comm | None = None,
                     max_samples: int | None = 1 << 36) -> Stage2Report:
    """Run-to-c.o.v. loop (not in the reference).

    Batch j is samples [j*H, (j+1)*H) of the generation-0 stream, so batch 0
    is exactly ``stage2_evaluate``; integer counts accumulate until the
    c.o.v. of the chosen side's estimate is <= ``target_cov``.  The loop also
    stops after ``max_batches`` batches or ``max_samples`` samples (an estimate
    that stays 0 has no c.o.v.), with a RuntimeWarning.
    """
    _check_threshold(model, threshold)
    if side not in ("lower", "upper"):
        raise ValueError(f"side must be 'lower' or 'upper', got {side!r}")
    if not target_cov > 0.0:
        raise ValueError("target_cov must be > 0")
    for s in (lower, upper):
        if s is not None and s.threshold != threshold:
            raise ValueError(f"reference set threshold {s.threshold} != requested m'={threshold}")
    comm = comm or Comm.single()
    h = batch_samples or config.stage2_samples or config.n_samples
    if h < 1:
        raise ValueError("batch_samples must be >= 1")
    limit = max_batches if max_samples is None else max(1, min(max_batches, max_samples // h))
    tot = np.zeros(3, dtype=np.int64)
    n = 0
    reached = False
    for j in range(limit):
        start, count = shard_range(h, comm.world, comm.rank)
        tot += _stage2_counts(model, dist, lower, upper, threshold, config.seed, j * h + start,
                              count, comm, config.rng)
        n += h
        p = (tot[0] if side == "lower" else tot[1]) / n
        c = cov(p, n)
        if c is not None and c <= target_cov:
            reached = True
            break
    if not reached:
        warnings.warn(f"stage2_until_cov stopped after {n} samples without reaching c.o.v. "
                      f"{target_cov} on the {side} estimate", RuntimeWarning, stacklevel=2)
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
    # thresholds share the sample stream: keep the drawn batches in HBM between them
    cache = None
    if (m_s > 2 and torch.cuda.is_available() and os.environ.get("RSR_BATCH_CACHE", "1") != "0"
            and dist.n_states == model.n_component_states
            and _abi.fp4_row_bytes(dist.n_components, dist.n_states) <= _abi.REFSET_MAX_ROW_BYTES):
        comm_ = comm or Comm.single()
        _, count = shard_range(config.n_samples, comm_.world, comm_.rank)
        cache = _BatchCache(count, _abi.fp4_row_bytes(dist.n_components, dist.n_states))
    for threshold in range(m_s - 1):
        s1 = stage1_find_references(model, dist, config, threshold, comm, _batch_cache=cache)
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
