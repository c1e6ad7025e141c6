#!/usr/bin/env python
"""Benchmark of the RSR dominance-classification hot path on B200.

Default workload (BASELINE.json configs[3] at its north-star point, "cfg4"):
S = 2^22 samples in total (Bernoulli(0.9), N = 295 components, drawn by the
device Philox sampler) against K = 5x10^5 random simple s-t path references
(upper side) on the 119-node / 295-edge config-3 graph.  Strong scaling: with
N GPUs each rank owns 2^22 / N samples of the same stream (start offsets) and
the whole reference set.  A step is one classification of the resident
samples against all K references: the support-compaction re-pack of the sample
plane (rsr_fp4_gather_columns: only the ~222 of 295 components some path uses can
add a violation, so rows shrink from 5 to 4 64-column K-steps; the library's cost
model decides, classify.fp4_compaction), rsr_classify_fp4_planar (tcgen05
block-scaled FP4 0/1 contraction, paired accumulators at 4 K-steps, fused any-zero
epilogue; the launches of rsr_classify_fp4_plan: L2-sized reference chunks at
K = 5x10^5) + rsr_finalize (labels + counts), plus an NCCL all-reduce of the counts
when N > 1.  Metric: classified samples x reference states per second (pairs/s).
`--method tc8` / `bits` time the int8 tcgen05 and bit-packed CUDA-core
variants instead.

Secondary keys of the default line: `cfg4_sweep` (K = 10^3, 10^4, 10^5),
`cfg2` (BASELINE configs[1]), `wall_time_to_cov` (config 3 loop to c.o.v.
0.05, with a same-run CPU slice of the reference loop) and the path's other
kernels.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N` (N > 1) without torchrun re-launches itself under
`python -m torch.distributed.run --nproc-per-node N` (127.0.0.1 rendezvous).
Other workloads for the profiles/ notes: --config cfg2 / cfg2_mixed / cfg4
--k K, --config cfg1 / cfg3 / cfg5 (full RSR loop wall time).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "classified samples·ref-states/sec"
UNIT = "pairs/s"
N_COMP = 295
REF_PKG = os.path.join(ROOT, "baseline", "_ref")


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="cfg4",
                   choices=["cfg4", "cfg2", "cfg2_mixed", "cfg1", "cfg3", "cfg5"])
    p.add_argument("--parallel-searches", type=int, default=64)
    p.add_argument("--shard-refs", action="store_true",
                   help="N>1: shard reference states across all ranks, OR-reduce hit flags")
    p.add_argument("--ref-shards", type=int, default=1,
                   help="N>1: G_k reference shards per sample shard (G_k divides N)")
    p.add_argument("--k", type=int, default=None,
                   help="refs per side (cfg2, default 10^4) / path refs (cfg4, default 5x10^5)")
    p.add_argument("--samples", type=int, default=None,
                   help="samples in total over all ranks (default 2^22 cfg4, 2^20 cfg2)")
    p.add_argument("--weak", action="store_true",
                   help="--samples per rank instead of in total (weak scaling)")
    p.add_argument("--method", choices=["tc", "tc8", "bits"], default="tc",
                   help="tc: FP4 (kind::mxf4) tensor cores; tc8: int8 tensor cores; bits: CUDA cores")
    p.add_argument("--rng", choices=["shared", "device"], default="shared",
                   help="loops: the reference's Philox4x64-10 stream or the independent device stream")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-loop", action="store_true",
                   help="skip the wall-time-to-c.o.v. loops attached to the default run")
    p.add_argument("--no-secondary", action="store_true",
                   help="skip cfg2 / sweep / secondary kernels of the default run")
    p.add_argument("--cpu-seconds", type=float, default=None,
                   help="CPU work per baseline slice (default: sized so the run takes minutes)")
    p.add_argument("--loop-cpu-reference", action="store_true",
                   help="loop CPU baseline: run the installed reference itself (minutes)")
    return p.parse_args(argv)


# ----------------------------------------------------------------- workloads

def workload(config: str, k: int | None, samples: int | None):
    """(p_survive, lower rows, upper rows, S_total, description).  cfg4's path rows
    come from a batched Bellman-Ford in torch on the GPU when one is present (setup
    data, not the measured path)."""
    from paper_2604_17066_b200 import workloads as W
    if config == "cfg2":
        k = k or 10_000
        lower, upper = W.cfg2_refs(0, N_COMP, k, k)
        S = samples or (1 << 20)
        desc = (f"cfg2: S=2^{int(np.log2(S))} x N=295 Bernoulli(0.9), K={len(upper)} upper "
                f"(15 ones) + {len(lower)} lower (10 zeros)")
        return 0.9, lower, upper, S, desc
    if config == "cfg2_mixed":
        k = k or 10_000
        lower, upper = W.cfg2_mixed_refs(0, N_COMP, k, k)
        S = samples or (1 << 20)
        return 0.5, lower, upper, S, f"cfg2-mixed: S={S}, p=0.5, 15-one upper / 14-zero lower"
    k = k or 500_000
    g = W.cfg3(0)
    upper = W.random_st_paths(g, k, seed=0)
    lower = np.zeros((0, N_COMP), dtype=np.uint8)
    S = samples or (1 << 22)
    return 0.9, lower, upper, S, (f"cfg4: S=2^{int(np.log2(S))} Bernoulli(0.9) x N=295, "
                                  f"K={len(upper)} s-t path refs (mean "
                                  f"{upper.sum(1).mean():.1f} edges), upper side")


# ------------------------------------------------------- CPU reference legs

def reference_pkg():
    """The unmodified reference package (`rsr`), installed into baseline/_ref by
    baseline/install_ref.sh (pip --target from /root/reference; it travels to the
    GPU box with the snapshot).  None when absent."""
    if not os.path.isdir(os.path.join(REF_PKG, "rsr")):
        return None
    if REF_PKG not in sys.path:
        sys.path.append(REF_PKG)
    import rsr
    return rsr


class CpuClassify:
    """The reference's classification (classify.py:187-249) on the host cores for
    bounded slices of the same workload.

    kind "reference": the installed reference itself.  Per slice: its
    `encode_batch` of the samples, then `_hits_for`'s work over the slice
    (classify.py:121-148: ThreadPoolExecutor(n_workers) over chunks, each chunk
    the reference's own `_chunk_hits` -> `_violation_block_packed`, popcount
    summed in int32) per side, and the lower-precedence partition.  The
    reference sets are encoded once (`encode_batch(...).packed_complement`):
    `classify` re-encodes them on every call, an O(K) cost (10 s at K = 5x10^5,
    mostly `ReferenceSet.as_array`) that a full-size single call amortises over
    2^22 samples, so it is measured once (`public_api`) and kept out of the rate.
    kind "port": the oracle restatement (oracle/core.py), when the reference is
    not installed.  n_workers = all host cores, chunk = rows / (4 cores)
    (SURVEY 8d); sample generation is outside the timing."""

    def __init__(self, p1, lower_rows, upper_rows):
        self.rsr = reference_pkg()
        self.kind = "reference" if self.rsr is not None else "port"
        self.cores = len(os.sched_getaffinity(0))
        self.lower = np.asarray(lower_rows, dtype=np.int64)
        self.upper = np.asarray(upper_rows, dtype=np.int64)
        self.K = len(self.lower) + len(self.upper)
        self.probs = np.tile([1 - p1, p1], (N_COMP, 1))
        if self.rsr is not None:
            r = self.rsr
            self.dist = r.ComponentDistribution(self.probs)
            self.rbar = {}
            for side, rows, kind in (("lower", self.lower, "lower_ref"),
                                     ("upper", self.upper, "upper_ref")):
                self.rbar[side] = (r.encode_batch(rows, 2, kind).packed_complement
                                   if len(rows) else None)

    def _samples(self, rows, start):
        if self.rsr is not None:
            return self.rsr.sample_batch(self.dist, rows, 0, 0, start).states
        import oracle
        return oracle.sample_states(self.probs, rows, 0, 0, start, fast=True)

    def chunk(self, rows):
        return max(1, rows // (4 * self.cores)) if self.cores > 1 else 65536

    def run(self, rows, start=0):
        """Classify `rows` samples starting at stream position `start`; returns
        (pairs/s, seconds, label counts)."""
        xs = self._samples(rows, start)
        ch = self.chunk(rows)
        t0 = time.perf_counter()
        if self.rsr is None:
            import oracle
            res = oracle.classify_labels(xs, self.lower, self.upper, 2, chunk_size=ch,
                                         n_workers=self.cores)
            labels = res["labels"]
        else:
            from concurrent.futures import ThreadPoolExecutor
            from rsr.classify import _chunk_hits
            enc = self.rsr.encode_batch(xs, 2, "sample").packed
            bounds = [(s, min(s + ch, rows)) for s in range(0, rows, ch)]
            hits = {}
            with ThreadPoolExecutor(max_workers=self.cores) as pool:
                for side in ("lower", "upper"):
                    rb = self.rbar[side]
                    if rb is None:
                        hits[side] = np.zeros(rows, dtype=bool)
                        continue
                    parts = list(pool.map(lambda b: _chunk_hits(enc[b[0]:b[1]], rb, False)[0],
                                          bounds))
                    hits[side] = np.concatenate(parts)
            labels = np.full(rows, 2, dtype=np.uint8)
            labels[hits["upper"]] = 1
            labels[hits["lower"]] = 0
        dt = time.perf_counter() - t0
        return rows * self.K / dt, dt, np.bincount(labels, minlength=3).tolist()

    def calibrate(self, target_s):
        """Rows per slice so that one slice takes about `target_s` seconds, in whole
        rounds of 4 x cores chunks of 16 rows (so both CPU legs -- this line's
        cpu_baseline and the reference arm -- land on the same slice size)."""
        quantum = 4 * self.cores * 16
        rate, dt, _ = self.run(quantum, start=1 << 40)
        rounds = max(1, round(rate * target_s / max(1, self.K) / quantum))
        return int(min(1 << 20, rounds * quantum))

    def public_api(self, rows):
        """One call of the reference's public `rsr.classify` on a slice, including
        its per-call reference-set conversion and encoding (diagnostic)."""
        r = self.rsr
        if r is None:
            return None
        lo = r.ReferenceSet(r.Side.LOWER, 0)
        up = r.ReferenceSet(r.Side.UPPER, 0)
        lo._members = list(map(tuple, self.lower.tolist()))  # recipe of BASELINE.md / SURVEY 8d
        up._members = list(map(tuple, self.upper.tolist()))
        b = r.sample_batch(self.dist, rows, 0, 0, 0)
        t0 = time.perf_counter()
        r.classify(b, lo, up, chunk_size=self.chunk(rows), n_workers=self.cores, n_states=2)
        t_rows = time.perf_counter() - t0
        b1 = r.sample_batch(self.dist, 1, 0, 0, 0)
        t0 = time.perf_counter()
        r.classify(b1, lo, up, chunk_size=1, n_workers=self.cores, n_states=2)
        t_fixed = time.perf_counter() - t0
        return {"rows": rows, "seconds": t_rows, "pairs_per_s_incl_fixed": rows * self.K / t_rows,
                "fixed_cost_s": t_fixed,
                "api": "rsr.classify(batch, lower, upper, chunk_size, n_workers, n_states=2)"}

    def describe(self, rows, desc):
        what = ("installed reference (baseline/_ref): encode_batch + classify.py:121-148 "
                "_hits_for work (ThreadPool over chunks of _chunk_hits), refs pre-encoded"
                if self.kind == "reference" else
                "oracle port of classify.py:99-148 (packbits + bitwise_count int32 sums)")
        return (f"{rows} samples/slice x {self.K} refs of {desc}; {what}, "
                f"n_workers={self.cores}, chunk={self.chunk(rows)}")


def cpu_slice_seconds(args, default):
    return args.cpu_seconds if args.cpu_seconds is not None else default


# ------------------------------------------------------------------- clocks

class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        """index: the CUDA device ordinal of this process; NVML is addressed by the
        device's PCI bus id (NVML ordinals ignore CUDA_VISIBLE_DEVICES)."""
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = None
            try:  # match the CUDA device's PCI location against NVML's devices
                prop = torch.cuda.get_device_properties(index)
                want = (int(prop.pci_domain_id), int(prop.pci_bus_id), int(prop.pci_device_id))
                for i in range(pynvml.nvmlDeviceGetCount()):
                    h = pynvml.nvmlDeviceGetHandleByIndex(i)
                    pci = pynvml.nvmlDeviceGetPciInfo(h)
                    if (int(pci.domain), int(pci.bus), int(pci.device)) == want:
                        self.h = h
                        break
            except Exception:
                self.h = None
            if self.h is None:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(
                    min(index, pynvml.nvmlDeviceGetCount() - 1))
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# -------------------------------------------------------------------- peaks

def secondary_kernels():
    """Device time of the path's other kernels on their config shapes (CUDA events,
    mean of 10 launches): the sampler (Philox4x64-10 + inverse CDF + FP4 operand,
    integer-multiply bound; HBM write rate reported against the measured copy
    bandwidth), Stage-2 Phi evaluation and the loop's boundary searches."""
    import numpy as np
    import torch

    import paper_2604_17066_b200 as P
    from paper_2604_17066_b200 import _abi, workloads as W

    def timed(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        e.synchronize()
        return s.elapsed_time(e) / reps

    out = {}
    S = 1 << 20
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs") or peaks.get("hbm_GBps") or peaks.get("copy_gbs")
    for m, probs in ((2, [0.1, 0.9]), (3, [0.05, 0.15, 0.8])):
        d = P.ComponentDistribution.iid(N_COMP, probs)
        rb = _abi.fp4_row_bytes(N_COMP, m)
        st = torch.empty((S, N_COMP), dtype=torch.uint8, device="cuda")
        a4 = torch.empty((S, 2 * rb), dtype=torch.uint8, device="cuda")
        pr = d.device_probs()
        for rng, code in (("shared", _abi.RNG_SHARED), ("device", _abi.RNG_DEVICE)):
            ms = timed(lambda: _abi.call("rsr_sample_fp4_ex", _abi.ptr(pr), N_COMP, m, 0, 1, 0, S,
                                         _abi.ptr(st), _abi.ptr(a4), rb, S * rb, code,
                                         _abi.stream_ptr()))
            wbytes = S * (N_COMP + 2 * rb)
            out[f"sample_rows_kernel_M{m}_{rng}"] = {
                "shape": f"2^20 x {N_COMP} draws", "ms": ms,
                "draws_per_s": S * N_COMP / (ms * 1e-3),
                "hbm_write_gbs": wbytes / (ms * 1e-3) / 1e9, "hbm_peak_gbs": hbm,
                "stream": ("Philox4x64-10 (reference stream, bit-exact)" if rng == "shared" else
                           "Philox4x32-10 (independent device stream)"),
                "bound": "integer multiply (FMA pipe), not HBM"}
        del st, a4
    g = W.cfg3(0)
    graph = P.Graph(g["n_nodes"], tuple(g["edges"]))
    phi = P.single_od_connectivity(graph, g["source"], g["target"])
    model = P.SystemModel(graph.n_edges, 2, 2, phi)
    rng = np.random.default_rng(0)
    x = torch.as_tensor((rng.random((4096, graph.n_edges)) < 0.9).astype(np.uint8)).cuda()
    vals = torch.empty(4096, dtype=torch.uint8, device="cuda")
    ms = timed(lambda: phi.eval_into(x, None, 4096, 2, vals))
    out["phi_eval (s-t, 119 nodes / 295 edges)"] = {"ms_per_4096": ms,
                                                      "phi_per_s": 4096 / (ms * 1e-3)}
    x0 = x[:64].contiguous()
    ms = timed(lambda: P.boundary_search_batch(model, x0, 0), reps=5)
    out["boundary_search (64 s-t searches, 119 / 295)"] = {"ms": ms,
                                                             "searches_per_s": 64 / (ms * 1e-3)}
    return out


def ncu_traffic(kernel: str, config: str, k: int, variant: str = ""):
    """DRAM bytes per launch of `kernel` on this workload from the committed ncu
    --set full capture (profiles/ncu_traffic.json: {kernel: {"cfg4_k500000": B, ...}}),
    if present."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            entry = json.load(f).get(kernel)
    except Exception:
        return None
    if isinstance(entry, dict):
        return entry.get(f"{config}_k{k}{variant}")
    return entry if config == "cfg2" else None


# --------------------------------------------------------------- reference arm

def run_reference(args):
    """The reference's own CPU classification of the same workload on all host
    cores (rank 0 only; other ranks exit without work)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    p1, lower, upper, S, desc = workload(args.config, args.k, args.samples)
    cpu = CpuClassify(p1, lower, upper)
    # each step one bounded slice; the whole --steps/--warmup run within a few minutes
    per_step = cpu_slice_seconds(args, min(6.0, max(1.0, 150.0 / (args.steps + args.warmup))))
    rows = cpu.calibrate(per_step)
    for w in range(args.warmup):
        cpu.run(rows, start=(1 << 41) + w * rows)
    times, counts = [], [0, 0, 0]
    for k in range(args.steps):
        _, dt, c = cpu.run(rows, start=k * rows)  # consecutive slices of the same stream
        times.append(dt)
        counts = [a + b for a, b in zip(counts, c)]
    value = rows * cpu.K * args.steps / sum(times)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8 (packed bits, int32 popcount sums)",
            "data": "synthetic",
            "config": {"workload": desc, "samples_per_step": rows, "ref_states": cpu.K,
                       "n_components": N_COMP,
                       "labels_over_steps": {"lower": counts[0], "upper": counts[1],
                                             "unclassified": counts[2]}},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu.cores, "kind": cpu.kind,
                             "sample": cpu.describe(rows, desc)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if cpu.kind == "reference" and cpu.K <= 100_000:
        line["public_api"] = cpu.public_api(rows)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- ours

def measure_classify(comm, config, k, samples, method, steps, warmup, *, weak=False,
                     ref_shards=1, e2e=False, encoded_e2e=False):
    """Time `steps` classification steps of one workload on every rank; returns the
    whole-job figures (rank 0 meaningful) plus the objects the e2e legs reuse."""
    import torch
    import torch.distributed as tdist

    import paper_2604_17066_b200 as P
    from paper_2604_17066_b200 import _abi
    from paper_2604_17066_b200.dist import shard_range

    rank, world = comm.rank, comm.world
    dev = torch.device("cuda", torch.cuda.current_device())
    p1, lower_rows, upper_rows, S_total, desc = workload(config, k, samples)
    K_job = len(lower_rows) + len(upper_rows)
    gk = ref_shards if world > 1 else 1
    shard_refs = gk > 1
    ref_comm, samp_comm = comm, comm
    n_sample_shards, sample_shard = world, rank
    if shard_refs:
        # process grid G = G_s x G_k: every rank of a reference group
        # classifies the same samples against its 1/G_k slice of each side; hit flags
        # are OR-reduced over the group (NCCL MAX on 0/1 planes), counts summed over
        # the sample groups
        ref_comm, samp_comm, sample_shard, ref_shard = comm.grid(gk)
        n_sample_shards = world // gk
        l0, lc = shard_range(len(lower_rows), gk, ref_shard)
        u0, uc = shard_range(len(upper_rows), gk, ref_shard)
        lower_rows, upper_rows = lower_rows[l0:l0 + lc], upper_rows[u0:u0 + uc]
    if weak:
        start, S = sample_shard * S_total, S_total
        S_job = n_sample_shards * S_total
    else:
        start, S = shard_range(S_total, n_sample_shards, sample_shard)
        S_job = S_total
    lower = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower_rows, trusted=True)
    upper = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper_rows, trusted=True)
    K = len(lower) + len(upper)
    dist = P.ComponentDistribution.iid(N_COMP, [1 - p1, p1])
    batch = P.sample_batch(dist, S, seed=0, generation_index=0, start=start)
    if method == "tc":
        A = batch.fp4(2)  # planar A_up / A_lo planes (sample_batch's default layout)
        plane = batch.fp4_plane_stride(2)
        bl, nl, al = lower.device_fp4_rows(2)
        bu, nu, au = upper.device_fp4_rows(2)
        width = _abi.fp4_row_bytes(N_COMP, 2)  # bytes per operand row
    else:
        A = batch.thermo(2)
        bl, nl = lower.device_thermo(2)
        bu, nu = upper.device_thermo(2)
        width = A.shape[1]
    sb = batch.thermo_bits(2) if method == "bits" else None
    lb, _ = lower.device_bits(2) if method == "bits" else (None, 0)
    ub, _ = upper.device_bits(2) if method == "bits" else (None, 0)
    a_bytes = A.numel()
    flags = torch.empty(S, dtype=torch.uint8, device=dev)
    labels = torch.empty(S, dtype=torch.uint8, device=dev)
    counts = torch.empty(4, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = _abi.stream_ptr()
    launches = 0
    # reference-chunked launches of the classifier (L2-resident B slices)
    if method == "tc":  # the library's own launch plan (tile width, chunked launches)
        classify_launches = max(1, _abi.fp4_plan(S, nl, nu, width)[1])
    else:
        tiles = {"tc8": lambda n: -(-n // 256), "bits": lambda n: 0}[method]
        per_launch = {"tc8": 256, "bits": 1}[method]
        classify_launches = max(1, -(-(tiles(nl) + tiles(nu)) // per_launch))

    # support compaction (classify.fp4_compaction): the library's cost model decides; when
    # it applies, every step re-packs the resident sample planes over the references'
    # column support (rsr_fp4_gather_columns, timed inside the step) and the classifier
    # runs on the narrower rows
    import importlib
    C = importlib.import_module("paper_2604_17066_b200.classify")
    cplan = C.fp4_compaction(S, N_COMP, 2, lower, upper) if method == "tc" else None
    cbuf = (torch.empty((2, S, cplan.row_bytes), dtype=torch.uint8, device=dev)
            if cplan is not None else None)
    if cplan is not None:
        classify_launches = max(1, _abi.fp4_plan(
            S, nl, cplan.n_pad if cplan.tail_tn and cplan.tail_ok else nu, cplan.row_bytes)[1])
    gev = []  # (start, end) events around the re-pack of each timed step

    def classify_kernel(kev=None):
        if method == "tc" and cplan is not None:
            evs = None
            if kev:  # re-pack start, classifier start (= re-pack end)
                gev.append((torch.cuda.Event(enable_timing=True), kev[0]))
                evs = gev[-1]
            C.fp4_classify_compacted(cplan, A, plane, S, width, 2, lower, upper, flags,
                                     out=cbuf, events=evs)
        elif method == "tc":
            _abi.call("rsr_classify_fp4_planar", _abi.ptr(A), plane, S, None, _abi.ptr(bl), nl, al,
                      _abi.ptr(bu), nu, au, width, _abi.ptr(flags), None, None, 0, stream)
        elif method == "tc8":
            _abi.call("rsr_classify_tc", _abi.ptr(A), S, _abi.ptr(bl), nl, _abi.ptr(bu), nu, width,
                      _abi.ptr(flags), 0, stream)
        else:
            _abi.call("rsr_classify_bits", _abi.ptr(sb), S, _abi.ptr(lb), nl, _abi.ptr(ub), nu,
                      sb.shape[1], _abi.ptr(flags), None, None, 0, stream)

    def step(kev=None):
        nonlocal launches
        if kev and cplan is None:
            kev[0].record()
        classify_kernel(kev)
        if kev:
            kev[1].record()
        if shard_refs:
            ref_comm.allreduce_or_hits(flags)  # OR of hit bits across the ref shards
        _abi.call("rsr_finalize", _abi.ptr(flags), S, _abi.ptr(labels), _abi.ptr(counts), stream)
        launches += classify_launches + 1 + (len(cplan.cols) if cplan is not None else 0)
        if samp_comm.distributed:
            tdist.all_reduce(counts, group=samp_comm.group)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    comm.barrier()
    launches = 0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    with ClockSampler(torch.cuda.current_device()) as clk:
        for i in range(steps):
            flush.zero_()  # L2 flush between timed steps (outside the step events)
            ev[i][0].record()
            step(kev[i])
            ev[i][1].record()
        torch.cuda.synchronize()
    comm.barrier()
    step_ms = sum(s.elapsed_time(e) for s, e in ev)
    kern_avg = sum(s.elapsed_time(e) for s, e in kev) / steps
    if world > 1:  # job time = slowest rank
        t = torch.tensor([step_ms, kern_avg], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        step_ms, kern_avg = (float(v) for v in t.tolist())
    ms_per_step = step_ms / steps
    value = S_job * K_job / (ms_per_step * 1e-3)
    final_counts = counts.cpu().tolist()
    gather_ms = sum(s.elapsed_time(e) for s, e in gev) / len(gev) if gev else 0.0
    if world > 1 and gev:
        t = torch.tensor([gather_ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        gather_ms = float(t.item())

    # ---- roofline of the dominant kernel (algorithmic ops per rank).  The contraction's
    # algorithmic work per pair is 2 x the thermometer columns it must inspect: all
    # N(M-1) without compaction, the reference side's column support with it (the
    # columns no reference uses cannot add a violation); the MMA issues 2 x 64 ops per
    # 64-column K-step of the padded row
    if cplan is not None:
        k_cols = max(c.size - 1 for c in cplan.cols.values())  # bias column not counted
        # shared tail: 7 of the 8 K-steps of a tile pair are issued
        mma_cols = cplan.row_bytes * 2 * (7 / 8 if cplan.tail_tn and cplan.tail_ok else 1)
    else:
        k_cols = N_COMP * (2 - 1)
        mma_cols = width * 2 if method == "tc" else width
    ops_per_pair = 2 * k_cols
    achieved = S * K * ops_per_pair / (kern_avg * 1e-3) / 1e12
    kname = {"tc": "classify_fp4_pair_kernel", "tc8": "classify_tc_pair_kernel",
             "bits": "classify_bits_kernel"}[method]
    # Denominators: dense tensor peaks of the pipe the kernel runs on -- FP4
    # (kind::mxf4) 9 POPS and int8 4.5 POPS (B200 spec), which our own tcgen05
    # issue-rate microbenchmarks reach on this pool (tools/mxf4_check.cu:
    # 8781-8931 TOPS, tools/mma_rate.cu: 4409-4544 TOPS at 1965 MHz);
    # MEASURED_PEAKS.json has neither figure.
    int8_peak = 4500.0
    peak = 9000.0 if method == "tc" else int8_peak
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS",
                "frac": achieved / peak, "traffic": ncu_traffic(kname, config, K,
                                       "" if cplan is None else f"_rb{cplan.row_bytes}" +
                                       ("_tail" if cplan.tail_tn and cplan.tail_ok else "")), "kernel": kname,
                "kernel_ms": kern_avg, "kernel_launches_per_step": classify_launches,
                "ops_per_pair": ops_per_pair, "pairs_per_rank_step": S * K,
                "peak_source": ("B200 dense FP4 spec = measured tcgen05 kind::mxf4 rate "
                                "(tools/mxf4_check.cu: 8781-8931 TOPS)" if method == "tc" else
                                "B200 dense int8 spec = measured tcgen05 kind::i8 rate "
                                "(tools/mma_rate.cu: 4409-4544 TOPS)") +
                               "; MEASURED_PEAKS.json has no int8/fp4 figure",
                "frac_of_int8_peak": achieved / int8_peak,
                "mma_ops_per_pair": 2 * mma_cols,
                "frac_mma_issued": S * K * 2 * mma_cols / (kern_avg * 1e-3) / 1e12 / peak,
                "support_compaction": (None if cplan is None else {
                    "columns": k_cols, "of": N_COMP * (2 - 1),
                    "row_bytes": [width, cplan.row_bytes],
                    "shared_tail_tile_n": cplan.tail_tn or None,
                    "repack_ms": gather_ms,
                    "kernel": "gather_columns_kernel (rsr_fp4_gather_columns)",
                    "repack_gbs": (S * len(cplan.cols) * (width + cplan.row_bytes) /
                                   (gather_ms * 1e-3) / 1e9) if gather_ms else None})}
    if method == "bits":
        # the CUDA-core variant is bound by the integer ALU pipe: one LOP3
        # (acc |= x & r) per 32-bit thermometer word and pair
        words = -(-N_COMP * (2 - 1) // 32)
        sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
        alu_peak = sm_count * 64 * 1.965e9 / 1e12  # 64 LOP3 lanes/clk/SM at 1965 MHz
        ach = S * K * words / (kern_avg * 1e-3) / 1e12
        roofline.update({"bound": "alu", "achieved": ach, "peak": alu_peak,
                         "unit": "T word-ops/s", "frac": ach / alu_peak, "ops_per_pair": words,
                         "peak_source": (f"ALU pipe: {sm_count} SMs x 64 LOP3/clk x 1965 MHz "
                                         "(B300_MICROARCH: alu rt_SMSP = 2)"),
                         "tensor_equivalent_tops": achieved})
    out = {"value": value, "ms_per_step": ms_per_step, "desc": desc, "S": S, "S_job": S_job,
           "K": K, "K_job": K_job, "launches": launches, "roofline": roofline,
           "clocks": clk.summary(), "counts": final_counts, "a_bytes": a_bytes,
           "shard_refs": shard_refs, "gk": gk, "p1": p1, "lower_rows": lower_rows,
           "upper_rows": upper_rows, "weak": weak}
    del flush
    if e2e:
        out["e2e"] = e2e_host(comm, batch, lower, upper, S, S_job, K_job, steps, method,
                              final_counts, shard_refs)
        if encoded_e2e and method == "tc" and not shard_refs:
            out["e2e"]["encoded_input"] = e2e_encoded_input(comm, batch, lower, upper, S, S_job,
                                                            K_job, steps)
    return out


def e2e_host(comm, batch, lower, upper, S, S_job, K_job, steps, method, final_counts, shard_refs):
    """The same metric end to end through the public API with host buffers:
    pinned host uint8 states of this rank's shard -> classify.classify_host (chunked
    H2D on a side stream overlapped with rsr_encode_samples_fp4 + rsr_classify_fp4,
    rsr_finalize) -> labels D2H, every step; max over ranks."""
    import torch
    from paper_2604_17066_b200.classify import classify_host
    if shard_refs:
        return None
    e2e_method = "tc8" if method == "tc8" else "tc"
    host = torch.empty((S, N_COMP), dtype=torch.uint8, pin_memory=True)
    host.copy_(batch.device_states())
    out = torch.empty(S, dtype=torch.uint8, pin_memory=True)
    for _ in range(2):
        classify_host(host, lower, upper, 2, labels_out=out, method=e2e_method)
    torch.cuda.synchronize()
    comm.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        _, c = classify_host(host, lower, upper, 2, labels_out=out, method=e2e_method)
    torch.cuda.synchronize()
    dt = _max_over_ranks(comm, time.perf_counter() - t0)
    assert list(c) == final_counts[:3] or comm.world > 1
    del host
    return {"value": S_job * K_job * steps / dt, "unit": UNIT, "h2d_bytes_per_step": S * N_COMP,
            "d2h_bytes_per_step": S + 32, "ms_per_step": 1e3 * dt / steps,
            "api": "paper_2604_17066_b200.classify.classify_host (pinned host uint8 states -> "
                   "labels), chunked H2D overlapped with " +
                   ("rsr_encode_samples + rsr_classify_tc" if e2e_method == "tc8" else
                    "rsr_encode_samples_fp4 + rsr_classify_fp4")}


def _max_over_ranks(comm, seconds):
    if comm.world == 1:
        return seconds
    import torch
    import torch.distributed as tdist
    t = torch.tensor([seconds], dtype=torch.float64, device=comm.device)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def e2e_encoded_input(comm, batch, lower, upper, S, S_job, K_job, steps):
    """Same metric end to end when the host holds the samples in the reference's
    own classification input format, EncodedBatch(kind="sample").packed
    (encoding.py:82-98: packed one-hot rows, 74 B/row at N=295, M=2):
    pinned host rows -> chunked H2D -> rsr_unpack_onehot_fp4 + rsr_classify_fp4
    -> labels D2H (classify.classify_host_encoded)."""
    import torch
    from paper_2604_17066_b200 import _abi
    from paper_2604_17066_b200.classify import classify_host_encoded
    m = 2
    dev = batch.device_states().device
    rows = torch.empty((S, N_COMP * m), dtype=torch.uint8, device=dev)
    _abi.call("rsr_encode_rows", _abi.ptr(batch.device_states()), S, N_COMP, m, 0, _abi.ptr(rows),
              _abi.stream_ptr())
    nb = (N_COMP * m + 7) // 8
    pk = torch.empty((S, nb), dtype=torch.uint8, device=dev)
    _abi.call("rsr_packbits_rows", _abi.ptr(rows), S, N_COMP * m, 0, _abi.ptr(pk), _abi.stream_ptr())
    del rows
    host = torch.empty((S, nb), dtype=torch.uint8, pin_memory=True)
    host.copy_(pk)
    del pk
    out = torch.empty(S, dtype=torch.uint8, pin_memory=True)
    for _ in range(2):
        classify_host_encoded(host, N_COMP, lower, upper, m, labels_out=out)
    torch.cuda.synchronize()
    comm.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        classify_host_encoded(host, N_COMP, lower, upper, m, labels_out=out)
    torch.cuda.synchronize()
    dt = _max_over_ranks(comm, time.perf_counter() - t0)
    return {"value": S_job * K_job * steps / dt, "unit": UNIT, "h2d_bytes_per_step": S * nb,
            "d2h_bytes_per_step": S + 32, "ms_per_step": 1e3 * dt / steps,
            "api": "paper_2604_17066_b200.classify.classify_host_encoded (pinned host rows of "
                   "EncodedBatch(kind='sample').packed, the reference's classification input "
                   "(encoding.py:82-98, classify.py:42-44) -> labels)"}


def _brief(r):
    """Secondary-workload summary of a measure_classify result."""
    rf = r["roofline"]
    return {"workload": r["desc"], "value": r["value"], "unit": UNIT, "ms_per_step": r["ms_per_step"],
            "kernel_ms": rf["kernel_ms"], "frac": rf["frac"], "achieved_tops": rf["achieved"],
            "peak_tops": rf["peak"], "kernel_launches_per_step": rf["kernel_launches_per_step"],
            "labels": r["counts"][:3]}


def run_ours(args):
    import torch

    from paper_2604_17066_b200.dist import Comm

    # RSR_DIST_BACKEND=gloo: functional check of the multi-rank path on one GPU
    comm = Comm.from_env(os.environ.get("RSR_DIST_BACKEND", "nccl"))
    rank, world = comm.rank, comm.world
    if world == 1:
        torch.cuda.set_device(0)
    gk = world if args.shard_refs else args.ref_shards
    steps, warmup = args.steps, args.warmup
    main = measure_classify(comm, args.config, args.k, args.samples, args.method, steps, warmup,
                            weak=args.weak, ref_shards=gk, e2e=not args.no_e2e,
                            encoded_e2e=True)
    default_run = args.config == "cfg4" and args.k is None and not args.no_secondary

    # reference-count sweep of config 4 (BASELINE configs[3]) on the same ranks
    sweep = None
    if default_run:
        sweep = []
        for kk in (1_000, 10_000, 100_000):
            r = measure_classify(comm, "cfg4", kk, args.samples, args.method, max(5, steps // 2), 3,
                                 weak=args.weak, ref_shards=gk)
            sweep.append({"k": kk, **_brief(r)})
        sweep.append({"k": main["K_job"], **_brief(main)})
    cfg2 = None
    if default_run and world == 1:
        cfg2 = _brief(measure_classify(comm, "cfg2", None, None, args.method, steps, warmup))

    kernels2 = secondary_kernels() if rank == 0 and world == 1 and default_run else None
    cov_loop = None
    if rank == 0 and world == 1 and default_run and not args.no_loop:
        cov_loop = {}
        for rng in ("shared", "device"):
            r = measure_loop("cfg3", args.parallel_searches, rng=rng)
            cov_loop[rng] = {"value": r["value"], "unit": "s", "workload": r["config"]["workload"],
                             "stages": r["stages"], "phi_evaluations": r["phi_evaluations"],
                             "clocks": r.get("clocks"), "trace": r.get("trace_s1")}
        cov_loop = {"metric": "wall-time to c.o.v.=0.05", "unit": "s", "higher_is_better": False,
                    "value": cov_loop["shared"]["value"], **cov_loop}

    # CPU baselines on rank 0 at N = 1 (measured after the GPU legs so the host
    # cores are idle for them)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c = CpuClassify(main["p1"], main["lower_rows"], main["upper_rows"])
        rows = c.calibrate(cpu_slice_seconds(args, 6.0))
        rates = [c.run(rows, start=i * rows)[0] for i in range(2)]
        cpu = {"value": float(np.mean(rates)), "unit": UNIT, "cores": c.cores, "kind": c.kind,
               "sample": c.describe(rows, main["desc"]) + "; mean of 2 slices"}
        if cov_loop is not None:
            cov_loop["cpu_baseline"] = loop_cpu_baseline(
                "cfg3", args.parallel_searches, cpu_slice_seconds(args, 15.0),
                cov_loop["shared"].pop("trace", None), reference=args.loop_cpu_reference)
    if cov_loop is not None:
        for rng in ("shared", "device"):
            cov_loop[rng].pop("trace", None)

    if rank == 0:
        rf = main["roofline"]
        S, K, counts = main["S"], main["K"], main["counts"]
        strong = not main["weak"]
        line = {"metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world,
                "steps": steps, "warmup": warmup, "ms_per_step": main["ms_per_step"],
                "higher_is_better": True, "scaling": "strong" if strong else "weak",
                "vs_baseline": None,
                "dtype": {"tc": "e2m1 (0/1, exact fp32 accumulate)", "tc8": "int8",
                          "bits": "u32 bitwise"}[args.method],
                "data": "synthetic",
                "config": {"workload": main["desc"], "samples_total": main["S_job"],
                           "samples_per_gpu": S, "ref_states": main["K_job"],
                           "ref_states_per_gpu": K, "n_components": N_COMP,
                           "method": args.method,
                           "parallelism": (f"samples x{world // main['gk']} by refs x{main['gk']} "
                                           f"(a reference group shares its samples; hit flags "
                                           f"OR-reduced with NCCL MAX on 0/1 planes)"
                                           if main["shard_refs"] else
                                           f"dp{world} (samples sharded by stream offset, refs "
                                           f"replicated, counts all-reduced)"),
                           "ranks": world,
                           "backend": (os.environ.get("RSR_DIST_BACKEND", "nccl")
                                       if world > 1 else None),
                           "l2": f"A operand {main['a_bytes'] / 1e6:.0f} MB per GPU > L2 and a "
                                 f"256 MB L2 flush between steps (outside the step events)",
                           "labels": {"lower": counts[0], "upper": counts[1],
                                      "unclassified": counts[2]}},
                "roofline": rf, "cpu_baseline": cpu, "e2e": main.get("e2e"),
                "gpu_launches": main["launches"], "clocks": main["clocks"]}
        if sweep is not None:
            line["cfg4_sweep"] = sweep
        if cfg2 is not None:
            line["cfg2"] = cfg2
        if cov_loop is not None:
            line["wall_time_to_cov"] = cov_loop
        if kernels2 is not None:
            line["secondary_kernels"] = kernels2
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as tdist
        tdist.destroy_process_group()


# --------------------------------------------------------------- full loops

def loop_problem(cfg: str, parallel_searches: int):
    """(model_spec, probs, RunConfig kwargs, thresholds, target) of cfg1/cfg3/cfg5."""
    from paper_2604_17066_b200 import workloads as W
    if cfg == "cfg1":
        g = W.cfg1(0)
        spec = {"kind": "st", "n_nodes": g["n_nodes"], "edges": g["edges"], "s": 0, "t": 24,
                "m": 2, "ms": 2}
        return spec, g["probs"], dict(n_samples=100_000, seed=0), [0], \
            "cfg1: 5x5 grid s-t, 10^5 samples, reference defaults (eps_u 1e-5, r_max 1e4, 1 search/it)"
    g = W.cfg3(0) if cfg == "cfg3" else W.cfg5(0)
    m = 2 if cfg == "cfg3" else 3
    spec = {"kind": "st" if cfg == "cfg3" else "widest", "n_nodes": g["n_nodes"],
            "edges": g["edges"], "s": g["source"], "t": g["target"], "m": m, "ms": m}
    kw = dict(n_samples=1 << 20, seed=0, eps_u=1e-5, r_max=10_000,
              parallel_searches=parallel_searches)
    thr = [0] if cfg == "cfg3" else [0, 1]
    desc = (f"{cfg}: 119-node/295-edge shortest-pairs graph, {'binary s-t' if m == 2 else 'M=3 widest path'}, "
            f"batches 2^20, eps_u 1e-5, r_max 1e4, {parallel_searches} searches/it, "
            f"Stage 2 to c.o.v. 0.05 on P(S<=m')")
    return spec, g["probs"], kw, thr, desc


def run_loop(args):
    """Wall time of the full RSR loop (Stage 1 + Stage 2 to c.o.v. 0.05).  Under torchrun
    the batch's samples shard across the ranks (same stream, start offsets; identical
    results to one GPU) and the per-iteration counts / picked rows are exchanged."""
    from paper_2604_17066_b200.dist import Comm
    comm = Comm.from_env(os.environ.get("RSR_DIST_BACKEND", "nccl"))
    out = measure_loop(args.config, args.parallel_searches, comm=comm, rng=args.rng)
    trace = out.pop("trace_s1", None)
    if comm.rank == 0 and comm.world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = loop_cpu_baseline(args.config, args.parallel_searches,
                                                cpu_slice_seconds(args, 15.0), trace,
                                                reference=args.loop_cpu_reference)
    if comm.rank == 0:
        print(json.dumps(out), flush=True)
    if comm.distributed:
        import torch.distributed as tdist
        tdist.destroy_process_group()


def measure_loop(config, parallel_searches, comm=None, rng="shared"):
    import torch

    import paper_2604_17066_b200 as P
    from paper_2604_17066_b200 import _abi
    from paper_2604_17066_b200.dist import shard_range
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _specs import device_model
    spec, probs, kw, thresholds, desc = loop_problem(config, parallel_searches)
    if rng != "shared":
        kw = {**kw, "rng": rng}
        desc += f", rng={rng}"
    dist = P.ComponentDistribution(probs)
    world = comm.world if comm is not None else 1
    if world == 1:
        torch.cuda.set_device(0)
    out = {"metric": "wall-time to c.o.v.=0.05", "unit": "s", "higher_is_better": False,
           "n_gpus": world, "dtype": "e2m1 classifier, u8 states", "data": "synthetic",
           "scaling": "strong",
           "config": {"workload": desc,
                      "parallelism": (f"dp{world}: each batch's samples sharded by stream offset, "
                                      "counts all-reduced, picked rows all-gathered, reference "
                                      "sets identical on every rank" if world > 1 else "dp1")}}
    from paper_2604_17066_b200.workflow import _BatchCache

    def run_all(model, cfg, stages):
        # thresholds share the sample stream: the drawn batches stay in HBM between
        # them, as in multistate_pmf (workflow._BatchCache)
        shard = shard_range(cfg.n_samples, world, comm.rank if comm is not None else 0)[1]
        cache = (_BatchCache(shard, _abi.fp4_row_bytes(dist.n_components, dist.n_states))
                 if len(thresholds) > 1 and os.environ.get("RSR_BATCH_CACHE", "1") != "0" else None)
        first = None
        for thr in thresholds:
            ts = time.perf_counter()
            s1 = P.stage1_find_references(model, dist, cfg, thr, comm, _batch_cache=cache)
            t1 = time.perf_counter()
            first = first or s1
            if config == "cfg1":
                rep = P.stage2_evaluate(model, dist, s1.lower, s1.upper, cfg, thr, comm)
            else:
                rep = P.stage2_until_cov(model, dist, s1.lower, s1.upper, cfg, thr, 0.05,
                                         side="lower", comm=comm)
            t2 = time.perf_counter()
            stages.append({"threshold": thr, "stage1_s": t1 - ts, "stage2_s": t2 - t1,
                           "refs": [len(s1.lower), len(s1.upper)], "iterations": s1.iterations,
                           "terminated_by": s1.terminated_by,
                           "p_unclassified_last": s1.trace[-1].p_unclassified,
                           "p_lower": rep.p_lower, "cov_lower": rep.cov_lower,
                           "stage2_samples": rep.n_samples})
        del cache
        return first

    # warm-up: the whole procedure once on another seed, so the timed run finds the CUDA
    # context, library state and the caching allocator's device buffers at full size
    # (reference sets grown to r_max, the multi-threshold batch cache filled); a short
    # warm-up left those first allocations inside the timed run (cfg3 device stream
    # 0.28 s vs 0.12 s, cfg5 0.54 s vs 0.25 s)
    run_all(device_model(spec), P.RunConfig(**{**kw, "seed": kw.get("seed", 0) + 1}), [])
    torch.cuda.synchronize()
    if comm is not None:
        comm.barrier()
    model = device_model(spec)
    cfg = P.RunConfig(**kw)
    stages = []
    clk = ClockSampler(torch.cuda.current_device())  # NVML init outside the timed region
    with clk:
        t0 = time.perf_counter()
        s1_first = run_all(model, cfg, stages)
        torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if comm is not None and comm.distributed:  # job wall time = slowest rank
        import torch.distributed as tdist
        t = torch.tensor([wall], dtype=torch.float64, device=comm.device)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        wall = float(t.item())
    out.update({"value": wall, "stages": stages, "phi_evaluations": model.evaluation_count,
                "clocks": clk.summary(), "rng": rng,
                "trace_s1": s1_first.trace if s1_first else None})
    return out


def loop_cpu_baseline(config, parallel_searches, budget, gpu_trace, reference=False):
    """Same-run CPU slice of the Stage-1 loop (workflow.py:122-195) on the host cores,
    compared with the GPU run's cumulative Stage-1 time at the same iteration count.

    Default: the oracle port (numpy Philox exactly as sampling.py, thread-pool
    classify over all cores, scalar union-find Phi) under a time budget.
    reference=True: the installed reference's own stage1_find_references
    (baseline/_ref; n_workers = all cores) stopped by r_max after its second
    iteration -- about a minute of host time at H = 2^20."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _specs import oracle_phi
    spec, probs, kw, thresholds, desc = loop_problem(config, parallel_searches)
    threshold = thresholds[0]
    cores = len(os.sched_getaffinity(0))
    kw2 = dict(kw)
    H = kw2.pop("n_samples")
    chunk = max(256, H // (4 * cores))
    rsr = reference_pkg() if reference else None
    if rsr is not None and spec["kind"] == "st":
        graph = rsr.Graph(spec["n_nodes"], tuple(tuple(e) for e in spec["edges"]))
        model = rsr.SystemModel(len(spec["edges"]), spec["m"], spec["ms"],
                                rsr.single_od_connectivity(graph, spec["s"], spec["t"]))
        cfg = rsr.RunConfig(n_samples=H, eps_u=kw2["eps_u"], r_max=1, seed=kw2["seed"],
                            parallel_searches=kw2["parallel_searches"], n_workers=cores,
                            chunk_size=chunk)
        res = rsr.stage1_find_references(model, rsr.ComponentDistribution(probs), cfg, threshold)
        times = [t.elapsed_seconds for t in res.trace]
        kind, what = "reference", "installed reference stage1_find_references (r_max=1: two iterations)"
    else:
        import oracle
        phi, n = oracle_phi(spec)
        ev = oracle.CountingPhi(phi, n, spec["m"], spec["ms"])
        res = oracle.stage1(ev, probs, threshold, H, n_workers=cores, chunk_size=chunk,
                            time_budget=budget, fast=True, **kw2)
        times = [t["elapsed"] for t in res["trace"] if "elapsed" in t]
        kind, what = "port", ("oracle port of workflow.py:122-195 with numpy Philox, ThreadPool "
                              "classify, scalar union-find Phi, time budget "
                              f"{budget:.0f} s")
    if not times:
        return None
    k = len(times) - 1 if kind == "reference" else len(times)
    cpu_s = times[-1]
    # GPU trace record k is taken at iteration k's classification, i.e. after k
    # complete iterations (sample, classify, searches, inserts) plus one sample+classify
    gpu_s = gpu_trace[k].elapsed_seconds if gpu_trace is not None and len(gpu_trace) > k else None
    return {"value": cpu_s, "unit": "s", "cores": cores, "kind": kind,
            "sample": f"first {k} Stage-1 iterations (threshold {threshold}) of the same run: "
                      f"{what} (n_workers={cores}, chunk={chunk})",
            "iterations": k, "gpu_seconds_same_iterations": gpu_s,
            "speedup_same_iterations": (cpu_s / gpu_s) if gpu_s else None}


def relaunch_under_torchrun(args) -> int | None:
    """`--gpus N` (N > 1) from a plain `python bench.py`: run N ranks under
    torch.distributed.run on 127.0.0.1 and return its exit code.  Under torchrun
    (WORLD_SIZE set) the world size must equal --gpus."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if args.gpus <= 1:
            return None
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        print(f"[bench] --gpus {args.gpus}: launching {args.gpus} ranks: {' '.join(cmd)}",
              file=sys.stderr, flush=True)
        return subprocess.call(cmd)
    if int(world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    return None


def main():
    args = parse()
    rc = relaunch_under_torchrun(args)
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference":
        run_reference(args)
    elif args.config in ("cfg1", "cfg3", "cfg5"):
        run_loop(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
