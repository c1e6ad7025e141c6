#!/usr/bin/env python
"""Benchmark of the RSR dominance-classification hot path on B200.

Default workload (BASELINE.json configs[1], "cfg2"): S = 2^20 samples x
N = 295 binary components (Bernoulli(0.9) via the device Philox sampler),
K = 10^4 upper refs (15 ones) + 10^4 lower refs (10 zeros).  A step is one
classification of the resident batch against all K refs: rsr_classify_tc
(tcgen05 int8 thermometer contraction with fused any-zero epilogue) +
rsr_finalize (labels + counts), plus an NCCL all-reduce of the counts when
N > 1.  Metric: classified samples x reference states per second (pairs/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        bench.py --gpus N ...

Other workloads for the profiles/ notes: --config cfg4 --k 500000 (path refs
sweep), --config cfg1 / cfg3 (full RSR loop wall time).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "classified samples·ref-states/sec"
UNIT = "pairs/s"
N_COMP = 295


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="cfg2",
                   choices=["cfg2", "cfg2_mixed", "cfg4", "cfg1", "cfg3", "cfg5"])
    p.add_argument("--parallel-searches", type=int, default=64)
    p.add_argument("--shard-refs", action="store_true",
                   help="N>1: shard reference states across all ranks, OR-reduce hit flags")
    p.add_argument("--ref-shards", type=int, default=1,
                   help="N>1: G_k reference shards per sample shard (G_k divides N)")
    p.add_argument("--k", type=int, default=10_000, help="refs per side (cfg2) / path refs (cfg4)")
    p.add_argument("--samples", type=int, default=None, help="samples per GPU")
    p.add_argument("--method", choices=["tc", "tc8", "bits"], default="tc",
                   help="tc: FP4 (kind::mxf4) tensor cores; tc8: int8 tensor cores; bits: CUDA cores")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-loop", action="store_true",
                   help="skip the cfg3 wall-time-to-c.o.v. loop attached to the default run")
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    return p.parse_args()


# ----------------------------------------------------------------- workloads

def workload(args):
    """(p_survive, lower rows, upper rows, S, description) -- numpy only."""
    from paper_2604_17066_b200 import workloads as W
    if args.config == "cfg2":
        lower, upper = W.cfg2_refs(0, N_COMP, args.k, args.k)
        S = args.samples or (1 << 20)
        desc = (f"cfg2: S=2^{int(np.log2(S))} x N=295 Bernoulli(0.9), K={len(upper)} upper "
                f"(15 ones) + {len(lower)} lower (10 zeros)")
        return 0.9, lower, upper, S, desc
    if args.config == "cfg2_mixed":
        lower, upper = W.cfg2_mixed_refs(0, N_COMP, args.k, args.k)
        S = args.samples or (1 << 20)
        return 0.5, lower, upper, S, f"cfg2-mixed: S={S}, p=0.5, 15-one upper / 14-zero lower"
    g = W.cfg3(0)
    upper = W.random_st_paths(g, args.k, seed=0)
    lower = np.zeros((0, N_COMP), dtype=np.uint8)
    S = args.samples or (1 << 22)
    return 0.9, lower, upper, S, (f"cfg4: S={S} Bernoulli(0.9), K={len(upper)} s-t path refs "
                                  f"(mean {upper.sum(1).mean():.1f} edges)")


def cpu_classify_rate(p1, lower, upper, rows, seed=0):
    """Reference algorithm (oracle port of classify.py:99-148) on host cores."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    probs = np.tile([1 - p1, p1], (N_COMP, 1))
    xs = oracle.sample_states(probs, rows, seed, 0, 0)
    chunk = max(256, rows // (4 * cores)) if cores > 1 else 65536
    t0 = time.perf_counter()
    oracle.classify_labels(xs, lower, upper, 2, chunk_size=chunk, n_workers=cores)
    dt = time.perf_counter() - t0
    return rows * (len(lower) + len(upper)) / dt, dt, cores, chunk


def calibrated_cpu_rows(p1, lower, upper, target_s):
    rate, _, _, _ = cpu_classify_rate(p1, lower, upper, 512)
    pairs = rate * target_s
    return int(max(512, min(1 << 18, pairs / max(1, len(lower) + len(upper)))))


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
        pr = _abi.ptr(d.device_probs())
        ms = timed(lambda: _abi.call("rsr_sample_fp4", pr, N_COMP, m, 0, 1, 0, S, _abi.ptr(st),
                                     _abi.ptr(a4), rb, _abi.stream_ptr()))
        wbytes = S * (N_COMP + 2 * rb)
        out[f"sample_rows_kernel_M{m}"] = {
            "shape": f"2^20 x {N_COMP} draws", "ms": ms, "draws_per_s": S * N_COMP / (ms * 1e-3),
            "hbm_write_gbs": wbytes / (ms * 1e-3) / 1e9, "hbm_peak_gbs": hbm,
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


def int8_peak_tops():
    """Measured dense int8 GEMM throughput (cuBLASLt via torch._int_mm), best of 10.

    MEASURED_PEAKS.json carries only the bf16 cuBLAS peak; this is the int8
    counterpart measured the same way on the same box.  Falls back to
    2 x bf16_tflops (int8 dense rate = 2 x bf16 on B200) if _int_mm fails.
    """
    import torch
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    try:
        n = 8192
        a = torch.randint(-8, 8, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-8, 8, (n, n), dtype=torch.int8, device="cuda").t()
        for _ in range(3):
            torch._int_mm(a, b)
        best = 0.0
        for _ in range(10):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch._int_mm(a, b)
            e.record()
            e.synchronize()
            best = max(best, 2 * n ** 3 / (s.elapsed_time(e) * 1e-3) / 1e12)
        del a, b
        return best, "measured: cuBLASLt int8 GEMM 8192^3 via torch._int_mm, best of 10 (burst)"
    except Exception as exc:  # pragma: no cover
        bf16 = peaks.get("bf16_tflops", 1590.0)
        return 2 * bf16, f"2 x bf16_tflops of MEASURED_PEAKS.json ({exc.__class__.__name__})"


def ncu_traffic(kernel: str):
    """dram bytes per launch from the committed ncu capture, if present."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


# --------------------------------------------------------------- reference arm

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    p1, lower, upper, S, desc = workload(args)
    rows = calibrated_cpu_rows(p1, lower, upper, 4.0)
    for _ in range(args.warmup):
        cpu_classify_rate(p1, lower, upper, rows, seed=1)
    rates, times = [], []
    cores = chunk = None
    for k in range(args.steps):
        r, dt, cores, chunk = cpu_classify_rate(p1, lower, upper, rows, seed=2 + k)
        rates.append(r)
        times.append(dt)
    value = rows * (len(lower) + len(upper)) * args.steps / sum(times)
    sample = (f"{rows} samples/step x {len(lower) + len(upper)} refs of {desc}; reference "
              f"algorithm (oracle/core.py port of classify.py:99-148, packbits + bitwise_count, "
              f"ThreadPool n_workers={cores}, chunk={chunk})")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": desc, "samples_per_step": rows,
                       "ref_states": int(len(lower) + len(upper)), "n_components": N_COMP},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- ours

def run_ours(args):
    import torch

    import paper_2604_17066_b200 as P
    from paper_2604_17066_b200 import _abi
    from paper_2604_17066_b200.dist import Comm

    # RSR_DIST_BACKEND=gloo: functional check of the multi-rank path on one GPU
    comm = Comm.from_env(os.environ.get("RSR_DIST_BACKEND", "nccl"))
    rank, world = comm.rank, comm.world
    if world == 1:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    p1, lower_rows, upper_rows, S, desc = workload(args)
    K_job = len(lower_rows) + len(upper_rows)
    # process grid G = G_s x G_k: G_k reference shards per sample shard
    gk = world if args.shard_refs else args.ref_shards
    shard_refs = gk > 1 and world > 1
    sample_shard, ref_comm, samp_comm = rank, comm, comm
    if shard_refs:
        # every rank of a reference group classifies the same S samples against its
        # 1/G_k slice of each side; hit flags are OR-reduced over the group (NCCL MAX
        # on 0/1 planes), counts summed over the sample groups
        from paper_2604_17066_b200.dist import shard_range
        ref_comm, samp_comm, sample_shard, ref_shard = comm.grid(gk)
        l0, lc = shard_range(len(lower_rows), gk, ref_shard)
        u0, uc = shard_range(len(upper_rows), gk, ref_shard)
        lower_rows, upper_rows = lower_rows[l0:l0 + lc], upper_rows[u0:u0 + uc]
    lower = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower_rows, trusted=True)
    upper = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper_rows, trusted=True)
    K = len(lower) + len(upper)
    dist = P.ComponentDistribution.iid(N_COMP, [1 - p1, p1])
    batch = P.sample_batch(dist, S, seed=0, generation_index=0, start=sample_shard * S)
    if args.method == "tc":
        A = batch.fp4(2)
        bl, nl, al = lower.device_fp4_rows(2)
        bu, nu, au = upper.device_fp4_rows(2)
        width = A.shape[1] // 2  # bytes per operand row
    else:
        A = batch.thermo(2)
        bl, nl = lower.device_thermo(2)
        bu, nu = upper.device_thermo(2)
        width = A.shape[1]
    sb = batch.thermo_bits(2) if args.method == "bits" else None
    lb, _ = lower.device_bits(2) if args.method == "bits" else (None, 0)
    ub, _ = upper.device_bits(2) if args.method == "bits" else (None, 0)
    a_bytes = A.shape[0] * A.shape[1]
    flags = torch.empty(S, dtype=torch.uint8, device=dev)
    labels = torch.empty(S, dtype=torch.uint8, device=dev)
    counts = torch.empty(4, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = _abi.stream_ptr()
    launches = 0
    # reference-chunked launches of the classifier (L2-resident B slices)
    tiles = {"tc": lambda n: -(-n // 240), "tc8": lambda n: -(-n // 256), "bits": lambda n: 0}[args.method]
    per_launch = {"tc": 512, "tc8": 256, "bits": 1}[args.method]
    classify_launches = max(1, -(-(tiles(nl) + tiles(nu)) // per_launch))
    import torch.distributed as tdist

    def classify_kernel():
        if args.method == "tc":
            _abi.call("rsr_classify_fp4_ex", _abi.ptr(A), S, None, _abi.ptr(bl), nl, al, _abi.ptr(bu),
                      nu, au, width, _abi.ptr(flags), None, None, 0, stream)
        elif args.method == "tc8":
            _abi.call("rsr_classify_tc", _abi.ptr(A), S, _abi.ptr(bl), nl, _abi.ptr(bu), nu, width,
                      _abi.ptr(flags), 0, stream)
        else:
            _abi.call("rsr_classify_bits", _abi.ptr(sb), S, _abi.ptr(lb), nl, _abi.ptr(ub), nu,
                      sb.shape[1], _abi.ptr(flags), None, None, 0, stream)

    def step(kev=None):
        nonlocal launches
        if kev:
            kev[0].record()
        classify_kernel()
        if kev:
            kev[1].record()
        if shard_refs:
            ref_comm.allreduce_or_hits(flags)  # OR of hit bits across the ref shards
        _abi.call("rsr_finalize", _abi.ptr(flags), S, _abi.ptr(labels), _abi.ptr(counts), stream)
        launches += classify_launches + 1
        if samp_comm.distributed:
            tdist.all_reduce(counts, group=samp_comm.group)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    comm.barrier()
    launches = 0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(torch.cuda.current_device()) as clk:
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the step events)
            ev[k][0].record()
            step(kev[k])
            ev[k][1].record()
        torch.cuda.synchronize()
    comm.barrier()
    step_ms = sum(s.elapsed_time(e) for s, e in ev)
    kern_ms = [s.elapsed_time(e) for s, e in kev]
    if world > 1:
        t = torch.tensor([step_ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        step_ms = float(t.item())
    ms_per_step = step_ms / args.steps
    # whole-job pairs per step: replicated refs -> world x S x K; G_s x G_k grid -> G_s x S x K_job
    job_pairs = (world // gk) * S * K_job if shard_refs else world * S * K
    value = job_pairs / (ms_per_step * 1e-3)
    final_counts = counts.cpu().tolist()

    # ---- roofline of the dominant kernel (algorithmic ops, unpadded K)
    ops_per_pair = 2 * N_COMP * (2 - 1)
    kern_avg = sum(kern_ms) / len(kern_ms)
    achieved = S * K * ops_per_pair / (kern_avg * 1e-3) / 1e12
    cublas_peak, cublas_src = int8_peak_tops()
    kname = {"tc": "classify_fp4_pair_kernel", "tc8": "classify_tc_pair_kernel",
             "bits": "classify_bits_kernel"}[args.method]
    # Denominators: dense tensor peaks of the pipe the kernel runs on -- FP4
    # (kind::mxf4) 9 POPS and int8 4.5 POPS (B200 spec), which our own tcgen05
    # issue-rate microbenchmarks reach on this pool (tools/mxf4_check.cu:
    # 8781-8931 TOPS, tools/mma_rate.cu: 4409-4544 TOPS at 1965 MHz);
    # MEASURED_PEAKS.json has neither figure.  cuBLASLt int8 (the best library
    # GEMM for this contraction) is reported alongside.
    int8_peak = 4500.0
    peak = 9000.0 if args.method == "tc" else int8_peak
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS",
                "frac": achieved / peak, "traffic": ncu_traffic(kname), "kernel": kname,
                "kernel_ms": kern_avg, "ops_per_pair": ops_per_pair,
                "peak_source": ("B200 dense FP4 spec = measured tcgen05 kind::mxf4 rate "
                                "(tools/mxf4_check.cu: 8781-8931 TOPS)" if args.method == "tc" else
                                "B200 dense int8 spec = measured tcgen05 kind::i8 rate "
                                "(tools/mma_rate.cu: 4409-4544 TOPS)") +
                               "; MEASURED_PEAKS.json has no int8/fp4 figure",
                "frac_of_int8_peak": achieved / int8_peak,
                "cublas_int8_tops": cublas_peak, "cublas_int8_source": cublas_src,
                "frac_of_cublas_int8": achieved / cublas_peak}
    if args.method == "bits":
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

    # ---- end to end through the public API with host buffers
    e2e = None
    e2e_method = "tc8" if args.method == "tc8" else "tc"
    if not args.no_e2e:
        host = torch.empty((S, N_COMP), dtype=torch.uint8, pin_memory=True)
        host.copy_(batch.device_states())
        out = torch.empty(S, dtype=torch.uint8, pin_memory=True)
        for _ in range(2):
            P.classify.__module__  # noqa: B018
            from paper_2604_17066_b200.classify import classify_host
            classify_host(host, lower, upper, 2, labels_out=out, method=e2e_method)
        torch.cuda.synchronize()
        comm.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            _, c = classify_host(host, lower, upper, 2, labels_out=out, method=e2e_method)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            dt = float(t.item())
        assert list(c) == final_counts[:3] or world > 1
        e2e_packed = e2e_encoded_input(args, batch, lower, upper, S, K, world, comm, dev)
        e2e = {"value": world * S * K * args.steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": S * N_COMP, "d2h_bytes_per_step": S + 32,
               "ms_per_step": 1e3 * dt / args.steps,
               "api": "paper_2604_17066_b200.classify.classify_host (pinned host uint8 states -> "
                      "labels), chunked H2D overlapped with " +
                      ("rsr_encode_samples + rsr_classify_tc" if e2e_method == "tc8" else
                       "rsr_encode_samples_fp4 + rsr_classify_fp4"),
               "encoded_input": e2e_packed}

    # second half of BASELINE.json's metric: wall time of the full RSR loop to
    # c.o.v. 0.05 on config 3 (one GPU; the loop has no data-parallel split);
    # measured before the CPU baseline keeps the host cores busy
    kernels2 = secondary_kernels() if rank == 0 and args.config == "cfg2" and not args.no_loop else None
    cov_loop = None
    if rank == 0 and world == 1 and args.config == "cfg2" and not args.no_loop:
        r = measure_loop("cfg3", args.parallel_searches)
        cov_loop = {"metric": "wall-time to c.o.v.=0.05", "value": r["value"], "unit": "s",
                    "higher_is_better": False, "workload": r["config"]["workload"],
                    "stages": r["stages"], "phi_evaluations": r["phi_evaluations"],
                    "cpu_baseline": "profiles/r1_loop_cfg3_fp4.json (oracle port of the reference "
                                    "loop at equal iteration count)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rows = calibrated_cpu_rows(p1, lower_rows, upper_rows, args.cpu_seconds)
        rate, dt, cores, chunk = cpu_classify_rate(p1, lower_rows, upper_rows, rows)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{rows} samples x {K} refs of the same workload ({dt:.1f} s); oracle port "
                         f"of the reference classify (packbits + bitwise_count, ThreadPool "
                         f"n_workers={cores}, chunk={chunk})"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong" if shard_refs else "weak",
                "vs_baseline": None,
                "dtype": {"tc": "e2m1 (0/1, exact fp32 accumulate)", "tc8": "int8",
                          "bits": "u32 bitwise"}[args.method],
                "data": "synthetic",
                "config": {"workload": desc, "samples_per_gpu": S, "ref_states": K_job,
                           "ref_states_per_gpu": K, "n_components": N_COMP, "method": args.method,
                           "parallelism": (f"samples x{world // gk} by refs x{gk} (a reference "
                                           f"group shares its samples; hit flags OR-reduced with "
                                           f"NCCL MAX on 0/1 planes)" if shard_refs else
                                           f"dp{world} (samples sharded by stream offset, refs "
                                           f"replicated, counts all-reduced)"),
                           "l2": f"A operand {a_bytes / 1e6:.0f} MB > L2 and 256 MB "
                                 f"L2 flush between steps (outside the step events)",
                           "labels": {"lower": final_counts[0], "upper": final_counts[1],
                                      "unclassified": final_counts[2]}},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary()}
        if cov_loop is not None:
            line["wall_time_to_cov"] = cov_loop
        if kernels2 is not None:
            line["secondary_kernels"] = kernels2
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()


def e2e_encoded_input(args, batch, lower, upper, S, K, world, comm, dev):
    """Same metric end to end when the host holds the samples in the reference's
    own classification input format, EncodedBatch(kind="sample").packed
    (encoding.py:82-98: packed one-hot rows, 74 B/row at N=295, M=2):
    pinned host rows -> chunked H2D -> rsr_unpack_onehot_fp4 + rsr_classify_fp4
    -> labels D2H (classify.classify_host_encoded)."""
    import torch
    from paper_2604_17066_b200 import _abi
    from paper_2604_17066_b200.classify import classify_host_encoded
    if args.method == "tc8":
        return None
    m = 2
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
    for _ in range(args.steps):
        classify_host_encoded(host, N_COMP, lower, upper, m, labels_out=out)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as tdist
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        dt = float(t.item())
    return {"value": world * S * K * args.steps / dt, "unit": UNIT, "h2d_bytes_per_step": S * nb,
            "d2h_bytes_per_step": S + 32, "ms_per_step": 1e3 * dt / args.steps,
            "api": "paper_2604_17066_b200.classify.classify_host_encoded (pinned host rows of "
                   "EncodedBatch(kind='sample').packed, the reference's classification input "
                   "(encoding.py:82-98, classify.py:42-44) -> labels)"}


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
    out = measure_loop(args.config, args.parallel_searches,
                       None if args.no_cpu_baseline or comm.world > 1 else args.cpu_seconds,
                       comm=comm)
    if comm.rank == 0:
        print(json.dumps(out), flush=True)
    if comm.distributed:
        import torch.distributed as tdist
        tdist.destroy_process_group()


def measure_loop(config, parallel_searches, cpu_seconds=None, comm=None):
    import torch

    import paper_2604_17066_b200 as P
    from paper_2604_17066_b200 import _abi
    from paper_2604_17066_b200.dist import shard_range
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _specs import device_model
    spec, probs, kw, thresholds, desc = loop_problem(config, parallel_searches)
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
    # warm-up on the same batch size (a few iterations + Stage 2), so the timed
    # run finds the CUDA context, library state and cached device buffers ready
    wm = device_model(spec)
    wcfg = P.RunConfig(**{**kw, "r_max": 5, "seed": kw.get("seed", 0) + 1})
    ws1 = P.stage1_find_references(wm, dist, wcfg, thresholds[0], comm)
    P.stage2_evaluate(wm, dist, ws1.lower, ws1.upper, wcfg, thresholds[0], comm)
    torch.cuda.synchronize()
    if comm is not None:
        comm.barrier()
    model = device_model(spec)
    cfg = P.RunConfig(**kw)
    stages = []
    s1_first = None
    clk = ClockSampler(torch.cuda.current_device())  # NVML init outside the timed region
    with clk:
        t0 = time.perf_counter()
        # thresholds share the sample stream: the drawn batches stay in HBM between
        # them, as in multistate_pmf (workflow._BatchCache)
        from paper_2604_17066_b200.workflow import _BatchCache
        shard = shard_range(cfg.n_samples, world, comm.rank if comm is not None else 0)[1]
        cache = (_BatchCache(shard, _abi.fp4_row_bytes(dist.n_components, dist.n_states))
                 if len(thresholds) > 1 and os.environ.get("RSR_BATCH_CACHE", "1") != "0" else None)
        for thr in thresholds:
            ts = time.perf_counter()
            s1 = P.stage1_find_references(model, dist, cfg, thr, comm, _batch_cache=cache)
            t1 = time.perf_counter()
            s1_first = s1_first or s1
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
        torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if comm is not None and comm.distributed:  # job wall time = slowest rank
        import torch.distributed as tdist
        t = torch.tensor([wall], dtype=torch.float64, device=comm.device)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        wall = float(t.item())
    out.update({"value": wall, "stages": stages, "phi_evaluations": model.evaluation_count,
                "clocks": clk.summary()})
    if cpu_seconds is not None:
        out["cpu_baseline"] = loop_cpu_baseline(spec, probs, kw, thresholds[0], cpu_seconds,
                                                gpu_trace=s1_first.trace if s1_first else None)
    return out


def loop_cpu_baseline(spec, probs, kw, threshold, budget, gpu_trace):
    """Reference Stage-1 loop (oracle port, numpy Philox as in sampling.py, thread-pool
    classify over all host cores, scalar union-find Phi) for `budget` seconds; compared
    with the GPU's cumulative Stage-1 time at the same iteration count."""
    import oracle
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _specs import oracle_phi
    phi, n = oracle_phi(spec)
    ev = oracle.CountingPhi(phi, n, spec["m"], spec["ms"])
    cores = len(os.sched_getaffinity(0))
    kw2 = dict(kw)
    H = kw2.pop("n_samples")
    res = oracle.stage1(ev, probs, threshold, H, n_workers=cores,
                        chunk_size=max(256, H // (4 * cores)), time_budget=budget, fast=True,
                        **kw2)
    done = [t for t in res["trace"] if "elapsed" in t]
    if not done:
        return None
    k = len(done)
    cpu_s = done[-1]["elapsed"]
    gpu_s = gpu_trace[k].elapsed_seconds if gpu_trace is not None and len(gpu_trace) > k else None
    return {"value": cpu_s, "unit": "s", "cores": cores, "kind": "port",
            "sample": f"first {k} Stage-1 iterations (threshold {threshold}) of the same run: "
                      f"oracle port of workflow.py:122-195 with numpy Philox, ThreadPool classify "
                      f"(n_workers={cores}), scalar union-find Phi",
            "iterations": k, "gpu_seconds_same_iterations": gpu_s,
            "speedup_same_iterations": (cpu_s / gpu_s) if gpu_s else None}


def main():
    args = parse()
    if args.config in ("cfg1", "cfg3", "cfg5"):
        run_loop(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
