"""CUDA-event timings of the non-classifier kernels on their config shapes."""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import workloads as W  # noqa: E402


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


def main():
    torch.cuda.set_device(0)
    for m, probs in ((2, [0.1, 0.9]), (3, [0.05, 0.15, 0.8])):
        d = P.ComponentDistribution.iid(295, probs)
        S = 1 << 20
        st = torch.empty((S, 295), dtype=torch.uint8, device="cuda")
        th = torch.empty((S, P._abi.thermo_kpad(295, m)), dtype=torch.int8, device="cuda")
        ms = timed(lambda: P.sample_batch(d, S, 0, 1, out_states=st, out_thermo=th))
        print(f"sample_batch+int8 thermo M={m} S=2^20 N=295: {ms:.3f} ms = {S * 295 / ms / 1e6:.1f} G draws/s")
        ms = timed(lambda: P.sample_batch(d, S, 0, 1, out_states=st))
        print(f"sample_batch M={m} S=2^20 N=295: {ms:.3f} ms = {S * 295 / ms / 1e6:.1f} G draws/s")
        rb = P._abi.fp4_row_bytes(295, m)
        a4 = torch.empty((S, 2 * rb), dtype=torch.uint8, device="cuda")
        ms = timed(lambda: P._abi.call("rsr_encode_samples_fp4", P._abi.ptr(st), S, 295, m,
                                       P._abi.ptr(a4), rb, P._abi.stream_ptr()))
        gbs = (S * 295 + S * 2 * rb) / ms / 1e6
        print(f"encode_samples_fp4 M={m} S=2^20: {ms:.3f} ms = {gbs:.0f} GB/s")
    g = W.cfg3(0)
    graph = P.Graph(g["n_nodes"], tuple(g["edges"]))
    for name, phi, m in (("st", P.single_od_connectivity(graph, g["source"], g["target"]), 2),
                         ("widest", P.widest_path_level(graph, g["source"], g["target"]), 3)):
        model = P.SystemModel(graph.n_edges, m, m, phi)
        rng = np.random.default_rng(0)
        x = torch.as_tensor(rng.integers(0, m, size=(4096, graph.n_edges)).astype(np.uint8)).cuda()
        out = torch.empty(4096, dtype=torch.uint8, device="cuda")
        ms = timed(lambda: phi.eval_into(x, None, 4096, m, out))
        print(f"phi {name} 4096 vectors: {ms:.3f} ms = {ms * 1e3 / 4096:.2f} us/vector")
        x0 = x[:64].contiguous()
        ms = timed(lambda: P.boundary_search_batch(model, x0, 0), reps=3)
        print(f"boundary_search {name} 64 searches: {ms:.3f} ms")


if __name__ == "__main__":
    main()


def classify_m3():
    """FP4 classifier at M = 3 (cfg5 shape): 2^20 x 2 x 10^4 refs, ops = 2 N (M-1) per pair."""
    from paper_2604_17066_b200.classify import classify_flags
    torch.cuda.set_device(0)
    n, m, k = 295, 3, 10_000
    rng = np.random.default_rng(5)
    d = P.ComponentDistribution.iid(n, [0.05, 0.15, 0.8])
    batch = P.sample_batch(d, 1 << 20, 0, 0)
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, rng.integers(1, 3, size=(k, n)), trusted=True)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, rng.integers(0, 2, size=(k, n)), trusted=True)
    ms = timed(lambda: classify_flags(batch, lo, up, m))
    tops = (1 << 20) * 2 * k * 2 * n * (m - 1) / ms / 1e9
    print(f"classify fp4 M=3 2^20 x 2x10^4: {ms:.3f} ms = {tops:.0f} TOPS = {tops / 9000:.3f} of FP4 peak")


if __name__ == "__main__" and os.environ.get("CLASSIFY_M3"):
    classify_m3()
