"""Classifier kernel time per state count M at N = 295 (timing experiment, not a test):
S = 2^20 samples x 10^4 lower + 10^4 upper references, FP4 tensor cores ("tc"; rows
past 416 bytes run one-sided launches per side) against the bit-packed CUDA-core kernel.
Algorithmic work 2 N (M-1) ops per (sample, reference) pair, as bench.py's roofline.

    python tools/wide_rows_bench.py [M ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200.classify import classify_flags  # noqa: E402

N, S, K = 295, 1 << 20, 10_000
ms = [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5]
for m in ms:
    rng = np.random.default_rng(m)
    probs = rng.dirichlet([1.0] * (m - 1) + [16.0], size=N)
    batch = P.sample_batch(P.ComponentDistribution(probs), S, seed=0)
    lower = rng.integers(1, m, size=(K, N))       # rarely dominate a sample from above
    upper = rng.integers(0, m - 1, size=(K, N)) * (rng.random((K, N)) < 0.9)
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower, trusted=True)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True)
    out = {}
    for method in ("tc", "bits"):
        for _ in range(2):
            classify_flags(batch, lo, up, m, method)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        s.record()
        for _ in range(reps):
            f, _, _ = classify_flags(batch, lo, up, m, method)
        e.record()
        e.synchronize()
        ms_ = s.elapsed_time(e) / reps
        out[method] = (ms_, f.clone())
    assert torch.equal(out["tc"][1], out["bits"][1]), f"M={m}: tc != bits"
    ops = 2.0 * S * 2 * K * N * (m - 1)
    t = out["tc"][0]
    print(f"M={m}: row bytes {P._abi.fp4_row_bytes(N, m)}, tc {t:.3f} ms = "
          f"{ops / (t * 1e-3) / 1e12:.0f} TOPS = {ops / (t * 1e-3) / 9e15:.3f} of 9 POPS; "
          f"bits {out['bits'][0]:.3f} ms ({out['bits'][0] / t:.1f}x slower); labels equal")
