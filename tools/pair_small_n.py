"""Paired vs unpaired FP4 classifier on rows of 1, 2, 3 and 4 K-steps (N = 40, 120, 180,
250 at M = 2): 2^22 samples x K upper references, kernel ms (CUDA events).
usage: python tools/pair_small_n.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import _abi, _device  # noqa: E402

S = 1 << 22
for n in (40, 120, 180, 250):
    for k in (1000, 20000):
        rng = np.random.default_rng(n)
        up = (rng.random((k, n)) < 8.0 / n).astype(np.uint8)
        up_s = P.ReferenceSet.from_array(P.Side.UPPER, 0, up, trusted=True)
        b = P.sample_batch(P.ComponentDistribution.iid(n, [0.05, 0.95]), S, seed=1)
        a, plane = b.fp4(2), b.fp4_plane_stride(2)
        bu, nu, au = up_s.device_fp4_rows(2)
        rb = _abi.fp4_row_bytes(n, 2)
        flags = torch.empty(S, dtype=torch.uint8, device=_device.device())
        res = {}
        for pair in ("0", "force", "force8"):
            os.environ["RSR_FP4_PAIR"] = pair[:5]
            os.environ["RSR_FP4_PAIR8"] = "1" if pair == "force8" else "0"
            tn = _abi.fp4_plan(S, 0, nu, rb)[0]
            run = lambda: _abi.call("rsr_classify_fp4_planar", _abi.ptr(a), plane, S, None, None, 0,
                                    0, _abi.ptr(bu), nu, au, rb, _abi.ptr(flags), None, None, 0,
                                    _device.stream())
            for _ in range(3):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(3, int(2e4 / k))
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            frac = S * k * 2 * 64 * (rb // 32) / (ms * 1e-3) / 9e15
            res[pair] = (tn, round(ms, 4), round(frac, 3))
        print(f"N={n} cq={rb // 32} K={k}: unpaired tn/ms/mma_frac {res['0']}  paired16 {res['force']}  paired8 {res['force8']}",
              flush=True)
