"""Sampler time per output set and stream (2^20 x 295, M = 2): states + FP4 operand, FP4 only,
states only -- where the time goes beyond the generator (tools/philox_rate.cu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import _abi  # noqa: E402

S, N = 1 << 20, 295
for m, probs in ((2, [0.1, 0.9]), (3, [0.05, 0.15, 0.8])):
    d = P.ComponentDistribution.iid(N, probs)
    rb = _abi.fp4_row_bytes(N, m)
    st = torch.empty((S, N), dtype=torch.uint8, device="cuda")
    a4 = torch.empty((2, S, rb), dtype=torch.uint8, device="cuda")
    pr = _abi.ptr(d.device_probs())
    for rng in (_abi.RNG_SHARED, _abi.RNG_DEVICE):
        row = []
        for name, so, fo in (("both", st, a4), ("fp4", None, a4), ("states", st, None)):
            def run():
                _abi.call("rsr_sample_fp4_ex", pr, N, m, 0, 1, 0, S, _abi.ptr(so), _abi.ptr(fo), rb,
                          S * rb if fo is not None else 0, rng, _abi.stream_ptr())
            run()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(20):
                run()
            e.record()
            e.synchronize()
            row.append(f"{name} {s.elapsed_time(e) / 20:.3f} ms")
        print(f"M={m} {'shared' if rng == 0 else 'device'}: " + ", ".join(row))
