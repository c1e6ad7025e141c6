"""Sampler phase costs: states + FP4 (default), FP4 only, states only (2^20 x 295, M=2)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import _abi  # noqa: E402

torch.cuda.set_device(0)
d = P.ComponentDistribution.iid(295, [0.1, 0.9])
S = 1 << 20
st = torch.empty((S, 295), dtype=torch.uint8, device="cuda")
rb = _abi.fp4_row_bytes(295, 2)
a4 = torch.empty((S, 2 * rb), dtype=torch.uint8, device="cuda")
pr = _abi.ptr(d.device_probs())


def run(states, fp4):
    _abi.call("rsr_sample_fp4", pr, 295, 2, 0, 1, 0, S, _abi.ptr(states) if states is not None else None,
              _abi.ptr(fp4) if fp4 is not None else None, rb, _abi.stream_ptr())


for name, args in (("states+fp4", (st, a4)), ("fp4 only", (None, a4)), ("states only", (st, None))) * 2:
    run(*args)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        run(*args)
    e.record()
    e.synchronize()
    print(f"{name:12s} {s.elapsed_time(e) / 10:.3f} ms")
