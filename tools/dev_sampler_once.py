"""One launch per output set of the device-stream sampler (2^20 x 295, M = 2 and 3):
states + FP4, FP4 only, states only -- for ncu captures (not a timing script)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import _abi  # noqa: E402

S, N = 1 << 20, 295
ms = [int(a) for a in sys.argv[1:]] or [2]
for m in ms:
    d = P.ComponentDistribution.iid(N, [0.1, 0.9] if m == 2 else [0.05, 0.15, 0.8])
    rb = _abi.fp4_row_bytes(N, m)
    st = torch.empty((S, N), dtype=torch.uint8, device="cuda")
    a4 = torch.empty((2, S, rb), dtype=torch.uint8, device="cuda")
    pr = _abi.ptr(d.device_probs())
    for so, fo in ((st, a4), (None, a4), (st, None)):
        _abi.call("rsr_sample_fp4_ex", pr, N, m, 0, 1, 0, S, _abi.ptr(so), _abi.ptr(fo), rb,
                  S * rb if fo is not None else 0, _abi.RNG_DEVICE, _abi.stream_ptr())
    torch.cuda.synchronize()
