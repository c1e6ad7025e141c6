"""rsr_encode_samples_fp4 time per 2^20 rows (N = 295, M = 2 / 3; planar output) -- the
host-fed (e2e) path's on-device encode."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import _abi  # noqa: E402

S, N = 1 << 20, 295
for m in (2, 3):
    st = torch.randint(0, m, (S, N), dtype=torch.uint8, device="cuda")
    rb = _abi.fp4_row_bytes(N, m)
    out = torch.empty((2, S, rb), dtype=torch.uint8, device="cuda")
    def run():
        _abi.call("rsr_encode_samples_fp4_ex", _abi.ptr(st), S, N, m, _abi.ptr(out), rb, S * rb,
                  _abi.stream_ptr())
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    gb = (S * N + 2 * S * rb) / 1e9
    print(f"M={m}: {ms:.3f} ms per 2^20 rows, {gb / ms * 1e3:.0f} GB/s")
