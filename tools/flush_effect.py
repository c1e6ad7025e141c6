"""FP4 classifier launch time with and without an L2 flush (256 MB memset) before each launch.
    K=2000 RSR_FP4_RESIDENT=0 RSR_FP4_TILE_N=240 python tools/flush_effect.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import _abi, workloads as W  # noqa: E402

K = int(os.environ.get("K", "2000"))
S = 1 << 22
upper = W.random_st_paths(W.cfg3(0), K, seed=0)
up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True)
t, n, avail = up.device_fp4_rows(2)
rb = _abi.fp4_row_bytes(295, 2)
batch = P.sample_batch(P.ComponentDistribution.iid(295, [0.1, 0.9]), S, seed=0)
a = batch.device_fp4(2) if hasattr(batch, "device_fp4") else None
if a is None:
    a = torch.empty((S, 2 * rb), dtype=torch.uint8, device="cuda")
    st = batch.device_states()
    _abi.call("rsr_encode_samples_fp4", _abi.ptr(st), S, 295, 2, _abi.ptr(a), rb, _abi.stream_ptr())
flags = torch.empty(S, dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def launch():
    _abi.call("rsr_classify_fp4_ex", _abi.ptr(a), S, None, None, 0, 0, _abi.ptr(t), n, avail, rb,
              _abi.ptr(flags), None, None, 0, _abi.stream_ptr())


for mode in ("flush", "no flush", "flush+sleep"):
    for _ in range(3):
        launch()
    ts = []
    for _ in range(10):
        if mode != "no flush":
            flush.zero_()
        if mode == "flush+sleep":
            torch.cuda._sleep(2_000_000)  # ~1 ms spin between the flush and the launch
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        launch()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print(f"K={K} {mode:12s} kernel ms median {np.median(ts):.4f} min {min(ts):.4f}")

# host cost of one launch call (enqueue only; the GPU is kept busy by a spin)
import time  # noqa: E402
torch.cuda._sleep(50_000_000)
hs = []
for _ in range(20):
    t0 = time.perf_counter()
    launch()
    hs.append((time.perf_counter() - t0) * 1e6)
torch.cuda.synchronize()
print(f"host enqueue us per launch: median {np.median(hs):.1f} min {min(hs):.1f} max {max(hs):.1f}")
