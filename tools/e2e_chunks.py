"""e2e classify_host step time vs H2D chunk size (cfg2 shape)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import workloads as W  # noqa: E402
from paper_2604_17066_b200.classify import classify_host, classify_host_encoded  # noqa: E402

torch.cuda.set_device(0)
lower, upper = W.cfg2_refs(0, 295, 10_000, 10_000)
lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower, trusted=True)
up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True)
S = 1 << 20
batch = P.sample_batch(P.ComponentDistribution.iid(295, [0.1, 0.9]), S, seed=0)
host = torch.empty((S, 295), dtype=torch.uint8, pin_memory=True)
host.copy_(batch.device_states())
out = torch.empty(S, dtype=torch.uint8, pin_memory=True)
m = 2
rows = torch.empty((S, 295 * m), dtype=torch.uint8, device="cuda")
P._abi.call("rsr_encode_rows", P._abi.ptr(batch.device_states()), S, 295, m, 0, P._abi.ptr(rows),
            P._abi.stream_ptr())
nb = (295 * m + 7) // 8
pk = torch.empty((S, nb), dtype=torch.uint8, device="cuda")
P._abi.call("rsr_packbits_rows", P._abi.ptr(rows), S, 295 * m, 0, P._abi.ptr(pk), P._abi.stream_ptr())
hpk = torch.empty((S, nb), dtype=torch.uint8, pin_memory=True)
hpk.copy_(pk)
for chunk in (1 << 15, 1 << 16, 1 << 17):
    for _ in range(2):
        classify_host_encoded(hpk, 295, lo, up, 2, labels_out=out, chunk_rows=chunk)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        classify_host_encoded(hpk, 295, lo, up, 2, labels_out=out, chunk_rows=chunk)
    torch.cuda.synchronize()
    print(f"encoded chunk {chunk:7d}: {1e3 * (time.perf_counter() - t) / 10:.3f} ms per step")
for chunk in (1 << 15, 1 << 16, 1 << 17, 1 << 18):
    for _ in range(2):
        classify_host(host, lo, up, 2, labels_out=out, chunk_rows=chunk)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        classify_host(host, lo, up, 2, labels_out=out, chunk_rows=chunk)
    torch.cuda.synchronize()
    print(f"chunk {chunk:7d}: {1e3 * (time.perf_counter() - t) / 10:.3f} ms per step")
