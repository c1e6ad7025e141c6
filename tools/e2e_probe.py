"""e2e probe: host-fed classification on the packed one-hot rows (classify_host_encoded), cfg2 shape."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2604_17066_b200 as P
from paper_2604_17066_b200 import _abi, workloads as W
from paper_2604_17066_b200.classify import classify_host_encoded
torch.cuda.set_device(0)
S, N, m = 1 << 20, 295, 2
lower, upper = W.cfg2_refs(0, N, 10_000, 10_000)
lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower, trusted=True)
up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True)
b = P.sample_batch(P.ComponentDistribution.iid(N, [0.1, 0.9]), S, 0)
rows = torch.empty((S, N * m), dtype=torch.uint8, device="cuda")
_abi.call("rsr_encode_rows", _abi.ptr(b.device_states()), S, N, m, 0, _abi.ptr(rows), _abi.stream_ptr())
nb = (N * m + 7) // 8
pk = torch.empty((S, nb), dtype=torch.uint8, device="cuda")
_abi.call("rsr_packbits_rows", _abi.ptr(rows), S, N * m, 0, _abi.ptr(pk), _abi.stream_ptr())
host = torch.empty((S, nb), dtype=torch.uint8, pin_memory=True); host.copy_(pk)
out = torch.empty(S, dtype=torch.uint8, pin_memory=True)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
print("H2D only %.3f ms" % t(lambda: pk.copy_(host, non_blocking=True)))
rb = _abi.fp4_row_bytes(N, m)
a4 = torch.empty((S, 2 * rb), dtype=torch.uint8, device="cuda")
print("unpack 2^20 %.3f ms" % t(lambda: _abi.call("rsr_unpack_onehot_fp4", _abi.ptr(pk), S, N, m, _abi.ptr(a4), rb, _abi.stream_ptr())))
for ch in (1 << 16, 1 << 17, 1 << 18, 1 << 19):
    print("chunk %d: e2e %.3f ms" % (ch, t(lambda: classify_host_encoded(host, N, lo, up, m, chunk_rows=ch, labels_out=out))))
