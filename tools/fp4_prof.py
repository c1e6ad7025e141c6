"""Per-role cycle counters of the FP4 classifier (instrumented build, timing
experiments only): make -C paper_2604_17066_b200/csrc prof, then
    RSR_LIB_OVERRIDE=tools/librsr_prof.so python tools/fp4_prof.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import _abi, workloads as W  # noqa: E402
from paper_2604_17066_b200.classify import classify_flags  # noqa: E402

lib = _abi.lib()
fn = lib.rsr_fp4_prof
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 24)()
K = int(os.environ.get("K", "10000"))
S = int(os.environ.get("S", str(1 << 20)))
M = int(os.environ.get("M", "2"))
if M == 2:
    lower, upper = W.cfg2_refs(0, 295, K, K)
    probs = [0.1, 0.9]
else:  # the M=3 classification shape of tools/time_kernels.py classify_m3
    rng = np.random.default_rng(5)
    lower, upper = rng.integers(1, 3, size=(K, 295)), rng.integers(0, 2, size=(K, 295))
    probs = [0.05, 0.15, 0.8]
if os.environ.get("REFS") == "paths":  # bench.py cfg4: s-t path references of the cfg3 graph
    lower, upper = lower[:0], W.random_st_paths(W.cfg3(0), K, seed=0)
if os.environ.get("UPPER_ONLY"):  # cfg4-like: survival references only
    lower = lower[:0]
lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower, trusted=True)
up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True)
batch = P.sample_batch(P.ComponentDistribution.iid(295, probs), S, seed=0)
for it in range(3):
    fn(buf, 1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    classify_flags(batch, lo, up, M)
    e.record()
    torch.cuda.synchronize()
    fn(buf, 0)
v = list(buf)
tiles = v[7]
print(f"kernel+encode {s.elapsed_time(e):.3f} ms; tiles (MMA warp) {tiles}")
names = ["b_full (MMA) / tmem load (epi)", "mma wait t_empty", "mma loop total", "epi wait t_full",
         "epi load+rel+min", "epi bookkeeping", "prod wait b_empty"]
E = int(os.environ.get("EPI_WARPS", "16")) * 2  # epilogue warps per tile (both CTAs)
per = [tiles + E * tiles, tiles, tiles, E * tiles, E * tiles, E * tiles, 2 * tiles]
for n, x, d in zip(names, v, per):
    print(f"{n:20s} {x / max(d, 1):8.1f} cycles per tile (per warp)")
groups = max(v[11], 1)
print(f"groups (MMA) {groups}, tiles per group {tiles / groups:.1f}; MMA-loop cycles per group "
      f"{v[2] / groups:.0f}")
print(f"epi group-end exchange {v[8] / (E * groups):8.1f} cycles per group (per warp)")
print(f"mma wait a_full        {v[9] / groups:8.1f} cycles per group")
print(f"prod wait a_empty      {v[10] / (2 * groups):8.1f} cycles per group")
ncl = max(v[12] and 74, 1)
print(f"MMA warp setup {v[12] / ncl:.0f} cycles, teardown wait {v[13] / ncl:.0f} cycles per cluster; "
      f"groups per cluster {groups / ncl:.1f}, MMA-loop cycles per cluster {v[2] / ncl:.0f}")
if v[14]:
    print(f"SM clock over the MMA warp's run: {v[15] / v[14]:.3f} GHz "
          f"({v[15] / ncl:.0f} cycles, {v[14] / ncl / 1e3:.1f} us per cluster)")
if v[20]:
    print(f"chain: commit issued -> epilogue (CTA 0) sees t_full {v[16] / v[20]:.0f} cycles; "
          f"CTA-0 release -> MMA warp sees t_empty {v[17] / max(v[21], 1):.0f}; "
          f"MMA issue of a tile {v[18] / max(tiles, 1):.0f}")
