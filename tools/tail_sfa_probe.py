"""Which A scale-factor word makes the shared-tail MMA (PAIR = 3) exact: runs the shared-tail
classifier with candidate RSR_FP4_TAIL_SFA words on cfg4-shaped data and compares the flags
with the unpaired kernel.  usage: python tools/tail_sfa_probe.py"""
import importlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import workloads as W  # noqa: E402

C = importlib.import_module("paper_2604_17066_b200.classify")
paths = W.random_st_paths(W.cfg3(0), 100_000, seed=0)
up = P.ReferenceSet.from_array(P.Side.UPPER, 0, paths, trusted=True)
lo = P.ReferenceSet(P.Side.LOWER, 0)
b = P.sample_batch(P.ComponentDistribution.iid(295, [0.15, 0.85]), 1 << 16, seed=5)
os.environ["RSR_FP4_COMPACT"] = "force"
os.environ["RSR_FP4_TAIL"] = "0"
ref = P.classify(b, lo, up, n_states=2).labels_device.cpu().numpy()
plan = C.fp4_compaction(1 << 16, 295, 2, lo, up, force=True)
print("support", up.device_fp4_support(2).size, "rb", plan.row_bytes)
os.environ["RSR_FP4_TAIL"] = "1"
plan = C.fp4_compaction(1 << 16, 295, 2, lo, up, force=True)
print("tail_tn", plan.tail_tn, "n_pad", plan.n_pad, "counts", np.bincount(ref, minlength=3))
for w in ("0x00001000", "0x00100000", "0x10000000", "0x00000010", "0x10001000"):
    os.environ["RSR_FP4_TAIL_SFA"] = w
    got = P.classify(b, lo, up, n_states=2).labels_device.cpu().numpy()
    print(w, "equal" if np.array_equal(got, ref) else f"DIFF {(got != ref).sum()}", flush=True)
