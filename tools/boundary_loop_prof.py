"""Graph boundary-search counters on the start vectors the cfg3 / cfg5 Stage-1 loops
actually search (instrumented build, experiments only):
    make -C paper_2604_17066_b200/csrc prof
    RSR_LIB_OVERRIDE=tools/librsr_prof.so python tools/boundary_loop_prof.py
"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import _abi  # noqa: E402
from _specs import device_model  # noqa: E402

sys.argv = ["bench.py"]
import bench  # noqa: E402

torch.cuda.set_device(0)
fn = _abi.lib().rsr_boundary_prof
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 8)()
captured = []
orig = _abi.call
state = {"i": 0}


def spy(name, *args):
    if name == "rsr_boundary_search":
        n, B = args[0]._obj.n_components, int(args[3])
        if state["i"] % 30 == 0:
            t = torch.empty((B, n), dtype=torch.uint8, device="cuda")
            ident = torch.arange(B, dtype=torch.int64, device="cuda")
            orig("rsr_gather_rows", args[2], n, ident.data_ptr(), B, t.data_ptr(), args[-1])
            captured.append((state["i"], int(args[1]), t))
        state["i"] += 1
    return orig(name, *args)


_abi.call = spy
for cfg in ("cfg3", "cfg5"):
    spec, probs, kw, thresholds, desc = bench.loop_problem(cfg, 64)
    dist = P.ComponentDistribution(probs)
    model = device_model(spec)
    captured.clear()
    state["i"] = 0
    P.stage1_find_references(model, dist, P.RunConfig(**kw), thresholds[0])
    _abi.call = orig
    for it, thr, x in captured:
        P.boundary_search_batch(model, x, thr)
        torch.cuda.synchronize()
        fn(buf, 1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        P.boundary_search_batch(model, x, thr)
        e.record()
        torch.cuda.synchronize()
        fn(buf, 0)
        v = list(buf)
        up = max(v[1], 1)
        print(f"{cfg} it {it:3d}: {s.elapsed_time(e):.3f} ms; searches {v[0]} (upper {v[1]}); per upper "
              f"search: BFS {v[2] / up:.1f}, levels/BFS {v[3] / max(v[2], 1):.1f}, cycles/BFS "
              f"{v[4] / max(v[2], 1):.0f}, trace cycles/BFS {v[5] / max(v[2], 1):.0f}; "
              f"cycles/search {v[7] / max(v[0], 1):.0f}")
    _abi.call = spy
