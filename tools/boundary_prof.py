"""Counters of the graph boundary search (instrumented build, experiments only):
    make -C paper_2604_17066_b200/csrc prof
    RSR_LIB_OVERRIDE=tools/librsr_prof.so python tools/boundary_prof.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import _abi, workloads as W  # noqa: E402

fn = _abi.lib().rsr_boundary_prof
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 8)()
g = W.cfg3(0)
graph = P.Graph(g["n_nodes"], tuple(g["edges"]))
rng = np.random.default_rng(0)
for name, m, thr, p_hi in (("st", 2, 0, 0.9), ("widest", 3, 0, 0.8), ("widest", 3, 1, 0.8)):
    phi = (P.single_od_connectivity(graph, g["source"], g["target"]) if name == "st"
           else P.widest_path_level(graph, g["source"], g["target"]))
    model = P.SystemModel(graph.n_edges, m, 2 if name == "st" else m, phi)
    lo = rng.random((64, graph.n_edges))
    xs = np.where(lo < p_hi, m - 1, rng.integers(0, m, size=lo.shape)).astype(np.uint8)
    xd = torch.as_tensor(xs).cuda()
    P.boundary_search_batch(model, xd, thr)
    torch.cuda.synchronize()
    fn(buf, 1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    P.boundary_search_batch(model, xd, thr)
    e.record()
    torch.cuda.synchronize()
    fn(buf, 0)
    v = list(buf)
    up = max(v[1], 1)
    if os.environ.get("RSR_BOUNDARY_MST", "1") != "0":  # closed-form upper side
        print(f"{name} m'={thr}: {s.elapsed_time(e):.3f} ms; searches {v[0]} (upper {v[1]}); per upper "
              f"search: spanning-forest cycles {v[2] / up:.0f}, tree BFS + trace cycles "
              f"{v[4] / up:.0f}; "
              f"init union-find cycles/search {v[6] / max(v[0], 1):.0f}; cycles/search "
              f"{v[7] / max(v[0], 1):.0f}")
        continue
    print(f"{name} m'={thr}: {s.elapsed_time(e):.3f} ms; searches {v[0]} (upper {v[1]}); per upper search: "
          f"BFS {v[2] / up:.1f}, levels/BFS {v[3] / max(v[2], 1):.1f}, cycles/BFS {v[4] / max(v[2], 1):.0f}, "
          f"trace cycles/BFS {v[5] / max(v[2], 1):.0f}, init union-find cycles/search {v[6] / max(v[0], 1):.0f}; "
          f"cycles/search {v[7] / max(v[0], 1):.0f}")
