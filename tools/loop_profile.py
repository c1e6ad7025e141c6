"""cProfile of the cfg3 Stage-1 loop (host time incl. synchronisation waits)."""
import cProfile
import os
import pstats
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2604_17066_b200 as P  # noqa: E402
from _specs import device_model  # noqa: E402

sys.argv = ["bench.py"]
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
spec, probs, kw, thresholds, desc = bench.loop_problem(os.environ.get("CFG", "cfg3"), 64)
dist = P.ComponentDistribution(probs)
torch.cuda.set_device(0)
wm = device_model(spec)
P.stage1_find_references(wm, dist, P.RunConfig(n_samples=1000, seed=1, r_max=5, eps_u=0.5),
                         thresholds[0])
torch.cuda.synchronize()
model = device_model(spec)
pr = cProfile.Profile()
pr.enable()
s1 = P.stage1_find_references(model, dist, P.RunConfig(**kw), thresholds[0])
torch.cuda.synchronize()
pr.disable()
print("iterations", s1.iterations)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
