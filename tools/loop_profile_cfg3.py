"""cProfile of the config-3 Stage-1 loop (host time incl. synchronisation waits), after a
full warm-up run: where the ~0.6 ms per iteration goes.  RNG=device|shared."""
import cProfile
import os
import pstats
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2604_17066_b200 as P  # noqa: E402
from _specs import device_model  # noqa: E402

sys.argv = ["bench.py"]
import bench  # noqa: E402

rng = os.environ.get("RNG", "device")
spec, probs, kw, thresholds, desc = bench.loop_problem("cfg3", 64)
kw = {**kw, "rng": rng}
dist = P.ComponentDistribution(probs)
torch.cuda.set_device(0)
P.stage1_find_references(device_model(spec), dist, P.RunConfig(**{**kw, "seed": 7}), 0)
torch.cuda.synchronize()
model = device_model(spec)
cfg = P.RunConfig(**kw)
t0 = time.perf_counter()
s = P.stage1_find_references(model, dist, cfg, 0)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"unprofiled: {t1 - t0:.4f} s, {s.iterations} it, {1e3 * (t1 - t0) / s.iterations:.3f} ms/it")
model = device_model(spec)
pr = cProfile.Profile()
pr.enable()
s = P.stage1_find_references(model, dist, cfg, 0)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
