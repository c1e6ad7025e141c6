"""cProfile of the config-5 Stage-1 loop at threshold 1, whose batches come from the HBM
batch cache filled at threshold 0 (no sampling: the serial classify -> search -> insert
chain and the host bookkeeping are what is left).  Host time incl. synchronisation waits."""
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
from paper_2604_17066_b200 import _abi  # noqa: E402
from paper_2604_17066_b200.workflow import _BatchCache  # noqa: E402
from _specs import device_model  # noqa: E402

sys.argv = ["bench.py"]
import bench  # noqa: E402

spec, probs, kw, thresholds, desc = bench.loop_problem("cfg5", 64)
dist = P.ComponentDistribution(probs)
torch.cuda.set_device(0)
wm = device_model(spec)
P.stage1_find_references(wm, dist, P.RunConfig(n_samples=1000, seed=1, r_max=5, eps_u=0.5), 0)
torch.cuda.synchronize()
model = device_model(spec)
cfg = P.RunConfig(**kw)
cache = _BatchCache(cfg.n_samples, _abi.fp4_row_bytes(dist.n_components, dist.n_states))
t0 = time.perf_counter()
s0 = P.stage1_find_references(model, dist, cfg, 0, _batch_cache=cache)
torch.cuda.synchronize()
t1 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
s1 = P.stage1_find_references(model, dist, cfg, 1, _batch_cache=cache)
torch.cuda.synchronize()
pr.disable()
t2 = time.perf_counter()
print(f"threshold 0: {t1 - t0:.4f} s, {s0.iterations} it; threshold 1 (cached): {t2 - t1:.4f} s, "
      f"{s1.iterations} it (profiled)")
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
