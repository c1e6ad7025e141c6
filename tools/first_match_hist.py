"""How early do samples find their first dominating upper reference? (cfg3 / cfg5 Stage-1
sets; guides the two-pass classification of the Stage-1 loop)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2604_17066_b200 as P  # noqa: E402
from _specs import device_model  # noqa: E402

sys.argv = ["bench.py"]
import bench  # noqa: E402

torch.cuda.set_device(0)
for cfg in ("cfg3", "cfg5"):
    spec, probs, kw, thresholds, desc = bench.loop_problem(cfg, 64)
    dist = P.ComponentDistribution(probs)
    model = device_model(spec)
    for thr in thresholds:
        s1 = P.stage1_find_references(model, dist, P.RunConfig(**kw), thr)
        batch = P.sample_batch(dist, 1 << 20, 0, 7)
        res = P.classify(batch, s1.lower, s1.upper, explain=True, n_states=dist.n_states)
        fu = res.first_match_upper
        fl = res.first_match_lower
        lab = res.labels_device.cpu().numpy()
        up = lab == 1
        print(cfg, thr, "refs", len(s1.lower), len(s1.upper), "labels", res.counts)
        for u1 in (240, 480, 960, 1920, 3840):
            rem = np.mean(up & (fu >= u1)) + np.mean(lab == 2)
            print(f"   upper prefix {u1:5d}: fraction still unresolved after pass 1 = {rem:.5f}")
