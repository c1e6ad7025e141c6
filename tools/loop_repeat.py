"""Run-to-run spread of the config-3 / config-5 loop wall time inside one process (the bench's
wall_time_to_cov measures one run after a short warm-up)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv = ["bench.py"]
import bench  # noqa: E402

cfg = os.environ.get("CFG", "cfg3")
for rng in ("shared", "device"):
    vals = []
    for _ in range(int(os.environ.get("REPS", "5"))):
        t0 = time.perf_counter()
        r = bench.measure_loop(cfg, 64, rng=rng)
        vals.append(round(r["value"], 4))
    print(cfg, rng, vals, flush=True)
