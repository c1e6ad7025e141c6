"""bench.py's multi-rank classification path on the one visible GPU (RSR_DIST_BACKEND=gloo:
host-side collectives, no kernel waits on another rank, so the ranks may share the device).
The driver's 8-GPU runs use NCCL with one GPU per rank; this checks the same code's
sharding, relaunch and JSON contract: strong scaling (2^22 samples split across the
ranks), replicated references with all-reduced counts, and the reference-sharded grid
with the OR-reduce of hit flags."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    env = dict(os.environ, RSR_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    return r, lines


BASE = ["--config", "cfg4", "--k", "3000", "--steps", "2", "--warmup", "3", "--no-cpu-baseline",
        "--no-secondary", "--no-loop"]


@pytest.fixture(scope="module")
def single():
    r, lines = _run(BASE)
    assert r.returncode == 0, r.stderr[-3000:]
    return lines[-1]


@pytest.mark.parametrize("extra", [[], ["--shard-refs"]])
def test_two_rank_bench_line_matches_one_rank(single, extra):
    r, lines = _run(["--gpus", "2"] + BASE + extra)
    assert r.returncode == 0, r.stderr[-3000:]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 prints the job's line
    line = lines[0]
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    cfg = line["config"]
    assert cfg["ranks"] == 2 and cfg["samples_total"] == single["config"]["samples_total"]
    # the union of the ranks' shards is the one-rank batch: identical label counts
    assert cfg["labels"] == single["config"]["labels"]
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert line["roofline"]["bound"] == "tensor"
    if extra:
        assert cfg["ref_states_per_gpu"] == cfg["ref_states"] // 2
