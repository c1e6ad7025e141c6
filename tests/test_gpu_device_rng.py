"""The independent device RNG mode (BASELINE north_star: "agree within 3 combined
standard errors under independent device RNG").

* the Philox4x32-10 device stream and its inverse CDF equal the oracle
  restatement (pinned by the Random123 known-answer vectors on CPU) bit for bit;
* its marginals match the component probabilities at full batch size, and it is
  independent of the reference's Philox4x64-10 stream;
* the Stage-1 / Stage-2 workflow with ``RunConfig(rng="device")`` equals the oracle
  workflow run on the same device stream (reference sets, traces, estimates);
* configs 3 and 5 run to c.o.v. 0.05 under both streams: each P-hat agrees with
  the shared-stream P-hat within 3 combined standard errors (workflow.py:234-245
  semantics: p = n / H, SE = sqrt(p (1 - p) / H)).
"""

import math
import os
import sys

import numpy as np
import pytest
import torch

import oracle
import paper_2604_17066_b200 as P
from paper_2604_17066_b200 import _abi
from paper_2604_17066_b200 import workloads as W

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _specs import device_model, oracle_phi  # noqa: E402


@pytest.mark.parametrize("seed,gen,start,count,n", [(0, 0, 0, 1, 4), (7, 3, 1, 4099, 295),
                                                     ((1 << 63) + 5, (1 << 40) + 1, 1 << 34, 1023,
                                                      7)])
def test_device_raw_matches_oracle(seed, gen, start, count, n):
    out = torch.empty(count * n, dtype=torch.int32, device="cuda")
    _abi.call("rsr_device_raw", seed, gen, start, count, n, _abi.ptr(out), _abi.stream_ptr())
    got = out.cpu().numpy().view(np.uint32).reshape(count, n)
    from oracle.philox import device_raw
    assert np.array_equal(got, device_raw(seed, gen, start, count, n))


@pytest.mark.parametrize("n,m,h,start", [(295, 2, 4099, 0), (295, 3, 2000, 12345),
                                         (40, 5, 3000, 1 << 20), (7, 2, 777, 3),
                                         (8, 2, 130, 0), (64, 3, 200, 9), (3, 4, 65, 1),
                                         (100, 2, 1, (1 << 32) + 3)])
@pytest.mark.parametrize("fp4", [True, False])
def test_device_stream_samples_match_oracle(n, m, h, start, fp4):
    rng = np.random.default_rng(n * m + h)
    raw = rng.random((n, m)) + 0.02
    probs = raw / raw.sum(1, keepdims=True)
    d = P.ComponentDistribution(probs)
    b = P.sample_batch(d, h, seed=11, generation_index=5, start=start, fp4=fp4, rng="device")
    want = oracle.sample_states(probs, h, 11, 5, start, rng="device")
    assert np.array_equal(b.device_states().cpu().numpy(), want)
    assert b.rng == "device"
    if fp4 and _abi.fp4_row_bytes(n, m) <= _abi.FP4_MAX_ROW_BYTES:
        # the fused FP4 operand equals the encoder's rows of the same states
        enc = P.SampleBatch(b.device_states().clone(), 0, 0, state_bound=m).fp4(m)
        assert torch.equal(b.fp4(m), enc)


def test_device_stream_marginals_and_independence():
    # full batch of config 4 (2^22 x 295 Bernoulli(0.9)): every component's frequency
    # within 5 SE of 0.9; the agreement rate with the shared stream is that of two
    # independent Bernoulli(0.9) draws (0.82), not 1
    S, n = 1 << 22, 295
    d = P.ComponentDistribution.iid(n, [0.1, 0.9])
    dev = P.sample_batch(d, S, seed=0, rng="device").device_states()
    freq = dev.float().mean(0).cpu().numpy()
    se = math.sqrt(0.9 * 0.1 / S)
    assert np.abs(freq - 0.9).max() < 5 * se
    shared = P.sample_batch(d, S, seed=0).device_states()
    agree = (dev == shared).float().mean().item()
    assert abs(agree - 0.82) < 1e-3
    # rows are independent of each other: adjacent-row agreement is also 0.82
    assert abs((dev[1:] == dev[:-1]).float().mean().item() - 0.82) < 1e-3


def test_device_rng_workflow_matches_oracle_on_same_stream():
    g = W.cfg1(0)
    spec = {"kind": "st", "n_nodes": g["n_nodes"], "edges": g["edges"], "s": 0, "t": 24,
            "m": 2, "ms": 2}
    cfg = dict(n_samples=6000, eps_u=1e-3, r_max=80, seed=2, parallel_searches=8)
    model = device_model(spec)
    dist = P.ComponentDistribution(g["probs"])
    s1 = P.stage1_find_references(model, dist, P.RunConfig(**cfg, rng="device"), 0)
    rep = P.stage2_evaluate(model, dist, s1.lower, s1.upper, P.RunConfig(**cfg, rng="device"), 0)
    phi, n = oracle_phi(spec)
    ev = oracle.CountingPhi(phi, n, 2, 2)
    o1 = oracle.stage1(ev, g["probs"], 0, rng="device", **cfg)
    o2 = oracle.stage2(ev, g["probs"], o1["lower"], o1["upper"], 0, cfg["n_samples"], cfg["seed"],
                       rng="device")
    assert s1.lower.members == o1["lower"] and s1.upper.members == o1["upper"]
    assert [(t.reference_count, t.phi_evaluations, t.p_lower, t.p_upper, t.p_unclassified)
            for t in s1.trace] == [(t["reference_count"], t["phi_evaluations"], t["p_lower"],
                                    t["p_upper"], t["p_unclassified"]) for t in o1["trace"]]
    assert (rep.p_lower, rep.p_upper, rep.unclassified_resolved) == (
        o2["p_lower"], o2["p_upper"], o2["unclassified_resolved"])
    assert model.evaluation_count == ev.count
    # and it is a different stream from the reference's
    o1s = oracle.stage1(oracle.CountingPhi(phi, n, 2, 2), g["probs"], 0, **cfg)
    assert [t["p_lower"] for t in o1s["trace"]] != [t["p_lower"] for t in o1["trace"]]


def _loop_estimates(cfg_name, rng):
    g = W.cfg3(0) if cfg_name == "cfg3" else W.cfg5(0)
    m = 2 if cfg_name == "cfg3" else 3
    spec = {"kind": "st" if m == 2 else "widest", "n_nodes": g["n_nodes"], "edges": g["edges"],
            "s": g["source"], "t": g["target"], "m": m, "ms": m}
    model = device_model(spec)
    dist = P.ComponentDistribution(g["probs"])
    cfg = P.RunConfig(n_samples=1 << 20, eps_u=1e-5, r_max=10_000, seed=0, parallel_searches=64,
                      rng=rng)
    out = []
    for thr in range(m - 1):
        s1 = P.stage1_find_references(model, dist, cfg, thr)
        rep = P.stage2_until_cov(model, dist, s1.lower, s1.upper, cfg, thr, 0.05, side="lower")
        out.append((rep.p_lower, rep.n_samples))
    return out


@pytest.mark.parametrize("cfg_name", ["cfg3", "cfg5"])
def test_loop_estimates_agree_within_3_combined_se(cfg_name):
    shared = _loop_estimates(cfg_name, "shared")
    device = _loop_estimates(cfg_name, "device")
    for (p1, n1), (p2, n2) in zip(shared, device):
        se = math.sqrt(p1 * (1 - p1) / n1 + p2 * (1 - p2) / n2)
        assert 0 < p1 < 1 and 0 < p2 < 1
        assert abs(p1 - p2) <= 3 * se, (cfg_name, p1, p2, se)
        assert p1 != p2  # independent streams


@pytest.mark.parametrize("stream", ["shared", "device"])
@pytest.mark.parametrize("n,m", [(1475, 2), (767, 3)])
def test_widest_rows_sample_like_the_oracle(stream, n, m):
    # rows whose 64-row staging buffers exceed shared memory run 16-row chunks (reference
    # stream) / row-aligned threads (device stream); both equal the oracle, FP4 operand
    # included (it equals the encoder's rows of the same states)
    rng = np.random.default_rng(n + m)
    raw = rng.random((n, m)) + 0.05
    probs = raw / raw.sum(1, keepdims=True)
    b = P.sample_batch(P.ComponentDistribution(probs), 300, seed=4, generation_index=2, start=77,
                       rng=stream)
    want = oracle.sample_states(probs, 300, 4, 2, 77, rng=stream)
    assert np.array_equal(b.device_states().cpu().numpy(), want)
    enc = P.SampleBatch(b.device_states().clone(), 0, 0, state_bound=m).fp4(m)
    assert torch.equal(b.fp4(m), enc)
