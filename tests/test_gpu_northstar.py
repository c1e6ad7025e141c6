"""Parity at the BASELINE north-star shapes (VERDICT r1 "Next round" item 1).

* config 4: S = 2^22 Bernoulli samples against K random simple s-t path references
  (upper side only, the default reference-chunked launches: 512 FP4 tiles per
  launch, i.e. 5 launches at K = 5x10^5).  Full-size FP4 tensor-core labels equal
  the bit-packed CUDA-core kernel's; three 2048-row slices (start / middle / end)
  equal the oracle restatement of classify.py:121-148.
* the run-to-c.o.v. loop (workflow.stage2_until_cov): batch 0 is
  stage2_evaluate (workflow.py:198-245), the accumulated counts equal the sum of
  oracle.stage2(start=j*H), and the loop stops at the first batch whose c.o.v. is
  within the target.
* configs 3 / 5 at the BASELINE batch size (2^20): the first Stage-1 iterations
  (workflow.py:122-195) against oracle.stage1 run on the host cores under a time
  budget -- ordered reference sets and every trace field.
"""

import os
import sys

import numpy as np
import pytest
import torch

import oracle
import paper_2604_17066_b200 as P
from paper_2604_17066_b200 import workloads as W

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _specs import device_model, oracle_phi  # noqa: E402

CORES = len(os.sched_getaffinity(0))
S4 = 1 << 22


@pytest.fixture(scope="module")
def cfg4_paths():
    g = W.cfg3(0)
    return W.random_st_paths(g, 500_000, seed=0)


@pytest.mark.parametrize("p1,k", [(0.9, 1_000), (0.9, 10_000), (0.9, 500_000),
                                  (0.8, 10_000), (0.8, 500_000)])
def test_cfg4_full_size_fp4_equals_bits_and_oracle_slices(cfg4_paths, p1, k):
    upper_rows = cfg4_paths[:k]
    assert len(upper_rows) == k
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper_rows, trusted=True)
    lo = P.ReferenceSet(P.Side.LOWER, 0)
    d = P.ComponentDistribution.iid(295, [1 - p1, p1])
    b = P.sample_batch(d, S4, seed=0)
    tc = P.classify(b, lo, up, n_states=2, method="tc")
    bits = P.classify(b, lo, up, n_states=2, method="bits")
    assert torch.equal(tc.labels_device, bits.labels_device)
    assert tc.counts == bits.counts and sum(tc.counts) == S4 and tc.counts[0] == 0
    if p1 == 0.8:  # mixed variant: both "survive" and "unclassified" occur in bulk
        assert min(tc.counts[1], tc.counts[2]) > S4 // 20
    states = b.device_states()
    rows = []
    for start in (0, S4 // 2 - 1024, S4 - 2048):
        rows.append(np.arange(start, start + 2048))
    idx = np.concatenate(rows)
    xs = states[torch.as_tensor(idx, device=states.device)].cpu().numpy()
    want = oracle.classify_labels(xs, np.zeros((0, 295), np.int64), upper_rows, 2,
                                  chunk_size=max(256, len(idx) // (4 * CORES)), n_workers=CORES)
    assert np.array_equal(tc.labels_device[torch.as_tensor(idx, device=states.device)].cpu().numpy(),
                          want["labels"])


def test_cfg4_first_match_chunked_launches(cfg4_paths):
    # explain=True at K = 2x10^5 (two reference-chunked launches of <= 122,880 rows):
    # the first 130,000 references carry ~200 extra ones and are almost never hit, so
    # the first match of most samples lies in the second launch; it must equal the
    # oracle's argmax over the whole set (classify.py:114-116)
    k, dense = 200_000, 130_000
    rng = np.random.default_rng(11)
    upper_rows = cfg4_paths[-k:].copy()
    upper_rows[:dense] |= (rng.random((dense, 295)) < 0.7).astype(np.uint8)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper_rows, trusted=True)
    d = P.ComponentDistribution.iid(295, [0.2, 0.8])
    b = P.sample_batch(d, 4096, seed=7, start=S4 - 4096)
    r = P.classify(b, None, up, n_states=2, explain=True)
    want = oracle.dominance_hits(b.device_states().cpu().numpy().astype(np.int64), upper_rows, 2,
                                 oracle.UPPER, chunk_size=256, n_workers=CORES, want_first=True)
    assert np.array_equal(r.first_match_upper, want[1])
    assert int((want[1] >= dense).sum()) > 500  # first matches in the second launch


@pytest.mark.parametrize("k_low,k_up", [(0, 3000), (1500, 1500), (0, 6000)])
def test_resident_chunked_launches_match_oracle(cfg4_paths, k_low, k_up, monkeypatch):
    # sets just past shared-memory residency run as resident-sized launches at the
    # north-star batch size (rsr_classify_fp4_plan); labels and first matches (explain)
    # must be those of one pass over the whole set: flags OR-accumulated, the earliest
    # chunk's match kept.  The oracle needs a small batch, which on its own would not
    # chunk (too few sample groups per CTA pair), so the 2^22-sample plan is forced.
    from paper_2604_17066_b200 import _abi
    rb = _abi.fp4_row_bytes(295, 2)
    assert _abi.fp4_plan(6144, k_low, k_up, rb)[1] == 1
    tn, launches = _abi.fp4_plan(1 << 22, k_low, k_up, rb, want_first=True)
    assert 2 <= launches <= 4, (tn, launches)
    nt_all = -(-k_low // tn) + -(-k_up // tn)
    monkeypatch.setenv("RSR_FP4_TILE_N", str(tn))
    monkeypatch.setenv("RSR_TC_CHUNK_TILES", str(-(-nt_all // launches)))
    rng = np.random.default_rng(k_low + k_up)
    upper_rows = cfg4_paths[:k_up].copy()
    # the earlier references rarely hit, so first matches fall in later launches too
    upper_rows[: k_up // 2] |= (rng.random((k_up // 2, 295)) < 0.05).astype(np.uint8)
    lower_rows = (rng.random((k_low, 295)) < 0.985).astype(np.uint8)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper_rows, trusted=True)
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower_rows, trusted=True)
    d = P.ComponentDistribution.iid(295, [0.1, 0.9])
    b = P.sample_batch(d, 6144, seed=3, start=1 << 20)
    r = P.classify(b, lo, up, n_states=2, explain=True)
    bits = P.classify(b, lo, up, n_states=2, method="bits")
    assert torch.equal(r.labels_device, bits.labels_device)
    xs = b.device_states().cpu().numpy().astype(np.int64)
    want_u = oracle.dominance_hits(xs, upper_rows, 2, oracle.UPPER, chunk_size=512,
                                   n_workers=CORES, want_first=True)
    assert np.array_equal(r.first_match_upper, want_u[1])
    nt = -(-k_low // tn) + -(-k_up // tn)
    first_launch_rows = -(-nt // launches) * tn - (-(-k_low // tn)) * tn  # upper rows in launch 1
    if first_launch_rows < k_up:
        assert int((want_u[1] >= max(first_launch_rows, 0)).sum()) > 50  # matches in later launches
    if k_low:
        want_l = oracle.dominance_hits(xs, lower_rows, 2, oracle.LOWER, chunk_size=512,
                                       n_workers=CORES, want_first=True)
        assert np.array_equal(r.first_match_lower, want_l[1])
        assert (want_l[1] >= 0).any()


# ----------------------------------------------------------- run-to-c.o.v. loop

def _grid():
    g = W.cfg1(0)
    spec = {"kind": "st", "n_nodes": g["n_nodes"], "edges": g["edges"], "s": 0, "t": 24,
            "m": 2, "ms": 2}
    return g, spec


@pytest.mark.parametrize("side", ["lower", "upper"])
def test_stage2_until_cov_matches_oracle_batches(side):
    g, spec = _grid()
    dist = P.ComponentDistribution(g["probs"])
    cfg = P.RunConfig(n_samples=3000, eps_u=1e-3, r_max=60, seed=4, parallel_searches=4)
    model = device_model(spec)
    s1 = P.stage1_find_references(model, dist, cfg, 0)
    h = 5000
    # P(S=0) ~ 0.017 here: c.o.v. 0.05 on it (0.001 on P(S=1)) needs ~2x10^4 samples
    target = 0.05 if side == "lower" else 0.001
    model.reset_evaluation_count()
    rep0 = P.stage2_evaluate(model, dist, s1.lower, s1.upper,
                             P.RunConfig(n_samples=h, seed=cfg.seed), 0)
    calls0 = model.evaluation_count
    model.reset_evaluation_count()
    rep = P.stage2_until_cov(model, dist, s1.lower, s1.upper, cfg, 0, target,
                             batch_samples=h, side=side)
    phi, n = oracle_phi(spec)
    ev = oracle.CountingPhi(phi, n, 2, 2)
    n_low = n_up = n_x = 0
    j = 0
    while True:
        o = oracle.stage2(ev, g["probs"], s1.lower.members, s1.upper.members, 0, h, cfg.seed,
                          start=j * h)
        if j == 0:  # batch 0 is the reference Stage 2
            assert (rep0.p_lower, rep0.p_upper, rep0.unclassified_resolved) == (
                o["p_lower"], o["p_upper"], o["unclassified_resolved"])
            assert calls0 == o["unclassified_resolved"]
        n_low, n_up, n_x = n_low + o["n_lower"], n_up + o["n_upper"], n_x + o["unclassified_resolved"]
        j += 1
        c = oracle.cov((n_low if side == "lower" else n_up) / (j * h), j * h)
        if c is not None and c <= target:
            break
    assert j >= 3
    assert rep.n_samples == j * h
    assert (rep.p_lower, rep.p_upper) == (n_low / (j * h), n_up / (j * h))
    assert rep.unclassified_resolved == n_x == model.evaluation_count
    assert rep.cov_lower == oracle.cov(n_low / (j * h), j * h)


def test_stage2_until_cov_validates_and_stops_on_budget():
    g, spec = _grid()
    model = device_model(spec)
    cfg = P.RunConfig(n_samples=1000, seed=0)
    lo, up = P.ReferenceSet(P.Side.LOWER, 0), P.ReferenceSet(P.Side.UPPER, 0)
    dist = P.ComponentDistribution(g["probs"])
    with pytest.raises(ValueError):
        P.stage2_until_cov(model, dist, lo, up, cfg, 0, 0.05, side="both")
    with pytest.raises(ValueError):
        P.stage2_until_cov(model, dist, lo, up, cfg, 0, 0.0)
    # every edge perfect: P(S=0) = 0, the estimate never leaves 0 and the loop must
    # stop at the sample budget instead of running 10^6 batches
    perfect = P.ComponentDistribution(np.tile([0.0, 1.0], (40, 1)))
    with pytest.warns(RuntimeWarning):
        rep = P.stage2_until_cov(model, perfect, lo, up, cfg, 0, 0.05, max_samples=20_000)
    assert rep.n_samples == 20_000 and rep.p_lower == 0.0 and rep.cov_lower is None


# ------------------------------------------------ configs 3 / 5 at full batch size

@pytest.mark.parametrize("cfg_name", ["cfg3", "cfg5"])
def test_full_batch_loop_prefix_vs_oracle(cfg_name):
    """Stage 1 at H = 2^20 with the bench protocol (eps_u 1e-5, 64 searches per
    iteration): the oracle runs on the host cores for a bounded time; the device loop,
    stopped by r_max at the oracle's final reference count, reproduces its ordered
    sets and every trace record of the iterations the oracle completed."""
    g = W.cfg3(0) if cfg_name == "cfg3" else W.cfg5(0)
    m = 2 if cfg_name == "cfg3" else 3
    spec = {"kind": "st" if m == 2 else "widest", "n_nodes": g["n_nodes"], "edges": g["edges"],
            "s": g["source"], "t": g["target"], "m": m, "ms": m}
    H = 1 << 20
    phi, n = oracle_phi(spec)
    ev = oracle.CountingPhi(phi, n, m, m)
    o1 = oracle.stage1(ev, g["probs"], 0, H, eps_u=1e-5, r_max=10_000, seed=0,
                       parallel_searches=64, n_workers=CORES,
                       chunk_size=max(256, H // (4 * CORES)), time_budget=60.0, fast=True)
    k = len(o1["trace"])
    # (the iteration count within the budget depends on the box's host cores)
    assert k >= 2 and o1["terminated_by"] == "budget"
    r_k = len(o1["lower"]) + len(o1["upper"])
    model = device_model(spec)
    cfg = P.RunConfig(n_samples=H, eps_u=1e-5, r_max=r_k, seed=0, parallel_searches=64)
    s1 = P.stage1_find_references(model, P.ComponentDistribution(g["probs"]), cfg, 0)
    assert s1.terminated_by == "r_max" and s1.iterations == k + 1
    assert s1.lower.members == o1["lower"] and s1.upper.members == o1["upper"]
    assert [(t.reference_count, t.phi_evaluations, t.p_lower, t.p_upper, t.p_unclassified)
            for t in s1.trace[:k]] == [(t["reference_count"], t["phi_evaluations"], t["p_lower"],
                                        t["p_upper"], t["p_unclassified"]) for t in o1["trace"]]
    assert s1.redundant_searches == o1["redundant_searches"]
    assert model.evaluation_count == ev.count


# --------------------------------------------- FP4 denormal-count self-check

@pytest.fixture
def fp4_selfcheck_reset():
    import importlib
    C = importlib.import_module("paper_2604_17066_b200.classify")
    saved = dict(C._FP4_EXACT)
    C._FP4_EXACT.clear()
    yield C
    C._FP4_EXACT.clear()
    C._FP4_EXACT.update(saved)


def test_fp4_selfcheck_passes_on_this_device(fp4_selfcheck_reset):
    assert fp4_selfcheck_reset.fp4_exact() is True


def test_fp4_selfcheck_failure_routes_to_int8_tensor_cores(fp4_selfcheck_reset, monkeypatch):
    """RSR_FP4_SELFCHECK=fail: the default classifier, the host-fed path and the
    Stage-1 loop run on the int8 tcgen05 kernel instead and still match the oracle."""
    C = fp4_selfcheck_reset
    monkeypatch.setenv("RSR_FP4_SELFCHECK", "fail")
    assert C.fp4_exact() is False
    calls = []
    from paper_2604_17066_b200 import _abi
    real = _abi.call

    def spy(name, *a):
        calls.append(name)
        return real(name, *a)
    monkeypatch.setattr(_abi, "call", spy)
    lower, upper = W.cfg2_mixed_refs(0, 295, 700, 700)
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower, trusted=True)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True)
    b = P.sample_batch(P.ComponentDistribution.iid(295, [0.5, 0.5]), 3000, seed=3)
    r = P.classify(b, lo, up, n_states=2)
    want = oracle.classify_labels(b.device_states().cpu().numpy(), lower, upper, 2)
    assert np.array_equal(r.labels_device.cpu().numpy(), want["labels"])
    from paper_2604_17066_b200.classify import classify_host
    labels, counts = classify_host(b.device_states().cpu(), lo, up, 2)
    assert np.array_equal(labels.numpy(), want["labels"])
    g, spec = _grid()
    cfg = dict(n_samples=3000, eps_u=1e-3, r_max=40, seed=1, parallel_searches=4)
    model = device_model(spec)
    s1 = P.stage1_find_references(model, P.ComponentDistribution(g["probs"]), P.RunConfig(**cfg), 0)
    phi, n = oracle_phi(spec)
    o1 = oracle.stage1(oracle.CountingPhi(phi, n, 2, 2), g["probs"], 0, **cfg)
    assert s1.lower.members == o1["lower"] and s1.upper.members == o1["upper"]
    assert "rsr_classify_tc" in calls
    assert not any(c.startswith("rsr_classify_fp4") for c in calls)


# ---------------------------------- wide multi-state rows on the tensor cores

@pytest.mark.parametrize("m", [4, 5])
def test_wide_multistate_rows_stay_on_tensor_cores(m, monkeypatch):
    """N = 295 at M = 4 / 5 (N(M-1) = 885 / 1180 > 831): the FP4 tensor-core kernel runs
    the lower and upper references as separate one-sided launches
    with labels and first matches equal to the oracle (classify.py:99-148)."""
    from paper_2604_17066_b200 import _abi
    n, h, k = 295, 3000, 700
    rng = np.random.default_rng(m)
    probs = rng.dirichlet([1.0] + [3.0] * (m - 2) + [16.0], size=n)
    samples = oracle.sample_states(probs, h, 5, 0, 0)
    lower = np.clip(samples[rng.integers(0, h, k)] + rng.integers(0, 2, (k, n)), 0, m - 1)
    upper = np.clip(samples[rng.integers(0, h, k)] - rng.integers(0, 2, (k, n)), 0, m - 1)
    want = oracle.classify_labels(samples, lower, upper, m, want_first=True, n_workers=CORES)
    assert len(set(want["labels"].tolist())) == 3
    from paper_2604_17066_b200.classify import fp4_exact
    assert fp4_exact()  # the one-time self-check runs the bit-packed kernel: before the spy
    calls = []
    real = _abi.call

    def spy(name, *a):
        calls.append(name)
        return real(name, *a)
    monkeypatch.setattr(_abi, "call", spy)
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower, trusted=True)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True)
    r = P.classify(P.SampleBatch(samples, 0, 0), lo, up, n_states=m, explain=True)
    assert np.array_equal(r.labels_device.cpu().numpy(), want["labels"])
    assert np.array_equal(r.first_match_lower, want["first_lower"])
    assert np.array_equal(r.first_match_upper, want["first_upper"])
    assert any(c.startswith("rsr_classify_fp4") for c in calls) and "rsr_classify_bits" not in calls
    # the device sampler's fused FP4 operand at this width, full classify path
    d = P.ComponentDistribution(probs)
    b = P.sample_batch(d, h, seed=9)
    r2 = P.classify(b, lo, up, n_states=m)
    want2 = oracle.classify_labels(oracle.sample_states(probs, h, 9, 0, 0), lower, upper, m,
                                   n_workers=CORES)
    assert np.array_equal(r2.labels_device.cpu().numpy(), want2["labels"])


def test_widest_rows_with_first_matches_leave_fp4_cleanly():
    # 768-byte FP4 rows (N(M-1) = 1475) fit shared memory without first matches but not
    # with them: explain=True must route to another tensor-core / CUDA-core kernel (the
    # planner reports tile_n 0) and still give the bit-packed kernel's answers
    from paper_2604_17066_b200 import _abi
    n, m, s = 1475, 2, 6000
    rb = _abi.fp4_row_bytes(n, m)
    assert rb == 768 and _abi.fp4_plan(s, 500, 300, rb, want_first=True)[0] == 0
    rng = np.random.default_rng(5)
    b = P.sample_batch(P.ComponentDistribution.iid(n, [0.03, 0.97]), s, seed=9)
    up = (rng.random((300, n)) < 0.002).astype(np.uint8)
    lo = 1 - (rng.random((500, n)) < 0.02).astype(np.uint8)
    uset = P.ReferenceSet.from_array(P.Side.UPPER, 0, up, trusted=True)
    lset = P.ReferenceSet.from_array(P.Side.LOWER, 0, lo, trusted=True)
    for explain in (False, True):
        r = P.classify(b, lset, uset, n_states=m, explain=explain)
        rb_ = P.classify(b, lset, uset, n_states=m, method="bits", explain=explain)
        assert torch.equal(r.labels_device, rb_.labels_device)
        if explain:
            assert np.array_equal(r.first_match_upper, rb_.first_match_upper)
            assert np.array_equal(r.first_match_lower, rb_.first_match_lower)
    assert min(r.counts) > 0 or r.counts[0] + r.counts[1] > 0
