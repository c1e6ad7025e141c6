"""Device path through the public API vs the reference's golden vectors and the oracle."""

import numpy as np
import pytest
import torch

import oracle
import paper_2604_17066_b200 as P
from _specs import device_model, load_json, load_npz

pytestmark = pytest.mark.gpu


def _set(side, thr, rows):
    s = P.ReferenceSet(side, thr)
    for v in rows:
        s.insert(P.ReferenceState(tuple(int(x) for x in v), side, thr))
    return s


# ---------------------------------------------------------------- sampling

def test_sample_batch_golden():
    g = load_npz("sampling.npz")
    for i, (n, seed, gen, start) in enumerate(g["specs"]):
        b = P.sample_batch(P.ComponentDistribution(g[f"probs{i}"]), n, seed, gen, start)
        assert np.array_equal(b.states, g[f"states{i}"])
        assert b.n_samples == n and b.n_components == g[f"probs{i}"].shape[0]


def test_uniform_field_golden():
    g = load_npz("philox.npz")
    for i, c in enumerate(g["ucases"]):
        assert np.array_equal(P.uniform_field(*c), g[f"uniform{i}"])


def test_sampling_properties():
    # reference test_sampling.py: degenerate rows, determinism, generation, chunking, marginal
    d1 = P.ComponentDistribution.iid(4, [0.0, 1.0])
    assert np.all(P.sample_batch(d1, 50, seed=1).states == 1)
    d0 = P.ComponentDistribution.iid(4, [1.0, 0.0])
    assert np.all(P.sample_batch(d0, 50, seed=1).states == 0)
    d = P.ComponentDistribution.iid(3, [0.2, 0.5, 0.3])
    full = P.sample_batch(d, 100, seed=4, generation_index=1)
    part = P.sample_batch(d, 40, seed=4, generation_index=1, start=37)
    assert np.array_equal(full.states[37:77], part.states)
    a = P.sample_batch(d, 1000, seed=9, generation_index=0).states
    b = P.sample_batch(d, 1000, seed=9, generation_index=1).states
    assert not np.array_equal(a, b)
    one = P.ComponentDistribution.iid(1, [0.1, 0.9])
    freq = float(np.mean(P.sample_batch(one, 1_000_000, seed=42).states == 0))
    assert abs(freq - 0.1) < 0.001
    with pytest.raises(ValueError):
        P.sample_batch(d, 0, seed=1)


def test_sampling_full_size_matches_oracle_slices():
    # cfg2 shape: S = 2^20, N = 295; check three slices bit-exactly against the oracle
    d = P.ComponentDistribution.iid(295, [0.1, 0.9])
    b = P.sample_batch(d, 1 << 20, seed=0, generation_index=0)
    st = b.device_states()
    for lo in (0, 517_001, (1 << 20) - 300):
        want = oracle.sample_states(d.probs, 300, 0, 0, lo)
        assert np.array_equal(st[lo:lo + 300].cpu().numpy(), want)


# ---------------------------------------------------------------- encodings

def test_encoding_worked_examples():
    assert np.array_equal(P.encode_lower_ref((1, 2), 5), [[1, 1, 0, 0, 0], [1, 1, 1, 0, 0]])
    assert np.array_equal(P.encode_upper_ref((1, 4), 5), [[0, 1, 1, 1, 1], [0, 0, 0, 0, 1]])
    assert np.array_equal(P.encode_upper_ref((4, 0), 5), [[0, 0, 0, 0, 1], [1, 1, 1, 1, 1]])
    assert np.array_equal(P.encode_sample((3, 0), 5), [[0, 0, 0, 1, 0], [1, 0, 0, 0, 0]])
    assert np.array_equal(P.encode_sample((0, 0, 0), 1), np.ones((3, 1)))
    with pytest.raises(ValueError):
        P.encode_sample((5,), 5)
    rng = np.random.default_rng(1)
    for m in (2, 3, 5):
        st = rng.integers(0, m, size=(7, 4))
        for kind in ("sample", "lower_ref", "upper_ref"):
            e = P.encode_batch(st, m, kind)
            assert np.array_equal(e.data, oracle.encode(st, m, kind))
            assert np.array_equal(e.packed, np.packbits(e.data, axis=1))
            assert np.array_equal(e.packed_complement, np.packbits(1 - e.data, axis=1))
            assert np.array_equal(e.decode_states(), st)


# ----------------------------------------------------------- classification

@pytest.mark.parametrize("method", ["tc", "tc8", "bits"])
def test_classify_golden(method):
    g = load_npz("classify.npz")
    for i, m in enumerate(g["n_states"]):
        m = int(m)
        batch = P.SampleBatch(g[f"samples{i}"], 0, 0)
        lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, g[f"lower{i}"], trusted=True)
        up = P.ReferenceSet.from_array(P.Side.UPPER, 0, g[f"upper{i}"], trusted=True)
        r = P.classify(batch, lo, up, n_states=m, method=method)
        assert np.array_equal(r.lower_indices, g[f"lo_idx{i}"])
        assert np.array_equal(r.upper_indices, g[f"up_idx{i}"])
        assert np.array_equal(r.unclassified_indices, g[f"un_idx{i}"])
        e = P.classify(batch, lo, up, n_states=m, explain=True, method=method)
        assert np.array_equal(e.first_match_lower, g[f"first_lo{i}"])
        assert np.array_equal(e.first_match_upper, g[f"first_up{i}"])


def test_violation_counts_golden():
    g = load_npz("classify.npz")
    s = P.encode_batch(g["viol_samples"], 3, "sample")
    for kind in ("lower_ref", "upper_ref"):
        got = P.violation_counts(s, P.encode_batch(g["viol_refs"], 3, kind))
        assert np.array_equal(got, g[f"viol_{kind}"])
    with pytest.raises(ValueError):
        P.violation_counts(s, s)


def test_classify_reference_examples():
    # reference test_classify.py:104-168 (counts 3/4/3, empty sets, precedence, strict, explain)
    states = np.array([[0, 0]] * 3 + [[4, 4]] * 4 + [[2, 2]] * 3)
    batch = P.SampleBatch(states, 0, 0)
    lower = _set(P.Side.LOWER, 0, [(1, 2)])
    upper = _set(P.Side.UPPER, 0, [(1, 4), (4, 0)])
    res = P.classify(batch, lower, upper, n_states=5)
    assert (res.p_lower, res.p_upper, res.p_unclassified) == (0.3, 0.4, 0.3)
    d = P.ComponentDistribution.iid(3, [0.5, 0.5])
    b20 = P.sample_batch(d, 20, seed=2)
    assert P.classify(b20, None, None, n_states=2).p_unclassified == 1.0
    assert P.classify(b20, _set(P.Side.LOWER, 0, [(1, 1, 1)]), None, n_states=2).p_lower == 1.0
    one = P.SampleBatch(np.array([[1, 1]]), 0, 0)
    lo, up = _set(P.Side.LOWER, 0, [(1, 1)]), _set(P.Side.UPPER, 0, [(1, 1)])
    r = P.classify(one, lo, up, n_states=2)
    assert r.lower_indices.size == 1 and r.upper_indices.size == 0
    with pytest.raises(P.InconsistentReferenceSets):
        P.classify(one, lo, up, strict=True, n_states=2)
    with pytest.raises(ValueError):
        P.classify(b20, _set(P.Side.LOWER, 0, [(0, 0, 0)]), _set(P.Side.UPPER, 1, [(1, 1, 1)]))
    ex = P.classify(P.SampleBatch(np.array([[0, 0], [4, 4], [2, 2]]), 0, 0), lower, upper,
                    explain=True, n_states=5)
    assert ex.first_match_lower[0] == 0 and ex.first_match_upper[1] >= 0
    assert ex.first_match_lower[2] == -1 and ex.first_match_upper[2] == -1
    with pytest.raises(ValueError):
        P.classify(batch, lower, upper, n_states=3)  # states out of range


@pytest.mark.parametrize("seed", range(6))
def test_classify_random_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    n, m = int(rng.integers(1, 40)), int(rng.integers(2, 6))
    h = int(rng.integers(1, 3000))
    samples = rng.integers(0, m, size=(h, n))
    lower = np.clip(samples[rng.integers(0, h, 30)] + rng.integers(0, 2, (30, n)), 0, m - 1)
    upper = np.clip(samples[rng.integers(0, h, 30)] - rng.integers(0, 2, (30, n)), 0, m - 1)
    want = oracle.classify_labels(samples, lower, upper, m)
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower, trusted=True)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True)
    for method in ("tc", "tc8", "bits"):
        r = P.classify(P.SampleBatch(samples, 0, 0), lo, up, n_states=m, method=method)
        assert np.array_equal(r.labels_device.cpu().numpy(), want["labels"])


@pytest.mark.parametrize("method", ["tc", "tc8"])
@pytest.mark.parametrize("chunk_tiles", ["1", "256"])
def test_explain_first_match_tensor_core_chunked(chunk_tiles, method, monkeypatch):
    # first-match indices from the tensor-core epilogue, also across chunked launches
    monkeypatch.setenv("RSR_TC_CHUNK_TILES", chunk_tiles)
    rng = np.random.default_rng(9)
    n, m, h = 60, 3, 3000
    samples = rng.integers(0, m, size=(h, n))
    lower = np.clip(samples[rng.integers(0, h, 700)] + rng.integers(0, 2, (700, n)), 0, m - 1)
    upper = np.clip(samples[rng.integers(0, h, 900)] - rng.integers(0, 2, (900, n)), 0, m - 1)
    want = oracle.classify_labels(samples, lower, upper, m, want_first=True)
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower, trusted=True)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True)
    r = P.classify(P.SampleBatch(samples, 0, 0), lo, up, n_states=m, explain=True, method=method)
    assert np.array_equal(r.labels_device.cpu().numpy(), want["labels"])
    assert np.array_equal(r.first_match_lower, want["first_lower"])
    assert np.array_equal(r.first_match_upper, want["first_upper"])


@pytest.mark.parametrize("n,m", [(300, 4), (400, 4), (700, 3), (800, 3)])
def test_classify_wide_rows_vs_oracle(n, m):
    # wide rows: N(M-1) = 900 / 1200 / 1400 run the FP4 tensor-core kernel as one-sided
    # launches per side; 1600 is past its limit (bit-packed CUDA-core path)
    rng = np.random.default_rng(n * m)
    h = 700
    samples = rng.integers(0, m, size=(h, n))
    lower = np.clip(samples[rng.integers(0, h, 25)] + rng.integers(0, 2, (25, n)), 0, m - 1)
    upper = np.clip(samples[rng.integers(0, h, 25)] - rng.integers(0, 2, (25, n)), 0, m - 1)
    want = oracle.classify_labels(samples, lower, upper, m, want_first=True)
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower, trusted=True)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True)
    r = P.classify(P.SampleBatch(samples, 0, 0), lo, up, n_states=m, explain=True)
    assert np.array_equal(r.labels_device.cpu().numpy(), want["labels"])
    assert np.array_equal(r.first_match_lower, want["first_lower"])
    assert np.array_equal(r.first_match_upper, want["first_upper"])


def _cfg2_sets(mixed, k=10_000, seed=0):
    from paper_2604_17066_b200 import workloads as W
    lower, upper = (W.cfg2_mixed_refs if mixed else W.cfg2_refs)(seed, 295, k, k)
    return (P.ReferenceSet.from_array(P.Side.LOWER, 0, lower, trusted=True),
            P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True), lower, upper)


@pytest.mark.parametrize("mixed", [False, True])
def test_cfg2_full_size_tc_equals_bits_and_slice_equals_oracle(mixed):
    p1 = 0.5 if mixed else 0.9
    d = P.ComponentDistribution.iid(295, [1 - p1, p1])
    lo, up, lower, upper = _cfg2_sets(mixed)
    b = P.sample_batch(d, 1 << 20, seed=0)
    tc = P.classify(b, lo, up, n_states=2, method="tc")
    tc8 = P.classify(b, lo, up, n_states=2, method="tc8")
    bits = P.classify(b, lo, up, n_states=2, method="bits")
    assert torch.equal(tc.labels_device, bits.labels_device)
    assert torch.equal(tc8.labels_device, bits.labels_device)
    assert tc.counts == bits.counts and sum(tc.counts) == 1 << 20
    if mixed:
        assert min(tc.counts) > 10_000  # all three labels are exercised
    # oracle on a bounded slice of the same samples
    sl = slice(123_456, 123_456 + 2048)
    want = oracle.classify_labels(b.device_states()[sl].cpu().numpy(), lower, upper, 2, n_workers=8)
    assert np.array_equal(tc.labels_device[sl].cpu().numpy(), want["labels"])


def test_reference_set_insert_examples_and_quadratic_oracle():
    s = _set(P.Side.LOWER, 0, [(1, 2)])
    assert s.insert(P.ReferenceState((3, 1), P.Side.LOWER, 0)) == "inserted"
    assert sorted(s.members) == [(1, 2), (3, 1)]
    s2 = _set(P.Side.LOWER, 0, [(3, 1)])
    assert s2.insert(P.ReferenceState((2, 1), P.Side.LOWER, 0)) == "redundant"
    s3 = _set(P.Side.LOWER, 0, [(2, 0), (0, 2)])
    assert s3.insert(P.ReferenceState((2, 2), P.Side.LOWER, 0)) == "inserted"
    assert s3.members == [(2, 2)]
    assert _set(P.Side.UPPER, 0, [(1, 1)]).insert(P.ReferenceState((1, 1), P.Side.UPPER, 0)) == "redundant"
    with pytest.raises(ValueError):
        P.ReferenceSet(P.Side.LOWER, 0).insert(P.ReferenceState((0, 0), P.Side.UPPER, 0))
    rng = np.random.default_rng(4)
    for trial in range(30):
        n, m = int(rng.integers(1, 7)), int(rng.integers(2, 5))
        for side in (P.Side.LOWER, P.Side.UPPER):
            vecs = [tuple(int(v) for v in rng.integers(0, m, size=n)) for _ in range(20)]
            dev = P.ReferenceSet(side, 0)
            ref = oracle.RefSet(side, 0)
            for v in vecs:
                assert dev.insert(P.ReferenceState(v, side, 0)) == ref.insert(v)
            assert dev.members == ref.members
            # batched insertion gives the same ordered list
            bat = P.ReferenceSet.from_array(side, 0, np.array(vecs))
            assert bat.members == ref.members


# ------------------------------------------------------------ Phi / search

def test_boundary_golden():
    for rec in load_json("boundary.json"):
        if rec["model"] == "fig_space":
            model = P.SystemModel(2, 5, 2, P.cone_sum([[(1, 4), (4, 0), (3, 2)]], 2))
        else:
            model = P.SystemModel(rec["n"], rec["m"], rec["ms"], P.cone_sum(rec["levels"], rec["n"]))
        model.reset_evaluation_count()
        r = P.boundary_search(model, rec["x0"], rec["threshold"])
        assert list(r.vector) == rec["vector"] and r.side == rec["side"]
        assert model.evaluation_count == rec["evals"]


def test_phi_kinds_vs_oracle():
    from paper_2604_17066_b200 import workloads as W
    g3 = W.cfg3(0)
    graph = P.Graph(g3["n_nodes"], tuple(g3["edges"]))
    s, t = g3["source"], g3["target"]
    rng = np.random.default_rng(0)
    xs2 = (rng.random((3000, graph.n_edges)) < 0.8).astype(np.int64)
    xs3 = rng.integers(0, 3, size=(3000, graph.n_edges))
    cases = [
        (P.single_od_connectivity(graph, s, t), oracle.phi_st(graph.n_nodes, graph.edges, s, t), xs2, 2),
        (P.global_connectivity(graph), oracle.phi_global(graph.n_nodes, graph.edges), xs2, 2),
        (P.widest_path_level(graph, s, t), oracle.phi_widest(graph.n_nodes, graph.edges, s, t, 3), xs3, 3),
        (P.k_out_of_n(40, graph.n_edges), oracle.phi_kofn(40, graph.n_edges), xs3, 3),
    ]
    for dev_phi, ref_phi, xs, m in cases:
        got = dev_phi.evaluate_device(xs, m)
        want = np.array([ref_phi(x) for x in xs])
        assert np.array_equal(got, want), dev_phi


# ----------------------------------------------------------------- workflow

_WORKFLOW_CASES = [("workflow.json", c["spec"]["name"]) for c in load_json("workflow.json")] + [
    ("cfg1_full.json", "cfg1_full")]  # BASELINE config 1 end to end (10^5 samples, 468 iterations)


@pytest.mark.parametrize("fname,case", _WORKFLOW_CASES)
@pytest.mark.parametrize("two_pass", [False, True])
def test_workflow_golden(fname, case, two_pass, monkeypatch):
    # two_pass: the Stage-1 loop's split classification (first 16 upper rows over
    # the batch, the rest over the samples still without a hit) from the first
    # iteration with more than 16 upper references
    if two_pass:
        monkeypatch.setenv("RSR_LOOP_PASS1_ROWS", "16")
        monkeypatch.setenv("RSR_LOOP_PASS2_MIN", "0")
    rec = next(c for c in load_json(fname) if c["spec"]["name"] == case)
    spec = rec["spec"]
    model = device_model(spec["model"])
    dist = P.ComponentDistribution(np.array(spec["probs"]))
    cfg = P.RunConfig(**spec["config"])
    for st in rec["stages"]:
        thr = st["threshold"]
        s1 = P.stage1_find_references(model, dist, cfg, thr)
        want = st["stage1"]
        assert [list(v) for v in s1.lower.members] == want["lower"]
        assert [list(v) for v in s1.upper.members] == want["upper"]
        got_trace = [[t.reference_count, t.phi_evaluations, t.p_lower, t.p_upper, t.p_unclassified]
                     for t in s1.trace]
        assert got_trace == want["trace"]
        assert (s1.iterations, s1.redundant_searches, s1.terminated_by) == (
            want["iterations"], want["redundant_searches"], want["terminated_by"])
        assert model.evaluation_count == want["phi_total"]
        rep = P.stage2_evaluate(model, dist, s1.lower, s1.upper, cfg, thr)
        w2 = st["stage2"]
        for k in ("p_lower", "p_upper", "cov_lower", "cov_upper", "n_samples",
                  "unclassified_resolved"):
            assert getattr(rep, k) == w2[k], k
        assert model.evaluation_count == w2["phi_total"]


def test_stage2_empty_sets_match_crude_mc():
    model = device_model({"kind": "kofn", "k": 3, "n": 3, "m": 2, "ms": 2})
    dist = P.ComponentDistribution.iid(3, [0.1, 0.9])
    cfg = P.RunConfig(n_samples=2000, eps_u=1e-3, r_max=50, seed=7)
    rep = P.stage2_evaluate(model, dist, None, None, cfg, 0)
    ev = oracle.CountingPhi(oracle.phi_kofn(3, 3), 3, 2, 2)
    want = oracle.stage2(ev, dist.probs, [], [], 0, 2000, 7)
    assert rep.p_lower == want["p_lower"] and rep.cov_lower == want["cov_lower"]
    assert rep.unclassified_resolved == 2000


def test_multistate_pmf_golden():
    g = load_json("pmf.json")
    model = P.SystemModel(3, 3, 3, P.k_out_of_n(2, 3))
    dist = P.ComponentDistribution.iid(3, [0.2, 0.3, 0.5])
    rep = P.multistate_pmf(model, dist, P.RunConfig(n_samples=40_000, eps_u=1e-3, r_max=200, seed=11))
    assert rep.pmf.tolist() == g["pmf"]
    assert rep.cumulative_lower.tolist() == g["cumulative_lower"]
    assert rep.max_chain_discrepancy == g["max_chain_discrepancy"]


@pytest.mark.parametrize("n,m,s", [(295, 2, 5000), (40, 3, 3000), (7, 5, 700)])
def test_classify_host_paths_match(n, m, s):
    # host-fed streaming paths (u8 states, reference packed one-hot rows, int8 variant)
    # give the same labels as the device batch path and the oracle
    from paper_2604_17066_b200.classify import classify_host, classify_host_encoded
    rng = np.random.default_rng(n + m)
    samples = rng.integers(0, m, size=(s, n))
    lower = np.clip(samples[rng.integers(0, s, 300)] + rng.integers(0, 2, (300, n)), 0, m - 1)
    upper = np.clip(samples[rng.integers(0, s, 200)] - rng.integers(0, 2, (200, n)), 0, m - 1)
    want = oracle.classify_labels(samples, lower, upper, m)["labels"]
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower, trusted=True)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True)
    u8 = samples.astype(np.uint8)
    lab, counts = classify_host(u8, lo, up, m, chunk_rows=1024)
    assert np.array_equal(lab.numpy(), want)
    assert counts == (int((want == 0).sum()), int((want == 1).sum()), int((want == 2).sum()))
    lab8, _ = classify_host(u8, lo, up, m, chunk_rows=777, method="tc8")
    assert np.array_equal(lab8.numpy(), want)
    packed = np.packbits(oracle.encode(samples, m, "sample"), axis=1)
    labp, countsp = classify_host_encoded(packed, n, lo, up, m, chunk_rows=1000)
    assert np.array_equal(labp.numpy(), want) and countsp == counts


@pytest.mark.parametrize("cache", ["1", "0", "partial"])
def test_multistate_pmf_batch_cache(cache, monkeypatch):
    """multistate_pmf keeps the drawn batches in HBM between thresholds (their picks
    decoded from the FP4 rows); every threshold's Stage 1 equals the golden run, also
    when only the first generations fit the cache."""
    monkeypatch.setenv("RSR_BATCH_CACHE", "0" if cache == "0" else "1")
    if cache == "partial":
        monkeypatch.setenv("RSR_BATCH_CACHE_MAX", "3")
    rec = next(c for c in load_json("workflow.json") if c["spec"]["name"] == "grid_widest_m3")
    spec = rec["spec"]
    model = device_model(spec["model"])
    dist = P.ComponentDistribution(np.array(spec["probs"]))
    cfg = P.RunConfig(**spec["config"])
    rep = P.multistate_pmf(model, dist, cfg)
    assert len(rep.stage1_results) == len(rec["stages"])
    for s1, st in zip(rep.stage1_results, rec["stages"]):
        want = st["stage1"]
        assert [list(v) for v in s1.lower.members] == want["lower"]
        assert [list(v) for v in s1.upper.members] == want["upper"]
        assert [[t.reference_count, t.phi_evaluations, t.p_lower, t.p_upper, t.p_unclassified]
                for t in s1.trace] == want["trace"]
    for r, st in zip(rep.stage2_reports, rec["stages"]):
        assert r.p_lower == st["stage2"]["p_lower"]
