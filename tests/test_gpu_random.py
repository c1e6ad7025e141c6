"""Randomised parity sweeps: device path vs the CPU oracle, bit-exact.

The oracle is pinned to the reference by tests/test_oracle_golden.py; here
random coherent systems (the reference suite's cone-sum construction,
tests/conftest.py:53-75), random distributions and random classifier shapes
exercise the device path far beyond the fixed golden cases.
"""

import numpy as np
import pytest

import oracle
import paper_2604_17066_b200 as P

pytestmark = pytest.mark.gpu


def _random_system(rng):
    n, m, ms = int(rng.integers(2, 9)), int(rng.integers(2, 5)), int(rng.integers(2, 4))
    levels = [[[int(v) for v in rng.integers(0, m, size=n)] for _ in range(int(rng.integers(1, 4)))]
              for _ in range(ms - 1)]
    raw = rng.random((n, m)) + 0.05
    probs = raw / raw.sum(1, keepdims=True)
    return n, m, ms, levels, probs


@pytest.mark.parametrize("loop", ["async", "sync"])
@pytest.mark.parametrize("seed", range(16))
def test_random_cone_systems_workflow(seed, loop, monkeypatch):
    # "async": device-resident reference sets (csrc/refset.cu, one host sync per
    # iteration); "sync": the host-resolved insertion path.  Seeds >= 12 search
    # wide batches without boundary search, where raw samples as references make
    # candidates redundant and drop members within and across batches.
    monkeypatch.setenv("RSR_SYNC_LOOP", "1" if loop == "sync" else "0")
    rng = np.random.default_rng(1000 + seed)
    n, m, ms, levels, probs = _random_system(rng)
    cfg = dict(n_samples=int(rng.integers(500, 4000)), eps_u=float(rng.choice([1e-2, 1e-3])),
               r_max=int(rng.integers(5, 200)), seed=int(rng.integers(0, 2**31)),
               parallel_searches=int(rng.integers(1, 9)),
               boundary_search_enabled=bool(rng.random() < 0.85))
    if seed >= 12:
        cfg.update(parallel_searches=int(rng.integers(16, 80)), boundary_search_enabled=False,
                   r_max=int(rng.integers(50, 400)))
    model = P.SystemModel(n, m, ms, P.cone_sum(levels, n))
    dist = P.ComponentDistribution(probs)
    ev = oracle.CountingPhi(oracle.phi_cones(levels), n, m, ms)
    for thr in range(ms - 1):
        s1 = P.stage1_find_references(model, dist, P.RunConfig(**cfg), thr)
        o1 = oracle.stage1(ev, probs, thr, **cfg)
        assert s1.lower.members == o1["lower"] and s1.upper.members == o1["upper"]
        assert [[t.reference_count, t.phi_evaluations, t.p_lower, t.p_upper, t.p_unclassified]
                for t in s1.trace] == [[t["reference_count"], t["phi_evaluations"], t["p_lower"],
                                        t["p_upper"], t["p_unclassified"]] for t in o1["trace"]]
        assert (s1.iterations, s1.redundant_searches, s1.terminated_by) == (
            o1["iterations"], o1["redundant_searches"], o1["terminated_by"])
        rep = P.stage2_evaluate(model, dist, s1.lower, s1.upper, P.RunConfig(**cfg), thr)
        o2 = oracle.stage2(ev, probs, o1["lower"], o1["upper"], thr, cfg["n_samples"], cfg["seed"])
        assert (rep.p_lower, rep.p_upper, rep.unclassified_resolved) == (
            o2["p_lower"], o2["p_upper"], o2["unclassified_resolved"])
        assert model.evaluation_count == ev.count


@pytest.mark.parametrize("seed", range(10))
def test_random_classifier_shapes(seed):
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.choice([1, 2, 7, 31, 33, 64, 100, 127, 128, 129, 295, 380]))
    m = int(rng.integers(2, 4)) if n > 200 else int(rng.integers(2, 6))
    h = int(rng.choice([1, 2, 255, 256, 257, 511, 1000, 3333]))
    kl, ku = int(rng.choice([0, 1, 255, 256, 257, 600])), int(rng.choice([0, 1, 255, 256, 257, 600]))
    samples = rng.integers(0, m, size=(h, n))
    base_l = samples[rng.integers(0, h, kl)] if kl else np.zeros((0, n), dtype=np.int64)
    base_u = samples[rng.integers(0, h, ku)] if ku else np.zeros((0, n), dtype=np.int64)
    lower = np.clip(base_l + rng.integers(0, 2, base_l.shape), 0, m - 1)
    upper = np.clip(base_u - rng.integers(0, 2, base_u.shape), 0, m - 1)
    want = oracle.classify_labels(samples, lower, upper, m)["labels"]
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lower, trusted=True)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, upper, trusted=True)
    batch = P.SampleBatch(samples, 0, 0)
    for method in ("tc", "tc8", "bits"):
        r = P.classify(batch, lo, up, n_states=m, method=method)
        assert np.array_equal(r.labels_device.cpu().numpy(), want), (method, n, m, h, kl, ku)
        assert r.counts == (int((want == 0).sum()), int((want == 1).sum()), int((want == 2).sum()))
        assert np.array_equal(r.unclassified_indices, np.flatnonzero(want == 2))


@pytest.mark.parametrize("seed", range(4))
def test_edge_disjoint_level_vs_oracle(seed):
    rng = np.random.default_rng(300 + seed)
    if seed == 0:  # multigraph (parallel edges add capacity)
        graph = P.Graph(5, ((0, 1), (0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (1, 3), (2, 4)))
    else:
        graph = P.random_geometric_graph(int(rng.integers(8, 16)), 0.5, seed=seed)
    for max_level in (1, 2, 3):
        phi = P.edge_disjoint_level(graph, max_level)
        ref = oracle.phi_edge_disjoint(graph.n_nodes, graph.edges, max_level)
        xs = (rng.random((300, graph.n_edges)) < 0.85).astype(np.int64)
        got = phi.evaluate_device(xs, 2)
        assert np.array_equal(got, np.array([ref(x) for x in xs]))
        model = P.SystemModel(graph.n_edges, 2, max_level + 1, phi)
        for thr in range(max_level):
            for x0 in xs[:4]:
                ev = oracle.CountingPhi(ref, graph.n_edges, 2, max_level + 1)
                vec, side = oracle.boundary_search(ev, x0, thr)
                model.reset_evaluation_count()
                r = P.boundary_search(model, x0, thr)
                assert r.vector == vec and r.side == side
                assert model.evaluation_count == ev.count


def test_sampling_random_tables_and_offsets():
    rng = np.random.default_rng(7)
    for _ in range(8):
        n, m = int(rng.integers(1, 60)), int(rng.integers(2, 7))
        raw = rng.random((n, m)) ** 3
        raw[rng.random((n, m)) < 0.2] = 0.0
        raw[:, 0] += 1e-3
        probs = raw / raw.sum(1, keepdims=True)
        count, start = int(rng.integers(1, 3000)), int(rng.integers(0, 10**6))
        seed, gen = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**40))
        b = P.sample_batch(P.ComponentDistribution(probs), count, seed, gen, start)
        assert np.array_equal(b.states, oracle.sample_states(probs, count, seed, gen, start))


@pytest.mark.parametrize("kind,m,p_hi", [("st", 2, 0.9), ("st", 2, 0.6), ("widest", 3, 0.8),
                                         ("widest", 4, 0.7)])
def test_boundary_graph_search_matches_bitset_walk(kind, m, p_hi, monkeypatch):
    """Union-find / witness-path boundary search (csrc/boundary_graph.cu) against the
    step-by-step bitset walk (csrc/phi_bits.cu) on 1024 random start vectors of the
    cfg3-shaped graph: identical references, sides and Phi-call counts; the oracle
    checks a slice."""
    import torch
    from paper_2604_17066_b200 import workloads as W
    g = W.cfg3(0)
    graph = P.Graph(g["n_nodes"], tuple(g["edges"]))
    phi = (P.single_od_connectivity(graph, g["source"], g["target"]) if kind == "st"
           else P.widest_path_level(graph, g["source"], g["target"]))
    ms = 2 if kind == "st" else m
    model = P.SystemModel(graph.n_edges, m, ms, phi)
    rng = np.random.default_rng(int(p_hi * 100) + m)
    lo = rng.random((1024, graph.n_edges))
    xs = np.where(lo < p_hi, m - 1, rng.integers(0, m, size=lo.shape)).astype(np.uint8)
    xd = torch.as_tensor(xs).cuda()
    ref = (oracle.phi_st(g["n_nodes"], g["edges"], g["source"], g["target"]) if kind == "st"
           else oracle.phi_widest(g["n_nodes"], g["edges"], g["source"], g["target"], m))
    for thr in range(ms - 1):
        out = {}
        for mode in ("1", "0"):
            monkeypatch.setenv("RSR_BOUNDARY_GRAPH", mode)
            r, sd, c = P.boundary_search_batch(model, xd, thr)
            out[mode] = (r.cpu().numpy(), sd.cpu().numpy(), c.cpu().numpy())
        for a, b in zip(out["1"], out["0"]):
            assert np.array_equal(a, b)
        assert 0 < int((out["1"][1] == 0).sum()) < 1024 or kind == "widest"
        for b in range(0, 1024, 97):
            ev = oracle.CountingPhi(ref, graph.n_edges, m, ms)
            vec, side = oracle.boundary_search(ev, xs[b].astype(np.int64), thr)
            assert tuple(out["1"][0][b].tolist()) == vec and int(out["1"][2][b]) == ev.count


@pytest.mark.parametrize("cfg_name", ["cfg3", "cfg5"])
def test_loop_paths_agree_on_config_graphs(cfg_name, monkeypatch):
    """Stage 1 on the BASELINE config 3 / 5 graphs at a reduced batch size: the
    one-sync loop (device reference sets, two-pass classification with the default
    480-row first pass) and the host-resolved loop give identical ordered sets,
    traces, redundant-search and Phi counts; the oracle checks the first iterations."""
    import torch  # noqa: F401
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from _specs import device_model
    from paper_2604_17066_b200 import workloads as W
    g = W.cfg3(0) if cfg_name == "cfg3" else W.cfg5(0)
    m = 2 if cfg_name == "cfg3" else 3
    spec = {"kind": "st" if m == 2 else "widest", "n_nodes": g["n_nodes"], "edges": g["edges"],
            "s": g["source"], "t": g["target"], "m": m, "ms": m}
    dist = P.ComponentDistribution(g["probs"])
    cfg = P.RunConfig(n_samples=1 << 14, eps_u=1e-5, r_max=1500, seed=3, parallel_searches=64)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("RSR_SYNC_LOOP", mode)
        model = device_model(spec)
        s1 = P.stage1_find_references(model, dist, cfg, 0)
        out[mode] = (s1.lower.members, s1.upper.members,
                     [(t.reference_count, t.phi_evaluations, t.p_lower, t.p_upper,
                       t.p_unclassified) for t in s1.trace],
                     s1.iterations, s1.redundant_searches, s1.terminated_by,
                     model.evaluation_count)
    assert out["0"] == out["1"]
    assert len(out["0"][1]) > 960  # the two-pass split was active
    from _specs import oracle_phi
    phi, n = oracle_phi(spec)
    ev = oracle.CountingPhi(phi, n, m, m)
    o1 = oracle.stage1(ev, g["probs"], 0, 1 << 14, eps_u=1e-5, r_max=100, seed=3,
                       parallel_searches=64, fast=True)
    k = len(o1["trace"])
    assert [(t["reference_count"], t["phi_evaluations"], t["p_lower"], t["p_upper"],
             t["p_unclassified"]) for t in o1["trace"]] == out["0"][2][:k]


def test_wide_row_system_workflow_vs_oracle():
    """A system too wide for the FP4 / int8 tensor-core rows (N(M-1) = 900 > 831): the
    Stage-1 loop falls back to the host-resolved path and the bit-packed classifier;
    results equal the oracle's."""
    n, k = 900, 890
    model = P.SystemModel(n, 2, 2, P.k_out_of_n(k, n))
    probs = np.tile([0.01, 0.99], (n, 1))
    dist = P.ComponentDistribution(probs)
    cfg = dict(n_samples=3000, eps_u=1e-3, r_max=40, seed=5, parallel_searches=4)
    s1 = P.stage1_find_references(model, dist, P.RunConfig(**cfg), 0)
    ev = oracle.CountingPhi(oracle.phi_kofn(k, n), n, 2, 2)
    o1 = oracle.stage1(ev, probs, 0, **cfg)
    assert s1.lower.members == o1["lower"] and s1.upper.members == o1["upper"]
    assert [[t.reference_count, t.phi_evaluations, t.p_lower, t.p_upper, t.p_unclassified]
            for t in s1.trace] == [[t["reference_count"], t["phi_evaluations"], t["p_lower"],
                                    t["p_upper"], t["p_unclassified"]] for t in o1["trace"]]
    assert model.evaluation_count == ev.count
