"""Host-side logic that needs no GPU: validation, estimates, bookkeeping, generators."""

import numpy as np
import pytest
import torch

import paper_2604_17066_b200 as P
from paper_2604_17066_b200 import workloads as W
from paper_2604_17066_b200.dist import global_pick_owners, shard_range


def test_run_config_validation():
    with pytest.raises(ValueError):
        P.RunConfig(n_samples=0)
    with pytest.raises(ValueError):
        P.RunConfig(eps_u=1.5)
    with pytest.raises(ValueError):
        P.RunConfig(r_max=0)
    with pytest.raises(ValueError):
        P.RunConfig(parallel_searches=0)


def test_cov_and_assemble_pmf():
    assert P.cov(1.0, 100) == 0.0
    assert P.cov(0.5, 100) == pytest.approx(0.1)
    assert P.cov(0.01, 1_000_000) == pytest.approx(0.0099498743710662, rel=1e-12)
    assert P.cov(0.0, 100) is None
    with pytest.raises(ValueError):
        P.cov(1.5, 100)
    with pytest.raises(ValueError):
        P.cov(0.5, 0)
    pmf, adj = P.assemble_pmf([0.3, 0.2999])
    assert np.all(pmf >= 0) and pmf.sum() == pytest.approx(1.0)
    assert adj == pytest.approx(0.0001, abs=1e-12)
    with pytest.raises(ValueError):
        P.assemble_pmf([-0.1])


def test_distribution_and_model_validation():
    with pytest.raises(ValueError):
        P.ComponentDistribution(np.array([[0.5, 0.4]]))
    with pytest.raises(ValueError):
        P.ComponentDistribution(np.array([0.5, 0.5]))
    d = P.ComponentDistribution.iid(3, [0.2, 0.8])
    assert d.n_components == 3 and d.n_states == 2
    with pytest.raises(ValueError):
        P.SystemModel(0, 2, 2, P.k_out_of_n(1, 1))
    with pytest.raises(ValueError):
        P.SystemModel(3, 1, 2, P.k_out_of_n(1, 3))
    with pytest.raises(ValueError):
        P.k_out_of_n(4, 3)
    m = P.SystemModel(3, 2, 2, lambda x: int(x.sum() == 3))
    with pytest.raises(TypeError, match="device-described"):
        m.device_phi()
    assert m.evaluate([1, 1, 1]) == 1 and m.evaluation_count == 1


def test_reference_state_and_set_validation():
    with pytest.raises(ValueError):
        P.ReferenceState((0, 1), "sideways", 0)
    with pytest.raises(ValueError):
        P.ReferenceSet("sideways", 0)
    s = P.ReferenceSet(P.Side.LOWER, 0)
    with pytest.raises(ValueError):
        s.insert(P.ReferenceState((0, 0), P.Side.UPPER, 0))
    with pytest.raises(ValueError):
        s.insert(P.ReferenceState((0, 0), P.Side.LOWER, 1))
    # first insertion into an empty set is pure bookkeeping (no device work)
    assert s.insert(P.ReferenceState((1, 0), P.Side.LOWER, 0)) == "inserted"
    assert s.members == [(1, 0)] and (1, 0) in s and len(s) == 1
    t = P.ReferenceSet.from_array(P.Side.UPPER, 0, np.array([[1, 0], [0, 1]]), trusted=True)
    assert t.members == [(1, 0), (0, 1)] and t.copy().members == t.members


def test_graph_utilities_match_reference_semantics():
    with pytest.raises(ValueError):
        P.Graph(2, ((0, 0),))
    g = P.random_geometric_graph(30, 0.35, seed=0)
    o, d = P.pick_od_pair(g)
    assert 0 <= o < g.n_nodes and 0 <= d < g.n_nodes and o != d
    with pytest.raises(ValueError):
        P.edge_disjoint_level(g, 0)
    assert P.edge_disjoint_level(g, 2).k == 2


def test_graph_utilities_vs_reference(reference_rsr):
    from rsr import sysfn
    for seed in range(3):
        a = P.random_geometric_graph(30, 0.35, seed=seed)
        b = sysfn.random_geometric_graph(30, 0.35, seed=seed)
        assert a.edges == b.edges and a.n_nodes == b.n_nodes
        assert P.pick_od_pair(a) == sysfn.pick_od_pair(b)


def test_workload_generators_are_deterministic():
    g1 = W.cfg1(0)
    assert g1["n_nodes"] == 25 and len(g1["edges"]) == 40
    assert np.all((g1["probs"][:, 0] >= 0.05) & (g1["probs"][:, 0] <= 0.15))
    g3 = W.cfg3(0)
    assert g3["n_nodes"] == 119 and len(g3["edges"]) == 295
    assert W.cfg3(0)["edges"] == g3["edges"]
    lo, up = W.cfg2_refs(0, 295, k_upper=400, k_lower=500)
    assert lo.shape == (500, 295) and up.shape == (400, 295)
    assert np.all((lo == 0).sum(1) == 10) and np.all(up.sum(1) == 15)
    g5 = W.cfg5(0)
    assert g5["probs"].shape == (295, 3) and np.allclose(g5["probs"].sum(1), 1.0)


def test_random_st_paths_are_distinct_simple_paths():
    g = W.cfg3(0)
    paths = W.random_st_paths(g, 200, seed=0, batch=256)
    assert len({p.tobytes() for p in paths}) == paths.shape[0] == 200
    import oracle
    phi = oracle.phi_st(g["n_nodes"], g["edges"], g["source"], g["target"])
    for p in paths[:50]:
        assert phi(p) == 1
        for e in np.flatnonzero(p)[:3]:  # minimal: removing any edge disconnects
            q = p.copy()
            q[e] = 0
            assert phi(q) == 0


def test_shard_ranges_cover_exactly():
    for n in (1, 7, 1 << 20, 1_000_003):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, w, r) for r in range(w)]
            assert parts[0][0] == 0
            assert all(a[0] + a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert parts[-1][0] + parts[-1][1] == n


def test_global_pick_owner_mapping():
    per = np.array([3, 0, 5, 2])
    owner, local = global_pick_owners(per, np.arange(10))
    assert owner.tolist() == [0, 0, 0, 2, 2, 2, 2, 2, 3, 3]
    assert local.tolist() == [0, 1, 2, 0, 1, 2, 3, 4, 0, 1]


@pytest.mark.parametrize("u", [1, 3, 5, 100, 20_000, 1_000_000])
def test_choice_positions_equal_choice_of_indices(u):
    # workflow.py:172-174 picks from the index array; the device path picks positions
    rng = np.random.default_rng(u)
    idx = np.sort(rng.choice(10 * u, size=u, replace=False))
    for it in range(3):
        k = min(64, u)
        a = np.random.default_rng([7, it]).choice(idx, size=k, replace=False)
        b = idx[np.random.default_rng([7, it]).choice(u, size=k, replace=False)]
        assert np.array_equal(a, b)


def test_device_calls_fail_loudly_without_cuda():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.sample_batch(P.ComponentDistribution.iid(3, [0.5, 0.5]), 10, seed=0)


@pytest.mark.timeout(180)
def _bench(args, env_extra=None, timeout=240):
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py")] + args, cwd=root, env=env,
                       capture_output=True, text=True, timeout=timeout)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    return r, lines


def test_bench_reference_arm_runs_on_cpu():
    """`bench.py --impl reference` (the driver's reference arm: the reference's own
    classification on the host cores) prints one well-formed JSON line."""
    r, lines = _bench(["--impl", "reference", "--config", "cfg2", "--steps", "1", "--warmup", "1",
                       "--cpu-seconds", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = lines[-1]
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "pairs/s"
    assert line["e2e"]["value"] == line["value"] and line["cpu_baseline"]["cores"] >= 1
    assert line["config"]["ref_states"] == 20_000
    assert line["cpu_baseline"]["kind"] in ("reference", "port")


def test_bench_gpus_flag_relaunches_under_torchrun():
    """`python bench.py --gpus 2` without torchrun runs two ranks (the reference arm:
    rank 0 prints, rank 1 exits without work); a WORLD_SIZE that disagrees with
    --gpus fails loudly instead of measuring another world size."""
    r, lines = _bench(["--impl", "reference", "--gpus", "2", "--config", "cfg4", "--k", "300",
                       "--steps", "1", "--warmup", "1", "--cpu-seconds", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert "launching 2 ranks" in r.stderr
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["config"]["ref_states"] == 300
    r, lines = _bench(["--impl", "reference", "--gpus", "2", "--steps", "1"],
                      env_extra={"WORLD_SIZE": "1"})
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr and not lines


def _msf_upper_walk(n_nodes, edges, s, t, x, L):
    """Closed form of the reference's upper-side boundary walk (boundary.py:116-147) used by
    csrc/boundary_graph.cu: keep the s-t path of the maximum spanning forest (weight =
    component index) of G_L = {e : x_e >= L}; path edges stop at L after x_e - L + 1 Phi
    calls, every other component drops to 0 after x_e calls."""
    par = list(range(n_nodes))

    def find(a):
        while par[a] != a:
            par[a] = par[par[a]]
            a = par[a]
        return a
    tree = [[] for _ in range(n_nodes)]
    for e in range(len(edges) - 1, -1, -1):
        if x[e] < L:
            continue
        u, v = edges[e]
        a, b = find(u), find(v)
        if a == b:
            continue
        par[a] = b
        tree[u].append((v, e))
        tree[v].append((u, e))
        if find(s) == find(t):
            break
    prev = {s: None}
    stack = [s]
    while stack:
        u = stack.pop()
        for v, e in tree[u]:
            if v not in prev:
                prev[v] = (u, e)
                stack.append(v)
    path = set()
    node = t
    while prev[node] is not None:
        node, e = prev[node]
        path.add(e)
    out, calls = [], 1
    for e, xe in enumerate(x):
        if xe >= L and e in path:
            out.append(L)
            calls += xe - L + 1
        else:
            out.append(0)
            calls += xe
    return tuple(out), calls


@pytest.mark.parametrize("seed", range(12))
def test_upper_boundary_walk_is_max_spanning_forest_path(seed):
    """The closed form the device's upper-side boundary search uses equals the reference
    walk (oracle restatement) on random graphs, states and thresholds: same reference
    state, same Phi-call count."""
    import oracle
    rng = np.random.default_rng(seed)
    n_nodes = int(rng.integers(6, 30))
    pairs = [(i, j) for i in range(n_nodes) for j in range(i + 1, n_nodes)]
    k = min(len(pairs), int(rng.integers(n_nodes, 3 * n_nodes)))
    edges = [pairs[i] for i in rng.choice(len(pairs), size=k, replace=False)]
    s, t = 0, n_nodes - 1
    m = int(rng.integers(2, 5))
    kinds = [("st", oracle.phi_st(n_nodes, edges, s, t), 2, 2)]
    kinds.append(("widest", oracle.phi_widest(n_nodes, edges, s, t, m), m, m))
    checked = 0
    for name, phi, mm, ms in kinds:
        for trial in range(40):
            x = rng.integers(0, mm, size=len(edges))
            x[rng.random(len(edges)) < 0.6] = mm - 1
            for thr in range(ms - 1):
                ev = oracle.CountingPhi(phi, len(edges), mm, ms)
                if ev(x) <= thr:
                    continue  # lower side: union-find walk (no closed form needed)
                ev.count = 0
                vec, side = oracle.boundary_search(ev, x, thr)
                assert side == oracle.UPPER
                got, calls = _msf_upper_walk(n_nodes, edges, s, t, [int(v) for v in x], thr + 1)
                assert got == vec and calls == ev.count, (name, thr, trial)
                checked += 1
    assert checked > 10


@pytest.mark.parametrize("m", [2, 3])
def test_support_compaction_preserves_violation_counts(m):
    """The identity behind the FP4 support compaction (csrc/fp4_compact.cu): dropping the
    thermometer columns no reference of a side uses leaves every violation count of that
    side unchanged (oracle.violation_counts, classify.py:57-96), so labels cannot change.
    Checked here on the oracle: components outside the references' support removed from
    samples and references alike."""
    import oracle
    rng = np.random.default_rng(m)
    n, h, k = 60, 300, 80
    x = rng.integers(0, m, size=(h, n))
    up = rng.integers(0, m, size=(k, n)) * (rng.random((k, n)) < 0.15)
    up[:, 10:25] = 0  # upper references never require these components
    lo = (m - 1) - rng.integers(0, m, size=(k, n)) * (rng.random((k, n)) < 0.15)
    lo[:, 40:] = m - 1  # lower references never fall below the top level here
    for refs, kind in ((up, "upper_ref"), (lo, "lower_ref")):
        keep = (refs > 0).any(0) if kind == "upper_ref" else (refs < m - 1).any(0)
        full = oracle.violation_counts(x, refs, m, kind)
        comp = oracle.violation_counts(x[:, keep], refs[:, keep], m, kind)
        assert not keep.all() and np.array_equal(full, comp)
