"""Differential checks of the oracle against the live reference (build container only)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.reference


@pytest.mark.parametrize("seed", range(8))
def test_sampling_and_classify_random(reference_rsr, seed):
    from rsr.boundary import ReferenceSet, Side
    from rsr.classify import classify
    from rsr.model import ComponentDistribution
    from rsr.sampling import sample_batch
    rng = np.random.default_rng(seed)
    n, m = int(rng.integers(1, 12)), int(rng.integers(2, 6))
    raw = rng.random((n, m)) + 0.02
    probs = raw / raw.sum(1, keepdims=True)
    h, gen, start = int(rng.integers(1, 400)), int(rng.integers(0, 50)), int(rng.integers(0, 99))
    b = sample_batch(ComponentDistribution(probs), h, seed, gen, start)
    xs = oracle.sample_states(probs, h, seed, gen, start)
    assert np.array_equal(b.states, xs)
    lower = np.clip(xs[rng.integers(0, h, 8)] + 1, 0, m - 1)
    upper = np.clip(xs[rng.integers(0, h, 8)] - 1, 0, m - 1)
    ls, us = ReferenceSet(Side.LOWER, 0), ReferenceSet(Side.UPPER, 0)
    ls._members = [tuple(int(v) for v in r) for r in lower]
    us._members = [tuple(int(v) for v in r) for r in upper]
    r = classify(b, ls, us, explain=True, n_states=m)
    o = oracle.classify_labels(xs, lower, upper, m, want_first=True)
    assert np.array_equal(r.lower_indices, o["lower_indices"])
    assert np.array_equal(r.upper_indices, o["upper_indices"])
    assert np.array_equal(r.first_match_lower, o["first_lower"])
    assert np.array_equal(r.first_match_upper, o["first_upper"])


@pytest.mark.parametrize("seed", range(4))
def test_rgg_st_stage1(reference_rsr, seed):
    from rsr.model import ComponentDistribution, SystemModel
    from rsr.sysfn import pick_od_pair, random_geometric_graph, single_od_connectivity
    from rsr.workflow import RunConfig, stage1_find_references
    g = random_geometric_graph(18, 0.4, seed=seed)
    s, t = pick_od_pair(g)
    model = SystemModel(g.n_edges, 2, 2, single_od_connectivity(g, s, t))
    dist = ComponentDistribution.iid(g.n_edges, [0.1, 0.9])
    cfg = RunConfig(n_samples=3000, eps_u=1e-3, r_max=300, seed=seed, parallel_searches=4)
    ref = stage1_find_references(model, dist, cfg, 0)
    ev = oracle.CountingPhi(oracle.phi_st(g.n_nodes, g.edges, s, t), g.n_edges, 2, 2)
    o = oracle.stage1(ev, dist.probs, 0, 3000, eps_u=1e-3, r_max=300, seed=seed,
                      parallel_searches=4)
    assert o["lower"] == ref.lower.members and o["upper"] == ref.upper.members
    assert o["iterations"] == ref.iterations and ev.count == model.evaluation_count


def test_model_api_matches_reference(reference_rsr):
    """SystemModel / ComponentDistribution / check_coherency behave as the reference's
    (model.py): same violations in the same order, same evaluation counts, same error
    messages."""
    import paper_2604_17066_b200 as P
    import rsr

    def phi(x):  # incoherent on purpose: component 0 helps, component 1 hurts
        return int(x[0] >= 1) if x[1] == 0 else 0

    for seed in range(3):
        mine = P.SystemModel(5, 3, 2, phi)
        ref = rsr.SystemModel(5, 3, 2, phi)
        a = P.check_coherency(mine, 40, seed)
        b = rsr.check_coherency(ref, 40, seed)
        assert len(a) == len(b) > 0
        assert all(np.array_equal(x, y) for p, q in zip(a, b) for x, y in zip(p, q))
        assert mine.evaluation_count == ref.evaluation_count == 80
    for args in ((0, 2, 2, phi), (3, 1, 2, phi), (3, 2, 1, phi)):
        with pytest.raises(ValueError) as e1:
            P.SystemModel(*args)
        with pytest.raises(ValueError) as e2:
            rsr.SystemModel(*args)
        assert str(e1.value) == str(e2.value)
    m1, m2 = P.SystemModel(3, 2, 2, phi), rsr.SystemModel(3, 2, 2, phi)
    for bad in ([0, 1], [0, 1, 2], [[0, 1, 1]]):
        with pytest.raises(ValueError) as e1:
            m1.evaluate(bad)
        with pytest.raises(ValueError) as e2:
            m2.evaluate(bad)
        assert str(e1.value) == str(e2.value)
    for probs in ([[0.5, 0.6]], [[1.5, -0.5]], [0.5, 0.5], [[0.3, 0.7], [0.2, 0.7]]):
        with pytest.raises(ValueError) as e1:
            P.ComponentDistribution(np.array(probs))
        with pytest.raises(ValueError) as e2:
            rsr.ComponentDistribution(np.array(probs))
        assert str(e1.value) == str(e2.value)
    d1 = P.ComponentDistribution.iid(4, [0.25, 0.75])
    d2 = rsr.ComponentDistribution.iid(4, [0.25, 0.75])
    assert np.array_equal(d1.probs, d2.probs) and (d1.n_components, d1.n_states) == (4, 2)
