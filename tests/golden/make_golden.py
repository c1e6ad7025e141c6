"""Generate golden vectors by running the REFERENCE package (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--full-cfg1]

Writes small fixtures next to this script.  They pin both the CPU oracle
(``oracle/``) and the device path on machines where the reference is absent
(the GPU box).  ``--full-cfg1`` additionally runs BASELINE config 1 end to end
(n_samples = 10^5, reference defaults; ~10 minutes single-threaded).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import rsr  # noqa: E402
from rsr import sampling as rs  # noqa: E402
from rsr.boundary import ReferenceSet, ReferenceState, Side, boundary_search  # noqa: E402
from rsr.classify import classify, violation_counts  # noqa: E402
from rsr.encoding import encode_batch  # noqa: E402
from rsr.model import ComponentDistribution, SystemModel  # noqa: E402
from rsr.sampling import SampleBatch, sample_batch  # noqa: E402
from rsr.sysfn import (Graph, edge_disjoint_level, k_out_of_n, random_geometric_graph,  # noqa: E402
                       single_od_connectivity)
from rsr.workflow import RunConfig, multistate_pmf, stage1_find_references, stage2_evaluate  # noqa: E402

from paper_2604_17066_b200 import workloads  # noqa: E402  (host-side generators only)


def _cone_phi(levels):
    """Cone-sum Phi (reference tests/conftest.py:53-75 shape) as a plain callable."""
    levels = [[tuple(int(v) for v in a) for a in lev] for lev in levels]

    def phi(x):
        s = 0
        for anchors in levels:
            if any(all(x[i] >= a[i] for i in range(len(a))) for a in anchors):
                s += 1
        return s
    return phi


def _widest_phi(graph: Graph, s: int, t: int, m: int):
    """Builder-defined widest-path level composed from the reference s-t Phi."""
    st = single_od_connectivity(graph, s, t)

    def phi(x):
        best = 0
        for k in range(1, m):
            if st((np.asarray(x) >= k).astype(np.int64)):
                best = k
        return best
    return phi


def gen_philox():
    cases = [(123, 0, 0, 8), (2**64 - 1, 5, 7, 33), (7, 2**63 + 5, 1001, 17), (0, 0, 3, 1)]
    raws = {}
    for i, (seed, gen, first, count) in enumerate(cases):
        bg = rs._philox(seed, gen)
        bg.advance(first // 4)
        raws[f"raw{i}"] = bg.random_raw(first % 4 + count)[first % 4:]
    ucases = [(123, 0, 0, 2, 3), (2**64 - 1, 5, 7, 33, 13), (7, 2**63 + 5, 1001, 17, 295)]
    for i, c in enumerate(ucases):
        raws[f"uniform{i}"] = rs.uniform_field(*c)
    np.savez(os.path.join(HERE, "philox.npz"), cases=np.array(cases, dtype=object),
             ucases=np.array(ucases, dtype=object), **raws)


def gen_sampling():
    out = {}
    specs = []
    rng = np.random.default_rng(2026)
    tables = [
        np.tile([0.1, 0.9], (295, 1)),
        rng.dirichlet([1.0, 3.0, 16.0], size=40),
        (lambda r: r / r.sum(1, keepdims=True))(rng.random((7, 5)) + 0.05),
        np.array([[1.0, 0.0], [0.0, 1.0], [0.5, 0.5]]),
        np.tile([0.1, 0.2, 0.7], (9, 1)),
    ]
    keys = [(257, 3, 1, 1001), (300, 5, 0, 0), (513, 2**63 + 11, 9, 17), (100, 1, 0, 0),
            (400, 42, 3, 5)]
    for i, (probs, (n, seed, gen, start)) in enumerate(zip(tables, keys)):
        b = sample_batch(ComponentDistribution(probs), n, seed, gen, start)
        out[f"probs{i}"] = probs
        out[f"states{i}"] = b.states.astype(np.uint8)
        specs.append([n, seed, gen, start])
    np.savez(os.path.join(HERE, "sampling.npz"), specs=np.array(specs, dtype=object), **out)


def _near_refs(rng, samples, k, m, up):
    base = samples[rng.integers(0, samples.shape[0], k)]
    delta = rng.integers(0, 2, base.shape)
    return np.clip(base - delta if up else base + delta, 0, m - 1)


def gen_classify():
    out = {}
    cases = []
    rng = np.random.default_rng(11)
    specs = [(300, 12, 2, 25, 30), (400, 9, 3, 20, 20), (250, 6, 4, 15, 15), (200, 5, 5, 10, 12),
             (500, 40, 2, 60, 0), (300, 40, 2, 0, 70), (64, 3, 2, 0, 0)]
    for i, (h, n, m, kl, ku) in enumerate(specs):
        samples = rng.integers(0, m, size=(h, n))
        lower = _near_refs(rng, samples, kl, m, False) if kl else np.zeros((0, n), dtype=np.int64)
        upper = _near_refs(rng, samples, ku, m, True) if ku else np.zeros((0, n), dtype=np.int64)
        ls = ReferenceSet(Side.LOWER, 0)
        us = ReferenceSet(Side.UPPER, 0)
        for v in lower:
            ls.insert(ReferenceState(tuple(v), Side.LOWER, 0))
        for v in upper:
            us.insert(ReferenceState(tuple(v), Side.UPPER, 0))
        res = classify(SampleBatch(samples, 0, 0), ls, us, explain=True, n_states=m)
        out[f"samples{i}"] = samples
        out[f"lower{i}"] = np.array(ls.members, dtype=np.int64).reshape(len(ls), n)
        out[f"upper{i}"] = np.array(us.members, dtype=np.int64).reshape(len(us), n)
        out[f"lo_idx{i}"] = res.lower_indices
        out[f"up_idx{i}"] = res.upper_indices
        out[f"un_idx{i}"] = res.unclassified_indices
        out[f"first_lo{i}"] = np.asarray(res.first_match_lower)
        out[f"first_up{i}"] = np.asarray(res.first_match_upper)
        cases.append(m)
    # violation counts
    samples = rng.integers(0, 3, size=(60, 9))
    refs = rng.integers(0, 3, size=(25, 9))
    s_enc = encode_batch(samples, 3, "sample")
    for kind in ("lower_ref", "upper_ref"):
        out[f"viol_{kind}"] = violation_counts(s_enc, encode_batch(refs, 3, kind))
    out["viol_samples"], out["viol_refs"] = samples, refs
    np.savez(os.path.join(HERE, "classify.npz"), n_states=np.array(cases), **out)


def fig_space_levels():
    return [[(1, 4), (4, 0), (3, 2)]]


def gen_boundary():
    recs = []
    model = SystemModel(2, 5, 2, _cone_phi(fig_space_levels()))
    for x0 in [(2, 0), (4, 4), (3, 1), (1, 4), (0, 0), (4, 0), (2, 3)]:
        model.reset_evaluation_count()
        r = boundary_search(model, x0, 0)
        recs.append({"model": "fig_space", "x0": list(x0), "threshold": 0, "vector": list(r.vector),
                     "side": r.side, "evals": model.evaluation_count})
    rng = np.random.default_rng(99)
    for case in range(25):
        n, m, ms = int(rng.integers(2, 7)), int(rng.integers(2, 5)), int(rng.integers(2, 4))
        levels = [[[int(v) for v in rng.integers(0, m, size=n)] for _ in range(int(rng.integers(1, 4)))]
                  for _ in range(ms - 1)]
        model = SystemModel(n, m, ms, _cone_phi(levels))
        for _ in range(4):
            x0 = [int(v) for v in rng.integers(0, m, size=n)]
            thr = int(rng.integers(0, ms - 1))
            model.reset_evaluation_count()
            r = boundary_search(model, x0, thr)
            recs.append({"model": "cones", "levels": levels, "n": n, "m": m, "ms": ms, "x0": x0,
                         "threshold": thr, "vector": list(r.vector), "side": r.side,
                         "evals": model.evaluation_count})
    with open(os.path.join(HERE, "boundary.json"), "w") as f:
        json.dump(recs, f)


def _s1_record(res, model):
    return {
        "lower": [list(v) for v in res.lower.members],
        "upper": [list(v) for v in res.upper.members],
        "trace": [[t.reference_count, t.phi_evaluations, t.p_lower, t.p_upper, t.p_unclassified]
                  for t in res.trace],
        "iterations": res.iterations, "redundant_searches": res.redundant_searches,
        "terminated_by": res.terminated_by, "phi_total": model.evaluation_count,
    }


def _s2_record(rep, model):
    return {"p_lower": rep.p_lower, "p_upper": rep.p_upper, "cov_lower": rep.cov_lower,
            "cov_upper": rep.cov_upper, "n_samples": rep.n_samples,
            "unclassified_resolved": rep.unclassified_resolved, "phi_total": model.evaluation_count}


def workflow_cases():
    """Case specs shared with the tests (model spec + RunConfig kwargs)."""
    g1 = workloads.cfg1(0)
    grid_m3 = workloads.cfg1(1)
    rng = np.random.default_rng(5)
    probs3 = rng.dirichlet([1.0, 3.0, 16.0], size=len(grid_m3["edges"]))
    cone_levels = [[[1, 0, 2, 1, 0, 1], [0, 2, 1, 1, 1, 0]], [[2, 1, 2, 2, 1, 1]]]
    rgg = random_geometric_graph(10, 0.55, seed=3)
    return [
        {"name": "series3", "model": {"kind": "kofn", "k": 3, "n": 3, "m": 2, "ms": 2},
         "probs": np.tile([0.1, 0.9], (3, 1)).tolist(),
         "config": dict(n_samples=2000, eps_u=1e-3, r_max=50, seed=7), "thresholds": [0]},
        {"name": "parallel3", "model": {"kind": "kofn", "k": 1, "n": 3, "m": 2, "ms": 2},
         "probs": np.tile([0.1, 0.9], (3, 1)).tolist(),
         "config": dict(n_samples=2000, eps_u=1e-3, r_max=50, seed=7), "thresholds": [0]},
        {"name": "series3_rmax1", "model": {"kind": "kofn", "k": 3, "n": 3, "m": 2, "ms": 2},
         "probs": np.tile([0.1, 0.9], (3, 1)).tolist(),
         "config": dict(n_samples=2000, eps_u=1e-3, r_max=1, seed=7), "thresholds": [0]},
        {"name": "series3_raw", "model": {"kind": "kofn", "k": 3, "n": 3, "m": 2, "ms": 2},
         "probs": np.tile([0.1, 0.9], (3, 1)).tolist(),
         "config": dict(n_samples=2000, eps_u=1e-3, r_max=30, seed=7,
                        boundary_search_enabled=False), "thresholds": [0]},
        {"name": "grid_st_small", "model": {"kind": "st", "n_nodes": g1["n_nodes"],
                                            "edges": g1["edges"], "s": 0, "t": 24, "m": 2, "ms": 2},
         "probs": g1["probs"].tolist(),
         "config": dict(n_samples=20_000, eps_u=1e-4, r_max=10_000, seed=0), "thresholds": [0]},
        {"name": "grid_st_b8", "model": {"kind": "st", "n_nodes": g1["n_nodes"],
                                         "edges": g1["edges"], "s": 0, "t": 24, "m": 2, "ms": 2},
         "probs": g1["probs"].tolist(),
         "config": dict(n_samples=20_000, eps_u=1e-4, r_max=10_000, seed=3, parallel_searches=8),
         "thresholds": [0]},
        {"name": "grid_widest_m3", "model": {"kind": "widest", "n_nodes": grid_m3["n_nodes"],
                                             "edges": grid_m3["edges"], "s": 0, "t": 24, "m": 3,
                                             "ms": 3},
         "probs": probs3.tolist(),
         "config": dict(n_samples=10_000, eps_u=1e-3, r_max=10_000, seed=1, parallel_searches=4),
         "thresholds": [0, 1]},
        {"name": "rgg_edge_disjoint", "model": {"kind": "edk", "n_nodes": rgg.n_nodes,
                                                "edges": [list(e) for e in rgg.edges], "max_level": 2,
                                                "m": 2, "ms": 3},
         "probs": np.tile([0.15, 0.85], (rgg.n_edges, 1)).tolist(),
         "config": dict(n_samples=3000, eps_u=1e-3, r_max=300, seed=5, parallel_searches=4),
         "thresholds": [0, 1]},
        {"name": "cones6", "model": {"kind": "cones", "levels": cone_levels, "n": 6, "m": 3, "ms": 3},
         "probs": np.tile([0.2, 0.3, 0.5], (6, 1)).tolist(),
         "config": dict(n_samples=5000, eps_u=1e-3, r_max=200, seed=11, parallel_searches=3),
         "thresholds": [0, 1]},
    ]


def build_reference_model(spec):
    m = spec["model"]
    if m["kind"] == "kofn":
        return SystemModel(m["n"], m["m"], m["ms"], k_out_of_n(m["k"], m["n"]))
    if m["kind"] in ("st", "widest"):
        g = Graph(m["n_nodes"], tuple(tuple(e) for e in m["edges"]))
        phi = single_od_connectivity(g, m["s"], m["t"]) if m["kind"] == "st" else \
            _widest_phi(g, m["s"], m["t"], m["m"])
        return SystemModel(len(m["edges"]), m["m"], m["ms"], phi)
    if m["kind"] == "cones":
        return SystemModel(m["n"], m["m"], m["ms"], _cone_phi(m["levels"]))
    if m["kind"] == "edk":
        g = Graph(m["n_nodes"], tuple(tuple(e) for e in m["edges"]))
        return SystemModel(len(m["edges"]), m["m"], m["ms"], edge_disjoint_level(g, m["max_level"]))
    raise ValueError(m["kind"])


def gen_workflow(specs, fname):
    out = []
    for spec in specs:
        model = build_reference_model(spec)
        dist = ComponentDistribution(np.array(spec["probs"]))
        cfg = RunConfig(**spec["config"])
        rec = {"spec": spec, "stages": []}
        for thr in spec["thresholds"]:
            s1 = stage1_find_references(model, dist, cfg, thr)
            r1 = _s1_record(s1, model)
            s2 = stage2_evaluate(model, dist, s1.lower, s1.upper, cfg, thr)
            rec["stages"].append({"threshold": thr, "stage1": r1, "stage2": _s2_record(s2, model)})
            print(spec["name"], thr, len(s1.lower), len(s1.upper), s1.iterations, flush=True)
        out.append(rec)
    with open(os.path.join(HERE, fname), "w") as f:
        json.dump(out, f)


def gen_refsets():
    """Reference-written rsr/1 set files and the member lists the reference loads."""
    from rsr.files import load_reference_sets, save_reference_sets
    import tempfile
    out = []
    rng = np.random.default_rng(77)
    docs = []
    # clean: a Stage-1 result of the 5x5 grid
    spec = next(c for c in workflow_cases() if c["name"] == "grid_st_small")
    model = build_reference_model(spec)
    s1 = stage1_find_references(model, ComponentDistribution(np.array(spec["probs"])),
                                RunConfig(**spec["config"]), 0)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "r.json")
        save_reference_sets(p, s1.lower, s1.upper, "grid-hash", seed=0)
        docs.append(json.loads(open(p).read()))
    # messy: duplicates and mutually dominated vectors, written raw
    vec = lambda k: [[int(v) for v in r] for r in rng.integers(0, 3, size=(k, 6))]  # noqa: E731
    lo, up = vec(80), vec(80)
    lo += lo[:5]
    up += up[3:9]
    docs.append({"format": "rsr/1", "threshold": 0, "model_hash": "messy",
                 "lower": {"format": "rsr/1", "side": "lower", "threshold": 0, "vectors": lo,
                           "model_hash": "messy"},
                 "upper": {"format": "rsr/1", "side": "upper", "threshold": 0, "vectors": up,
                           "model_hash": "messy"}})
    for doc in docs:
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "r.json")
            with open(p, "w") as f:
                json.dump(doc, f)
            lower, upper = load_reference_sets(p, doc["model_hash"])
        out.append({"file": doc, "lower": [list(v) for v in lower.members],
                    "upper": [list(v) for v in upper.members]})
    with open(os.path.join(HERE, "refsets.json"), "w") as f:
        json.dump(out, f)


from _cli_cases import run_cli  # noqa: E402  (shared with tests/test_cli.py)


def gen_cli():
    import tempfile
    from rsr.cli import main
    with tempfile.TemporaryDirectory() as d:
        outs = run_cli(main, d)
    with open(os.path.join(HERE, "cli.json"), "w") as f:
        json.dump(outs, f)


def gen_pmf():
    model = SystemModel(3, 3, 3, k_out_of_n(2, 3))
    dist = ComponentDistribution.iid(3, [0.2, 0.3, 0.5])
    cfg = RunConfig(n_samples=40_000, eps_u=1e-3, r_max=200, seed=11)
    rep = multistate_pmf(model, dist, cfg)
    with open(os.path.join(HERE, "pmf.json"), "w") as f:
        json.dump({"pmf": rep.pmf.tolist(), "cumulative_lower": rep.cumulative_lower.tolist(),
                   "max_chain_discrepancy": rep.max_chain_discrepancy,
                   "renormalization_adjustment": rep.renormalization_adjustment,
                   "n_refs": [[len(s.lower), len(s.upper)] for s in rep.stage1_results]}, f)


if __name__ == "__main__":
    if "--full-cfg1" in sys.argv:
        g = workloads.cfg1(0)
        spec = {"name": "cfg1_full", "model": {"kind": "st", "n_nodes": g["n_nodes"],
                                               "edges": g["edges"], "s": 0, "t": 24, "m": 2,
                                               "ms": 2},
                "probs": g["probs"].tolist(), "config": dict(n_samples=100_000, seed=0),
                "thresholds": [0]}
        gen_workflow([spec], "cfg1_full.json")
        sys.exit(0)
    gen_philox()
    gen_sampling()
    gen_classify()
    gen_boundary()
    gen_pmf()
    gen_refsets()
    gen_cli()
    gen_workflow(workflow_cases(), "workflow.json")
    print("rsr", rsr.__version__, "numpy", np.__version__)
