"""Randomised workflow parity (evidence, not a unit test): Stage 1 + Stage 2 on random small
systems (random connected graphs with s-t or widest-path Phi, k-out-of-n) and random
RunConfigs against the oracle restatement of workflow.py:122-245, on both sample streams:
ordered reference sets, every trace field, redundant searches, Phi-call counts, estimates.

    python tools/fuzz_workflow.py [seconds]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_2604_17066_b200 as P  # noqa: E402
from _specs import device_model, oracle_phi  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(os.environ.get("SEED", "3")))
t_end = time.time() + budget
cases = 0
n_pmf = 0


def random_graph(n_nodes, n_edges):
    edges = set()
    order = rng.permutation(n_nodes)
    for i in range(1, n_nodes):  # random spanning tree: connected
        edges.add(tuple(sorted((int(order[i]), int(order[rng.integers(0, i)])))))
    while len(edges) < n_edges:
        u, v = rng.choice(n_nodes, 2, replace=False)
        edges.add(tuple(sorted((int(u), int(v)))))
    return sorted(edges)


while time.time() < t_end:
    kind = rng.choice(["st", "widest", "kofn"])
    m = 2 if kind == "st" else int(rng.integers(2, 4))
    if kind == "kofn":
        n = int(rng.integers(3, 30))
        spec = {"kind": "kofn", "k": int(rng.integers(1, n + 1)), "n": n, "m": 2, "ms": 2}
        m = 2
    else:
        nn = int(rng.integers(4, 14))
        edges = random_graph(nn, int(rng.integers(nn - 1, min(3 * nn, nn * (nn - 1) // 2) + 1)))
        s, t = (int(x) for x in rng.choice(nn, 2, replace=False))
        spec = {"kind": kind, "n_nodes": nn, "edges": [list(e) for e in edges], "s": s, "t": t,
                "m": m, "ms": m}
        n = len(edges)
    probs = rng.dirichlet([1.0] * (m - 1) + [float(rng.uniform(3, 20))], size=n)
    cfg = dict(n_samples=int(rng.integers(500, 6000)), eps_u=float(rng.choice([1e-2, 1e-3])),
               r_max=int(rng.integers(5, 80)), seed=int(rng.integers(1 << 30)),
               parallel_searches=int(rng.choice([1, 4, 16])))
    stream = "device" if rng.random() < 0.4 else "shared"
    thr = int(rng.integers(0, m - 1))
    model = device_model(spec)
    dist = P.ComponentDistribution(probs)
    if m > 2 and rng.random() < 0.3:  # the whole PMF (thresholds share the batch cache)
        try:
            rep = P.multistate_pmf(model, dist, P.RunConfig(**cfg, rng=stream))
            err = None
        except ValueError as e:
            rep, err = None, str(e)
        phi, nc = oracle_phi(spec)
        ev = oracle.CountingPhi(phi, nc, m, m)
        try:
            want = oracle.multistate_pmf(ev, probs, rng=stream, **cfg)
            werr = None
        except ValueError as e:
            want, werr = None, str(e)
        if (err is None) != (werr is None) or (rep is not None and (
                not np.array_equal(rep.pmf, want["pmf"])
                or not np.array_equal(rep.cumulative_lower, want["cumulative_lower"])
                or [(r.lower.members, r.upper.members) for r in rep.stage1_results]
                != [(o["lower"], o["upper"]) for o in want["stage1"]]
                or model.evaluation_count != ev.count)):
            print("MISMATCH pmf", spec, cfg, stream, err, werr, flush=True)
            sys.exit(1)
        cases += 1
        n_pmf += 1
        continue
    s1 = P.stage1_find_references(model, dist, P.RunConfig(**cfg, rng=stream), thr)
    rep = P.stage2_evaluate(model, dist, s1.lower, s1.upper, P.RunConfig(**cfg, rng=stream), thr)
    phi, nc = oracle_phi(spec)
    ev = oracle.CountingPhi(phi, nc, m, m)
    o1 = oracle.stage1(ev, probs, thr, rng=stream, **cfg)
    o2 = oracle.stage2(ev, probs, o1["lower"], o1["upper"], thr, cfg["n_samples"], cfg["seed"],
                       rng=stream)
    got = (s1.lower.members, s1.upper.members,
           [(t.reference_count, t.phi_evaluations, t.p_lower, t.p_upper, t.p_unclassified)
            for t in s1.trace], s1.redundant_searches, rep.p_lower, rep.p_upper,
           rep.unclassified_resolved, model.evaluation_count)
    want = (o1["lower"], o1["upper"],
            [(t["reference_count"], t["phi_evaluations"], t["p_lower"], t["p_upper"],
              t["p_unclassified"]) for t in o1["trace"]], o1["redundant_searches"],
            o2["p_lower"], o2["p_upper"], o2["unclassified_resolved"], ev.count)
    if got != want:
        print("MISMATCH", spec, cfg, stream, thr, flush=True)
        for g_, w_ in zip(got, want):
            if g_ != w_:
                print(" got ", str(g_)[:300], "\n want", str(w_)[:300])
        sys.exit(1)
    cases += 1
print(f"fuzz workflow: {cases} random cases ({n_pmf} whole multistate PMFs, the rest Stage 1 + "
      f"Stage 2) equal to the oracle "
      f"({budget:.0f} s, seed {os.environ.get('SEED', '3')})")
