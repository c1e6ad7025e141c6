"""numpy restatement of the RSR hot path -- TEST INFRASTRUCTURE ONLY.

Every function cites the reference function it restates (paths relative to
``/root/reference/pkg/src/rsr/``).  The restatement is deliberately written in
a functional style over plain arrays so it shares no code with the product
package; it is pinned against golden vectors produced by the reference itself
(``tests/golden/make_golden.py``) and, where the reference is importable, by
live differential tests.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .philox import uniform_field

__all__ = [
    "sample_states", "encode", "dominance_hits", "classify_labels", "violation_counts",
    "cov", "UnionFind", "phi_st", "phi_global", "phi_kofn", "phi_widest", "phi_cones",
    "phi_edge_disjoint",
    "CountingPhi", "boundary_search", "RefSet", "stage1", "stage2", "assemble_pmf",
    "multistate_pmf", "LOWER", "UPPER",
]

LOWER = "lower"
UPPER = "upper"

# -------------------------------------------------------------------- sampling


def sample_states(probs: np.ndarray, n_samples: int, seed: int, generation_index: int = 0,
                  start: int = 0, fast: bool = False, rng: str = "shared") -> np.ndarray:
    """Inverse-CDF draw on the Philox field (``sampling.py:69-90``).

    state[i, n] = #{m : cumsum(probs[n])[m] <= u[i, n]} clipped to M-1, which is
    ``np.searchsorted(cum[n], u, side="right")`` for the non-decreasing cum.
    ``fast`` uses numpy's own Philox as the reference does (timing runs).
    ``rng="device"``: the independent device stream (not in the reference), u =
    raw32 * 2^-32 from row-aligned Philox4x32-10 (philox.device_raw), same inverse CDF.
    """
    if n_samples < 1:
        raise ValueError("n_samples must be >= 1")
    probs = np.asarray(probs, dtype=np.float64)
    n, m = probs.shape
    if rng == "device":
        from .philox import device_raw
        u = device_raw(seed, generation_index, start, n_samples, n).astype(np.float64) * 2.0 ** -32
    elif rng == "shared":
        u = uniform_field(seed, generation_index, start, n_samples, n, fast=fast)
    else:
        raise ValueError(f"rng must be 'shared' or 'device', got {rng!r}")
    cum = np.cumsum(probs, axis=1)
    out = np.empty((n_samples, n), dtype=np.int64)
    for comp in range(n):
        out[:, comp] = (u[:, comp, None] >= cum[comp][None, :]).sum(axis=1)
    np.minimum(out, m - 1, out=out)
    return out


# -------------------------------------------------------------------- encoding


def encode(states: np.ndarray, n_states: int, kind: str) -> np.ndarray:
    """Flattened N x M one-hot / prefix / suffix rows (``encoding.py:138-153``)."""
    arr = np.asarray(states, dtype=np.int64)
    if arr.size and (arr.min() < 0 or arr.max() >= n_states):
        raise ValueError(f"states must lie in [0, {n_states - 1}]")
    levels = np.arange(n_states)[None, None, :]
    cube = arr[:, :, None]
    if kind == "sample":
        bits = levels == cube
    elif kind == "lower_ref":
        bits = levels <= cube
    elif kind == "upper_ref":
        bits = levels >= cube
    else:
        raise ValueError(kind)
    return bits.reshape(arr.shape[0], -1).astype(np.uint8)


# -------------------------------------------------------------- classification

_BLOCK_BYTES = 1 << 26  # classify.py:34-35 working-set bound per ref block


def _zero_violation(sample_bits: np.ndarray, refbar_bits: np.ndarray,
                    want_first: bool) -> tuple[np.ndarray, np.ndarray | None]:
    """Any-zero of popcount(sample & ~ref) over a ref block loop (``classify.py:99-118``)."""
    rows, width = sample_bits.shape
    hit = np.zeros(rows, dtype=bool)
    first = np.full(rows, -1, dtype=np.int64) if want_first else None
    step = max(1, min(refbar_bits.shape[0], _BLOCK_BYTES // max(1, rows * width)))
    for r0 in range(0, refbar_bits.shape[0], step):
        blk = refbar_bits[r0:r0 + step]
        viol = np.bitwise_count(sample_bits[:, None, :] & blk[None, :, :]).sum(axis=2, dtype=np.int32)
        z = viol == 0
        zh = z.any(axis=1)
        if want_first:
            new = zh & ~hit
            first[new] = np.argmax(z[new], axis=1) + r0
        hit |= zh
    return hit, first


def dominance_hits(samples: np.ndarray, refs: np.ndarray, n_states: int, side: str,
                   chunk_size: int = 65536, n_workers: int = 1,
                   want_first: bool = False) -> tuple[np.ndarray, np.ndarray | None]:
    """hit[h] = exists r with x_h dominated (lower) / dominating (upper) (``classify.py:121-148``)."""
    h = samples.shape[0]
    refs = np.asarray(refs, dtype=np.int64).reshape(-1, samples.shape[1])
    if refs.shape[0] == 0:
        return np.zeros(h, dtype=bool), (np.full(h, -1, dtype=np.int64) if want_first else None)
    kind = "lower_ref" if side == LOWER else "upper_ref"
    sbits = np.packbits(encode(samples, n_states, "sample"), axis=1)
    rbar = np.packbits(1 - encode(refs, n_states, kind), axis=1)
    bounds = [(a, min(a + chunk_size, h)) for a in range(0, h, chunk_size)]

    def run(b):
        return _zero_violation(sbits[b[0]:b[1]], rbar, want_first)

    if n_workers > 1 and len(bounds) > 1:
        with ThreadPoolExecutor(max_workers=n_workers) as pool:
            parts = list(pool.map(run, bounds))
    else:
        parts = [run(b) for b in bounds]
    hit = np.concatenate([p[0] for p in parts])
    first = np.concatenate([p[1] for p in parts]) if want_first else None
    return hit, first


def classify_labels(samples: np.ndarray, lower_refs: np.ndarray, upper_refs: np.ndarray,
                    n_states: int, chunk_size: int = 65536, n_workers: int = 1,
                    want_first: bool = False) -> dict:
    """Three-way partition with lower precedence (``classify.py:187-249``).

    ``labels`` uses the device convention 0 = lower, 1 = upper, 2 = unclassified.
    """
    samples = np.asarray(samples, dtype=np.int64)
    hl, fl = dominance_hits(samples, lower_refs, n_states, LOWER, chunk_size, n_workers, want_first)
    hu, fu = dominance_hits(samples, upper_refs, n_states, UPPER, chunk_size, n_workers, want_first)
    labels = np.full(samples.shape[0], 2, dtype=np.uint8)
    labels[hu] = 1
    labels[hl] = 0
    return {
        "labels": labels,
        "lower_indices": np.flatnonzero(hl),
        "upper_indices": np.flatnonzero(hu & ~hl),
        "unclassified_indices": np.flatnonzero(~(hl | hu)),
        "both": np.flatnonzero(hl & hu),
        "first_lower": fl,
        "first_upper": fu,
    }


def violation_counts(samples: np.ndarray, refs: np.ndarray, n_states: int, kind: str) -> np.ndarray:
    """Full H x R int32 count of violated encoding positions (``classify.py:57-96``).

    Restated as the unpacked integer product ``classify.py:47-49``.
    """
    s = encode(samples, n_states, "sample").astype(np.int32)
    r = encode(refs, n_states, kind).astype(np.int32)
    return s @ (1 - r).T


def cov(p_hat: float, n_samples: int) -> float | None:
    """sqrt((1-p)/(H p)), None at p = 0 (``classify.py:265-277``)."""
    if n_samples < 1:
        raise ValueError("n_samples must be >= 1")
    if not 0.0 <= p_hat <= 1.0:
        raise ValueError("p_hat must lie in [0, 1]")
    if p_hat == 0.0:
        return None
    return math.sqrt((1.0 - p_hat) / (n_samples * p_hat))


# ---------------------------------------------------------------- system Phi


class UnionFind:
    """Path-halving union-find (``sysfn.py:62-76``)."""

    def __init__(self, n: int) -> None:
        self.p = list(range(n))

    def find(self, a: int) -> int:
        p = self.p
        while p[a] != a:
            p[a] = p[p[a]]
            a = p[a]
        return a

    def union(self, a: int, b: int) -> None:
        ra, rb = self.find(a), self.find(b)
        if ra != rb:
            self.p[rb] = ra


def _alive_uf(n_nodes, edges, x, level=1):
    uf = UnionFind(n_nodes)
    for e, (u, v) in enumerate(edges):
        if x[e] >= level:
            uf.union(u, v)
    return uf


def phi_st(n_nodes: int, edges, s: int, t: int):
    """s-t connectivity over edges with x_e >= 1 (``sysfn.py:79-98``)."""
    def phi(x):
        uf = _alive_uf(n_nodes, edges, x)
        return int(uf.find(s) == uf.find(t))
    return phi


def phi_global(n_nodes: int, edges):
    """All nodes connected over alive edges (``sysfn.py:101-109``)."""
    def phi(x):
        uf = _alive_uf(n_nodes, edges, x)
        r = uf.find(0)
        return int(all(uf.find(v) == r for v in range(1, n_nodes)))
    return phi


def _unit_max_flow(n_nodes: int, arcs, s: int, t: int, cap_limit: int) -> int:
    """Edge-disjoint s-t path count by BFS augmentation, stopped at cap_limit (``sysfn.py:112-137``).

    ``arcs`` is a list of (tail, head); arc 2e and 2e+1 are the two directions of
    edge e (unit capacity each); augmenting along arc a moves one unit to a ^ 1.
    """
    res = [1] * len(arcs)
    flow = 0
    while flow < cap_limit:
        parent = [-1] * n_nodes
        parent[s] = -2
        frontier = [s]
        while frontier and parent[t] == -1:
            nxt = []
            for a, (u, v) in enumerate(arcs):
                if res[a] > 0 and parent[v] == -1 and parent[u] != -1 and u in frontier:
                    parent[v] = a
                    nxt.append(v)
            frontier = nxt
        if parent[t] == -1:
            break
        v = t
        while v != s:
            a = parent[v]
            res[a] -= 1
            res[a ^ 1] += 1
            v = arcs[a][0]
        flow += 1
    return flow


def phi_edge_disjoint(n_nodes: int, edges, max_level: int):
    """Min over targets of capped unit max-flows from node 0 (``sysfn.py:140-174``)."""
    if max_level < 1 or n_nodes < 2:
        raise ValueError("bad edge_disjoint_level parameters")

    def phi(x):
        arcs = []
        for e, (u, v) in enumerate(edges):
            if x[e] >= 1:
                arcs += [(u, v), (v, u)]
        level = max_level
        for t in range(1, n_nodes):
            level = min(level, _unit_max_flow(n_nodes, arcs, 0, t, level))
            if level == 0:
                return 0
        return level
    return phi


def phi_kofn(k: int, n: int):
    """k-th largest component state (``sysfn.py:177-185``)."""
    def phi(x):
        return int(np.sort(np.asarray(x))[n - k])
    return phi


def phi_widest(n_nodes: int, edges, s: int, t: int, n_states: int):
    """Widest-path level: max{k : s-t connected on edges with x_e >= k}.

    Not in the reference; composed from the reference s-t connectivity applied to
    the level sets ``x >= k`` (``sysfn.py:79-98``).
    """
    def phi(x):
        best = 0
        for k in range(1, n_states):
            uf = _alive_uf(n_nodes, edges, x, level=k)
            if uf.find(s) == uf.find(t):
                best = k
        return best
    return phi


def phi_cones(levels):
    """Sum over levels of [x dominates any anchor] (reference ``tests/conftest.py:53-75``)."""
    levels = [np.asarray(a, dtype=np.int64).reshape(len(a), -1) for a in levels]

    def phi(x):
        x = np.asarray(x)
        return int(sum(bool(np.any(np.all(x[None, :] >= a, axis=1))) for a in levels))
    return phi


class CountingPhi:
    """Validated, counted evaluation (``model.py:88-97``)."""

    def __init__(self, phi, n_components: int, n_states: int, n_system_states: int):
        self.phi, self.n, self.m, self.ms = phi, n_components, n_states, n_system_states
        self.count = 0

    def __call__(self, x) -> int:
        arr = np.asarray(x, dtype=np.int64)
        if arr.shape != (self.n,) or (arr.size and (arr.min() < 0 or arr.max() >= self.m)):
            raise ValueError("bad component-state vector")
        self.count += 1
        s = int(self.phi(arr))
        if not 0 <= s < self.ms:
            raise ValueError("performance out of range")
        return s


# ----------------------------------------------------------- boundary search


def boundary_search(ev: CountingPhi, x0, threshold: int) -> tuple[tuple[int, ...], str]:
    """Unit-step componentwise walk to the boundary (``boundary.py:116-147``)."""
    if not 0 <= threshold <= ev.ms - 2:
        raise ValueError("threshold out of range")
    x = np.array(x0, dtype=np.int64)
    if ev(x) <= threshold:
        side, step, limit = LOWER, 1, ev.m - 1
    else:
        side, step, limit = UPPER, -1, 0
    for n in range(ev.n):
        while x[n] != limit:
            x[n] += step
            s = ev(x)
            if (s > threshold) if side == LOWER else (s <= threshold):
                x[n] -= step
                break
    return tuple(int(v) for v in x), side


def _covers(side: str, a, b) -> bool:
    """a is redundant given b (``boundary.py:50-54``)."""
    if side == LOWER:
        return all(p <= q for p, q in zip(a, b))
    return all(p >= q for p, q in zip(a, b))


class RefSet:
    """Ordered non-dominated member list (``boundary.py:57-113``)."""

    def __init__(self, side: str, threshold: int):
        self.side, self.threshold = side, threshold
        self.members: list[tuple[int, ...]] = []

    def insert(self, vec) -> str:
        vec = tuple(int(v) for v in vec)
        if any(_covers(self.side, vec, m) for m in self.members):
            return "redundant"
        self.members = [m for m in self.members if not _covers(self.side, m, vec)]
        self.members.append(vec)
        return "inserted"

    def array(self, n: int) -> np.ndarray:
        return np.array(self.members, dtype=np.int64).reshape(len(self.members), n)

    def __len__(self):
        return len(self.members)


# ----------------------------------------------------------------- workflow


def stage1(ev: CountingPhi, probs: np.ndarray, threshold: int, n_samples: int,
           eps_u: float = 1e-5, r_max: int = 10_000, seed: int = 0,
           parallel_searches: int = 1, boundary_search_enabled: bool = True,
           chunk_size: int = 65536, n_workers: int = 1, time_budget: float | None = None,
           fast: bool = False, rng: str = "shared") -> dict:
    """Reference discovery loop (``workflow.py:122-195``).

    Trace records omit elapsed time and RSS (host-dependent); everything else
    is restated field for field.  ``time_budget`` (seconds) stops the loop
    early for CPU-baseline timing (terminated_by = "budget"); each trace
    record then also carries the cumulative ``elapsed`` seconds.
    """
    import time
    if not 0 <= threshold <= ev.ms - 2:
        raise ValueError("threshold out of range")
    lower, upper = RefSet(LOWER, threshold), RefSet(UPPER, threshold)
    trace, redundant, phi0, it = [], 0, ev.count, 0
    terminated_by = "r_max"
    t0 = time.perf_counter()
    while True:
        if time_budget is not None and trace and time.perf_counter() - t0 > time_budget:
            terminated_by = "budget"
            break
        xs = sample_states(probs, n_samples, seed, it, fast=fast, rng=rng)
        res = classify_labels(xs, lower.array(ev.n), upper.array(ev.n), ev.m,
                              chunk_size, n_workers)
        n_l, n_u = res["lower_indices"].size, res["upper_indices"].size
        n_x = res["unclassified_indices"].size
        trace.append({
            "reference_count": len(lower) + len(upper),
            "phi_evaluations": ev.count - phi0,
            "p_lower": n_l / n_samples,
            "p_upper": n_u / n_samples,
            "p_unclassified": n_x / n_samples,
        })
        if n_x / n_samples <= eps_u:
            terminated_by = "eps_u"
            break
        if len(lower) + len(upper) >= r_max:
            break
        gen = np.random.default_rng([seed, it])
        picks = gen.choice(res["unclassified_indices"], size=min(parallel_searches, n_x),
                           replace=False)
        for idx in picks:
            x0 = xs[int(idx)]
            if boundary_search_enabled:
                vec, side = boundary_search(ev, x0, threshold)
            else:
                side = LOWER if ev(x0) <= threshold else UPPER
                vec = tuple(int(v) for v in x0)
            tgt = lower if side == LOWER else upper
            if tgt.insert(vec) == "redundant":
                redundant += 1
        if time_budget is not None:
            trace[-1]["elapsed"] = time.perf_counter() - t0
        it += 1
    return {"lower": list(lower.members), "upper": list(upper.members), "trace": trace,
            "iterations": it + 1, "redundant_searches": redundant,
            "terminated_by": terminated_by}


def stage2(ev: CountingPhi, probs: np.ndarray, lower_members, upper_members, threshold: int,
           n_samples: int, seed: int = 0, chunk_size: int = 65536, n_workers: int = 1,
           start: int = 0, rng: str = "shared") -> dict:
    """One generation-0 batch, Phi on the unclassified (``workflow.py:198-245``).

    ``start`` extends the generation-0 index space for the run-to-c.o.v. loop
    (SURVEY a16); start = 0 is exactly the reference Stage 2.
    """
    xs = sample_states(probs, n_samples, seed, 0, start, rng=rng)
    lo = np.array(lower_members, dtype=np.int64).reshape(-1, ev.n)
    up = np.array(upper_members, dtype=np.int64).reshape(-1, ev.n)
    res = classify_labels(xs, lo, up, ev.m, chunk_size, n_workers)
    n_low, n_up = res["lower_indices"].size, res["upper_indices"].size
    for idx in res["unclassified_indices"]:
        if ev(xs[int(idx)]) <= threshold:
            n_low += 1
        else:
            n_up += 1
    return {"p_lower": n_low / n_samples, "p_upper": n_up / n_samples,
            "cov_lower": cov(n_low / n_samples, n_samples),
            "cov_upper": cov(n_up / n_samples, n_samples), "n_samples": n_samples,
            "n_lower": n_low, "n_upper": n_up,
            "unclassified_resolved": int(res["unclassified_indices"].size),
            "threshold": threshold, "seed": seed}


def assemble_pmf(cumulative) -> tuple[np.ndarray, float]:
    """diff / clamp / renormalise (``workflow.py:258-271``)."""
    c = np.asarray(cumulative, dtype=np.float64)
    if c.size and (c.min() < 0.0 or c.max() > 1.0):
        raise ValueError("cumulative probabilities must lie in [0, 1]")
    raw = np.diff(np.concatenate([[0.0], c, [1.0]]))
    kept = np.clip(raw, 0.0, None)
    return kept / kept.sum(), float(np.abs(kept - raw).sum())


def multistate_pmf(ev: CountingPhi, probs: np.ndarray, **cfg) -> dict:
    """All thresholds, 4-sigma monotonicity check, PMF + chain cross-check (``workflow.py:274-321``)."""
    s1s, s2s = [], []
    for thr in range(ev.ms - 1):
        s1 = stage1(ev, probs, thr, **cfg)
        s2 = stage2(ev, probs, s1["lower"], s1["upper"], thr, cfg["n_samples"],
                    cfg.get("seed", 0), cfg.get("chunk_size", 65536), cfg.get("n_workers", 1),
                    rng=cfg.get("rng", "shared"))
        s1s.append(s1)
        s2s.append(s2)
    cum = np.array([r["p_lower"] for r in s2s])
    sig = np.array([math.sqrt(r["p_lower"] * (1 - r["p_lower"]) / r["n_samples"]) for r in s2s])
    for i in range(1, len(cum)):
        if cum[i] < cum[i - 1] - 4.0 * (sig[i] + sig[i - 1]):
            raise ValueError("cumulative estimates non-monotone beyond tolerance")
    pmf, adj = assemble_pmf(cum)
    surv = np.concatenate([[1.0], [r["p_upper"] for r in s2s], [0.0]])
    pmf_up, _ = assemble_pmf(np.cumsum(-np.diff(surv))[:-1])
    return {"pmf": pmf, "cumulative_lower": cum, "stage1": s1s, "stage2": s2s,
            "max_chain_discrepancy": float(np.max(np.abs(pmf - pmf_up))),
            "renormalization_adjustment": adj}
