"""Seeded synthetic inputs for the BASELINE.json configurations (host-side setup).

No public dataset is involved: the paper's Graph 1 / Graph 2 edge lists are
not published (reference SPEC.md:157), so configs 3-5 use synthetic graphs of
the stated size.  Everything here is deterministic given the seed and is
plain numpy; it builds inputs, it does not compute any hot-path result.

* cfg1: 5 x 5 grid, 40 edges (horizontal row-major, then vertical), s = 0,
  t = 24, p_fail ~ U[0.05, 0.15].
* cfg2: S = 2^20 samples of Bernoulli(0.9) over N = 295 components,
  10^4 upper refs with exactly 15 ones, 10^4 lower refs with exactly 10 zeros.
  ``cfg2_mixed`` (p = 0.5, 15-one upper / 14-zero lower) exercises all labels.
* cfg3: 119 nodes uniform in the unit square, the 295 globally shortest pairs
  as edges; placement re-seeded until that edge set is connected (SURVEY B2
  option (i) -- the literal recipe is infeasible); s, t = Euclidean-farthest
  pair; p_fail ~ U[0.01, 0.10].
* cfg4: cfg3-shaped graph; upper refs = distinct simple s-t paths (shortest
  paths under random log-normal edge weights).
* cfg5: cfg3-shaped graph, M = 3, per-edge Dirichlet(1, 3, 16) probabilities,
  widest-path Phi, M_S = 3.
"""

from __future__ import annotations

import numpy as np

__all__ = ["grid_graph", "cfg1", "nn_graph", "cfg3", "cfg5", "cfg2_refs", "cfg2_mixed_refs",
           "random_st_paths"]


def grid_graph(rows: int = 5, cols: int = 5) -> tuple[int, list[tuple[int, int]]]:
    edges = [(r * cols + c, r * cols + c + 1) for r in range(rows) for c in range(cols - 1)]
    edges += [(r * cols + c, (r + 1) * cols + c) for r in range(rows - 1) for c in range(cols)]
    return rows * cols, edges


def cfg1(seed: int = 0) -> dict:
    n_nodes, edges = grid_graph(5, 5)
    rng = np.random.default_rng(seed)
    p_fail = rng.uniform(0.05, 0.15, size=len(edges))
    probs = np.stack([p_fail, 1.0 - p_fail], axis=1)
    return {"n_nodes": n_nodes, "edges": edges, "source": 0, "target": n_nodes - 1,
            "probs": probs}


def _connected(n: int, edges) -> bool:
    parent = list(range(n))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for u, v in edges:
        parent[find(u)] = find(v)
    return len({find(v) for v in range(n)}) == 1


def nn_graph(seed: int = 0, n_nodes: int = 119, n_edges: int = 295) -> dict:
    """Shortest-pairs graph, re-seeded until connected (see module docstring)."""
    for attempt in range(10_000):
        rng = np.random.default_rng([seed, attempt])
        pos = rng.random((n_nodes, 2))
        iu, ju = np.triu_indices(n_nodes, k=1)
        d = np.hypot(pos[iu, 0] - pos[ju, 0], pos[iu, 1] - pos[ju, 1])
        order = np.argsort(d, kind="stable")[:n_edges]
        edges = [(int(iu[k]), int(ju[k])) for k in order]
        if _connected(n_nodes, edges):
            far = int(np.argmax(d))
            return {"n_nodes": n_nodes, "edges": edges, "source": int(iu[far]),
                    "target": int(ju[far]), "positions": pos, "attempts": attempt + 1}
    raise RuntimeError("no connected placement found")


def cfg3(seed: int = 0) -> dict:
    g = nn_graph(seed)
    rng = np.random.default_rng([seed, 3])
    p_fail = rng.uniform(0.01, 0.10, size=len(g["edges"]))
    g["probs"] = np.stack([p_fail, 1.0 - p_fail], axis=1)
    return g


def cfg5(seed: int = 0) -> dict:
    g = nn_graph(seed)
    rng = np.random.default_rng([seed, 5])
    g["probs"] = rng.dirichlet([1.0, 3.0, 16.0], size=len(g["edges"]))
    return g


def _fixed_weight_rows(rng: np.random.Generator, k: int, n: int, n_hot: int, hot: int) -> np.ndarray:
    """k distinct rows of length n with exactly n_hot entries equal to `hot`."""
    rows = np.full((k, n), 1 - hot, dtype=np.uint8)
    keys = np.argsort(rng.random((k, n)), axis=1)[:, :n_hot]
    np.put_along_axis(rows, keys, hot, axis=1)
    _, first = np.unique(rows, axis=0, return_index=True)
    return rows[np.sort(first)]


def cfg2_refs(seed: int = 0, n: int = 295, k_upper: int = 10_000, k_lower: int = 10_000):
    """Upper refs: exactly 15 ones; lower refs: exactly 10 zeros (mutually non-dominated)."""
    rng = np.random.default_rng([seed, 2])
    upper = _fixed_weight_rows(rng, k_upper, n, 15, 1)
    lower = _fixed_weight_rows(rng, k_lower, n, 10, 0)
    return lower, upper


def cfg2_mixed_refs(seed: int = 0, n: int = 295, k_upper: int = 10_000, k_lower: int = 10_000):
    """Mixed-label variant for p = 0.5 samples: 15-one upper, 14-zero lower refs."""
    rng = np.random.default_rng([seed, 22])
    upper = _fixed_weight_rows(rng, k_upper, n, 15, 1)
    lower = _fixed_weight_rows(rng, k_lower, n, 14, 0)
    return lower, upper


def random_st_paths(graph: dict, k: int, seed: int = 0, sigma: float = 1.5,
                    batch: int = 4096) -> np.ndarray:
    """Up to k distinct simple s-t paths as edge-indicator rows (uint8 [K, E]).

    Shortest paths under i.i.d. log-normal edge weights, computed with a
    vectorised Bellman-Ford over a batch of weight draws.  Distinct simple
    s-t paths are mutually non-dominated as upper reference states.
    """
    try:
        import torch
        if torch.cuda.is_available():
            return _random_st_paths_torch(graph, k, seed, sigma)
    except ImportError:  # pragma: no cover
        pass
    n_nodes, edges = graph["n_nodes"], graph["edges"]
    s, t = graph["source"], graph["target"]
    eu = np.array([e[0] for e in edges])
    ev = np.array([e[1] for e in edges])
    E = len(edges)
    # directed arcs (both orientations) grouped by head node for reduceat
    tail = np.concatenate([eu, ev])
    head = np.concatenate([ev, eu])
    arc_edge = np.concatenate([np.arange(E), np.arange(E)])
    order = np.argsort(head, kind="stable")
    tail, head, arc_edge = tail[order], head[order], arc_edge[order]
    starts = np.flatnonzero(np.r_[True, head[1:] != head[:-1]])
    heads = head[starts]
    rng = np.random.default_rng([seed, 4])
    found: dict[bytes, None] = {}
    rounds = 0
    while len(found) < k and rounds < 10_000:
        rounds += 1
        w = np.exp(sigma * rng.standard_normal((batch, E)))[:, arc_edge]
        dist = np.full((batch, n_nodes), np.inf)
        dist[:, s] = 0.0
        for _ in range(n_nodes):
            cand = dist[:, tail] + w
            best = np.minimum.reduceat(cand, starts, axis=1)
            new = dist.copy()
            new[:, heads] = np.minimum(dist[:, heads], best)
            new[:, s] = 0.0
            if np.array_equal(new, dist):
                break
            dist = new
        # predecessor arc of every node: an incoming arc achieving dist[head]
        tight = np.isclose(dist[:, tail] + w, dist[:, head], rtol=0, atol=1e-12) & \
            np.isfinite(dist[:, tail])
        pred = np.full((batch, n_nodes), -1, dtype=np.int64)
        arc_ids = np.where(tight, np.arange(tail.size)[None, :], -1)
        pred[:, heads] = np.maximum.reduceat(arc_ids, starts, axis=1)  # any tight arc
        rows = np.zeros((batch, E), dtype=np.uint8)
        node = np.full(batch, t)
        ok = np.isfinite(dist[:, t])
        for _ in range(n_nodes):
            active = ok & (node != s)
            if not active.any():
                break
            a = pred[np.arange(batch), node]
            bad = active & (a < 0)
            ok &= ~bad
            active &= ~bad
            rows[active, arc_edge[a[active]]] = 1
            node = np.where(active, tail[a], node)
        for r in rows[ok & (node == s)]:
            found.setdefault(r.tobytes(), None)
            if len(found) >= k:
                break
    out = np.frombuffer(b"".join(found.keys()), dtype=np.uint8).reshape(-1, E)
    return out[:k].copy()


def _random_st_paths_torch(graph: dict, k: int, seed: int, sigma: float,
                           batch: int = 1 << 16) -> np.ndarray:
    """Same construction as ``random_st_paths`` with the batched Bellman-Ford on
    the GPU (setup data only: cfg4 needs up to 5 x 10^5 distinct paths)."""
    import torch
    dev = torch.device("cuda")
    n_nodes, edges = graph["n_nodes"], graph["edges"]
    s, t = graph["source"], graph["target"]
    E = len(edges)
    eu = torch.tensor([e[0] for e in edges], device=dev)
    ev = torch.tensor([e[1] for e in edges], device=dev)
    tail = torch.cat([eu, ev])
    head = torch.cat([ev, eu])
    arc_edge = torch.cat([torch.arange(E, device=dev)] * 2)
    A = tail.numel()
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed) * 1_000_003 + 4)
    found = None
    rounds = 0
    while (found is None or found.shape[0] < k) and rounds < 1000:
        rounds += 1
        w = torch.exp(sigma * torch.randn((batch, E), generator=gen, device=dev,
                                          dtype=torch.float64))[:, arc_edge]
        dist = torch.full((batch, n_nodes), float("inf"), device=dev, dtype=torch.float64)
        dist[:, s] = 0.0
        hidx = head.unsqueeze(0).expand(batch, A)
        for _ in range(n_nodes):
            cand = dist[:, tail] + w
            new = dist.scatter_reduce(1, hidx, cand, reduce="amin", include_self=True)
            if torch.equal(new, dist):
                break
            dist = new
        tight = (dist[:, tail] + w == dist[:, head]) & torch.isfinite(dist[:, tail])
        arc_ids = torch.where(tight, torch.arange(A, device=dev).unsqueeze(0), -1)
        pred = torch.full((batch, n_nodes), -1, dtype=torch.int64, device=dev)
        pred = pred.scatter_reduce(1, hidx, arc_ids, reduce="amax", include_self=True)
        rows = torch.zeros((batch, E), dtype=torch.uint8, device=dev)
        node = torch.full((batch,), t, dtype=torch.int64, device=dev)
        ok = torch.isfinite(dist[:, t])
        ar = torch.arange(batch, device=dev)
        for _ in range(n_nodes):
            active = ok & (node != s)
            if not bool(active.any()):
                break
            a = pred[ar, node]
            ok &= ~(active & (a < 0))
            active &= a >= 0
            rows[ar[active], arc_edge[a[active]]] = 1
            node = torch.where(active, tail[a.clamp(min=0)], node)
        rows = rows[ok & (node == s)]
        found = rows if found is None else torch.cat([found, rows])
        found = torch.unique(found, dim=0)
    return found[:k].cpu().numpy()
