"""Device-described system functions Phi (mirror of reference ``sysfn.py``).

The reference's performance functions are opaque Python closures
(sysfn.py:87-185).  Here each factory returns a ``DevicePerformance``: a
structured descriptor (kind, graph edge list, s, t, k, anchors) that the CUDA
kernels in ``csrc/phi.cu`` evaluate, one warp per vector.  Calling the object
on a vector evaluates it on the device.

Kinds (``include/rsr_b200.h``):
  * ``single_od_connectivity`` -- s-t connected over edges with x_e >= 1
    (sysfn.py:87-98);
  * ``widest_path_level`` -- max k such that s, t connect over x_e >= k
    (BASELINE cfg5; not in the reference);
  * ``global_connectivity`` (sysfn.py:101-109);
  * ``k_out_of_n`` -- k-th largest state (sysfn.py:177-185);
  * ``edge_disjoint_level`` -- capped edge connectivity (sysfn.py:112-174);
  * ``cone_sum`` -- number of levels whose anchor set has a member dominated
    by x: the coherent-by-construction test system of the reference suite
    (tests/conftest.py:53-75).

``Graph``, ``random_geometric_graph`` and ``pick_od_pair`` are host-side
graph construction utilities with the reference semantics
(sysfn.py:32-59, 188-269).
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np
import torch

from . import _abi, _device
from .model import SystemModel

__all__ = [
    "Graph", "DevicePerformance", "single_od_connectivity", "widest_path_level",
    "global_connectivity", "edge_disjoint_level", "k_out_of_n", "cone_sum",
    "random_geometric_graph", "pick_od_pair", "build_graph_model",
]

_RGG_MAX_RETRIES = 100


@dataclass(frozen=True)
class Graph:
    """Undirected graph; immutable after construction (sysfn.py:32-59)."""

    n_nodes: int
    edges: tuple[tuple[int, int], ...]
    node_positions: tuple[tuple[float, float], ...] | None = None
    metadata: dict = field(default_factory=dict, compare=False)

    def __post_init__(self) -> None:
        if self.n_nodes < 1:
            raise ValueError("n_nodes must be positive")
        edges = tuple((int(u), int(v)) for u, v in self.edges)
        object.__setattr__(self, "edges", edges)
        for u, v in edges:
            if not (0 <= u < self.n_nodes and 0 <= v < self.n_nodes):
                raise ValueError(f"edge ({u}, {v}) out of range for {self.n_nodes} nodes")
            if u == v:
                raise ValueError(f"self-loop at node {u}")
        if self.node_positions is not None:
            pos = tuple((float(x), float(y)) for x, y in self.node_positions)
            if len(pos) != self.n_nodes:
                raise ValueError("node_positions length must equal n_nodes")
            object.__setattr__(self, "node_positions", pos)

    @property
    def n_edges(self) -> int:
        return len(self.edges)


class DevicePerformance:
    """A performance function Phi evaluated by ``rsr_phi_eval`` on the device."""

    def __init__(self, kind: int, n_components: int, *, graph: Graph | None = None,
                 source: int = 0, target: int = 0, k: int = 0,
                 anchors: np.ndarray | None = None, anchor_level: np.ndarray | None = None,
                 name: str = ""):
        self.kind = kind
        self.n_components = int(n_components)
        self.graph = graph
        self.source, self.target, self.k = int(source), int(target), int(k)
        self.anchors = anchors
        self.anchor_level = anchor_level
        self.name = name
        self._cache: dict = {}

    def __repr__(self) -> str:
        return f"DevicePerformance({self.name})"

    def descriptor(self, n_states: int) -> _abi.PhiDesc:
        """ctypes descriptor with device arrays (cached per device and M)."""
        dev = _device.device()
        key = (str(dev), int(n_states))
        hit = self._cache.get(key)
        if hit is not None:
            return hit[0]
        keep = []
        eu = ev = an = al = None
        n_nodes = 0
        if self.graph is not None:
            eu = _device.to_device(np.array([e[0] for e in self.graph.edges], dtype=np.int32))
            ev = _device.to_device(np.array([e[1] for e in self.graph.edges], dtype=np.int32))
            n_nodes = self.graph.n_nodes
            keep += [eu, ev]
        n_anchors = 0
        if self.anchors is not None and len(self.anchors):
            an = _device.to_device(np.asarray(self.anchors, dtype=np.uint8))
            al = _device.to_device(np.asarray(self.anchor_level, dtype=np.int32))
            n_anchors = an.shape[0]
            keep += [an, al]
        flags = 0
        if self.graph is not None:
            pairs = {(min(u, v), max(u, v)) for u, v in self.graph.edges}
            if len(pairs) == len(self.graph.edges):
                flags |= _abi.PHI_FLAG_SIMPLE  # bitset-BFS kernels (csrc/phi_bits.cu)
        d = _abi.PhiDesc(self.kind, self.n_components, int(n_states), n_nodes, self.source,
                         self.target, self.k, n_anchors, _abi.ptr(eu), _abi.ptr(ev),
                         _abi.ptr(an), _abi.ptr(al), flags)
        self._cache[key] = (d, keep)
        return d

    def evaluate_device(self, rows, n_states: int) -> np.ndarray:
        """Phi of each row (host or device input), as a host uint8 array."""
        xs = _device.u8_rows(rows, self.n_components, n_states)
        out = torch.empty(xs.shape[0], dtype=torch.uint8, device=xs.device)
        self.eval_into(xs, None, xs.shape[0], n_states, out)
        return out.cpu().numpy()

    def eval_into(self, states: torch.Tensor, idx: torch.Tensor | None, count: int, n_states: int,
                  out: torch.Tensor | None, threshold: int = 0,
                  count_leq: torch.Tensor | None = None) -> None:
        d = self.descriptor(n_states)
        import ctypes
        _abi.call("rsr_phi_eval", ctypes.byref(d), _abi.ptr(states), _abi.ptr(idx), int(count),
                  _abi.ptr(out), int(threshold), _abi.ptr(count_leq), _device.stream())

    def __call__(self, x) -> int:
        n_states = int(np.max(np.asarray(x))) + 1 if np.asarray(x).size else 2
        return int(self.evaluate_device(np.asarray(x)[None, :], max(2, n_states))[0])


def single_od_connectivity(graph: Graph, origin: int, destination: int) -> DevicePerformance:
    """Binary s-t connectivity over surviving edges x_e >= 1 (sysfn.py:87-98)."""
    if not (0 <= origin < graph.n_nodes and 0 <= destination < graph.n_nodes):
        raise ValueError("origin/destination out of range")
    if origin == destination:
        raise ValueError("origin and destination must differ")
    return DevicePerformance(_abi.PHI_ST, graph.n_edges, graph=graph, source=origin,
                             target=destination, name=f"st({origin},{destination})")


def widest_path_level(graph: Graph, origin: int, destination: int) -> DevicePerformance:
    """max{k : origin, destination connected over edges with x_e >= k} (M_S = M)."""
    if not (0 <= origin < graph.n_nodes and 0 <= destination < graph.n_nodes):
        raise ValueError("origin/destination out of range")
    if origin == destination:
        raise ValueError("origin and destination must differ")
    return DevicePerformance(_abi.PHI_WIDEST, graph.n_edges, graph=graph, source=origin,
                             target=destination, name=f"widest({origin},{destination})")


def global_connectivity(graph: Graph) -> DevicePerformance:
    """State 1 iff the surviving subgraph connects all nodes (sysfn.py:101-109)."""
    return DevicePerformance(_abi.PHI_GLOBAL, graph.n_edges, graph=graph, name="global")


def k_out_of_n(k: int, n_components: int) -> DevicePerformance:
    """Generalised multi-state k-out-of-N:G, the k-th largest state (sysfn.py:177-185)."""
    if not 1 <= k <= n_components:
        raise ValueError(f"k must lie in [1, {n_components}]")
    return DevicePerformance(_abi.PHI_KOFN, n_components, k=k, name=f"{k}-out-of-{n_components}")


def cone_sum(levels: Sequence[Sequence[Sequence[int]]], n_components: int) -> DevicePerformance:
    """Phi(x) = #{levels l : x >= some anchor of l} (coherent by construction)."""
    rows, lev = [], []
    for li, anchors in enumerate(levels):
        for a in anchors:
            rows.append([int(v) for v in a])
            lev.append(li)
    if len(levels) > 31:
        raise ValueError("at most 31 levels")
    arr = np.array(rows, dtype=np.uint8).reshape(len(rows), n_components)
    return DevicePerformance(_abi.PHI_CONES, n_components, anchors=arr,
                             anchor_level=np.array(lev, dtype=np.int32), name="cone_sum")


def edge_disjoint_level(graph: Graph, max_level: int) -> DevicePerformance:
    """Min over node pairs of edge-disjoint path counts, capped (sysfn.py:140-174), M_S = max_level + 1.

    Device: unit-capacity max-flow from node 0 to every other node by BFS
    augmentation, one warp per vector (csrc/phi.cu).
    """
    if max_level < 1:
        raise ValueError("max_level must be >= 1")
    if graph.n_nodes < 2:
        raise ValueError("need at least two nodes")
    return DevicePerformance(_abi.PHI_EDGE_DISJOINT, graph.n_edges, graph=graph, k=max_level,
                             name=f"edge_disjoint_level({max_level})")


class _UnionFind:
    def __init__(self, n: int) -> None:
        self.parent = list(range(n))

    def find(self, a: int) -> int:
        p = self.parent
        while p[a] != a:
            p[a] = p[p[a]]
            a = p[a]
        return a

    def union(self, a: int, b: int) -> None:
        ra, rb = self.find(a), self.find(b)
        if ra != rb:
            self.parent[rb] = ra


def random_geometric_graph(n_nodes: int, radius: float, seed: int) -> Graph:
    """Unit-square RGG with connectivity retries (sysfn.py:188-241), host-side setup."""
    if n_nodes < 2:
        raise ValueError("n_nodes must be >= 2")
    if not 0.0 < radius <= 1.0:
        raise ValueError("radius must lie in (0, 1]")
    for attempt in range(_RGG_MAX_RETRIES):
        rng = np.random.default_rng([seed, attempt])
        pos = rng.random((n_nodes, 2))
        d2 = np.sum((pos[:, None, :] - pos[None, :, :]) ** 2, axis=2)
        iu, ju = np.triu_indices(n_nodes, k=1)
        mask = d2[iu, ju] <= radius * radius
        edges = tuple((int(u), int(v)) for u, v in zip(iu[mask], ju[mask]))
        uf = _UnionFind(n_nodes)
        for u, v in edges:
            uf.union(u, v)
        roots = [uf.find(v) for v in range(n_nodes)]
        if len(set(roots)) == 1:
            return Graph(n_nodes, edges, node_positions=tuple(map(tuple, pos.tolist())),
                         metadata={"seed": seed, "radius": radius, "attempts": attempt + 1})
    counts: dict[int, int] = {}
    for r in roots:
        counts[r] = counts.get(r, 0) + 1
    keep_root = max(counts, key=lambda r: (counts[r], -r))
    keep = [v for v in range(n_nodes) if roots[v] == keep_root]
    relabel = {old: new for new, old in enumerate(keep)}
    sub_edges = tuple((relabel[u], relabel[v]) for u, v in edges if u in relabel and v in relabel)
    return Graph(len(keep), sub_edges, node_positions=tuple(tuple(pos[v]) for v in keep),
                 metadata={"seed": seed, "radius": radius, "attempts": _RGG_MAX_RETRIES,
                           "largest_component_of": n_nodes})


def pick_od_pair(graph: Graph) -> tuple[int, int]:
    """Most-connected origin, BFS-farthest destination (sysfn.py:244-269)."""
    degree = [0] * graph.n_nodes
    adj: list[list[int]] = [[] for _ in range(graph.n_nodes)]
    for u, v in graph.edges:
        degree[u] += 1
        degree[v] += 1
        adj[u].append(v)
        adj[v].append(u)
    origin = max(range(graph.n_nodes), key=lambda v: (degree[v], -v))
    dist = [-1] * graph.n_nodes
    dist[origin] = 0
    q = deque([origin])
    while q:
        u = q.popleft()
        for v in adj[u]:
            if dist[v] == -1:
                dist[v] = dist[u] + 1
                q.append(v)
    reach = max(d for d in dist if d >= 0)
    return origin, min(v for v in range(graph.n_nodes) if dist[v] == reach)


def build_graph_model(graph: Graph, performance: Callable, n_component_states: int = 2,
                      n_system_states: int = 2) -> SystemModel:
    """Wrap a graph performance function as a component-per-edge model (sysfn.py:272-284)."""
    return SystemModel(n_components=graph.n_edges, n_component_states=n_component_states,
                       n_system_states=n_system_states, performance=performance)
