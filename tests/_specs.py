"""Shared loaders for the golden fixtures (no reference import needed)."""

from __future__ import annotations

import json
import os

import numpy as np

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_npz(name: str):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=True)


def load_json(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def oracle_phi(spec_model: dict):
    """Oracle Phi (plain callable) of a workflow-case model spec."""
    m = spec_model
    if m["kind"] == "kofn":
        return oracle.phi_kofn(m["k"], m["n"]), m["n"]
    if m["kind"] == "st":
        edges = [tuple(e) for e in m["edges"]]
        return oracle.phi_st(m["n_nodes"], edges, m["s"], m["t"]), len(edges)
    if m["kind"] == "widest":
        edges = [tuple(e) for e in m["edges"]]
        return oracle.phi_widest(m["n_nodes"], edges, m["s"], m["t"], m["m"]), len(edges)
    if m["kind"] == "cones":
        return oracle.phi_cones(m["levels"]), m["n"]
    if m["kind"] == "edk":
        edges = [tuple(e) for e in m["edges"]]
        return oracle.phi_edge_disjoint(m["n_nodes"], edges, m["max_level"]), len(edges)
    raise ValueError(m["kind"])


def device_model(spec_model: dict):
    """Device SystemModel of a workflow-case model spec."""
    import paper_2604_17066_b200 as P
    m = spec_model
    if m["kind"] == "kofn":
        return P.SystemModel(m["n"], m["m"], m["ms"], P.k_out_of_n(m["k"], m["n"]))
    if m["kind"] in ("st", "widest"):
        g = P.Graph(m["n_nodes"], tuple(tuple(e) for e in m["edges"]))
        f = P.single_od_connectivity if m["kind"] == "st" else P.widest_path_level
        return P.SystemModel(len(m["edges"]), m["m"], m["ms"], f(g, m["s"], m["t"]))
    if m["kind"] == "cones":
        return P.SystemModel(m["n"], m["m"], m["ms"], P.cone_sum(m["levels"], m["n"]))
    if m["kind"] == "edk":
        g = P.Graph(m["n_nodes"], tuple(tuple(e) for e in m["edges"]))
        return P.SystemModel(len(m["edges"]), m["m"], m["ms"], P.edge_disjoint_level(g, m["max_level"]))
    raise ValueError(m["kind"])
