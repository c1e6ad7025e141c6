"""rsr/1 persistence: interoperability with the reference's files.py."""

import json

import numpy as np
import pytest

import paper_2604_17066_b200 as P
from paper_2604_17066_b200 import files as F
from _specs import load_json


def _model_docs(tmp_path):
    grid = {"format": "rsr/1", "n_nodes": 4, "edges": [[0, 1], [1, 2], [2, 3], [3, 0], [0, 2]]}
    (tmp_path / "g.json").write_text(json.dumps(grid))
    return {
        "kofn": {"format": "rsr/1", "n_components": 3, "n_component_states": 3,
                 "n_system_states": 3, "distribution": [[0.2, 0.3, 0.5]] * 3,
                 "system_function": {"name": "k_out_of_n", "k": 2}},
        "st_inline": {"format": "rsr/1", "n_components": 5, "n_component_states": 2,
                      "n_system_states": 2, "distribution": [[0.1, 0.9]] * 5,
                      "system_function": {"name": "single_od_connectivity", "graph": grid,
                                          "origin": 0, "destination": 2}},
        "st_file_auto_od": {"format": "rsr/1", "n_components": 5, "n_component_states": 2,
                            "n_system_states": 2, "distribution": [[0.1, 0.9]] * 5,
                            "system_function": {"name": "single_od_connectivity",
                                                "graph_file": "g.json"}},
        "edk": {"format": "rsr/1", "n_components": 5, "n_component_states": 2,
                "n_system_states": 3, "distribution": [[0.1, 0.9]] * 5,
                "system_function": {"name": "edge_disjoint_level", "graph": grid,
                                    "max_level": 2}},
        "global": {"format": "rsr/1", "n_components": 5, "n_component_states": 2,
                   "n_system_states": 2, "distribution": [[0.1, 0.9]] * 5,
                   "system_function": {"name": "global_connectivity", "graph_file": "g.json"}},
    }


def test_model_files_load_like_the_reference(tmp_path, reference_rsr):
    from rsr import files as RF
    for name, doc in _model_docs(tmp_path).items():
        p = tmp_path / f"{name}.json"
        p.write_text(json.dumps(doc))
        m, d, h = F.load_model(p)
        rm, rd, rh = RF.load_model(p)
        assert h == rh == F.model_hash(doc), name
        assert (m.n_components, m.n_component_states, m.n_system_states) == (
            rm.n_components, rm.n_component_states, rm.n_system_states)
        assert np.array_equal(d.probs, rd.probs)
        if name == "st_file_auto_od":  # OD picked like the reference (files.py:146-149)
            from rsr.sysfn import pick_od_pair
            g = RF.load_graph(tmp_path / "g.json")
            assert (m.performance.source, m.performance.target) == pick_od_pair(g)


def test_model_file_validation_errors(tmp_path):
    docs = _model_docs(tmp_path)
    bad = dict(docs["kofn"], n_system_states=2)
    (tmp_path / "b1.json").write_text(json.dumps(bad))
    with pytest.raises(ValueError):
        F.load_model(tmp_path / "b1.json")
    bad = dict(docs["kofn"], format="rsr/0")
    (tmp_path / "b2.json").write_text(json.dumps(bad))
    with pytest.raises(ValueError):
        F.load_model(tmp_path / "b2.json")
    bad = dict(docs["st_inline"], n_components=4, distribution=[[0.1, 0.9]] * 4)
    (tmp_path / "b3.json").write_text(json.dumps(bad))
    with pytest.raises(ValueError):
        F.load_model(tmp_path / "b3.json")


def test_model_hash_ignores_presentation():
    doc = {"n_components": 2, "n_component_states": 2, "n_system_states": 2,
           "distribution": [[0.5, 0.5]] * 2, "system_function": {"name": "k_out_of_n", "k": 1}}
    assert F.model_hash(doc) == F.model_hash(dict(doc, manifest={"x": 1}, format="rsr/1"))
    assert F.model_hash(doc) != F.model_hash(dict(doc, n_system_states=3))


def test_saved_sets_load_in_the_reference(tmp_path, reference_rsr):
    from rsr import files as RF
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, np.array([[0, 1, 1], [1, 0, 1]]), trusted=True)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, np.array([[1, 1, 1]]), trusted=True)
    path = tmp_path / "refs.json"
    F.save_reference_sets(path, lo, up, "abc123", seed=7)
    rl, ru = RF.load_reference_sets(path, "abc123")
    assert rl.members == lo.members and ru.members == up.members
    doc = json.loads(path.read_text())
    assert doc["format"] == "rsr/1" and doc["lower"]["seed"] == 7
    with pytest.raises(ValueError):
        F.load_reference_sets(path, "other-model")
    with pytest.raises(ValueError):
        F.save_reference_sets(tmp_path / "x.json", lo, P.ReferenceSet(P.Side.UPPER, 1), "h")


def test_graph_round_trip(tmp_path, reference_rsr):
    from rsr import files as RF
    g = P.random_geometric_graph(12, 0.4, seed=1)
    F.save_graph(tmp_path / "g.json", g)
    rg = RF.load_graph(tmp_path / "g.json")
    assert rg.edges == g.edges and rg.n_nodes == g.n_nodes
    assert F.load_graph(tmp_path / "g.json").edges == g.edges


@pytest.mark.gpu
def test_reference_written_sets_load_with_insert_semantics():
    # tests/golden/refsets.json: files written by the reference (one clean, one with
    # duplicates and dominated vectors) and the member lists the reference loaded
    for case in load_json("refsets.json"):
        import os
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "r.json")
            with open(p, "w") as f:
                json.dump(case["file"], f)
            lo, up = F.load_reference_sets(p, case["file"]["model_hash"])
        assert [list(v) for v in lo.members] == case["lower"]
        assert [list(v) for v in up.members] == case["upper"]
