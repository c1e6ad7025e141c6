"""Pin the CPU oracle against golden vectors produced by the reference itself.

The fixtures come from ``tests/golden/make_golden.py`` run against the
reference package in the build container; these tests run anywhere (CPU).
"""

import numpy as np
import pytest

import oracle
from _specs import load_json, load_npz, oracle_phi


def test_philox_raw_and_uniform_golden():
    g = load_npz("philox.npz")
    for i, (seed, gen, first, count) in enumerate(g["cases"]):
        assert np.array_equal(oracle.random_raw(seed, gen, first, count), g[f"raw{i}"])
    for i, c in enumerate(g["ucases"]):
        assert np.array_equal(oracle.uniform_field(*c), g[f"uniform{i}"])


def test_survey_appendix_a_vectors():
    # Philox(key=[123, 0]).random_raw(8) and uniform_field(123,0,0,2,3)
    want = [0x845a748f4852c9a3, 0x2f0d8aae69b255ba, 0x367c80c2347e0a9b, 0x35c08aae20fba324,
            0x5ce186961ac0d00e, 0x1b371a64654599de, 0xed174403995b0bdc, 0x76205c46ff469dd2]
    assert [int(v) for v in oracle.random_raw(123, 0, 0, 8)] == want
    u = oracle.uniform_field(123, 0, 0, 2, 3)
    assert u.tolist() == [[0.5170052385149787, 0.18380038030745394, 0.2128372644551676],
                          [0.20996920348350878, 0.3628162495103908, 0.10630955649437224]]


def test_philox_matches_numpy_bit_generator():
    for seed, gen in [(0, 0), (5, 9), (2**64 - 1, 2**63)]:
        bg = np.random.Philox(key=np.array([seed, gen], dtype=np.uint64))
        bg.advance(3)
        assert np.array_equal(bg.random_raw(50), oracle.random_raw(seed, gen, 12, 50))


def test_sampling_golden():
    g = load_npz("sampling.npz")
    for i, (n, seed, gen, start) in enumerate(g["specs"]):
        got = oracle.sample_states(g[f"probs{i}"], n, seed, gen, start)
        assert np.array_equal(got, g[f"states{i}"])


def test_classify_golden():
    g = load_npz("classify.npz")
    for i, m in enumerate(g["n_states"]):
        r = oracle.classify_labels(g[f"samples{i}"], g[f"lower{i}"], g[f"upper{i}"], int(m),
                                   want_first=True)
        assert np.array_equal(r["lower_indices"], g[f"lo_idx{i}"])
        assert np.array_equal(r["upper_indices"], g[f"up_idx{i}"])
        assert np.array_equal(r["unclassified_indices"], g[f"un_idx{i}"])
        assert np.array_equal(r["first_lower"], g[f"first_lo{i}"])
        assert np.array_equal(r["first_upper"], g[f"first_up{i}"])
    for kind in ("lower_ref", "upper_ref"):
        got = oracle.violation_counts(g["viol_samples"], g["viol_refs"], 3, kind)
        assert np.array_equal(got, g[f"viol_{kind}"])


def test_boundary_golden():
    for rec in load_json("boundary.json"):
        if rec["model"] == "fig_space":
            phi, n, m, ms = oracle.phi_cones([[(1, 4), (4, 0), (3, 2)]]), 2, 5, 2
        else:
            phi, n, m, ms = oracle.phi_cones(rec["levels"]), rec["n"], rec["m"], rec["ms"]
        ev = oracle.CountingPhi(phi, n, m, ms)
        vec, side = oracle.boundary_search(ev, rec["x0"], rec["threshold"])
        assert list(vec) == rec["vector"] and side == rec["side"] and ev.count == rec["evals"]


@pytest.mark.parametrize("case", [c["spec"]["name"] for c in load_json("workflow.json")])
def test_workflow_golden(case):
    rec = next(c for c in load_json("workflow.json") if c["spec"]["name"] == case)
    spec = rec["spec"]
    phi, n = oracle_phi(spec["model"])
    ev = oracle.CountingPhi(phi, n, spec["model"]["m"], spec["model"]["ms"])
    probs = np.array(spec["probs"])
    cfg = dict(spec["config"])
    for st in rec["stages"]:
        thr = st["threshold"]
        s1 = oracle.stage1(ev, probs, thr, **cfg)
        want = st["stage1"]
        assert [list(v) for v in s1["lower"]] == want["lower"]
        assert [list(v) for v in s1["upper"]] == want["upper"]
        got_trace = [[t["reference_count"], t["phi_evaluations"], t["p_lower"], t["p_upper"],
                      t["p_unclassified"]] for t in s1["trace"]]
        assert got_trace == want["trace"]
        assert (s1["iterations"], s1["redundant_searches"], s1["terminated_by"]) == (
            want["iterations"], want["redundant_searches"], want["terminated_by"])
        assert ev.count == want["phi_total"]
        s2 = oracle.stage2(ev, probs, s1["lower"], s1["upper"], thr, cfg["n_samples"],
                           cfg.get("seed", 0))
        w2 = st["stage2"]
        for k in ("p_lower", "p_upper", "cov_lower", "cov_upper", "n_samples",
                  "unclassified_resolved"):
            assert s2[k] == w2[k], k
        assert ev.count == w2["phi_total"]


def test_pmf_golden():
    g = load_json("pmf.json")
    ev = oracle.CountingPhi(oracle.phi_kofn(2, 3), 3, 3, 3)
    rep = oracle.multistate_pmf(ev, np.tile([0.2, 0.3, 0.5], (3, 1)), n_samples=40_000,
                                eps_u=1e-3, r_max=200, seed=11)
    assert rep["pmf"].tolist() == g["pmf"]
    assert rep["cumulative_lower"].tolist() == g["cumulative_lower"]
    assert rep["max_chain_discrepancy"] == g["max_chain_discrepancy"]


def test_assemble_pmf_and_cov_known_answers():
    # reference test_workflow.py:103-120 and test_classify.py:205-213 known answers
    pmf, adj = oracle.assemble_pmf([0.2, 0.7])
    assert np.allclose(pmf, [0.2, 0.5, 0.3]) and adj == 0.0
    pmf, adj = oracle.assemble_pmf([2.47e-3, 1.04e-1])
    assert abs(pmf[1] - 1.02e-1) <= 5e-4 and abs(pmf[2] - 8.96e-1) <= 5e-4
    assert oracle.cov(1.0, 100) == 0.0
    assert oracle.cov(0.5, 100) == pytest.approx(0.1)
    assert oracle.cov(0.01, 1_000_000) == pytest.approx(0.0099498743710662, rel=1e-12)
    assert oracle.cov(0.0, 100) is None
    with pytest.raises(ValueError):
        oracle.cov(1.5, 100)
    with pytest.raises(ValueError):
        oracle.cov(0.5, 0)


def test_fast_sampler_equals_restatement():
    # the timing path draws with numpy's own Philox (as the reference does)
    probs = np.tile([0.2, 0.5, 0.3], (11, 1))
    for seed, gen, start in [(0, 0, 0), (5, 3, 17), (2**64 - 1, 2**40, 1001)]:
        a = oracle.sample_states(probs, 77, seed, gen, start)
        b = oracle.sample_states(probs, 77, seed, gen, start, fast=True)
        assert np.array_equal(a, b)


def test_stage1_time_budget_records_elapsed():
    ev = oracle.CountingPhi(oracle.phi_kofn(3, 3), 3, 2, 2)
    r = oracle.stage1(ev, np.tile([0.1, 0.9], (3, 1)), 0, 2000, eps_u=1e-3, r_max=50, seed=7,
                      time_budget=1e-9)
    assert r["terminated_by"] == "budget" and "elapsed" in r["trace"][0]


def test_device_stream_philox4x32_known_answers():
    # Random123 known-answer vectors of Philox4x32-10 (the independent device
    # stream, include/rsr_b200.h RSR_RNG_DEVICE, is not part of the reference)
    from oracle.philox import device_raw, philox4x32_blocks
    f = 0xFFFFFFFF
    kat = [((0, 0, 0, 0, 0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((f, f, f, f, f, f), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for args, want in kat:
        assert tuple(int(v) for v in philox4x32_blocks(*args)) == want
    # stream layout: draw (row R, component n) of (seed, gen) is word n % 4 of the block
    # with counter [n // 4, R lo, R hi, gen lo], key [seed lo ^ gen hi, seed hi]
    seed, gen = (1 << 63) + 12345, (1 << 40) + 7
    row, q = (1 << 33) + 5, 3
    blk = philox4x32_blocks(q, row & f, row >> 32, gen & f, (seed & f) ^ (gen >> 32), seed >> 32)
    got = device_raw(seed, gen, row - 1, 2, 14)
    assert got.shape == (2, 14) and np.array_equal(got[1, 12:], blk[:2])
    # rows are whole blocks: row R's draws do not depend on N beyond truncation
    assert np.array_equal(device_raw(seed, gen, row, 1, 9)[0], device_raw(seed, gen, row, 1, 14)[0, :9])
    # the generation's high word feeds the key, so gen and gen + 2^32 differ
    assert not np.array_equal(device_raw(1, 5, 0, 1, 8), device_raw(1, 5 + (1 << 32), 0, 1, 8))
    # inverse CDF at 2^-32 resolution on the same fp64 cumsum
    probs = np.array([[0.25, 0.5, 0.25], [0.1, 0.0, 0.9]])
    xs = oracle.sample_states(probs, 1000, 3, 2, 17, rng="device")
    raw = device_raw(3, 2, 17, 1000, 2).astype(np.float64)
    cum = np.cumsum(probs, axis=1)
    want = np.minimum((raw[:, :, None] >= np.ceil(cum * 2.0 ** 32)[None]).sum(2), 2)
    assert np.array_equal(xs, want)
    with pytest.raises(ValueError):
        oracle.sample_states(probs, 4, 0, rng="numpy")
