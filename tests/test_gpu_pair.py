"""Paired accumulators in the FP4 classifier (csrc/classify_fp4.cu, kSfbHiCol).

Rows of at most 4 K-steps (N(M-1) < 256) classified without first matches can run two
reference tiles per TMEM accumulator buffer (by default: streamed sets at 4 K-steps;
RSR_FP4_PAIR=force pairs every such plan, which these tests use): the second tile's products carry 2^16, so
each accumulator holds c1 + 2^16 c2.  Labels must equal the unpaired kernel
(RSR_FP4_PAIR=0), the bit-packed kernel and the oracle (classify.py:121-148) for

* odd and even tile counts per side (the last buffer of a side may hold one tile),
* one- and two-sided calls, resident and streamed / chunked reference sets,
* reference buffers without pad rows (columns past the last reference masked),
* the largest counts the trick allows (255 violated columns, samples all-failed),
* 1..4 K-steps (N = 40 .. 255 at M = 2, M = 3 and 4).
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2604_17066_b200 as P
from paper_2604_17066_b200 import _abi, _device

pytestmark = pytest.mark.gpu


def _refs(rng, k, n, m, density, side):
    r = rng.integers(1, m, size=(k, n)) * (rng.random((k, n)) < density)
    return r if side == "upper" else (m - 1) - r


def _classify(batch, lo, up, m, pair, monkeypatch, method="tc"):
    """pair: False (unpaired), True / 16 (c1 + 2^16 c2), 8 (packed c1 + 2^8 c2)."""
    monkeypatch.setenv("RSR_FP4_PAIR", "force" if pair else "0")
    monkeypatch.setenv("RSR_FP4_PAIR8", "1" if pair == 8 else "0")
    monkeypatch.setenv("RSR_FP4_COMPACT", "0")
    r = P.classify(batch, lo, up, n_states=m, method=method)
    return r.labels_device.cpu().numpy(), r.counts


@pytest.mark.parametrize("n,m,kl,ku,p_top", [
    (40, 2, 0, 1, 0.9), (40, 2, 300, 500, 0.9), (200, 2, 0, 449, 0.95),
    (200, 2, 225, 225, 0.95), (255, 2, 673, 0, 0.9), (100, 3, 1000, 1300, 0.8),
    (63, 4, 224, 447, 0.8), (200, 2, 0, 20_000, 0.97), (120, 2, 9000, 7001, 0.96)])
def test_paired_equals_unpaired_bits_and_oracle(n, m, kl, ku, p_top, monkeypatch):
    rng = np.random.default_rng(n * 1000 + kl + ku)
    assert _abi.fp4_row_bytes(n, m) <= 128  # <= 4 K-steps: the paired kernel runs
    lo_rows = _refs(rng, kl, n, m, 6.0 / n, "lower") if kl else np.zeros((0, n), np.int64)
    up_rows = _refs(rng, ku, n, m, 6.0 / n, "upper") if ku else np.zeros((0, n), np.int64)
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lo_rows, trusted=True)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, up_rows, trusted=True)
    probs = np.full(m, (1 - p_top) / (m - 1))
    probs[-1] = p_top
    d = P.ComponentDistribution.iid(n, probs.tolist())
    b = P.sample_batch(d, 70_001, seed=n + m)
    paired, cp = _classify(b, lo, up, m, True, monkeypatch)
    paired8, cp8 = _classify(b, lo, up, m, 8, monkeypatch)
    plain, c0 = _classify(b, lo, up, m, False, monkeypatch)
    bits, cb = _classify(b, lo, up, m, False, monkeypatch, method="bits")
    assert np.array_equal(paired, plain) and cp == c0
    assert np.array_equal(paired8, plain) and cp8 == c0
    assert np.array_equal(paired, bits)
    xs = b.device_states()[:1500].cpu().numpy()
    want = oracle.classify_labels(xs, lo_rows, up_rows, m)
    assert np.array_equal(paired[:1500], want["labels"])


@pytest.mark.parametrize("n,k", [(40, 1), (40, 225), (255, 449), (160, 3000)])
def test_paired_unpadded_reference_buffers(n, k, monkeypatch):
    """rsr_classify_fp4 on reference buffers of exactly k rows (no never-hit pad rows):
    the TMA box reads zeros past row k and the paired epilogue masks both halves."""
    dev = _device.device()
    rng = np.random.default_rng(k)
    up_rows = _refs(rng, k, n, 2, 5.0 / n, "upper").astype(np.uint8)
    rb = _abi.fp4_row_bytes(n, 2)
    bu = torch.empty((k, rb), dtype=torch.uint8, device=dev)
    st = torch.from_numpy(up_rows).to(dev)
    _abi.call("rsr_encode_refs_fp4", _abi.ptr(st), k, k, n, 2, _abi.SIDE_UPPER, _abi.ptr(bu), rb,
              _device.stream())
    d = P.ComponentDistribution.iid(n, [0.05, 0.95])
    b = P.SampleBatch(P.sample_batch(d, 9001, seed=k).device_states().clone(), k, 0, state_bound=2)
    a = b.fp4(2)
    plane = b.fp4_plane_stride(2)
    out = {}
    for pair in ("force", "force8", "0"):
        monkeypatch.setenv("RSR_FP4_PAIR", pair[:5])
        monkeypatch.setenv("RSR_FP4_PAIR8", "1" if pair == "force8" else "0")
        flags = torch.empty(9001, dtype=torch.uint8, device=dev)
        _abi.call("rsr_classify_fp4_planar", _abi.ptr(a), plane, 9001, None, None, 0, 0,
                  _abi.ptr(bu), k, k, rb, _abi.ptr(flags), None, None, 0, _device.stream())
        out[pair] = flags.cpu().numpy()
    assert np.array_equal(out["force"], out["0"]) and np.array_equal(out["force8"], out["0"])
    want = oracle.classify_labels(b.device_states()[:2000].cpu().numpy(),
                                  np.zeros((0, n), np.int64), up_rows, 2)
    got = np.where(out["force"][:2000] & _abi.HIT_UPPER, 1, 2)
    assert np.array_equal(got, want["labels"])


def test_paired_largest_counts(monkeypatch):
    """N = 255, M = 2: an all-ones upper reference against all-zero samples violates all
    255 columns (c = 255 in both halves of a buffer, the most the trick allows), next to
    references the samples do dominate."""
    n = 255
    up_rows = np.ones((480, n), dtype=np.uint8)
    up_rows[::7] = 0  # every 7th reference all zero: dominated by every sample
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, up_rows, trusted=True)
    lo = P.ReferenceSet(P.Side.LOWER, 0)
    states = np.zeros((4096, n), dtype=np.uint8)
    states[::2, ::3] = 1
    b = P.SampleBatch(states, 0, 0)
    for mode in (16, 8):
        paired, cp = _classify(b, lo, up, 2, mode, monkeypatch)
        assert cp[1] == 4096 and (paired == 1).all()
        up2 = P.ReferenceSet.from_array(P.Side.UPPER, 0, np.ones((481, n), np.uint8), trusted=True)
        paired2, cp2 = _classify(b, lo, up2, 2, mode, monkeypatch)
        plain2, _ = _classify(b, lo, up2, 2, False, monkeypatch)
        assert cp2[1] == 0 and np.array_equal(paired2, plain2)


def test_plan_reports_paired_widths(monkeypatch):
    """The launch-plan query never picks a width without TMEM room for the second scale
    when the paired kernel applies (RSR_FP4_PAIR=force: every plan of rows <= 4 K-steps;
    by default only streamed sets at 4 K-steps, e.g. config 4's 5x10^5 paths)."""
    monkeypatch.setenv("RSR_FP4_PAIR", "force")
    for k in (1, 224, 1000, 30_000, 500_000):
        tn, launches = _abi.fp4_plan(1 << 22, 0, k, 128)
        assert tn in (176, 192, 208, 224) and launches >= 1


def test_paired_selfcheck_passes(monkeypatch):
    """classify._fp4_pair_selfcheck (run by fp4_exact on first use): counts of 128..249 in
    the second tile of a buffer (fp32 normal range) read back exactly, so pairing stays on."""
    import importlib
    import os
    C = importlib.import_module("paper_2604_17066_b200.classify")
    monkeypatch.delenv("RSR_FP4_PAIR", raising=False)
    monkeypatch.delenv("RSR_FP4_TAIL", raising=False)
    C._fp4_pair_selfcheck(np.random.default_rng(20260419))
    assert os.environ.get("RSR_FP4_PAIR") is None  # pairing stays on
    assert os.environ.get("RSR_FP4_TAIL") is None  # and the shared tail
