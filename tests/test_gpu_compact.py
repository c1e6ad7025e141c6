"""Support compaction of the FP4 contraction (csrc/fp4_compact.cu, classify.fp4_compaction).

A thermometer column in which no reference of a side is 1 adds 0 to every violation
count of that side (classify.py:42-44 on the encodings of encoding.py:138-153), so the
FP4 classifier may run over each side's column support.  These tests check

* rsr_fp4_or_rows / rsr_fp4_gather_columns against numpy nibble arithmetic (ragged
  counts, strides, maps shorter than the output row, empty inputs);
* labels and first matches with compaction forced on equal compaction off, the
  bit-packed kernel and the oracle (classify.py:121-148 / 99-118): s-t path references
  (config 4's shape), multi-state rows with both sides present, interleaved and planar
  sample operands, a side whose support is empty (bias column only);
* the cost model: no compaction for small reference sets, compaction for config 4.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2604_17066_b200 as P
from paper_2604_17066_b200 import _abi, _device
import importlib
C = importlib.import_module("paper_2604_17066_b200.classify")
from paper_2604_17066_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _nibbles(rows: np.ndarray) -> np.ndarray:
    return np.stack([rows & 0xF, rows >> 4], axis=-1).reshape(rows.shape[0], 2 * rows.shape[1])


def _pack(nib: np.ndarray) -> np.ndarray:
    nib = nib.reshape(nib.shape[0], nib.shape[1] // 2, 2)
    return (nib[..., 0] | (nib[..., 1] << 4)).astype(np.uint8)


@pytest.mark.parametrize("count,src_rb,src_stride,dst_rb,n_cols", [
    (1, 160, 160, 128, 214), (1000, 160, 320, 128, 200), (4097, 96, 96, 64, 70),
    (63, 32, 48, 32, 64), (65, 384, 384, 160, 1), (300, 768, 768, 768, 1000), (130, 160, 160, 160, 0), (0, 160, 160, 128, 5)])
def test_gather_columns_matches_numpy(count, src_rb, src_stride, dst_rb, n_cols):
    dev = _device.device()
    rng = np.random.default_rng(count + n_cols)
    src = rng.integers(0, 256, size=(max(count, 1), src_stride), dtype=np.uint8)
    cols = np.sort(rng.choice(2 * src_rb, size=n_cols, replace=n_cols > 2 * src_rb)).astype(np.int32)
    s_d = torch.from_numpy(src).to(dev)
    c_d = torch.from_numpy(cols).to(dev)
    dst_stride = dst_rb + 16
    out = torch.full((max(count, 1), dst_stride), 0xAB, dtype=torch.uint8, device=dev)
    _abi.call("rsr_fp4_gather_columns", _abi.ptr(s_d), src_stride, count, src_rb, _abi.ptr(c_d),
              n_cols, _abi.ptr(out), dst_stride, dst_rb, _device.stream())
    got = out.cpu().numpy()[:count]
    nib = _nibbles(src[:count, :src_rb])
    want = np.zeros((count, 2 * dst_rb), dtype=np.uint8)
    want[:, :n_cols] = nib[:, cols]
    assert np.array_equal(got[:, :dst_rb], _pack(want))
    assert (got[:, dst_rb:] == 0xAB).all()  # bytes past the row untouched


def test_gather_columns_rejects_bad_arguments():
    dev = _device.device()
    a = torch.zeros((4, 160), dtype=torch.uint8, device=dev)
    c = torch.zeros(10, dtype=torch.int32, device=dev)
    with pytest.raises(ValueError):  # n_cols past the output row
        _abi.call("rsr_fp4_gather_columns", _abi.ptr(a), 160, 4, 160, _abi.ptr(c), 300,
                  _abi.ptr(a), 160, 128, _device.stream())
    with pytest.raises(ValueError):  # stride not a multiple of 16
        _abi.call("rsr_fp4_gather_columns", _abi.ptr(a), 100, 1, 96, _abi.ptr(c), 10,
                  _abi.ptr(a), 160, 128, _device.stream())


@pytest.mark.parametrize("rows,rb", [(1, 160), (239, 32), (500_000, 160), (0, 64)])
def test_or_rows_matches_numpy(rows, rb):
    dev = _device.device()
    rng = np.random.default_rng(rows)
    b = (rng.random((max(rows, 1), rb)) < (3.0 / max(rows, 1))) * rng.integers(1, 256, (max(rows, 1), rb))
    b = b.astype(np.uint8)
    b_d = torch.from_numpy(b).to(dev)
    out = torch.full((rb // 4,), -1, dtype=torch.int32, device=dev)
    _abi.call("rsr_fp4_or_rows", _abi.ptr(b_d), rows, rb, _abi.ptr(out), _device.stream())
    want = np.bitwise_or.reduce(b[:rows], axis=0) if rows else np.zeros(rb, np.uint8)
    assert np.array_equal(np.frombuffer(out.cpu().numpy().tobytes(), np.uint8), want)


def _labels(batch, lo, up, m, force, want_first=False, monkeypatch=None):
    monkeypatch.setenv("RSR_FP4_COMPACT", "force" if force else "0")
    r = P.classify(batch, lo, up, n_states=m, method="tc", explain=want_first)
    return r.labels_device.cpu().numpy(), r.counts, r


@pytest.fixture(scope="module")
def paths():
    return W.random_st_paths(W.cfg3(0), 3000, seed=1)


@pytest.mark.parametrize("k", [1, 240, 3000])
def test_compacted_paths_equal_full_bits_and_oracle(paths, k, monkeypatch):
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, paths[:k], trusted=True)
    lo = P.ReferenceSet(P.Side.LOWER, 0)
    cols = up.device_fp4_support(2)
    assert np.array_equal(cols, np.flatnonzero(paths[:k].any(0)))
    d = P.ComponentDistribution.iid(295, [0.2, 0.8])
    b = P.sample_batch(d, 20_000, seed=3)
    full, cf, _ = _labels(b, lo, up, 2, False, monkeypatch=monkeypatch)
    comp, cc, _ = _labels(b, lo, up, 2, True, monkeypatch=monkeypatch)
    assert np.array_equal(full, comp) and cf == cc
    monkeypatch.setenv("RSR_FP4_COMPACT", "0")
    bits = P.classify(b, lo, up, n_states=2, method="bits").labels_device.cpu().numpy()
    assert np.array_equal(comp, bits)
    xs = b.device_states()[:3000].cpu().numpy()
    want = oracle.classify_labels(xs, np.zeros((0, 295), np.int64), paths[:k], 2)
    assert np.array_equal(comp[:3000], want["labels"])
    if k > 1:
        assert 0 < cc[1] < 20_000 and cc[2] > 0


@pytest.mark.parametrize("m", [2, 3, 4])
def test_compacted_two_sided_multistate_first_match(m, monkeypatch):
    """Both sides present with different supports (upper refs never touch the first 40
    components, lower refs never go below the top level on the last 60): labels and the
    first matching reference of each side are unchanged (classify.py:99-118)."""
    rng = np.random.default_rng(m)
    N, K = 150, 700
    up = rng.integers(0, m, size=(K, N)) * (rng.random((K, N)) < 0.04)
    up[:, :40] = 0
    lo = np.full((K, N), m - 1) - rng.integers(0, m, size=(K, N)) * (rng.random((K, N)) < 0.05)
    lo[:, -60:] = m - 1
    up_s = P.ReferenceSet.from_array(P.Side.UPPER, 0, up, trusted=True)
    lo_s = P.ReferenceSet.from_array(P.Side.LOWER, 0, lo, trusted=True)
    probs = np.full(m, 0.5 / (m - 1))
    probs[-1] = 0.5
    d = P.ComponentDistribution.iid(N, probs.tolist())
    b = P.sample_batch(d, 12_345, seed=m)
    plan = C.fp4_compaction(b.n_samples, N, m, lo_s, up_s, force=True)
    assert plan is not None and plan.row_bytes < _abi.fp4_row_bytes(N, m)
    monkeypatch.setenv("RSR_FP4_COMPACT", "0")
    r0 = P.classify(b, lo_s, up_s, n_states=m, method="tc", explain=True)
    monkeypatch.setenv("RSR_FP4_COMPACT", "force")
    r1 = P.classify(b, lo_s, up_s, n_states=m, method="tc", explain=True)
    assert np.array_equal(r0.labels_device.cpu().numpy(), r1.labels_device.cpu().numpy())
    assert r0.counts == r1.counts
    assert np.array_equal(np.asarray(r0.first_match_lower), np.asarray(r1.first_match_lower))
    assert np.array_equal(np.asarray(r0.first_match_upper), np.asarray(r1.first_match_upper))
    xs = b.device_states()[:2000].cpu().numpy()
    want = oracle.classify_labels(xs, lo, up, m)
    assert np.array_equal(r1.labels_device[:2000].cpu().numpy(), want["labels"])


def test_compacted_interleaved_operand_and_empty_support(monkeypatch):
    """An interleaved sample operand (batch.fp4(out=...)) and an upper side whose only
    member is all zeros (support = the bias column alone: every sample dominates it)."""
    N = 295
    d = P.ComponentDistribution.iid(N, [0.1, 0.9])
    b = P.SampleBatch(P.sample_batch(d, 5000, seed=9).device_states().clone(), 9, 0, state_bound=2)
    rb = _abi.fp4_row_bytes(N, 2)
    buf = torch.empty((5000, 2 * rb), dtype=torch.uint8, device=_device.device())
    b.fp4(2, out=buf)
    assert b.fp4_plane_stride(2) == 0
    rng = np.random.default_rng(0)
    lo_rows = np.ones((300, N), dtype=np.uint8)
    for r in lo_rows:
        r[rng.choice(N // 2, 12, replace=False)] = 0
    lo = P.ReferenceSet.from_array(P.Side.LOWER, 0, lo_rows, trusted=True)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, np.zeros((1, N), np.uint8), trusted=True)
    assert up.device_fp4_support(2).size == 0
    monkeypatch.setenv("RSR_FP4_COMPACT", "0")
    r0 = P.classify(b, lo, up, n_states=2, method="tc")
    monkeypatch.setenv("RSR_FP4_COMPACT", "force")
    r1 = P.classify(b, lo, up, n_states=2, method="tc")
    assert np.array_equal(r0.labels_device.cpu().numpy(), r1.labels_device.cpu().numpy())
    assert r1.counts[0] + r1.counts[1] == 5000 and r1.counts[1] > 0


def test_cost_model_picks_compaction_for_config4_only(paths):
    up_small = P.ReferenceSet.from_array(P.Side.UPPER, 0, paths[:500], trusted=True)
    # 3x10^4 rows (the fixture's paths repeated: duplicates are harmless here)
    up_big = P.ReferenceSet.from_array(P.Side.UPPER, 0, np.tile(paths, (10, 1)), trusted=True)
    assert C.fp4_compaction(1 << 22, 295, 2, None, up_small) is None
    plan = C.fp4_compaction(1 << 22, 295, 2, None, up_big)
    ncols = up_big.device_fp4_support(2).size + 1  # + bias column
    assert plan is not None and plan.row_bytes == (ncols + 63) // 64 * 32 < 160
    assert C.fp4_compaction(1 << 22, 295, 2, None, up_big, force=False) is None


@pytest.mark.parametrize("k,p1", [(60_001, 0.85), (100_000, 0.9)])
def test_shared_tail_layout_equals_plain_bits_and_oracle(k, p1, monkeypatch):
    """Shared-tail pairs (csrc/classify_fp4.cu PAIR = 3): 193..224 compacted columns, the
    last K-step of each tile pair shared by both tiles (per-K-block A scales), odd tile
    counts padded with a never-hit tile.  Labels equal the plain compacted kernel, the
    uncompacted one, the bit-packed kernel and the oracle."""
    paths = W.random_st_paths(W.cfg3(0), k, seed=0)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, paths, trusted=True)
    lo = P.ReferenceSet(P.Side.LOWER, 0)
    H = 1 << 16
    b = P.sample_batch(P.ComponentDistribution.iid(295, [1 - p1, p1]), H, seed=k)
    monkeypatch.setenv("RSR_FP4_COMPACT", "force")
    monkeypatch.setenv("RSR_FP4_TAIL", "1")
    plan = C.fp4_compaction(H, 295, 2, lo, up)
    assert plan is not None and plan.tail_tn > 0 and plan.n_pad % (2 * plan.tail_tn) == 0
    tail = P.classify(b, lo, up, n_states=2)
    monkeypatch.setenv("RSR_FP4_TAIL", "0")
    plain = P.classify(b, lo, up, n_states=2)
    monkeypatch.setenv("RSR_FP4_COMPACT", "0")
    full = P.classify(b, lo, up, n_states=2)
    bits = P.classify(b, lo, up, n_states=2, method="bits")
    t = tail.labels_device.cpu().numpy()
    assert np.array_equal(t, plain.labels_device.cpu().numpy())
    assert np.array_equal(t, full.labels_device.cpu().numpy())
    assert np.array_equal(t, bits.labels_device.cpu().numpy())
    assert tail.counts == full.counts and min(tail.counts[1], tail.counts[2]) > 0
    xs = b.device_states()[-2000:].cpu().numpy()
    want = oracle.classify_labels(xs, np.zeros((0, 295), np.int64), paths, 2)
    assert np.array_equal(t[-2000:], want["labels"])


def test_shared_tail_host_fed_chunks(monkeypatch):
    """classify_host with a shared-tail plan: the host-fed chunks are smaller than the job,
    so each chunk re-checks the library's plan and falls back to the plain compacted layout
    where it differs.  Labels equal the uncompacted classification."""
    from paper_2604_17066_b200.classify import classify_host
    paths = W.random_st_paths(W.cfg3(0), 60_001, seed=0)
    up = P.ReferenceSet.from_array(P.Side.UPPER, 0, paths, trusted=True)
    lo = P.ReferenceSet(P.Side.LOWER, 0)
    H = 300_001
    b = P.sample_batch(P.ComponentDistribution.iid(295, [0.12, 0.88]), H, seed=11)
    host = b.device_states().cpu().pin_memory()
    monkeypatch.setenv("RSR_FP4_COMPACT", "force")
    labels, counts = classify_host(host, lo, up, 2)
    monkeypatch.setenv("RSR_FP4_COMPACT", "0")
    want = P.classify(b, lo, up, n_states=2)
    assert np.array_equal(labels.numpy()[:H], want.labels_device.cpu().numpy())
    assert counts == want.counts
