"""(2)+(5) Dominance classification and estimates (mirror of reference ``classify.py``).

``classify`` keeps the reference signature and semantics (classify.py:187-249):
lower takes precedence over upper, ``strict`` raises on overlap,
``explain`` records the first matching reference per sample.  The work is
done on the device:

* default (``method="tc"``): ``rsr_classify_fp4`` -- thermometer contraction
  on block-scaled FP4 tcgen05 tensor cores (kind::mxf4, exact for 0/1
  operands, twice the int8 rate) with the any-zero epilogue fused, the S x K
  violation matrix never materialised; rows wider than the FP4 kernel keeps
  resident use the int8 kernel, wider still the bit-packed one;
* ``method="tc8"``: ``rsr_classify_tc`` -- the same contraction on int8
  tcgen05 tensor cores (comparison variant);
* ``method="bits"``: ``rsr_classify_bits`` -- bit-packed AND/OR-reduce on CUDA
  cores (comparison variant);
* first-match indices (``explain`` / ``strict``) come from the same kernels'
  epilogues (``*_explain`` entry points);
* then ``rsr_finalize`` (labels + counts) and, lazily, ``rsr_compact``
  (order-preserving index arrays, np.flatnonzero semantics).

``chunk_size`` and ``n_workers`` are accepted for API compatibility; the
results are invariant to them as in the reference (the device kernels tile
internally).
"""

from __future__ import annotations

import math
import os
from typing import TYPE_CHECKING

import numpy as np
import torch

from . import _abi, _device
from .boundary import ReferenceSet, Side
from .encoding import EncodedBatch
from .sampling import SampleBatch

if TYPE_CHECKING:  # pragma: no cover
    pass

__all__ = ["ClassificationResult", "InconsistentReferenceSets", "violation_counts", "classify",
           "cov", "DEFAULT_CHUNK_SIZE", "classify_flags", "classify_host", "classify_host_encoded"]

DEFAULT_CHUNK_SIZE = 65536
# widest thermometer row the tensor-core kernel keeps resident (6 x 128 bytes);
# wider rows (N(M-1) > ~760) go to the bit-packed kernel
TC_MAX_KPAD = 768


class InconsistentReferenceSets(ValueError):
    """A sample matched both a lower and an upper reference in strict mode."""


_FP4_EXACT: dict[int, bool] = {}


def _fp4_pair_selfcheck(rng) -> None:
    """Known answer for the paired accumulators (csrc/classify_fp4.cu kSfbHiCol): the
    second tile of a buffer counts in bits 16..23 of the fp32 accumulator, which leaves
    the denormal range once that count reaches 128.  N = 250 rows (4 K-steps), 481
    references with up to 250 ones (counts 0..~250 in both halves, the three tiles an
    odd count), paired kernel forced, flags compared with the bit-packed kernel.  On a
    mismatch pairing is switched off for the process (RSR_FP4_PAIR=0)."""
    import os
    n, h, k = 250, 512, 481
    x = (rng.random((h, n)) < 0.5).astype(np.uint8)
    up = np.zeros((k, n), dtype=np.uint8)
    for j in range(k):
        w = (1 + j % 3) if j % 2 else 150 + j % 100
        up[j, rng.choice(n, size=w, replace=False)] = 1
    x[:64] = rng.random((64, n)) < 0.1  # mostly-failed samples: counts of 128..249
    x[64:, :5] = 1  # some samples dominate some sparse references
    batch = SampleBatch(_device.to_device(x), 0, 0, state_bound=2)
    uset = ReferenceSet.from_array(Side.UPPER, 0, up, trusted=True)
    prev = os.environ.get("RSR_FP4_PAIR")
    os.environ["RSR_FP4_PAIR"] = "force"
    try:
        f4, _, _ = classify_flags(batch, None, uset, 2, "fp4")
    finally:
        if prev is None:
            del os.environ["RSR_FP4_PAIR"]
        else:
            os.environ["RSR_FP4_PAIR"] = prev
    fb, _, _ = classify_flags(batch, None, uset, 2, "bits")
    if not np.array_equal(f4.cpu().numpy(), fb.cpu().numpy()):
        import warnings
        warnings.warn("FP4 paired-accumulator self-check failed: pairing disabled",
                      RuntimeWarning)
        os.environ["RSR_FP4_PAIR"] = "0"
        return
    # shared tail (rsr_classify_fp4_tail): references using 210 of the 250 components, so
    # the compacted rows have 211 columns = 192 main + a 19-column tail shared per tile pair
    # (per-K-block A scales); on mismatch the shared tail is switched off
    n2 = 295  # 160-byte rows, so the compaction to 128 bytes applies
    tup = np.zeros((k, n2), dtype=np.uint8)
    tup[:, :n] = up
    tup[:, 210:] = 0
    tup[:8, :210] = 1  # every support column used
    x2 = np.ones((h, n2), dtype=np.uint8)
    x2[:, :n] = x
    batch = SampleBatch(_device.to_device(x2), 0, 0, state_bound=2)
    tset = ReferenceSet.from_array(Side.UPPER, 0, tup, trusted=True)
    saved = {k: os.environ.get(k) for k in ("RSR_FP4_PAIR", "RSR_FP4_COMPACT", "RSR_FP4_TAIL")}
    os.environ.update(RSR_FP4_PAIR="force", RSR_FP4_COMPACT="force", RSR_FP4_TAIL="1")
    try:
        plan = fp4_compaction(h, n2, 2, None, tset)
        used = plan is not None and plan.tail_tn > 0
        ft, _, _ = classify_flags(batch, None, tset, 2, "fp4")
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    fbt, _, _ = classify_flags(batch, None, tset, 2, "bits")
    if not used or not np.array_equal(ft.cpu().numpy(), fbt.cpu().numpy()):
        import warnings
        warnings.warn("FP4 shared-tail self-check failed: shared tail disabled", RuntimeWarning)
        os.environ["RSR_FP4_TAIL"] = "0"


def fp4_exact() -> bool:
    """Known-answer self-check of the FP4 classifier, once per device.

    The FP4 kernel reads violation counts out of fp32 *denormals* (scale factors
    2^-127 x 2^-22 make every 0/1 product 2^-149; csrc/classify_fp4.cu), so a part
    or driver that flushed accumulator denormals would read every count as 0 and
    label every sample a hit.  This runs the FP4 kernel on 512 samples x 2 x 240
    references whose minimum violation counts include exactly 1 (the smallest
    denormal) and compares its hit flags with the bit-packed CUDA-core kernel's.
    On a mismatch the default classifier (``method="tc"``) uses the int8 tcgen05
    kernel instead -- on the device, there is no CPU fallback.
    ``RSR_FP4_SELFCHECK=fail`` forces the failure branch (tests)."""
    dev = _device.device()
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    ok = _FP4_EXACT.get(key)
    if ok is not None:
        return ok
    import os
    if os.environ.get("RSR_FP4_SELFCHECK") == "fail":
        _FP4_EXACT[key] = False
        return False
    rng = np.random.default_rng(20260419)
    n, h, k = 64, 512, 240
    x = (rng.random((h, n)) < 0.5).astype(np.uint8)
    x[0], x[1] = 0, 1
    up = np.zeros((k, n), dtype=np.uint8)
    lo = np.ones((k, n), dtype=np.uint8)
    for j in range(k):  # 1-3 ones (upper) / zeros (lower): many counts of exactly 1
        up[j, rng.choice(n, size=1 + j % 3, replace=False)] = 1
        lo[j, rng.choice(n, size=1 + j % 3, replace=False)] = 0
    batch = SampleBatch(_device.to_device(x), 0, 0, state_bound=2)
    lset = ReferenceSet.from_array(Side.LOWER, 0, lo, trusted=True)
    uset = ReferenceSet.from_array(Side.UPPER, 0, up, trusted=True)
    f4, _, _ = classify_flags(batch, lset, uset, 2, "fp4")
    fb, _, _ = classify_flags(batch, lset, uset, 2, "bits")
    got, want = f4.cpu().numpy(), fb.cpu().numpy()
    # the data must exercise count-1 non-hits on both sides
    min_up = (up[None, :, :] & (1 - x[:, None, :])).sum(2).min(1)
    min_lo = ((1 - lo[None, :, :]) & x[:, None, :]).sum(2).min(1)
    assert (min_up == 1).any() and (min_lo == 1).any() and (want == 3).any()
    ok = bool(np.array_equal(got, want))
    if ok:
        _fp4_pair_selfcheck(rng)
    _FP4_EXACT[key] = ok
    if not ok:
        import warnings
        warnings.warn("FP4 classifier self-check failed (accumulator denormals not exact on "
                      "this device): using the int8 tcgen05 classifier", RuntimeWarning)
    return ok


def violation_counts(samples: EncodedBatch, refs: EncodedBatch, chunk_size: int = DEFAULT_CHUNK_SIZE,
                     method: str = "packed") -> np.ndarray:
    """Full H x R violation matrix (classify.py:57-96), ``rsr_violation_counts_rows``."""
    if samples.kind != "sample":
        raise ValueError("samples batch must have kind='sample'")
    if refs.kind not in ("lower_ref", "upper_ref"):
        raise ValueError("refs batch must have kind 'lower_ref' or 'upper_ref'")
    if (samples.n_components, samples.n_states) != (refs.n_components, refs.n_states):
        raise ValueError("samples and refs must share N and M")
    if len(refs) == 0:
        raise ValueError("refs batch is empty")
    if chunk_size < 1:
        raise ValueError("chunk_size must be >= 1")
    if method not in ("packed", "unpacked"):
        raise ValueError("method must be 'packed' or 'unpacked'")
    h, r = len(samples), len(refs)
    out = torch.empty((max(h, 1), r), dtype=torch.int32, device=_device.device())
    if h:
        _abi.call("rsr_violation_counts_rows", _abi.ptr(samples.device_rows()), h,
                  _abi.ptr(refs.device_rows()), r, samples.data.shape[1], _abi.ptr(out),
                  _device.stream())
    return out[:h].cpu().numpy()


class ClassificationResult:
    """Partition of sample indices plus probability estimates (classify.py:151-184).

    Counts are host integers; the index arrays are compacted on the device
    and copied to the host on first access.
    """

    def __init__(self, lower_indices=None, upper_indices=None, unclassified_indices=None,
                 n_samples: int = 0, first_match_lower=None, first_match_upper=None, *,
                 counts: tuple[int, int, int] | None = None, labels: torch.Tensor | None = None):
        self.n_samples = int(n_samples)
        self.first_match_lower = first_match_lower
        self.first_match_upper = first_match_upper
        self._labels = labels
        self._idx = {0: lower_indices, 1: upper_indices, 2: unclassified_indices}
        if counts is None:
            counts = tuple(int(np.asarray(self._idx[k]).size) for k in range(3))
        self.counts = tuple(int(c) for c in counts)
        self._dev_idx: dict[int, torch.Tensor] = {}

    @property
    def labels_device(self) -> torch.Tensor | None:
        """uint8 labels on the device: 0 lower, 1 upper, 2 unclassified."""
        return self._labels

    def indices_device(self, label: int) -> torch.Tensor:
        """Sorted int64 indices with the given label, compacted on the device."""
        t = self._dev_idx.get(label)
        if t is None:
            if self._labels is None:
                t = _device.to_device(np.asarray(self._idx[label], dtype=np.int64))
            else:
                n = self.counts[label]
                S = self.n_samples
                t = torch.empty(max(n, 1), dtype=torch.int64, device=self._labels.device)
                cnt = torch.empty(1, dtype=torch.int64, device=self._labels.device)
                scratch = torch.empty(_abi.call("rsr_compact_scratch", S), dtype=torch.int64,
                                      device=self._labels.device)
                _abi.call("rsr_compact", _abi.ptr(self._labels), S, label, _abi.ptr(t), _abi.ptr(cnt),
                          _abi.ptr(scratch), _device.stream())
                t = t[:n]
            self._dev_idx[label] = t
        return t

    def _host(self, label: int) -> np.ndarray:
        v = self._idx[label]
        if v is None:
            v = self.indices_device(label).cpu().numpy()
            self._idx[label] = v
        return np.asarray(v)

    @property
    def lower_indices(self) -> np.ndarray:
        return self._host(0)

    @property
    def upper_indices(self) -> np.ndarray:
        return self._host(1)

    @property
    def unclassified_indices(self) -> np.ndarray:
        return self._host(2)

    @property
    def p_lower(self) -> float:
        return self.counts[0] / self.n_samples

    @property
    def p_upper(self) -> float:
        return self.counts[1] / self.n_samples

    @property
    def p_unclassified(self) -> float:
        return self.counts[2] / self.n_samples

    @property
    def cov_lower(self) -> float | None:
        return cov(self.p_lower, self.n_samples)

    @property
    def cov_upper(self) -> float | None:
        return cov(self.p_upper, self.n_samples)


# Support compaction (csrc/fp4_compact.cu): a thermometer column in which no reference of
# a side is 1 adds nothing to that side's violation counts, so the FP4 contraction may run
# over the side's column support only.  It pays when the K-steps it saves on the tensor
# cores outweigh re-packing the sample planes (HBM): the plan below compares the two.
# RSR_FP4_COMPACT: "1" (default) cost model, "0" never, "force" whenever columns drop
_FP4_COMPACT = os.environ.get("RSR_FP4_COMPACT", "1")
_MMA_OPS_PER_S = 8.8e15     # kind::mxf4 rate of the classifier's issued K-steps
_REPACK_BYTES_PER_S = 2.5e12  # gather kernel: read + write of the sample planes


def _fp4_step_cost(cq: int) -> float:
    """Classifier time per reference tile in K-step units for rows of cq 64-column K-steps.
    Below 5 K-steps a tile's MMAs no longer cover the accumulator round trip (commit ->
    epilogue TMEM load -> release -> issuer, two buffers), so the time stops shrinking
    in proportion (cfg4, tools/compact_tile_sweep.sh: issued-MMA fraction 0.98 at 5
    K-steps, 0.855 at 4, 0.69 at 3)."""
    return {1: 3.5, 2: 4.0, 3: 4.35, 4: 4.68}.get(cq, cq / 0.98)
_COLS_DEV: dict = {}


class Fp4Compaction:
    """Column maps (bias column kdim last) of the non-empty sides and the compacted row
    width; ``cols[side]`` is host int32, ``dev[side]`` the device copy."""

    def __init__(self, row_bytes: int, cols: dict):
        self.row_bytes = row_bytes
        self.cols = cols
        self.tail_tn = 0  # > 0: shared-tail layout (rsr_classify_fp4_tail) of tile_n tiles
        self.n_pad = 0
        self.tail_cols = None  # (sample map, reference map)
        self.tail_checked, self.tail_ok = -1, False  # batch size the plan was checked for
        self.dev = {}
        for side, c in cols.items():
            key = (_device.device().index, c.tobytes())
            t = _COLS_DEV.get(key)
            if t is None:
                if len(_COLS_DEV) > 64:
                    _COLS_DEV.clear()
                t = torch.from_numpy(c).to(_device.device())
                _COLS_DEV[key] = t
            self.dev[side] = t


def fp4_compaction(n_samples: int, n_components: int, n_states: int,
                   lower_set: ReferenceSet | None, upper_set: ReferenceSet | None,
                   force: bool | None = None, want_first: bool = False) -> Fp4Compaction | None:
    """The support-compaction plan of one FP4 classification, or None when it would not
    save time (``force`` True / False overrides the cost model; RSR_FP4_COMPACT=0 turns
    it off).  Labels, first matches and counts are the same either way."""
    if force is None:
        mode = os.environ.get("RSR_FP4_COMPACT", _FP4_COMPACT)
        if mode == "0":
            return None
        if mode == "force":
            force = True
    if force is False:
        return None
    rb = _abi.fp4_row_bytes(n_components, n_states)
    kdim = n_components * (n_states - 1)
    cols, k_total, rb_out = {}, 0, 32
    for side, s in ((Side.LOWER, lower_set), (Side.UPPER, upper_set)):
        if s is None or not len(s):
            continue
        sup = s.device_fp4_support(n_states)
        c = np.concatenate([sup, np.array([kdim], dtype=np.int32)]).astype(np.int32)
        cols[side] = c
        k_total += len(s)
        rb_out = max(rb_out, (c.size + 63) // 64 * 32)
    if not cols or rb_out >= rb:
        return None
    if force is None:
        saved = (n_samples * k_total * 128 / _MMA_OPS_PER_S *
                 (_fp4_step_cost(rb // 32) - _fp4_step_cost(rb_out // 32)))
        cost = n_samples * len(cols) * (rb + rb_out) / _REPACK_BYTES_PER_S + 20e-6
        if saved <= cost:
            return None
    plan = Fp4Compaction(rb_out, cols)
    if not want_first and list(cols) == [Side.UPPER] and rb_out == 128:
        _fp4_tail_layout(plan, n_samples, len(upper_set), n_components * (n_states - 1))
    return plan


def _fp4_tail_layout(plan: Fp4Compaction, n_samples: int, n_refs: int, kdim: int) -> None:
    """Shared-tail layout (csrc/classify_fp4.cu PAIR = 3) when the compacted upper rows have
    193..224 columns and the library pairs this set's accumulators: 192 main columns (the
    bias first) plus a tail of <= 32 that tile pairs share in one MMA (7 MMAs per pair
    instead of 8, and the odd tiles stream 3 of their 4 K-steps: cfg4 K = 5x10^5 121.3 ->
    118.5 ms, profiles/r2_pair_sweep.txt).  RSR_FP4_TAIL=0 turns it off."""
    c = plan.cols[Side.UPPER]
    if os.environ.get("RSR_FP4_TAIL", "1") == "0" or not (192 < c.size <= 224):
        return
    tn, _, paired = _abi.fp4_plan_ex(n_samples, 0, n_refs, 128)
    if not paired:
        return
    n_pad = -(-n_refs // (2 * tn)) * 2 * tn
    tn2, _, paired2 = _abi.fp4_plan_ex(n_samples, 0, n_pad, 128)
    if not paired2 or tn2 != tn:
        return
    sup = c[:-1]
    main = np.concatenate([np.array([kdim], np.int32), sup[:191]])
    tail = np.full(32, -1, np.int32)
    tail[: sup.size - 191] = sup[191:]
    plan.tail_tn, plan.n_pad = tn, n_pad
    plan.tail_checked, plan.tail_ok = n_samples, True
    plan.tail_cols = (np.concatenate([main, tail, tail]).astype(np.int32),
                      np.concatenate([main, tail, np.full(32, -1, np.int32)]).astype(np.int32))
    key = (_device.device().index, plan.tail_cols[0].tobytes())
    t = _COLS_DEV.get(key)
    if t is None:
        t = torch.from_numpy(plan.tail_cols[0]).to(_device.device())
        _COLS_DEV[key] = t
    plan.dev["tail"] = t


def fp4_classify_compacted(plan: Fp4Compaction, a: torch.Tensor, plane: int, n_samples: int,
                           row_bytes: int, n_states: int, lower_set, upper_set,
                           flags: torch.Tensor, first_lower=None, first_upper=None,
                           out: torch.Tensor | None = None, accumulate: int = 0,
                           events=None) -> None:
    """Re-pack the samples over the plan's column maps and run the classifier on them
    (rsr_classify_fp4_tail for the shared-tail layout, else rsr_classify_fp4_planar).
    ``events``: optional (re-pack start, classifier start) CUDA events (bench.py)."""
    st = _device.stream()
    H = n_samples
    if events:
        events[0].record()
    tail = plan.tail_tn > 0
    if tail and H != plan.tail_checked:
        # the library re-plans per call: the shared-tail layout needs the same paired plan
        # for this batch size (host-fed chunks are smaller than the job)
        tn, _, paired = _abi.fp4_plan_ex(H, 0, plan.n_pad, 128)
        plan.tail_ok = paired and tn == plan.tail_tn
        plan.tail_checked = H
    if tail and plan.tail_ok:
        if out is None or out.numel() < H * 128:
            out = torch.empty((1, max(H, 1), 128), dtype=torch.uint8, device=a.device)
        stride = row_bytes if plane else 2 * row_bytes
        c = plan.dev["tail"]
        _abi.call("rsr_fp4_gather_columns", _abi.ptr(a), stride, H, row_bytes, _abi.ptr(c),
                  c.numel(), _abi.ptr(out), 128, 128, st)
        bu = upper_set.device_fp4_tail(n_states, plan.tail_cols[1], plan.tail_tn, plan.n_pad)
        if events:
            events[1].record()
        _abi.call("rsr_classify_fp4_tail", _abi.ptr(out), H * 128, H, _abi.ptr(bu), plan.n_pad,
                  128, plan.tail_tn, _abi.ptr(flags), accumulate, st)
        return
    a2, pl2, rb2, (bl, nl, al), (bu, nu, au) = fp4_compact_operands(
        plan, a, plane, H, row_bytes, n_states, lower_set, upper_set, out=out)
    if events:
        events[1].record()
    _abi.call("rsr_classify_fp4_planar", _abi.ptr(a2), pl2, H, None, _abi.ptr(bl), nl, al,
              _abi.ptr(bu), nu, au, rb2, _abi.ptr(flags), _abi.ptr(first_lower),
              _abi.ptr(first_upper), accumulate, st)


def fp4_compact_operands(plan: Fp4Compaction, a: torch.Tensor, plane: int, n_samples: int,
                         row_bytes: int, n_states: int, lower_set, upper_set,
                         out: torch.Tensor | None = None):
    """Gather the sample planes (planar output [2, H, rb_out]) and the reference rows over
    the plan's column maps.  Returns (A, plane_stride, row_bytes, (bl, nl, al), (bu, nu, au))
    for rsr_classify_fp4_planar."""
    rbo = plan.row_bytes
    H = n_samples
    planes = 2 if Side.LOWER in plan.cols else 1  # upper alone reads only the A_up plane
    if out is None or out.numel() < planes * H * rbo:
        out = torch.empty((planes, max(H, 1), rbo), dtype=torch.uint8, device=a.device)
    st = _device.stream()
    stride = row_bytes if plane else 2 * row_bytes
    lo_off = plane if plane else row_bytes
    base, obase = _abi.ptr(a), _abi.ptr(out)
    for side, off, ooff in ((Side.UPPER, 0, 0), (Side.LOWER, lo_off, H * rbo)):
        if side in plan.dev:
            c = plan.dev[side]
            _abi.call("rsr_fp4_gather_columns", base + off, stride, H, row_bytes, _abi.ptr(c),
                      c.numel(), obase + ooff, rbo, rbo, st)
    bl = (lower_set.device_fp4_compact(n_states, plan.cols[Side.LOWER], rbo)
          if Side.LOWER in plan.cols else (None, 0, 0))
    bu = (upper_set.device_fp4_compact(n_states, plan.cols[Side.UPPER], rbo)
          if Side.UPPER in plan.cols else (None, 0, 0))
    return out, H * rbo, rbo, bl, bu


def _infer_n_states(batch: SampleBatch, lower_set, upper_set) -> int:
    """Largest state in samples or refs + 1 (classify.py:252-262)."""
    if batch._host is not None:
        top = int(batch._host.max(initial=0))
    else:
        top = int(batch.device_states().max().item()) if batch.n_samples else 0
    for s in (lower_set, upper_set):
        if s is not None and len(s):
            top = max(top, s.max_state)
    return top + 1


def _check_range(batch: SampleBatch, sets, n_states: int) -> None:
    """encode_batch's range check (encoding.py:35-39) without a host copy when avoidable."""
    if batch.state_bound > n_states:
        top = (int(batch._host.max(initial=0)) if batch._host is not None
               else int(batch.device_states().max().item()))
        if top >= n_states:
            raise ValueError(f"states must lie in [0, {n_states - 1}]")
    for s in sets:
        if s is not None and len(s) and s.max_state >= n_states:
            raise ValueError(f"states must lie in [0, {n_states - 1}]")


def classify_flags(batch: SampleBatch, lower_set: ReferenceSet | None,
                   upper_set: ReferenceSet | None, n_states: int, method: str = "tc",
                   flags: torch.Tensor | None = None, want_first: bool = False):
    """Run one classifier; returns (flags[u8 H], first_lower, first_upper) on device."""
    H = batch.n_samples
    dev = _device.device()
    if flags is None:
        flags = torch.empty(H, dtype=torch.uint8, device=dev)
    m_eff = max(2, n_states, batch.state_bound)
    fl = fu = None
    st = _device.stream()
    if method not in ("tc", "tc8", "fp4", "bits"):
        raise ValueError("method must be 'tc', 'tc8', 'fp4' or 'bits'")
    rb4 = _abi.fp4_row_bytes(batch.n_components, m_eff)
    fp4_ok = rb4 <= _abi.FP4_MAX_ROW_BYTES
    if fp4_ok and rb4 > _abi.REFSET_MAX_ROW_BYTES:
        # the widest rows: ask the planner whether a tile width fits shared memory (768-byte
        # rows with first matches do not); otherwise the int8 / bit-packed kernels run
        nl0 = len(lower_set) if lower_set is not None else 0
        nu0 = len(upper_set) if upper_set is not None else 0
        fp4_ok = _abi.fp4_plan(H, nl0, nu0, rb4, want_first)[0] > 0
    tc_ok = _abi.thermo_kpad(batch.n_components, m_eff) <= TC_MAX_KPAD
    if fp4_ok and (method == "fp4" or (method == "tc" and fp4_exact())):
        a = batch.fp4(m_eff)
        plane = batch.fp4_plane_stride(m_eff)
        rb = _abi.fp4_row_bytes(batch.n_components, m_eff)
        cplan = fp4_compaction(H, batch.n_components, m_eff, lower_set, upper_set,
                               want_first=want_first)
        if cplan is not None:
            if want_first:
                fl = torch.empty(H, dtype=torch.int64, device=dev)
                fu = torch.empty(H, dtype=torch.int64, device=dev)
            fp4_classify_compacted(cplan, a, plane, H, rb, m_eff, lower_set, upper_set, flags,
                                   fl, fu)
            return flags, fl, fu
        else:
            bl, nl, al = lower_set.device_fp4_rows(m_eff) if lower_set is not None else (None, 0, 0)
            bu, nu, au = upper_set.device_fp4_rows(m_eff) if upper_set is not None else (None, 0, 0)
        if want_first:
            fl = torch.empty(H, dtype=torch.int64, device=dev)
            fu = torch.empty(H, dtype=torch.int64, device=dev)
        if plane:
            _abi.call("rsr_classify_fp4_planar", _abi.ptr(a), plane, H, None, _abi.ptr(bl), nl, al,
                      _abi.ptr(bu), nu, au, rb, _abi.ptr(flags), _abi.ptr(fl), _abi.ptr(fu), 0, st)
        else:
            _abi.call("rsr_classify_fp4_ex", _abi.ptr(a), H, None, _abi.ptr(bl), nl, al,
                      _abi.ptr(bu), nu, au, rb, _abi.ptr(flags), _abi.ptr(fl), _abi.ptr(fu), 0, st)
    elif method in ("tc", "tc8", "fp4") and tc_ok:
        a = batch.thermo(m_eff)
        bl, nl = lower_set.device_thermo(m_eff) if lower_set is not None else (None, 0)
        bu, nu = upper_set.device_thermo(m_eff) if upper_set is not None else (None, 0)
        if want_first:  # first-match indices from the tensor-core epilogue
            fl = torch.empty(H, dtype=torch.int64, device=dev)
            fu = torch.empty(H, dtype=torch.int64, device=dev)
            _abi.call("rsr_classify_tc_explain", _abi.ptr(a), H, _abi.ptr(bl), nl, _abi.ptr(bu),
                      nu, a.shape[1], _abi.ptr(flags), _abi.ptr(fl), _abi.ptr(fu), 0, st)
        else:
            _abi.call("rsr_classify_tc", _abi.ptr(a), H, _abi.ptr(bl), nl, _abi.ptr(bu), nu,
                      a.shape[1], _abi.ptr(flags), 0, st)
    else:
        sb = batch.thermo_bits(m_eff)
        lb, nl = lower_set.device_bits(m_eff) if lower_set is not None else (None, 0)
        ub, nu = upper_set.device_bits(m_eff) if upper_set is not None else (None, 0)
        if want_first:
            fl = torch.empty(H, dtype=torch.int64, device=dev)
            fu = torch.empty(H, dtype=torch.int64, device=dev)
        _abi.call("rsr_classify_bits", _abi.ptr(sb), H, _abi.ptr(lb), nl, _abi.ptr(ub), nu,
                  sb.shape[1], _abi.ptr(flags), _abi.ptr(fl), _abi.ptr(fu), 0, st)
    return flags, fl, fu


def classify(batch: SampleBatch, lower_set: ReferenceSet | None, upper_set: ReferenceSet | None,
             chunk_size: int = DEFAULT_CHUNK_SIZE, n_workers: int = 1, strict: bool = False,
             explain: bool = False, n_states: int | None = None, *,
             method: str = "tc") -> ClassificationResult:
    """Partition a sample batch against lower and upper reference sets (classify.py:187-249)."""
    if lower_set is not None and upper_set is not None:
        if lower_set.threshold != upper_set.threshold:
            raise ValueError(f"threshold mismatch: lower m'={lower_set.threshold}, "
                             f"upper m'={upper_set.threshold}")
    if lower_set is not None and lower_set.side != Side.LOWER:
        raise ValueError("lower_set must have side 'lower'")
    if upper_set is not None and upper_set.side != Side.UPPER:
        raise ValueError("upper_set must have side 'upper'")
    if not isinstance(batch, SampleBatch):
        raise TypeError("batch must be a SampleBatch")
    for s in (lower_set, upper_set):
        if s is not None and len(s) and s._width != batch.n_components:
            raise ValueError("reference vectors and samples must share N")
    H = batch.n_samples
    if n_states is None:
        n_states = _infer_n_states(batch, lower_set, upper_set)
    else:
        _check_range(batch, (lower_set, upper_set), n_states)
    want_first = bool(explain or strict)
    flags, fl, fu = classify_flags(batch, lower_set, upper_set, n_states, method,
                                   want_first=want_first)
    dev = flags.device
    labels = torch.empty(H, dtype=torch.uint8, device=dev)
    counts_d = torch.empty(4, dtype=torch.int64, device=dev)
    _abi.call("rsr_finalize", _abi.ptr(flags), H, _abi.ptr(labels), _abi.ptr(counts_d),
              _device.stream())
    counts = counts_d.cpu().tolist()
    if strict and counts[3] > 0:
        idx = torch.empty(counts[3], dtype=torch.int64, device=dev)
        cnt = torch.empty(1, dtype=torch.int64, device=dev)
        scratch = torch.empty(_abi.call("rsr_compact_scratch", H), dtype=torch.int64, device=dev)
        _abi.call("rsr_compact", _abi.ptr(flags), H, _abi.HIT_LOWER | _abi.HIT_UPPER, _abi.ptr(idx),
                  _abi.ptr(cnt), _abi.ptr(scratch), _device.stream())
        first = int(idx[0].item())
        raise InconsistentReferenceSets(
            f"sample {first} matches both a lower and an upper reference")
    return ClassificationResult(
        n_samples=H, counts=(counts[0], counts[1], counts[2]), labels=labels,
        first_match_lower=fl.cpu().numpy() if (explain and fl is not None) else None,
        first_match_upper=fu.cpu().numpy() if (explain and fu is not None) else None)


def classify_host(states, lower_set: ReferenceSet | None, upper_set: ReferenceSet | None,
                  n_states: int, *, chunk_rows: int | None = None,
                  labels_out: torch.Tensor | None = None,
                  method: str = "tc") -> tuple[torch.Tensor, tuple[int, int, int]]:
    """Classify host-resident uint8 samples, streaming them through the GPU.

    ``states`` is a (preferably pinned) host uint8 tensor/array [S, N].  Chunks
    are copied on a side stream while the previous chunk is encoded and
    classified (rsr_encode_samples_fp4 + rsr_classify_fp4; ``method="tc8"``:
    rsr_encode_samples + rsr_classify_tc), then rsr_finalize runs once and the
    uint8 labels (0 lower / 1 upper / 2 unclassified) come back into
    ``labels_out`` (host).  Returns (labels_out, counts).
    """
    host = states if isinstance(states, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(states))
    if host.dtype != torch.uint8 or host.dim() != 2:
        raise ValueError("states must be a uint8 S x N host matrix")
    if method not in ("tc", "tc8"):
        raise ValueError("method must be 'tc' or 'tc8'")
    return _classify_host_stream(host, host.shape[1], n_states, lower_set, upper_set, chunk_rows,
                                 labels_out, "tc8" if method == "tc8" else "states")


def classify_host_encoded(packed, n_components: int, lower_set: ReferenceSet | None,
                          upper_set: ReferenceSet | None, n_states: int, *,
                          chunk_rows: int | None = None,
                          labels_out: torch.Tensor | None = None
                          ) -> tuple[torch.Tensor, tuple[int, int, int]]:
    """Classify host samples given in the reference's own classification input:
    rows of ``encode_batch(states, M, "sample").packed`` (encoding.py:82-98, the
    packed one-hot rows classify.py:42-44 consumes; ceil(N*M/8) bytes per row).
    Same streaming as ``classify_host``; the device decodes each chunk straight
    into the FP4 operand (rsr_unpack_onehot_fp4)."""
    host = packed if isinstance(packed, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(packed))
    m_eff = max(2, n_states)
    if host.dtype != torch.uint8 or host.dim() != 2 or host.shape[1] != (n_components * m_eff + 7) // 8:
        raise ValueError("packed must be a uint8 S x ceil(N*M/8) host matrix")
    return _classify_host_stream(host, n_components, n_states, lower_set, upper_set, chunk_rows,
                                 labels_out, "onehot")


_STREAM_CACHE: dict = {}


def _stream_buffers(dev, chunk, width_in, opnd_shape, opnd_dtype):
    """Copy stream, double buffers and events of the host-fed path, reused across
    calls with the same geometry (creating them per call costs more than a chunk)."""
    key = (dev.index, chunk, width_in, opnd_shape, opnd_dtype)
    ent = _STREAM_CACHE.get(key)
    if ent is None:
        if len(_STREAM_CACHE) > 4:
            _STREAM_CACHE.clear()
        ent = (torch.cuda.Stream(),
               [torch.empty((chunk, width_in), dtype=torch.uint8, device=dev) for _ in range(2)],
               [torch.empty((chunk,) + opnd_shape, dtype=opnd_dtype, device=dev) for _ in range(2)],
               [torch.cuda.Event() for _ in range(2)], [torch.cuda.Event() for _ in range(2)])
        _STREAM_CACHE[key] = ent
    # the previous call's copies and kernels must be done with the buffers
    ent[0].wait_stream(torch.cuda.current_stream())
    return ent


def _classify_host_stream(host, N, n_states, lower_set, upper_set, chunk_rows, labels_out, mode):
    S = host.shape[0]
    width_in = host.shape[1]
    dev = _device.device()
    m_eff = max(2, n_states)
    for s in (lower_set, upper_set):
        if s is not None and len(s) and s.max_state >= m_eff:
            raise ValueError(f"states must lie in [0, {n_states - 1}]")
    fp4 = mode != "tc8" and _abi.fp4_row_bytes(N, m_eff) <= _abi.FP4_MAX_ROW_BYTES
    if mode == "onehot" and not fp4:
        raise ValueError("encoded input needs the FP4 classifier (N(M-1) <= 831)")
    if fp4 and not fp4_exact():
        if mode == "onehot":
            raise RuntimeError("encoded input needs the FP4 classifier, whose self-check "
                               "failed on this device")
        fp4 = False  # int8 tcgen05 classifier
    if fp4:
        width = _abi.fp4_row_bytes(N, m_eff)
        opnd_shape, opnd_dtype = (2 * width,), torch.uint8
        bl, nl, al = lower_set.device_fp4_rows(m_eff) if lower_set is not None else (None, 0, 0)
        bu, nu, au = upper_set.device_fp4_rows(m_eff) if upper_set is not None else (None, 0, 0)
        # support compaction: each encoded chunk is re-packed over the sides' column
        # supports before the classifier (fp4_compaction decides for the whole job)
        cplan = fp4_compaction(S, N, m_eff, lower_set, upper_set)
    else:
        width = _abi.thermo_kpad(N, m_eff)
        if width > TC_MAX_KPAD:
            raise ValueError("rows too wide for the tensor-core classifiers")
        opnd_shape, opnd_dtype = (width,), torch.int8
        bl, nl = lower_set.device_thermo(m_eff) if lower_set is not None else (None, 0)
        bu, nu = upper_set.device_thermo(m_eff) if upper_set is not None else (None, 0)
    comp = torch.cuda.current_stream()
    wave = 256 * max(1, _abi.device_sm_count() // 2)  # one sample group per CTA pair
    if chunk_rows is None:
        # whole waves of the persistent classifier, 16 per chunk.  A chunk of 2^16 rows
        # is 256 groups = 3.46 waves of 74 pairs, so a quarter of every chunk's last wave
        # idled (cfg4 K = 5x10^5 e2e: 183 ms for a 151 ms kernel).  The first chunks ramp
        # up from one wave (1, 2, 4, 8, 16): the copy of the first chunk is the part of
        # the transfer nothing overlaps
        chunk_rows = 16 * wave
        sizes, tot, k = [], 0, 1
        while tot < S:
            n = min(k * wave, chunk_rows, S - tot)
            sizes.append(n)
            tot += n
            k = min(2 * k, 16)
    else:
        sizes = [min(chunk_rows, S - lo) for lo in range(0, S, chunk_rows)]
    chunk = max(1, min(chunk_rows, S))
    copy, bufs, opnd, ready, free = _stream_buffers(dev, chunk, width_in, opnd_shape, opnd_dtype)
    # encoded chunks are planar (A_up plane, A_lo plane of `chunk` rows): a one-sided
    # classification streams only its half
    plane = chunk * width if (fp4 and mode != "onehot") else 0
    flags = torch.empty(max(S, 1), dtype=torch.uint8, device=dev)
    st = _device.stream()
    cbuf = None
    if fp4 and cplan is not None:  # one buffer: the gather and the classifier share `comp`
        cbuf = torch.empty((2, chunk, cplan.row_bytes), dtype=torch.uint8, device=dev)
    lo = 0
    for i, n_rows in enumerate(sizes):
        hi = lo + n_rows
        slot = i & 1
        with torch.cuda.stream(copy):
            if i >= 2:
                copy.wait_event(free[slot])
            bufs[slot][: hi - lo].copy_(host[lo:hi], non_blocking=True)
            ready[slot].record(copy)
        comp.wait_event(ready[slot])
        if mode == "onehot":
            _abi.call("rsr_unpack_onehot_fp4", _abi.ptr(bufs[slot]), hi - lo, N, m_eff,
                      _abi.ptr(opnd[slot]), width, st)
        elif fp4:
            _abi.call("rsr_encode_samples_fp4_ex", _abi.ptr(bufs[slot]), hi - lo, N, m_eff,
                      _abi.ptr(opnd[slot]), width, plane, st)
        else:
            _abi.call("rsr_encode_samples", _abi.ptr(bufs[slot]), hi - lo, N, m_eff,
                      _abi.ptr(opnd[slot]), width, st)
        if cbuf is not None:
            fp4_classify_compacted(cplan, opnd[slot], plane, hi - lo, width, m_eff, lower_set,
                                   upper_set, flags[lo:hi], out=cbuf)
        elif fp4 and plane:
            _abi.call("rsr_classify_fp4_planar", _abi.ptr(opnd[slot]), plane, hi - lo, None,
                      _abi.ptr(bl), nl, al, _abi.ptr(bu), nu, au, width, _abi.ptr(flags[lo:hi]),
                      None, None, 0, st)
        elif fp4:
            _abi.call("rsr_classify_fp4_ex", _abi.ptr(opnd[slot]), hi - lo, None, _abi.ptr(bl), nl,
                      al, _abi.ptr(bu), nu, au, width, _abi.ptr(flags[lo:hi]), None, None, 0, st)
        else:
            _abi.call("rsr_classify_tc", _abi.ptr(opnd[slot]), hi - lo, _abi.ptr(bl), nl,
                      _abi.ptr(bu), nu, width, _abi.ptr(flags[lo:hi]), 0, st)
        free[slot].record(comp)
        lo = hi
    labels = torch.empty(max(S, 1), dtype=torch.uint8, device=dev)
    counts_d = torch.empty(4, dtype=torch.int64, device=dev)
    _abi.call("rsr_finalize", _abi.ptr(flags), S, _abi.ptr(labels), _abi.ptr(counts_d), st)
    if labels_out is None:
        labels_out = torch.empty(S, dtype=torch.uint8, pin_memory=True)
    labels_out[:S].copy_(labels[:S], non_blocking=True)
    counts = counts_d.cpu().tolist()  # synchronises the stream
    return labels_out, (counts[0], counts[1], counts[2])


def cov(p_hat: float, n_samples: int) -> float | None:
    """sqrt((1 - p) / (H p)); None at p = 0 (classify.py:265-277)."""
    if n_samples < 1:
        raise ValueError("n_samples must be >= 1")
    if not 0.0 <= p_hat <= 1.0:
        raise ValueError("p_hat must lie in [0, 1]")
    if p_hat == 0.0:
        return None
    return math.sqrt((1.0 - p_hat) / (n_samples * p_hat))
