"""(4) Boundary search and non-dominated reference sets (mirror of reference ``boundary.py``).

``ReferenceSet`` keeps the reference's ordered member list semantics
(boundary.py:57-113) and mirrors it on the device: a uint8 state matrix plus,
per component-state count M, the packed e2m1 rows the FP4 tensor-core
classifier streams (``rsr_encode_refs_fp4``; rows padded to 240-row tiles with
never-hit rows), the int8 thermometer rows of the int8 variant
(``rsr_encode_refs``, 256-row tiles) and the packed bits of the CUDA-core
variant.  Appends encode only the
new rows; a drop (a new member dominating old ones) rebuilds the mirror.

Redundancy checks run on the device (``rsr_dominance_scan``), for a single
``insert`` as for the batched ``insert_batch`` used by the Stage-1 loop.
``boundary_search`` / ``boundary_search_batch`` run ``rsr_boundary_search``:
one warp per start vector, the reference's unit-step walk (boundary.py:
116-147) with the same evaluation count.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _abi, _device
from .model import SystemModel, validate_vector

__all__ = ["Side", "ReferenceState", "ReferenceSet", "boundary_search", "boundary_search_batch"]


class Side:
    LOWER = "lower"
    UPPER = "upper"


def _side_code(side: str) -> int:
    return _abi.SIDE_LOWER if side == Side.LOWER else _abi.SIDE_UPPER


@dataclass(frozen=True)
class ReferenceState:
    """(boundary.py:26-47)"""

    vector: tuple[int, ...]
    side: str
    threshold: int

    def __post_init__(self) -> None:
        if self.side not in (Side.LOWER, Side.UPPER):
            raise ValueError(f"side must be '{Side.LOWER}' or '{Side.UPPER}'")
        object.__setattr__(self, "vector", tuple(int(v) for v in self.vector))

    @classmethod
    def checked(cls, model: SystemModel, vector: Sequence[int], side: str,
                threshold: int) -> "ReferenceState":
        s = model.evaluate(vector)
        if side == Side.LOWER and s > threshold:
            raise ValueError(f"lower reference has system state {s} > m'={threshold}")
        if side == Side.UPPER and s <= threshold:
            raise ValueError(f"upper reference has system state {s} <= m'={threshold}")
        return cls(tuple(vector), side, threshold)


_TILE = 256  # reference rows per classifier tile (CTA-pair kernel: 2 x 128)
_TILE4 = _abi.FP4_TILE_ROWS  # reference rows per FP4 classifier tile (2 x 120)


class ReferenceSet:
    """Non-dominated set of reference vectors for one side and threshold."""

    def __init__(self, side: str, threshold: int, members: Iterable[Sequence[int]] = ()) -> None:
        if side not in (Side.LOWER, Side.UPPER):
            raise ValueError(f"side must be '{Side.LOWER}' or '{Side.UPPER}'")
        self.side = side
        self.threshold = int(threshold)
        self._rows = np.zeros((0, 0), dtype=np.uint8)  # capacity x N
        self._n = 0
        self._width: int | None = None
        self._max_state = -1
        self._dev_rows: torch.Tensor | None = None
        self._dev_n = 0
        self._thermo: dict[int, list] = {}  # M -> [tensor, encoded_rows]
        self._bits: dict[int, list] = {}
        self._fp4: dict[int, list] = {}  # M -> [tensor, encoded_rows]
        self._fp4c: dict = {}  # support-compaction caches (device_fp4_support / _compact)
        for m in members:
            self.insert(ReferenceState(tuple(m), side, threshold))

    # -- reference API -----------------------------------------------------
    @property
    def members(self) -> list[tuple[int, ...]]:
        return [tuple(int(v) for v in r) for r in self._rows[: self._n]]

    def __len__(self) -> int:
        return self._n

    def __contains__(self, vector: Sequence[int]) -> bool:
        if self._n == 0:
            return False
        v = np.asarray([int(x) for x in vector])
        if v.shape[0] != self._width:
            return False
        return bool(np.any(np.all(self._rows[: self._n] == v[None, :], axis=1)))

    def as_array(self) -> np.ndarray:
        if self._n == 0:
            return np.zeros((0, 0), dtype=np.int64)
        return self._rows[: self._n].astype(np.int64)

    def copy(self) -> "ReferenceSet":
        new = ReferenceSet(self.side, self.threshold)
        if self._n:
            new._set_rows(self._rows[: self._n].copy())
        return new

    def insert(self, candidate: ReferenceState) -> str:
        """Insert keeping non-dominance (boundary.py:87-108); device dominance scan."""
        if candidate.side != self.side:
            raise ValueError(f"candidate side {candidate.side!r} != set side {self.side!r}")
        if candidate.threshold != self.threshold:
            raise ValueError(f"candidate threshold {candidate.threshold} != set threshold "
                             f"{self.threshold}")
        vec = np.asarray(candidate.vector, dtype=np.int64)
        self._check_width(vec.shape[0])
        if vec.size and (vec.min() < 0 or vec.max() > 255):
            raise ValueError("reference states must lie in [0, 255]")
        row = vec.astype(np.uint8)[None, :]
        if self._n == 0:
            self._append_host(row)
            return "inserted"
        return self.insert_batch(_device.to_device(row), row)[0]

    # -- batched device insertion (Stage-1 hot path) ------------------------
    def insert_batch(self, cands_dev: torch.Tensor, cands_host: np.ndarray) -> list[str]:
        """Insert B candidates in order; same outcome as B sequential ``insert`` calls.

        Redundancy against the current members and the candidate x candidate
        relation come from two ``rsr_dominance_scan`` launches; the ordered
        list updates are then resolved exactly as boundary.py:100-108 does
        one candidate at a time (transitivity makes the pre-batch scan exact).
        """
        B = int(cands_host.shape[0])
        if B == 0:
            return []
        self._check_width(cands_host.shape[1])
        N = self._width
        side = _side_code(self.side)
        st = _device.stream()
        dev = cands_dev.device
        # covered [B] | covers [B] | rel [B x B] in one buffer: one device->host copy
        scan = torch.zeros(2 * B + B * B, dtype=torch.uint8, device=dev)
        covered, covers, rel = scan[:B], scan[B: 2 * B], scan[2 * B:].view(B, B)
        if self._n:
            mem = self.device_rows()
            _abi.call("rsr_dominance_scan", _abi.ptr(cands_dev), B, _abi.ptr(mem), self._n, N, side,
                      _abi.ptr(covered), _abi.ptr(covers), -1, None, st)
        if B > 1:
            _abi.call("rsr_dominance_scan", _abi.ptr(cands_dev), B, _abi.ptr(cands_dev), B, N, side,
                      None, None, -1, _abi.ptr(rel), st)
        scan_h = scan.cpu().numpy()
        covered_h = scan_h[:B].astype(bool)
        covers_h = scan_h[B: 2 * B].astype(bool)
        rel_h = scan_h[2 * B:].reshape(B, B)
        if not covers_h.any() and not np.tril(rel_h, -1).any():
            # common case (e.g. bulk loads of non-dominated sets): no candidate relates
            # to an earlier one and none drops a member -> inserted iff not covered
            keep = np.flatnonzero(~covered_h)
            if keep.size:
                idx = torch.as_tensor(keep, dtype=torch.int64, device=dev)
                self._append_device(cands_dev.index_select(0, idx), cands_host[keep])
            return ["redundant" if c else "inserted" for c in covered_h]
        outcome: list[str] = []
        inserted: list[int] = []
        alive: list[bool] = []
        drop_members = np.zeros(self._n, dtype=bool)
        for c in range(B):
            if covered_h[c] or any(rel_h[c, j] & 2 for j in inserted):
                outcome.append("redundant")
                continue
            if covers_h[c]:
                mask = torch.zeros(self._n, dtype=torch.uint8, device=dev)
                _abi.call("rsr_dominance_scan", _abi.ptr(cands_dev), B, _abi.ptr(self.device_rows()),
                          self._n, N, side, None, None, c, _abi.ptr(mask), st)
                drop_members |= mask.cpu().numpy().astype(bool)
            for pos, j in enumerate(inserted):
                if alive[pos] and (rel_h[c, j] & 1):
                    alive[pos] = False
            inserted.append(c)
            alive.append(True)
            outcome.append("inserted")
        keep_new = [j for j, a in zip(inserted, alive) if a]
        if drop_members.any() or len(keep_new) != len(inserted):
            old = self._rows[: self._n] if self._n else np.zeros((0, N), dtype=np.uint8)
            rows = np.concatenate([old[~drop_members],
                                   cands_host[keep_new].astype(np.uint8)], axis=0)
            self._set_rows(rows)
        elif keep_new:
            idx = torch.as_tensor(keep_new, dtype=torch.int64, device=dev)
            self._append_device(cands_dev.index_select(0, idx), cands_host[keep_new])
        return outcome

    # -- internals ---------------------------------------------------------
    def _check_width(self, n: int) -> None:
        if self._width is None:
            self._width = int(n)
        elif n != self._width:
            raise ValueError(f"reference vector length {n} != set width {self._width}")

    def _reserve(self, n_total: int) -> None:
        cap = self._rows.shape[0]
        if n_total > cap or self._rows.shape[1] != self._width:
            new_cap = max(64, n_total, 2 * cap)
            rows = np.zeros((new_cap, self._width), dtype=np.uint8)
            if self._n:
                rows[: self._n] = self._rows[: self._n]
            self._rows = rows

    def _append_host(self, rows: np.ndarray) -> None:
        self._check_width(rows.shape[1])
        self._reserve(self._n + rows.shape[0])
        self._rows[self._n: self._n + rows.shape[0]] = rows
        self._n += rows.shape[0]
        self._max_state = max(self._max_state, int(rows.max()) if rows.size else -1)

    def _append_device(self, rows_dev: torch.Tensor, rows_host: np.ndarray) -> None:
        before = self._n
        self._append_host(rows_host.astype(np.uint8))
        if self._dev_rows is not None and self._dev_n == before:
            self._ensure_dev_capacity(self._n)
            self._dev_rows[before: self._n].copy_(rows_dev)
            self._dev_n = self._n

    def _set_rows(self, rows: np.ndarray) -> None:
        """Replace the member list (after drops): the device mirror is rebuilt."""
        self._n = 0
        self._max_state = -1
        if rows.shape[0]:
            self._append_host(rows)
        self._dev_rows = None
        self._dev_n = 0
        self._thermo.clear()
        self._bits.clear()
        self._fp4.clear()
        self._fp4c.clear()

    def _ensure_dev_capacity(self, n: int) -> None:
        cap = 0 if self._dev_rows is None else self._dev_rows.shape[0]
        if n > cap:
            new = torch.empty((max(256, n, 2 * cap), self._width), dtype=torch.uint8,
                              device=_device.device())
            if self._dev_rows is not None and self._dev_n:
                new[: self._dev_n].copy_(self._dev_rows[: self._dev_n])
            self._dev_rows = new

    @property
    def max_state(self) -> int:
        return self._max_state

    def device_rows(self) -> torch.Tensor:
        """uint8 [n, N] device mirror of the members (uploads what is missing)."""
        if self._n == 0:
            return torch.empty((0, self._width or 0), dtype=torch.uint8, device=_device.device())
        if self._dev_rows is None or self._dev_n < self._n:
            self._ensure_dev_capacity(self._n)
            lo = self._dev_n
            self._dev_rows[lo: self._n].copy_(torch.from_numpy(self._rows[lo: self._n]))
            self._dev_n = self._n
        return self._dev_rows[: self._n]

    def device_thermo(self, n_states: int) -> tuple[torch.Tensor | None, int]:
        """int8 thermometer B rows (padded to 128-row tiles) and the member count."""
        if self._n == 0:
            return None, 0
        rows_dev = self.device_rows()
        N = self._width
        kpad = _abi.thermo_kpad(N, n_states)
        need = (self._n + _TILE - 1) // _TILE * _TILE
        ent = self._thermo.get(n_states)
        if ent is None or ent[0].shape[0] < need:
            cap = max(need, 2 * (ent[0].shape[0] if ent else 0), _TILE)
            cap = (cap + _TILE - 1) // _TILE * _TILE
            t = torch.empty((cap, kpad), dtype=torch.int8, device=rows_dev.device)
            if ent is not None and ent[1]:
                t[: ent[1]].copy_(ent[0][: ent[1]])
            ent = [t, ent[1] if ent else 0]
            self._thermo[n_states] = ent
        t, done = ent
        if done < self._n:
            _abi.call("rsr_encode_refs", _abi.ptr(rows_dev[done:]), self._n - done, need - done, N,
                      n_states, _side_code(self.side), _abi.ptr(t[done:]), kpad, _device.stream())
            ent[1] = self._n
        return t, self._n

    def device_fp4(self, n_states: int) -> tuple[torch.Tensor | None, int]:
        """FP4 B rows ([r < k] lower / [r >= k] upper as packed e2m1) and the number
        of rows to stream: the members padded to whole 240-row tiles with never-hit
        rows, so the classifier's epilogue needs no column masking."""
        if self._n == 0:
            return None, 0
        rows_dev = self.device_rows()
        N = self._width
        rb = _abi.fp4_row_bytes(N, n_states)
        need = (self._n + _TILE4 - 1) // _TILE4 * _TILE4
        ent = self._fp4.get(n_states)
        if ent is None or ent[0].shape[0] < need:
            cap = max(need, 2 * (ent[0].shape[0] if ent else 0), _TILE4)
            cap = (cap + _TILE4 - 1) // _TILE4 * _TILE4
            t = torch.empty((cap, rb), dtype=torch.uint8, device=rows_dev.device)
            if ent is not None and ent[1]:
                t[: ent[1]].copy_(ent[0][: ent[1]])
            ent = [t, ent[1] if ent else 0]
            self._fp4[n_states] = ent
        t, done = ent
        if done < self._n:
            _abi.call("rsr_encode_refs_fp4", _abi.ptr(rows_dev[done:]), self._n - done, need - done,
                      N, n_states, _side_code(self.side), _abi.ptr(t[done:]), rb, _device.stream())
            ent[1] = self._n
        return t, need

    def device_fp4_rows(self, n_states: int) -> tuple[torch.Tensor | None, int, int]:
        """FP4 B rows, the member count and the readable rows (members plus the
        never-hit tile padding) -- the (B, n, avail) triple of rsr_classify_fp4_ex."""
        t, need = self.device_fp4(n_states)
        return t, self._n, need

    def device_fp4_support(self, n_states: int) -> np.ndarray:
        """Thermometer columns (< kdim) in which some member's FP4 row is 1: the only
        columns that can add a violation for this side (classify.py:42-44), from an OR
        of the encoded rows on the device (rsr_fp4_or_rows).  Cached per member count."""
        key = ("support", n_states)
        ent = self._fp4c.get(key)
        if ent is not None and ent[0] == self._n:
            return ent[1]
        t, _ = self.device_fp4(n_states)
        kdim = self._width * (n_states - 1)
        if t is None:
            cols = np.zeros(0, dtype=np.int32)
        else:
            rb = t.shape[1]
            words = torch.empty(rb // 4, dtype=torch.int32, device=t.device)
            _abi.call("rsr_fp4_or_rows", _abi.ptr(t), self._n, rb, _abi.ptr(words), _device.stream())
            nib = np.frombuffer(words.cpu().numpy().tobytes(), dtype=np.uint8)
            nib = np.stack([nib & 0xF, nib >> 4], axis=1).reshape(-1)
            cols = np.flatnonzero(nib[:kdim]).astype(np.int32)
        self._fp4c[key] = (self._n, cols)
        return cols

    def device_fp4_compact(self, n_states: int, cols: np.ndarray, row_bytes: int
                           ) -> tuple[torch.Tensor | None, int, int]:
        """(B, n, avail) of device_fp4_rows over the column map ``cols`` (host int32,
        bias column kdim last) in rows of ``row_bytes`` (rsr_fp4_gather_columns);
        cached for one map per member count."""
        t, need = self.device_fp4(n_states)
        if t is None:
            return None, 0, 0
        key = ("compact", n_states)
        ent = self._fp4c.get(key)
        sig = (self._n, row_bytes, np.asarray(cols, dtype=np.int32).tobytes())
        if ent is not None and ent[0] == sig:
            return ent[1], self._n, need
        cols_dev = torch.from_numpy(np.asarray(cols, dtype=np.int32)).to(t.device)
        out = torch.empty((need, row_bytes), dtype=torch.uint8, device=t.device)
        _abi.call("rsr_fp4_gather_columns", _abi.ptr(t), t.shape[1], need, t.shape[1],
                  _abi.ptr(cols_dev), cols_dev.numel(), _abi.ptr(out), row_bytes, row_bytes,
                  _device.stream())
        self._fp4c[key] = (sig, out, cols_dev)
        return out, self._n, need

    def device_fp4_tail(self, n_states: int, cols: np.ndarray, tile_n: int, n_pad: int
                        ) -> torch.Tensor:
        """Reference rows in the shared-tail layout of rsr_classify_fp4_tail: the FP4 rows
        re-packed over ``cols`` ([bias + 191 main | 32 tail | 32 unused], host int32, -1 =
        empty), ``n_pad`` rows (whole pairs of ``tile_n``-row tiles; rows past the members
        never-hit), and in every even tile the last 16 bytes (columns 224..255) holding the
        next tile's tail (columns 192..223).  Cached for one layout per member count."""
        t, need = self.device_fp4(n_states)
        key = ("tail", n_states)
        sig = (self._n, tile_n, n_pad, np.asarray(cols, dtype=np.int32).tobytes())
        ent = self._fp4c.get(key)
        if ent is not None and ent[0] == sig:
            return ent[1]
        dev = t.device
        out = torch.zeros((n_pad, 128), dtype=torch.uint8, device=dev)
        out[:, 0] = 0x02  # never-hit pad rows: the bias column (column 0) only
        cols_dev = torch.from_numpy(np.asarray(cols, dtype=np.int32)).to(dev)
        rows = min(need, n_pad)
        _abi.call("rsr_fp4_gather_columns", _abi.ptr(t), t.shape[1], rows, t.shape[1],
                  _abi.ptr(cols_dev), cols_dev.numel(), _abi.ptr(out), 128, 128, _device.stream())
        v = out.view(n_pad // (2 * tile_n), 2, tile_n, 128)
        v[:, 0, :, 112:128] = v[:, 1, :, 96:112]
        self._fp4c[key] = (sig, out, cols_dev)
        return out

    def device_bits(self, n_states: int) -> tuple[torch.Tensor | None, int]:
        """Packed thermometer bits ([r < k] lower / [r >= k] upper) and count."""
        if self._n == 0:
            return None, 0
        rows_dev = self.device_rows()
        N = self._width
        w = _abi.thermo_words(N, n_states)
        ent = self._bits.get(n_states)
        if ent is None or ent[0].shape[0] < self._n:
            cap = max(self._n, 2 * (ent[0].shape[0] if ent else 0), 64)
            t = torch.empty((cap, w), dtype=torch.int32, device=rows_dev.device)
            if ent is not None and ent[1]:
                t[: ent[1]].copy_(ent[0][: ent[1]])
            ent = [t, ent[1] if ent else 0]
            self._bits[n_states] = ent
        t, done = ent
        if done < self._n:
            invert = 1 if self.side == Side.UPPER else 0
            _abi.call("rsr_pack_thermo_bits", _abi.ptr(rows_dev[done:]), self._n - done, N, n_states,
                      invert, _abi.ptr(t[done:]), w, _device.stream())
            ent[1] = self._n
        return t, self._n

    @classmethod
    def from_array(cls, side: str, threshold: int, rows: np.ndarray,
                   trusted: bool = False) -> "ReferenceSet":
        """Bulk construction.  ``trusted`` skips the dominance filter for inputs
        known to be mutually non-dominated (the reference benchmark recipe
        assigns ``_members`` directly); otherwise rows are inserted
        in order through the batched device path."""
        s = cls(side, threshold)
        rows = np.asarray(rows)
        if rows.size and (rows.min() < 0 or rows.max() > 255):
            raise ValueError("reference states must lie in [0, 255]")
        rows = rows.astype(np.uint8)
        if trusted:
            s._check_width(rows.shape[1])
            s._append_host(rows)
            return s
        for lo in range(0, rows.shape[0], 4096):
            chunk = rows[lo: lo + 4096]
            s._check_width(chunk.shape[1])
            s.insert_batch(_device.to_device(chunk), chunk)
        return s


def _validate_threshold(model: SystemModel, threshold: int) -> None:
    if not 0 <= threshold <= model.n_system_states - 2:
        raise ValueError(f"threshold must lie in [0, {model.n_system_states - 2}]")


def boundary_search_batch(model: SystemModel, x0_dev: torch.Tensor, threshold: int):
    """B independent searches (one warp each); returns device (refs, side, calls).

    Adds the exact number of Phi evaluations (sum over searches, each equal to
    the reference's count for that start vector) to the model's counter.
    """
    _validate_threshold(model, threshold)
    phi = model.device_phi()
    d = phi.descriptor(model.n_component_states)
    B = int(x0_dev.shape[0])
    refs = torch.empty_like(x0_dev)
    side = torch.empty(B, dtype=torch.uint8, device=x0_dev.device)
    calls = torch.empty(B, dtype=torch.int64, device=x0_dev.device)
    _abi.call("rsr_boundary_search", ctypes.byref(d), int(threshold), _abi.ptr(x0_dev), B,
              _abi.ptr(refs), _abi.ptr(side), _abi.ptr(calls), _device.stream())
    return refs, side, calls


def boundary_search(model: SystemModel, x0: Sequence[int], threshold: int) -> ReferenceState:
    """Walk x0 to the system-state boundary (boundary.py:116-147), on the device."""
    _validate_threshold(model, threshold)
    x = validate_vector(x0, model.n_components, model.n_component_states)
    xd = _device.to_device(x.astype(np.uint8)[None, :])
    refs, side, calls = boundary_search_batch(model, xd, threshold)
    model.add_evaluations(int(calls.item()))
    s = Side.LOWER if int(side.item()) == _abi.SIDE_LOWER else Side.UPPER
    return ReferenceState(tuple(int(v) for v in refs[0].cpu().tolist()), s, threshold)
