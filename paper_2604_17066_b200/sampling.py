"""(1) Device-resident Monte Carlo batches (mirror of reference ``sampling.py``).

``sample_batch`` runs ``rsr_sample_fp4``: numpy-compatible Philox4x64-10
keyed by (seed, generation_index), flat draw index (start+i)*N + n, inverse
CDF on the cumulative probabilities (sampling.py:39-90), bit-exact with the
reference.  The kernel writes the uint8 state matrix and, fused, the FP4
sample operand of the default classifier (``rsr_sample`` with the int8
thermometer rows fused serves the int8 variant).  The batch stays in HBM; the
host ``states`` array (int64, as in the reference) is materialised lazily.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _abi, _device
from .model import ComponentDistribution

__all__ = ["SampleBatch", "sample_batch", "uniform_field"]


class SampleBatch:
    """H component-state vectors plus the keys that regenerate them (sampling.py:22-36).

    ``states`` may be a host array (any integer dtype) or a CUDA uint8 tensor.
    """

    def __init__(self, states, seed: int, generation_index: int, *, state_bound: int | None = None,
                 rng: str = "shared"):
        self.seed = int(seed)
        self.generation_index = int(generation_index)
        self.rng = rng  # the stream that regenerates the batch (sample_batch)
        self._host: np.ndarray | None = None
        self._dev: torch.Tensor | None = None
        self._thermo: dict[int, torch.Tensor] = {}
        self._bits: dict[int, torch.Tensor] = {}
        self._fp4: dict[int, torch.Tensor] = {}
        self._fp4_plane: dict[int, int] = {}  # FP4 layout per M: 0 interleaved, > 0 planar
        if isinstance(states, torch.Tensor):
            if states.dim() != 2:
                raise ValueError("states must be an H x N matrix")
            self._dev = states
            self._shape = tuple(states.shape)
            self._bound = state_bound
        else:
            arr = np.asarray(states)
            if arr.ndim != 2:
                raise ValueError("states must be an H x N matrix")
            self._host = arr
            self._shape = arr.shape
            self._bound = state_bound
            if self._bound is None and arr.size:
                if arr.min() < 0:
                    raise ValueError("states must be non-negative")
                self._bound = int(arr.max()) + 1

    # -- reference API -----------------------------------------------------
    @property
    def states(self) -> np.ndarray:
        if self._host is None:
            self._host = self._dev.cpu().numpy().astype(np.int64)
        return self._host

    @property
    def n_samples(self) -> int:
        return self._shape[0]

    @property
    def n_components(self) -> int:
        return self._shape[1]

    # -- device views ------------------------------------------------------
    @property
    def state_bound(self) -> int:
        """Exclusive upper bound of the states (M of the sampler, or max+1)."""
        if self._bound is None:
            self._bound = int(self.device_states().max().item()) + 1 if self.n_samples else 1
        return self._bound

    def device_states(self) -> torch.Tensor:
        if self._dev is None:
            arr = self._host
            if arr.size and (arr.min() < 0 or arr.max() > 255):
                raise ValueError("device states must lie in [0, 255]")
            self._dev = _device.to_device(arr.astype(np.uint8, copy=False))
        return self._dev

    def thermo(self, n_states: int) -> torch.Tensor:
        """int8 thermometer rows [H, Kpad] (A operand of the classifier), cached per M."""
        t = self._thermo.get(n_states)
        if t is None:
            n = self.n_components
            kpad = _abi.thermo_kpad(n, n_states)
            st = self.device_states()
            t = torch.empty((self.n_samples, kpad), dtype=torch.int8, device=st.device)
            _abi.call("rsr_encode_samples", _abi.ptr(st), self.n_samples, n, n_states,
                      _abi.ptr(t), kpad, _device.stream())
            self._thermo[n_states] = t
        return t

    def fp4(self, n_states: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """FP4 sample operand (A operand of the FP4 classifier, include/rsr_b200.h), cached
        per M: planar [2, H, row_bytes] (A_up plane, A_lo plane) by default, or
        interleaved rows [H, 2 * row_bytes] = [A_up | A_lo] written into ``out``.
        ``fp4_plane_stride`` tells which."""
        t = self._fp4.get(n_states)
        if t is None:
            n = self.n_components
            rb = _abi.fp4_row_bytes(n, n_states)
            st = self.device_states()
            if out is not None:
                if out.dtype != torch.uint8 or out.shape[0] < self.n_samples or out.shape[1] != 2 * rb:
                    raise ValueError("fp4 buffer must be uint8 [>= H, 2 * row_bytes]")
                t, plane = out[: self.n_samples], 0
            else:
                t = torch.empty((2, self.n_samples, rb), dtype=torch.uint8, device=st.device)
                plane = self.n_samples * rb
            _abi.call("rsr_encode_samples_fp4_ex", _abi.ptr(st), self.n_samples, n, n_states,
                      _abi.ptr(t), rb, plane, _device.stream())
            self._fp4[n_states] = t
            self._fp4_plane[n_states] = plane
        return t

    def fp4_plane_stride(self, n_states: int) -> int:
        """Layout of ``fp4(n_states)``: 0 = interleaved rows, else the byte offset of the
        A_lo plane (planar; a one-sided classification then reads only its half)."""
        self.fp4(n_states)
        return self._fp4_plane[n_states]

    def thermo_bits(self, n_states: int) -> torch.Tensor:
        """Packed thermometer bits [H, words] (bit-packed classifier operand)."""
        t = self._bits.get(n_states)
        if t is None:
            n = self.n_components
            w = _abi.thermo_words(n, n_states)
            st = self.device_states()
            t = torch.empty((max(1, self.n_samples), w), dtype=torch.int32, device=st.device)
            _abi.call("rsr_pack_thermo_bits", _abi.ptr(st), self.n_samples, n, n_states, 0,
                      _abi.ptr(t), w, _device.stream())
            self._bits[n_states] = t
        return t

    def release_thermo(self) -> None:
        self._thermo.clear()
        self._bits.clear()
        self._fp4.clear()


def uniform_field(seed: int, generation_index: int, start: int, count: int,
                  n_components: int) -> np.ndarray:
    """Uniform(0,1) field of samples [start, start+count) (sampling.py:45-66), on device."""
    out = torch.empty((count, n_components), dtype=torch.float64, device=_device.device())
    mask = (1 << 64) - 1
    _abi.call("rsr_uniform_field", seed & mask, generation_index & mask, start, count,
              n_components, _abi.ptr(out), _device.stream())
    return out.cpu().numpy()


RNG_KINDS = {"shared": _abi.RNG_SHARED, "device": _abi.RNG_DEVICE}


def rng_code(rng: str) -> int:
    try:
        return RNG_KINDS[rng]
    except KeyError:
        raise ValueError(f"rng must be 'shared' or 'device', got {rng!r}") from None


def sample_batch(dist: ComponentDistribution, n_samples: int, seed: int,
                 generation_index: int = 0, start: int = 0, *, encode: bool = False,
                 fp4: bool | None = None,
                 out_states: torch.Tensor | None = None,
                 out_thermo: torch.Tensor | None = None,
                 out_fp4: torch.Tensor | None = None,
                 rng: str = "shared") -> SampleBatch:
    """Inverse-CDF draw on the counter-based stream (sampling.py:69-90), on device.

    By default (``fp4`` None -> on whenever the FP4 classifier handles the row
    width) one kernel, ``rsr_sample_fp4``, writes the uint8 states and the FP4
    sample operand of the default classifier.  ``encode`` (or ``out_thermo``)
    instead runs ``rsr_sample`` with the int8 thermometer rows fused.
    ``out_*`` let callers reuse preallocated buffers.  ``rng="shared"`` is the
    reference's Philox4x64-10 stream (bit-exact); ``rng="device"`` the independent
    Philox4x32-10 device stream (include/rsr_b200.h RSR_RNG_DEVICE).
    """
    if n_samples < 1:
        raise ValueError("n_samples must be >= 1")
    code = rng_code(rng)
    n, m = dist.n_components, dist.n_states
    dev = _device.device()
    states = out_states if out_states is not None else torch.empty(
        (n_samples, n), dtype=torch.uint8, device=dev)
    mask = (1 << 64) - 1
    int8_path = encode or out_thermo is not None
    rb = _abi.fp4_row_bytes(n, m)
    if fp4 is None:
        fp4 = (not int8_path) and rb <= _abi.FP4_MAX_ROW_BYTES
    if fp4 and not int8_path:
        if out_fp4 is not None:  # caller's interleaved rows [H, 2 * row_bytes]
            a4, plane = out_fp4[:n_samples], 0
            if a4.dtype != torch.uint8 or a4.shape != (n_samples, 2 * rb):
                raise ValueError("fp4 buffer must be uint8 [>= H, 2 * row_bytes]")
        else:  # planar: one-sided classifications stream only their half
            a4 = torch.empty((2, n_samples, rb), dtype=torch.uint8, device=dev)
            plane = n_samples * rb
        _abi.call("rsr_sample_fp4_ex", _abi.ptr(dist.device_probs()), n, m, seed & mask,
                  generation_index & mask, start, n_samples, _abi.ptr(states), _abi.ptr(a4), rb,
                  plane, code, _device.stream())
        batch = SampleBatch(states, seed, generation_index, state_bound=m, rng=rng)
        batch._fp4[m] = a4
        batch._fp4_plane[m] = plane
        return batch
    thermo = None
    kpad = _abi.thermo_kpad(n, m)
    if int8_path:
        thermo = out_thermo if out_thermo is not None else torch.empty(
            (n_samples, kpad), dtype=torch.int8, device=dev)
    _abi.call("rsr_sample_ex", _abi.ptr(dist.device_probs()), n, m, seed & mask,
              generation_index & mask, start, n_samples, _abi.ptr(states), _abi.ptr(thermo),
              kpad, code, _device.stream())
    batch = SampleBatch(states, seed, generation_index, state_bound=m, rng=rng)
    if thermo is not None:
        batch._thermo[m] = thermo
    if out_fp4 is not None:
        batch.fp4(m, out=out_fp4)
    return batch
