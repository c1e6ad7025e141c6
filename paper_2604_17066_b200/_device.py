"""Device plumbing: cached uploads, scratch buffers, host<->device transfers.

PyTorch is used only for device memory and streams; all hot-path compute is
in ``librsr_b200.so`` (see ``_abi``).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _abi

__all__ = ["device", "to_device", "cached_tensor", "stream", "u8_rows"]


def device() -> torch.device:
    return _abi.require_device()


def stream() -> int:
    return _abi.stream_ptr()


def to_device(arr: np.ndarray, dtype: torch.dtype | None = None) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device(), non_blocking=False)


def cached_tensor(owner, attr: str, arr: np.ndarray, dtype: torch.dtype | None = None) -> torch.Tensor:
    """Upload ``arr`` once per (owner, device) and cache it on the owner."""
    dev = device()
    cache = owner.__dict__.get(attr)
    if cache is None or cache.device != dev:
        cache = to_device(arr, dtype)
        object.__setattr__(owner, attr, cache)
    return cache


def u8_rows(x, n_components: int, n_states: int) -> torch.Tensor:
    """Validated uint8 device matrix of component-state rows."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.dim() == 1:
            t = t.unsqueeze(0)
        if t.dtype != torch.uint8:
            if t.numel() and (int(t.min()) < 0 or int(t.max()) >= n_states):
                raise ValueError(f"component states must lie in [0, {n_states - 1}]")
            t = t.to(torch.uint8)
        return t.to(device()).contiguous()
    a = np.asarray(x)
    if a.ndim == 1:
        a = a[None, :]
    if a.ndim != 2 or a.shape[1] != n_components:
        raise ValueError(f"expected rows of length {n_components}")
    if a.size and (a.min() < 0 or a.max() >= n_states):
        raise ValueError(f"component states must lie in [0, {n_states - 1}]")
    return to_device(a.astype(np.uint8))
