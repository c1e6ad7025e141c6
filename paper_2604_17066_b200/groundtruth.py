"""Ground-truth engines of the reference (``oracle.py``) on the device, for the CLI.

``exact_probabilities`` enumerates all M^N vectors (guarded at 2^24 like
oracle.py:30-38) with ``rsr_enumerate_states``, evaluates Phi with
``rsr_phi_eval`` and accumulates the per-state mass with ``rsr_state_mass``
in enumeration order (bit-exact float64 sums).  ``crude_monte_carlo`` is the
generation-0 batch resolved entirely by Phi (oracle.py:82-101), i.e. Stage 2
with empty reference sets.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi, _device
from .dist import Comm
from .model import ComponentDistribution, SystemModel

__all__ = ["ExactResult", "exact_probabilities", "crude_monte_carlo", "MAX_ENUM_VECTORS"]

MAX_ENUM_VECTORS = 1 << 24
_CHUNK = 1 << 20


@dataclass(frozen=True)
class ExactResult:
    cumulative: np.ndarray
    state_count: np.ndarray


def exact_probabilities(model: SystemModel, dist: ComponentDistribution) -> ExactResult:
    """Enumerate all M^N vectors (oracle.py:49-63)."""
    n, m = model.n_components, model.n_component_states
    if m ** n > MAX_ENUM_VECTORS:
        raise ValueError(f"{m}**{n} vectors exceed the enumeration guard of {MAX_ENUM_VECTORS}")
    phi = model.device_phi()
    dev = _device.device()
    total = m ** n
    mass = torch.zeros(model.n_system_states, dtype=torch.float64, device=dev)
    counts = torch.zeros(model.n_system_states, dtype=torch.int64, device=dev)
    chunk = min(_CHUNK, total)
    states = torch.empty((chunk, n), dtype=torch.uint8, device=dev)
    probs = torch.empty(chunk, dtype=torch.float64, device=dev)
    vals = torch.empty(chunk, dtype=torch.uint8, device=dev)
    st = _device.stream()
    for first in range(0, total, chunk):
        c = min(chunk, total - first)
        _abi.call("rsr_enumerate_states", _abi.ptr(dist.device_probs()), n, m, first, c,
                  _abi.ptr(states), _abi.ptr(probs), st)
        phi.eval_into(states, None, c, m, vals)
        _abi.call("rsr_state_mass", _abi.ptr(vals), _abi.ptr(probs), c, model.n_system_states,
                  _abi.ptr(mass), _abi.ptr(counts), st)
    model.add_evaluations(total)
    if int(counts.sum().item()) != total:
        raise ValueError("performance function returned a state outside [0, n_system_states)")
    return ExactResult(cumulative=np.cumsum(mass.cpu().numpy()), state_count=counts.cpu().numpy())


def crude_monte_carlo(model: SystemModel, dist: ComponentDistribution, n_samples: int, seed: int,
                      threshold: int) -> tuple[float, float | None]:
    """Plain MC estimate of P(S <= m') on generation 0 (oracle.py:82-101)."""
    from .workflow import _stage2_counts
    if n_samples < 1:
        raise ValueError("n_samples must be >= 1")
    n_low, _, n_x = (int(v) for v in _stage2_counts(model, dist, None, None, threshold, seed, 0,
                                                     n_samples, Comm.single()))
    model.add_evaluations(n_x)
    p_hat = n_low / n_samples
    if p_hat == 0.0:
        return 0.0, None
    return p_hat, math.sqrt((1.0 - p_hat) / (n_samples * p_hat))
