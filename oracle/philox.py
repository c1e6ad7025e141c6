"""Philox4x64-10 counter stream, restated in plain numpy uint64 arithmetic.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The reference draws its uniforms from ``numpy.random.Philox`` (numpy 2.3.5,
the reference's only runtime dependency, ``pkg/pyproject.toml:9``) keyed by
``[seed, generation_index]`` (``sampling.py:39-42``) and positions the stream
at flat index ``(start+i)*N + n`` via ``advance(first // 4)`` plus a discard
of ``first % 4`` raws (``sampling.py:45-66``).

numpy's Philox is the Random123 Philox4x64 with 10 rounds.  Its state starts
with counter 0 and an empty 4-word buffer, so the first raw draw increments
the counter *before* generating: flat draw ``f`` is word ``f % 4`` of the
block generated from counter ``f // 4 + 1`` (256-bit counter, low word
first).  ``advance(d)`` adds ``d`` to the counter without touching the buffer.
"""

from __future__ import annotations

import numpy as np

_M32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)

PHILOX_M0 = np.uint64(0xD2E7470EE14C6C93)
PHILOX_M1 = np.uint64(0xCA5A826395121157)
PHILOX_W0 = np.uint64(0x9E3779B97F4A7C15)
PHILOX_W1 = np.uint64(0xBB67AE8584CAA73B)


def _mulhilo(a: np.uint64, b: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """64x64 -> 128 multiply split as (hi, lo) using 32-bit limbs."""
    a_lo, a_hi = a & _M32, a >> _S32
    b_lo, b_hi = b & _M32, b >> _S32
    with np.errstate(over="ignore"):
        lo = a * b  # wraps mod 2**64
        p0 = a_lo * b_lo
        p1 = a_lo * b_hi
        p2 = a_hi * b_lo
        p3 = a_hi * b_hi
        mid = (p0 >> _S32) + (p1 & _M32) + (p2 & _M32)
        hi = p3 + (p1 >> _S32) + (p2 >> _S32) + (mid >> _S32)
    return hi, lo


def philox4x64_blocks(counters: np.ndarray, key0: int, key1: int) -> np.ndarray:
    """Philox4x64-10 of 64-bit block counters ``counters`` (upper counter words 0).

    Returns a ``len(counters) x 4`` uint64 array.
    """
    c0 = np.asarray(counters, dtype=np.uint64).copy()
    c1 = np.zeros_like(c0)
    c2 = np.zeros_like(c0)
    c3 = np.zeros_like(c0)
    k0 = np.uint64(key0 & ((1 << 64) - 1))
    k1 = np.uint64(key1 & ((1 << 64) - 1))
    with np.errstate(over="ignore"):
        for rnd in range(10):
            if rnd:
                k0 = k0 + PHILOX_W0
                k1 = k1 + PHILOX_W1
            hi0, lo0 = _mulhilo(PHILOX_M0, c0)
            hi1, lo1 = _mulhilo(PHILOX_M1, c2)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return np.stack([c0, c1, c2, c3], axis=1)


def random_raw(seed: int, generation_index: int, first: int, count: int) -> np.ndarray:
    """Raw uint64 draws ``first .. first+count-1`` of the (seed, gen) stream."""
    if count <= 0:
        return np.zeros(0, dtype=np.uint64)
    b_lo = first // 4
    b_hi = (first + count - 1) // 4
    blocks = philox4x64_blocks(np.arange(b_lo, b_hi + 1, dtype=np.uint64) + np.uint64(1),
                               seed, generation_index)
    flat = blocks.reshape(-1)
    off = first - 4 * b_lo
    return flat[off:off + count]


def uniform_field(seed: int, generation_index: int, start: int, count: int,
                  n_components: int, fast: bool = False) -> np.ndarray:
    """u[i, n] = (raw >> 11) * 2**-53 at flat index (start+i)*N + n (``sampling.py:45-66``).

    ``fast`` draws the raws from ``numpy.random.Philox`` itself, exactly as the
    reference does (used when *timing* the reference path; the restatement
    above is what pins correctness, and tests check the two agree).
    """
    if fast:
        mask = (1 << 64) - 1
        bg = np.random.Philox(key=np.array([seed & mask, generation_index & mask],
                                           dtype=np.uint64))
        first = start * n_components
        bg.advance(first // 4)
        raw = bg.random_raw(first % 4 + count * n_components)[first % 4:]
    else:
        raw = random_raw(seed, generation_index, start * n_components, count * n_components)
    u = (raw >> np.uint64(11)).astype(np.float64) * float(2.0 ** -53)
    return u.reshape(count, n_components)


# ------------------------------------------------- independent device stream
# Not in the reference: the north_star's "independent device RNG" mode
# (include/rsr_b200.h RSR_RNG_DEVICE).  Philox4x32-10 is the published
# Random123 generator (Salmon et al., SC'11): 32-bit multipliers
# 0xD2511F53 / 0xCD9E8D57, Weyl key increments 0x9E3779B9 / 0xBB67AE85.  The
# restatement is pinned by the Random123 known-answer vectors in
# tests/test_oracle_golden.py.

P32_M0, P32_M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
P32_W0, P32_W1 = 0x9E3779B9, 0xBB67AE85
_M32 = np.uint64(0xFFFFFFFF)


def philox4x32_blocks(c0, c1, c2, c3, k0: int, k1: int) -> np.ndarray:
    """Philox4x32-10 of counter arrays (c0..c3) under key (k0, k1): uint32 [n, 4]."""
    c = [np.asarray(x, dtype=np.uint64) & _M32 for x in (c0, c1, c2, c3)]
    c0, c1, c2, c3 = np.broadcast_arrays(*c)
    k0, k1 = k0 & 0xFFFFFFFF, k1 & 0xFFFFFFFF
    for r in range(10):
        if r:
            k0 = (k0 + P32_W0) & 0xFFFFFFFF
            k1 = (k1 + P32_W1) & 0xFFFFFFFF
        p0 = P32_M0 * c0  # < 2^64: exact in uint64
        p1 = P32_M1 * c2
        c0, c1, c2, c3 = ((p1 >> np.uint64(32)) ^ c1 ^ np.uint64(k0), p1 & _M32,
                          (p0 >> np.uint64(32)) ^ c3 ^ np.uint64(k1), p0 & _M32)
    return np.stack([c0, c1, c2, c3], axis=-1).astype(np.uint32)


def device_raw(seed: int, generation_index: int, start: int, count: int,
               n_components: int) -> np.ndarray:
    """uint32 draws [count, n_components] of rows start..start+count-1 of the device
    stream (seed, gen): draw (row R, component n) is word n % 4 of the block with
    counter [n // 4, R lo, R hi, gen lo] and key [seed lo ^ gen hi, seed hi]
    (include/rsr_b200.h, csrc/philox.cuh device_row_block)."""
    if count <= 0:
        return np.zeros((0, n_components), dtype=np.uint32)
    mask = (1 << 64) - 1
    seed, gen = seed & mask, generation_index & mask
    qb = (n_components + 3) // 4
    rows = np.arange(start, start + count, dtype=np.uint64)[:, None]
    q = np.arange(qb, dtype=np.uint64)[None, :]
    blocks = philox4x32_blocks(q, rows & _M32, rows >> np.uint64(32), gen & 0xFFFFFFFF,
                               (seed & 0xFFFFFFFF) ^ (gen >> 32), seed >> 32)
    return blocks.reshape(count, 4 * qb)[:, :n_components]
