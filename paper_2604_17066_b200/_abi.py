"""ctypes binding of ``librsr_b200.so`` (declared in ``include/rsr_b200.h``).

The library is loaded lazily on the first device call so that the host-side
API (models, distributions, reference-set bookkeeping) imports on machines
without a GPU.  There is no CPU fallback: every hot-path call goes through
this module and raises if the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

__all__ = ["lib", "call", "stream_ptr", "ptr", "PhiDesc", "RefsetDev", "LIB_PATH", "require_device",
           "SIDE_LOWER", "SIDE_UPPER", "HIT_LOWER", "HIT_UPPER", "LABEL_LOWER", "LABEL_UPPER",
           "LABEL_UNCLASSIFIED", "PHI_ST", "PHI_WIDEST", "PHI_GLOBAL", "PHI_KOFN", "PHI_CONES",
           "thermo_kpad", "thermo_words", "fp4_row_bytes", "FP4_TILE_ROWS",
           "FP4_MAX_ROW_BYTES", "REFSET_MAX_ROW_BYTES", "EXPORTED"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "librsr_b200.so")
# timing experiments (tools/fp4_prof.py) may load an instrumented build instead
LIB_PATH = os.environ.get("RSR_LIB_OVERRIDE", LIB_PATH)

RSR_OK, RSR_EINVAL, RSR_ECUDA, RSR_EUNSUPPORTED, RSR_ENCCL = 0, 1, 2, 3, 4
SIDE_LOWER, SIDE_UPPER = 0, 1
HIT_LOWER, HIT_UPPER = 1, 2
RNG_SHARED, RNG_DEVICE = 0, 1  # reference Philox4x64-10 stream / independent Philox4x32-10
LABEL_LOWER, LABEL_UPPER, LABEL_UNCLASSIFIED = 0, 1, 2
PHI_ST, PHI_WIDEST, PHI_GLOBAL, PHI_KOFN, PHI_CONES, PHI_EDGE_DISJOINT = 0, 1, 2, 3, 4, 5


class PhiDesc(ctypes.Structure):
    """Mirror of ``rsr_phi_desc`` (include/rsr_b200.h)."""

    _fields_ = [
        ("kind", ctypes.c_int32),
        ("n_components", ctypes.c_int32),
        ("n_states", ctypes.c_int32),
        ("n_nodes", ctypes.c_int32),
        ("source", ctypes.c_int32),
        ("target", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("n_anchors", ctypes.c_int32),
        ("edge_u", ctypes.c_void_p),
        ("edge_v", ctypes.c_void_p),
        ("anchors", ctypes.c_void_p),
        ("anchor_level", ctypes.c_void_p),
        ("flags", ctypes.c_int32),
    ]


PHI_FLAG_SIMPLE = 1


class RefsetDev(ctypes.Structure):
    """Mirror of ``rsr_refset_dev`` (include/rsr_b200.h)."""

    _fields_ = [
        ("rows", ctypes.c_void_p),
        ("fp4", ctypes.c_void_p),
        ("alive", ctypes.c_void_p),
        ("ctr", ctypes.c_void_p),
        ("cap", ctypes.c_int64),
        ("n_bound", ctypes.c_int64),
    ]


_P, _I, _I64, _U64, _D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double

# name -> (restype, argtypes); the full exported surface of include/rsr_b200.h
EXPORTED = {
    "rsr_version": (_I, []),
    "rsr_last_error": (ctypes.c_char_p, []),
    "rsr_thermo_kpad": (_I, [_I, _I]),
    "rsr_device_info": (_I, [_P, _P, _P]),
    "rsr_philox_raw": (_I, [_U64, _U64, _I64, _I64, _P, _P]),
    "rsr_uniform_field": (_I, [_U64, _U64, _I64, _I64, _I, _P, _P]),
    "rsr_sample": (_I, [_P, _I, _I, _U64, _U64, _I64, _I64, _P, _P, _I, _P]),
    "rsr_sample_fp4": (_I, [_P, _I, _I, _U64, _U64, _I64, _I64, _P, _P, _I, _P]),
    "rsr_sample_ex": (_I, [_P, _I, _I, _U64, _U64, _I64, _I64, _P, _P, _I, _I, _P]),
    "rsr_sample_fp4_ex": (_I, [_P, _I, _I, _U64, _U64, _I64, _I64, _P, _P, _I, _I64, _I, _P]),
    "rsr_device_raw": (_I, [_U64, _U64, _I64, _I64, _I, _P, _P]),
    "rsr_comm_unique_id": (_I, [_P]),
    "rsr_comm_init": (_I, [_P, _I, _I, _P]),
    "rsr_comm_destroy": (_I, [_P]),
    "rsr_allreduce_counts": (_I, [_P, _P, _I, _P]),
    "rsr_allgather_refs": (_I, [_P, _P, _I64, _P, _P]),
    "rsr_or_reduce_flags": (_I, [_P, _P, _I64, _P, _P]),
    "rsr_encode_samples": (_I, [_P, _I64, _I, _I, _P, _I, _P]),
    "rsr_encode_refs": (_I, [_P, _I64, _I64, _I, _I, _I, _P, _I, _P]),
    "rsr_encode_rows": (_I, [_P, _I64, _I, _I, _I, _P, _P]),
    "rsr_packbits_rows": (_I, [_P, _I64, _I, _I, _P, _P]),
    "rsr_classify_tc": (_I, [_P, _I64, _P, _I64, _P, _I64, _I, _P, _I, _P]),
    "rsr_classify_tc_explain": (_I, [_P, _I64, _P, _I64, _P, _I64, _I, _P, _P, _P, _I, _P]),
    "rsr_fp4_row_bytes": (_I, [_I, _I]),
    "rsr_encode_samples_fp4": (_I, [_P, _I64, _I, _I, _P, _I, _P]),
    "rsr_encode_samples_fp4_ex": (_I, [_P, _I64, _I, _I, _P, _I, _I64, _P]),
    "rsr_encode_refs_fp4": (_I, [_P, _I64, _I64, _I, _I, _I, _P, _I, _P]),
    "rsr_unpack_onehot_fp4": (_I, [_P, _I64, _I, _I, _P, _I, _P]),
    "rsr_classify_fp4": (_I, [_P, _I64, _P, _I64, _P, _I64, _I, _P, _I, _P]),
    "rsr_classify_fp4_planar": (_I, [_P, _I64, _I64, _P, _P, _I64, _I64, _P, _I64, _I64, _I, _P,
                                     _P, _P, _I, _P]),
    "rsr_classify_fp4_explain": (_I, [_P, _I64, _P, _I64, _P, _I64, _I, _P, _P, _P, _I, _P]),
    "rsr_classify_fp4_plan": (_I, [_I64, _I64, _I64, _I, _I, _P, _P]),
    "rsr_fp4_or_rows": (_I, [_P, _I64, _I, _P, _P]),
    "rsr_classify_fp4_tail": (_I, [_P, _I64, _I64, _P, _I64, _I, _I, _P, _I, _P]),
    "rsr_classify_fp4_plan_ex": (_I, [_I64, _I64, _I64, _I, _I, _P, _P, _P]),
    "rsr_fp4_gather_columns": (_I, [_P, _I64, _I64, _I, _P, _I, _P, _I64, _I, _P]),
    "rsr_pack_thermo_bits": (_I, [_P, _I64, _I, _I, _I, _P, _I, _P]),
    "rsr_classify_bits": (_I, [_P, _I64, _P, _I64, _P, _I64, _I, _P, _P, _P, _I, _P]),
    "rsr_finalize": (_I, [_P, _I64, _P, _P, _P]),
    "rsr_compact_scratch": (_I64, [_I64]),
    "rsr_compact": (_I, [_P, _I64, _I, _P, _P, _P, _P]),
    "rsr_violation_counts": (_I, [_P, _I64, _P, _I64, _I, _I, _P, _P]),
    "rsr_violation_counts_rows": (_I, [_P, _I64, _P, _I64, _I, _P, _P]),
    "rsr_phi_eval": (_I, [ctypes.POINTER(PhiDesc), _P, _P, _I64, _P, _I, _P, _P]),
    "rsr_boundary_search": (_I, [ctypes.POINTER(PhiDesc), _I, _P, _I64, _P, _P, _P, _P]),
    "rsr_gather_rows": (_I, [_P, _I, _P, _I64, _P, _P]),
    "rsr_enumerate_states": (_I, [_P, _I, _I, _I64, _I64, _P, _P, _P]),
    "rsr_state_mass": (_I, [_P, _P, _I64, _I, _P, _P, _P]),
    "rsr_dominance_scan": (_I, [_P, _I64, _P, _I64, _I, _I, _P, _P, _I, _P, _P]),
    "rsr_refset_scratch": (_I64, [_I64, _I]),
    "rsr_refset_insert": (_I, [_P, _P, _I64, _I, _I, ctypes.POINTER(RefsetDev),
                               ctypes.POINTER(RefsetDev), _P, _P, _P, _P, _P]),
    "rsr_gather_picks": (_I, [_P, _I, _P, _P, _I64, _P, _P]),
    "rsr_gather_picks_fp4": (_I, [_P, _I, _I, _I, _P, _P, _I64, _P, _P]),
    "rsr_gather_rows_dev": (_I, [_P, _I64, _I, _P, _P, _I64, _P, _I64, _P]),
    "rsr_scatter_or_dev": (_I, [_P, _P, _P, _I64, _P, _P]),
    "rsr_classify_fp4_dev": (_I, [_P, _I64, _P, _P, _I64, _P, _I64, _I, _P, _I, _P]),
    "rsr_classify_fp4_ex": (_I, [_P, _I64, _P, _P, _I64, _I64, _P, _I64, _I64, _I, _P, _P, _P, _I,
                                 _P]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def lib() -> ctypes.CDLL:
    """Load and type the shared library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                        "g.build()'` (no CPU fallback exists for the RSR device path)")
                handle = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in EXPORTED.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


_CUDA_OK: bool | None = None
_DEVICES: dict[int, torch.device] = {}


def require_device() -> torch.device:
    global _CUDA_OK
    if not _CUDA_OK:  # checked once; torch.cuda.is_available() is slow in hot loops
        _CUDA_OK = torch.cuda.is_available()
        if not _CUDA_OK:
            raise RuntimeError("the RSR hot path runs on CUDA devices only (no CPU fallback); "
                               "torch.cuda.is_available() is False")
    idx = torch._C._cuda_getDevice()
    dev = _DEVICES.get(idx)
    if dev is None:
        dev = _DEVICES[idx] = torch.device("cuda", idx)
    return dev


_FN: dict = {}
_VALUE_RESULT = frozenset(("rsr_compact_scratch", "rsr_thermo_kpad", "rsr_version",
                           "rsr_fp4_row_bytes", "rsr_refset_scratch"))


def call(name: str, *args) -> int:
    """Invoke an entry point, mapping status codes to Python exceptions."""
    fn = _FN.get(name)
    if fn is None:
        fn = _FN[name] = getattr(lib(), name)
    rc = fn(*args)
    if rc == RSR_OK or name in _VALUE_RESULT:
        return rc
    msg = (lib().rsr_last_error() or b"").decode(errors="replace")
    if rc in (RSR_EINVAL, RSR_EUNSUPPORTED):
        raise ValueError(f"{name}: {msg}")
    raise RuntimeError(f"{name}: {msg}")


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    if stream is not None:
        return stream.cuda_stream
    # raw cudaStream_t of the current stream without torch.cuda.current_stream()'s
    # per-call device-index bookkeeping (this runs once per library call)
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device pointer expected")
    return t.data_ptr()


def thermo_kpad(n: int, m: int) -> int:
    """Kpad of the thermometer layout (mirrors rsr_thermo_kpad; pure arithmetic)."""
    kdim = n * (m - 1)
    nb = (kdim + 126) // 127
    return (kdim + nb + 31) // 32 * 32


FP4_TILE_ROWS = 240
FP4_MAX_ROW_BYTES = 768      # classifier (include/rsr_b200.h)
REFSET_MAX_ROW_BYTES = 416   # Stage-1 loop's device reference sets


def fp4_row_bytes(n: int, m: int) -> int:
    """Bytes per operand row of the FP4 layout (mirrors rsr_fp4_row_bytes)."""
    return (n * (m - 1) + 1 + 63) // 64 * 32


def fp4_plan(n_samples: int, n_lower: int, n_upper: int, row_bytes: int,
             want_first: bool = False) -> tuple[int, int]:
    """(MMA N per reference tile, kernel launches) of an rsr_classify_fp4* call over
    n_samples samples with these reference counts (rsr_classify_fp4_plan; host only)."""
    tn = ctypes.c_int(0)
    launches = ctypes.c_int64(0)
    call("rsr_classify_fp4_plan", n_samples, n_lower, n_upper, row_bytes, int(want_first),
         ctypes.addressof(tn), ctypes.addressof(launches))
    return tn.value, launches.value


def fp4_plan_ex(n_samples: int, n_lower: int, n_upper: int, row_bytes: int,
                want_first: bool = False) -> tuple[int, int, bool]:
    """(tile_n, launches, paired) of rsr_classify_fp4_plan_ex (host only)."""
    tn, nl, pr = ctypes.c_int(0), ctypes.c_int64(0), ctypes.c_int(0)
    call("rsr_classify_fp4_plan_ex", n_samples, n_lower, n_upper, row_bytes, int(want_first),
         ctypes.addressof(tn), ctypes.addressof(nl), ctypes.addressof(pr))
    return tn.value, nl.value, bool(pr.value)


def thermo_words(n: int, m: int) -> int:
    return (n * (m - 1) + 31) // 32


_SM_COUNT: dict = {}


def device_sm_count() -> int:
    """SM count of the current device (rsr_device_info), cached per device."""
    idx = require_device().index
    n = _SM_COUNT.get(idx)
    if n is None:
        sm, ma, mi = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        call("rsr_device_info", ctypes.byref(sm), ctypes.byref(ma), ctypes.byref(mi))
        n = _SM_COUNT[idx] = int(sm.value)
    return n
