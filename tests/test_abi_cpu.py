"""The C-ABI library loads without a GPU and exports every declared entry point."""

import ctypes
import os
import re

import pytest

from paper_2604_17066_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rsr_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rsr_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_surface():
    names = _declared()
    assert "rsr_classify_tc" in names and "rsr_sample" in names and "rsr_boundary_search" in names
    assert set(names) == set(_abi.EXPORTED), set(names) ^ set(_abi.EXPORTED)


def test_library_loads_and_exports_every_symbol():
    if not os.path.exists(_abi.LIB_PATH):
        pytest.fail("librsr_b200.so not built; run __graft_entry__.build()")
    lib = _abi.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.rsr_version() == 1
    assert lib.rsr_thermo_kpad(295, 2) == _abi.thermo_kpad(295, 2) == 320
    assert lib.rsr_thermo_kpad(295, 3) == _abi.thermo_kpad(295, 3) == 608
    assert lib.rsr_thermo_kpad(40, 2) == 64


def test_bad_arguments_fail_before_any_device_work():
    lib = _abi.lib()
    # argument validation happens on the host side of the ABI: no GPU needed
    with pytest.raises(ValueError, match="n_samples"):
        _abi.call("rsr_sample", None, 4, 2, 0, 0, 0, 0, None, None, 0, None)
    with pytest.raises(ValueError, match="Kpad"):
        _abi.call("rsr_classify_tc", None, 10, None, 0, None, 0, 48, None, 0, None)
    with pytest.raises(ValueError):
        _abi.call("rsr_encode_rows", None, 1, 3, 2, 7, None, None)
    assert lib.rsr_last_error()


def test_shared_object_is_sm100a_only():
    # the fatbin must carry sm_100a SASS (cuobjdump lists the ELF arch)
    import shutil
    import subprocess
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True)
    archs = set(re.findall(r"sm_\d+a?", out.stdout))
    assert archs == {"sm_100a"}, archs


def test_fp4_launch_plan_is_host_only():
    # the planner runs on the host (no device needed): tile width and launch count of
    # the FP4 classifier for the cfg4 sweep's reference counts (one side, 160-byte rows)
    rb = _abi.fp4_row_bytes(295, 2)
    S = 1 << 22
    assert _abi.fp4_plan(S, 0, 1000, rb) == (208, 1)       # 5 resident tiles of 208
    tn, n = _abi.fp4_plan(S, 0, 3000, rb)                   # past residency: 2 resident launches
    assert n == 2 and tn in (208, 224, 240)
    tn, n = _abi.fp4_plan(S, 0, 10_000, rb)                 # resident-sized launches up to ~2x10^4
    assert n >= 4
    tn, n = _abi.fp4_plan(S, 0, 500_000, rb)                # L2-sized chunks of 512 tiles
    assert n == -(-(-(-500_000 // tn)) // (122880 // tn))
    # a small batch has few sample groups per CTA pair: extra launches do not pay
    assert _abi.fp4_plan(4096, 0, 10_000, rb)[1] == 1
    assert _abi.fp4_plan(S, 0, 0, rb)[1] == 0
    # the widest rows (768 bytes, N(M-1) up to 1535) fit without first matches only
    assert _abi.fp4_plan(S, 3000, 700, 768)[0] > 0
    assert _abi.fp4_plan(S, 3000, 700, 768, want_first=True) == (0, 0)
    assert _abi.fp4_plan(S, 3000, 700, 736, want_first=True)[0] > 0
    with pytest.raises(ValueError):
        _abi.fp4_plan(S, -1, 0, rb)
