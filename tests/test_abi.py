"""CPU checks of the drop-in boundary: libspdkfac.so loads, exports exactly
the entry points include/spdkfac.h declares, and the ctypes signatures used by
the host API cover all of them (no compute calls -- no GPU here)."""

import pathlib
import re
import subprocess

import pytest

from paper_2107_06533_b200 import _lib as L

ROOT = pathlib.Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "spdkfac.h"


def declared():
    text = HEADER.read_text()
    return set(re.findall(r"SPDKFAC_API\s+[\w\s\*]+?\b(spdkfac_\w+)\s*\(", text))


def test_header_declares_abi():
    names = declared()
    assert "spdkfac_factor_plan_run" in names and "spdkfac_inverse_plan_run" in names
    assert len(names) == 53


def test_library_exports_every_declared_symbol():
    if not L.LIB_PATH.exists():
        pytest.skip("library not built")
    out = subprocess.run(["nm", "-D", "--defined-only", str(L.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (spdkfac_\w+)", out))
    assert declared() <= exported
    assert exported <= declared()  # nothing undeclared leaks out


def test_ctypes_binds_all_symbols():
    if not L.LIB_PATH.exists():
        pytest.skip("library not built")
    lib = L.load()
    assert set(L.SIGNATURES) == declared()
    assert lib.spdkfac_version() >= 100
    # no device in this container: the library reports unsupported instead of crashing
    assert lib.spdkfac_device_supported() in (0, 1)


def test_kernels_are_sm100a_tcgen05():
    if not L.LIB_PATH.exists():
        pytest.skip("library not built")
    sass = subprocess.run(["cuobjdump", "-sass", str(L.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA tensor loads
    assert "LDTM" in sass     # tcgen05.ld (TMEM -> registers)
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(L.LIB_PATH)], capture_output=True, text=True).stdout


def test_error_mapping():
    with pytest.raises(ValueError):
        L.check(L.ERR_ARG)
    with pytest.raises(ValueError):
        L.check(L.ERR_SHAPE)
    with pytest.raises(L.LibraryError):
        L.check(L.ERR_CUDA)
