"""The C-ABI library loads without a GPU and exports every symbol that
include/aderdg_b200.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO
from paper_1801_08682_b200 import _lib

HEADER = os.path.join(REPO, "include", "aderdg_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(adg_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    _lib.load_library()


def test_library_is_sm100a():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(_lib.DeviceError):
        _lib.load_library(str(tmp_path / "nope.so"))


def test_struct_layouts_match_header():
    # adg_step_record: 2 ints + 4 doubles + 2 long long = 56 bytes
    assert ctypes.sizeof(_lib.AdgStepRecord) == 56
    assert ctypes.sizeof(_lib.AdgConfig) == 80
