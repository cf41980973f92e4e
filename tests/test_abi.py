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


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the C structs agree with the C compiler's layout."""
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "aderdg_b200.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu\\n", sizeof(adg_config), sizeof(adg_step_record),'
                   ' sizeof(adg_layout), offsetof(adg_config, driver_mode), offsetof(adg_step_record, predicts));'
                   'return 0;}\n')
    exe = tmp_path / "sz"
    r = subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(src), "-o", str(exe)],
                       capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("gcc unavailable: " + r.stderr[:200])
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert vals == [ctypes.sizeof(_lib.AdgConfig), ctypes.sizeof(_lib.AdgStepRecord),
                    ctypes.sizeof(_lib.AdgLayout), _lib.AdgConfig.driver_mode.offset,
                    _lib.AdgStepRecord.predicts.offset]
