"""The C-ABI library loads and exports every symbol include/*.h declares
(no GPU needed: loading does not touch a device)."""

import ctypes
import glob
import os
import re

import pytest

from conftest import REPO
from paper_2601_22344_b200 import _ffi


def _declared_functions():
    names = set()
    for h in glob.glob(os.path.join(REPO, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:int|const char\*|void)\s+(rplu_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return sorted(names)


def test_header_declares_entry_points():
    names = _declared_functions()
    for must in ("rplu_dense_run", "rplu_ctx_create", "rplu_last_error", "rplu_sample_index"):
        assert must in names


def test_library_exports_all_declared_symbols():
    lib = _ffi.load_library()
    for name in _declared_functions():
        assert hasattr(lib, name), f"{name} declared in include/ but not exported"
    assert lib.rplu_abi_version() == 1


def test_ffi_signatures_cover_header():
    assert set(_declared_functions()) <= set(_ffi.SIGNATURES)


def test_library_is_sm100a():
    # the fatbin carries sm_100a SASS (checked via cuobjdump when available)
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", _ffi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    # rplu_dense_args: 2 int32 + 4 int64 + double + 3 ptr + int64 + ptr + int64 + ptr
    assert ctypes.sizeof(_ffi.DenseArgs) == 8 + 8 * 4 + 8 + 8 * 3 + 8 + 8 + 8 + 8 + 8
    assert ctypes.sizeof(_ffi.DenseOut) == 8 * 2 + 8 * 3 + 4 * 2 + 8 * 2 + 8 * 4 + 8 * 2
