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
        for m in re.finditer(r"^\s*(?:int|int64_t|const char\*|void)\s+(rplu_\w+)\s*\(", src, flags=re.M):
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
    assert lib.rplu_abi_version() == 2


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


def _c_layouts(structs):
    """sizeof / offsetof of the header's structs, from a C program built with gcc."""
    import shutil
    import subprocess
    import tempfile
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    lines = ["#include <stddef.h>", "#include <stdio.h>", '#include "rplu_b200.h"',
             "int main(void) {"]
    for cname, pystruct in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in pystruct._fields_:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["  return 0;", "}"]
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "l.c"), os.path.join(d, "l")
        with open(src, "w") as fh:
            fh.write("\n".join(lines))
        subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), src, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    res = {}
    for ln in out.splitlines():
        c, f, v = ln.split()
        res[(c, f)] = int(v)
    return res


def test_ctypes_structs_match_c_layout():
    """Every ctypes mirror has the header struct's size and field offsets."""
    from paper_2601_22344_b200.operators import _GaussOpStruct
    structs = {"rplu_dense_args": _ffi.DenseArgs, "rplu_dense_out": _ffi.DenseOut,
               "rplu_cauchy_args": _ffi.CauchyArgs, "rplu_cauchy_out": _ffi.CauchyOut,
               "rplu_shard_args": _ffi.ShardArgs, "rplu_cauchy_shard_args": _ffi.CauchyShardArgs,
               "rplu_tree_plan": _ffi.TreePlan, "rplu_gauss_op": _GaussOpStruct}
    lay = _c_layouts(structs)
    for cname, py in structs.items():
        assert lay[(cname, "size")] == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert lay[(cname, f)] == getattr(py, f).offset, (cname, f)
