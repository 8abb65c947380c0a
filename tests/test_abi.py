"""The C-ABI library loads and exports every symbol include/dmst.h declares.
No compute calls (no GPU here): only sizes and argument validation, which
return before touching the device."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

from paper_2401_06089_b200 import _lib
from paper_2401_06089_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build()
    return _lib.load()


def declared_symbols() -> set[str]:
    text = open(os.path.join(ROOT, "include", "dmst.h")).read()
    return set(re.findall(r"\b(dmst_[a-z0-9_]+)\s*\(", text))


def test_header_and_binding_agree():
    assert declared_symbols() == set(_lib.EXPORTS)


def test_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_stats_struct_layout_matches_header(tmp_path):
    # the ctypes mirror agrees with the C compiler's layout of dmst_stats, field by field
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    names = [f[0] for f in _lib.DmstStats._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "dmst.h"\nint main(void) {\n'
                   '  printf("%zu\\n", sizeof(dmst_stats));\n'
                   + "".join(f'  printf("%zu\\n", offsetof(dmst_stats, {n}));\n' for n in names)
                   + "  return 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got[0] == ctypes.sizeof(_lib.DmstStats)
    assert got[1:] == [getattr(_lib.DmstStats, n).offset for n in names]


def test_workspace_bytes(lib):
    assert lib.dmst_workspace_bytes(0, 1) == 0
    small = lib.dmst_workspace_bytes(1, 2)
    big = lib.dmst_workspace_bytes(128_000_000, 128_000_001)
    assert 0 < small < big
    # ~ (64 sort + 8 euv + 8 ptr/q + 1 ret + 16 views + 12 maps) bytes/edge
    assert big < 128 * 128_000_000


def test_invalid_arguments_return_einval(lib):
    ws = ctypes.create_string_buffer(16)
    rc = lib.dmst_build(None, None, None, 0, 1, None, None, None, None, None, ws, 16, None)
    assert rc == _lib.DMST_EINVAL
    assert b"n_edges" in lib.dmst_last_error()
    rc = lib.dmst_build(None, None, None, 5, 9, None, None, None, None, None, ws, 16, None)
    assert rc == _lib.DMST_EINVAL and b"n_vertices" in lib.dmst_last_error()
    rc = lib.dmst_pandora(None, None, 5, 6, None, None, None, ws, 16, None)
    assert rc == _lib.DMST_EINVAL and b"workspace too small" in lib.dmst_last_error()
    with pytest.raises(ValueError):
        _lib.check(_lib.DMST_EINVAL)


def test_version(lib):
    assert lib.dmst_version().startswith(b"dmst")


def test_library_is_sm100a(lib):
    # the in-tree .so carries sm_100a SASS (cuobjdump lists the arch)
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
