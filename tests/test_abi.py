"""C-ABI boundary (no GPU): libsinn.so loads and exports every symbol include/sinn.h declares,
and the Python binding mirrors the header one to one (argument marshalling only)."""
import os
import re
import subprocess

import paper_2301_10622_b200 as sinn
from paper_2301_10622_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "sinn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sinn_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_every_header_symbol():
    so = _build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (sinn_[a-z0-9_]+)", out))
    declared = header_functions()
    assert declared, "no functions parsed from sinn.h"
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    L = sinn.lib()  # dlopen works without a GPU
    for f in declared:
        assert hasattr(L, f)
    assert sinn.version().startswith("sinn-b200")


def test_binding_mirrors_header():
    assert sorted(sinn.SIGNATURES) == header_functions()


def test_library_is_sm100a_only():
    so = _build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_create_rejects_bad_arguments_without_gpu_work():
    import ctypes
    import numpy as np
    L = sinn.lib()
    h = ctypes.c_void_p()
    table = np.zeros(4, np.int32)
    assert L.sinn_create(0, 4, 1, table.ctypes.data, 0, None, ctypes.byref(h)) == sinn.EINVAL
    assert L.sinn_create(4, 0, 1, table.ctypes.data, 0, None, ctypes.byref(h)) == sinn.EINVAL
    assert L.sinn_create(4, 4, 9, table.ctypes.data, 0, None, ctypes.byref(h)) == sinn.EINVAL
    bad = np.array([0, 1, 2, 4], np.int32)  # 4 >= m
    assert L.sinn_create(4, 4, 1, bad.ctypes.data, 0, None, ctypes.byref(h)) == sinn.EINVAL
    assert L.sinn_create(4, 4, 1, table.ctypes.data, 8, None, ctypes.byref(h)) == sinn.EINVAL  # unknown flag
    # n above 2^27: term ids would wrap in the packed (j << 5) | d index entries (sinn.h SINN_MAX_N);
    # rejected before the table is read, so a 4-entry table suffices
    assert L.sinn_create((1 << 27) + 1, 4, 1, table.ctypes.data, 0, None, ctypes.byref(h)) == sinn.EINVAL
    assert h.value is None
