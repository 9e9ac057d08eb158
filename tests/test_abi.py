"""The C-ABI library builds, loads without a GPU and exports every symbol
include/csvd_b200.h declares; the ctypes struct mirrors match the header."""

import ctypes
import os
import re

from paper_2511_21702_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "csvd_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char \*)\s*(csvd_\w+)\(", src, re.M)))


def test_header_declarations_are_exported():
    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.EXPORTS)


def test_struct_sizes_match_header():
    lib = _lib.load()
    v = [ctypes.c_int32() for _ in range(4)]
    assert lib.csvd_test_sizes(*[ctypes.byref(x) for x in v]) == 0
    assert ctypes.sizeof(_lib.Config) == v[0].value
    assert ctypes.sizeof(_lib.Result) == v[1].value
    assert ctypes.sizeof(_lib.TableDesc) == v[2].value
    assert ctypes.sizeof(_lib.IndexDesc) == v[3].value


def test_strerror_on_null():
    lib = _lib.load()
    assert lib.csvd_strerror(None) == b"null context"
