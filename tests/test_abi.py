"""The C-ABI library loads and exports every entry point include/sbx.h declares
(no compute calls: runs without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sbx.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sbx_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    from paper_2109_03592_b200 import _lib

    names = declared_symbols()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(_lib.lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2109_03592_b200", "libsbx.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data


def test_version():
    from paper_2109_03592_b200 import _lib

    assert b"sm_100a" in _lib.lib.sbx_version()
