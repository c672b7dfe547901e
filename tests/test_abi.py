"""The C-ABI library loads without a GPU and exports every symbol the public
header declares (no compute calls here)."""

import os
import re

from conftest import ROOT
from paper_2605_19951_b200 import _lib


def header_symbols():
    src = open(os.path.join(ROOT, "include", "rba_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rba_[A-Za-z0-9_]+)\s*\(", src)))


def test_library_exports_header():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)


def test_error_path_without_gpu():
    lib = _lib.load()
    assert lib.rba_version() == 1
    rc = lib.rba_symbolic_analyze(0, None, None, None, 64, None)
    assert rc == 1
    assert b"null" in lib.rba_last_error()
