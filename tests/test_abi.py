"""The C-ABI boundary without a GPU: libevo.so loads, exports every entry point that
include/evo.h declares, and the ctypes binding (_lib._SIGS) covers exactly that set.
No compute call is made (there is no device here)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "evo.h")
LIB = os.path.join(ROOT, "paper_2203_00854_b200", "libevo.so")


def declared():
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\**\s*(evo_\w+)\s*\(", src, re.M)))


def test_header_parses():
    names = declared()
    assert "evo_gated_attention_fwd" in names and "evo_bgemm" in names and len(names) >= 20


@pytest.mark.skipif(not os.path.exists(LIB), reason="libevo.so not built (run __graft_entry__.build())")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.evo_version() != 0


def test_binding_covers_header():
    from paper_2203_00854_b200 import _lib
    assert sorted(set(_lib.exported_symbols())) == declared()


@pytest.mark.skipif(not os.path.exists(LIB), reason="libevo.so not built")
def test_attention_desc_layout_matches_header():
    """the ctypes struct mirrors EvoAttnDesc field by field (flags is the last member)"""
    from paper_2203_00854_b200 import _lib
    names = [f[0] for f in _lib.EvoAttnDesc._fields_]
    assert names[-1] == "flags" and names[-2] == "scale"
    src = open(HEADER).read()
    body = src[src.index("typedef struct EvoAttnDesc"):src.index("} EvoAttnDesc;")]
    assert "int flags;" in body
