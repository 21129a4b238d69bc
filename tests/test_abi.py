"""The C-ABI library loads and exports every symbol include/gconn.h declares
(no compute calls: this runs without a GPU)."""
import ctypes as C
import re
from pathlib import Path

from paper_2008_11839_b200 import _native

HEADER = Path(__file__).resolve().parent.parent / "include" / "gconn.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gc_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = C.CDLL(str(_native.LIB_PATH))
    names = declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert set(declared()) <= set(_native.exported_symbols())


def test_version_and_workspace_query():
    lib = _native.lib()
    assert b"sm_100a" in lib.gc_version()
    s = _native.Spec()
    s.sample, s.finish, s.find, s.splice = 1, 4, 2, 3
    assert lib.gc_workspace_size(1 << 20, 1 << 24, C.byref(s)) > 4 * (1 << 20)
