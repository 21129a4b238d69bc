"""The ctypes mirrors of the C-ABI structs (paper_2008_11839_b200/_native.py)
match include/gconn.h field for field: a small C program compiled with gcc
prints sizeof / offsetof of every field and the test compares them with the
ctypes layout (CPU only; no library call)."""
import ctypes as C
import shutil
import subprocess
from pathlib import Path

import pytest

from paper_2008_11839_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent
STRUCTS = {"gc_csr": N.Csr, "gc_spec": N.Spec, "gc_stats": N.Stats}


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_struct_layouts_match_header(tmp_path):
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "gconn.h"', "int main(void) {"]
    for cname, cls in STRUCTS.items():
        lines.append(f'  printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {}
    for line in filter(None, out):
        cname, key, val = line.split()
        got[(cname, key)] = int(val)
    for cname, cls in STRUCTS.items():
        assert got[(cname, "sizeof")] == C.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[(cname, fname)] == getattr(cls, fname).offset, (cname, fname)
