"""CPU checks of the C-ABI boundary: the library loads and exports every
symbol declared in include/qtt_b200.h (no compute calls without a GPU)."""

import ctypes
import os
import re

from paper_2501_07778_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "qtt_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(qtt_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_lib.EXPORTS)


def test_layout_struct_matches_header():
    # int32 d, int32 is_matrix, then 4 int64 arrays
    assert ctypes.sizeof(_lib.Layout) == 8 + 8 * (65 + 64 * 3)
    lay = _lib.Layout()
    lay.d = 3
    for l in range(3):
        lay.ranks[l] = 1 if l == 0 else 2
        lay.rows[l] = 2
        lay.cols[l] = 1
        lay.offsets[l] = 32 * l
    lay.ranks[3] = 1
    assert _lib.load().qtt_layout_size(ctypes.byref(lay)) == 64 + 2 * 2 * 1
    assert b"sm_100a" in _lib.load().qtt_version()


def test_shared_object_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.library_path()], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
