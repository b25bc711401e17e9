"""C ABI checks that need no GPU: libmhdg.so loads, exports every function
declared in include/mhdg.h, and the ctypes mirrors of the structs have the
C layout (sizes and field offsets compared against a gcc-compiled probe)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2402_11361_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mhdg.h")
TUNING = os.path.join(ROOT, "paper_2402_11361_b200", "csrc", "mhdg_tuning.h")


def declared_functions(path=HEADER):
    text = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:int|long long|void)\s+(mhdg_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 15
    lib = _lib.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED)


def test_tuning_knobs_stay_out_of_the_public_header():
    """The A/B knobs are process-global diagnostics: exported, declared only in
    the internal csrc/mhdg_tuning.h, never in the drop-in header."""
    knobs = declared_functions(TUNING)
    assert set(knobs) == set(_lib.TUNING)
    assert not set(knobs) & set(declared_functions())
    lib = _lib.lib()
    for n in knobs:
        assert hasattr(lib, n), n


def test_packed_factor_size():
    lib = _lib.lib()
    for n in (20, 175, 364):
        assert lib.mhdg_packed_lu_size(n) >= n * n


STRUCTS = {"mhdg_disc": _lib.Disc, "mhdg_flow": _lib.Flow, "mhdg_stage": _lib.Stage,
           "mhdg_blocks": _lib.Blocks, "mhdg_frozen": _lib.Frozen, "mhdg_factors": _lib.Factors}


def test_struct_layout_matches_header(tmp_path):
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void) {"]
    for cname, py in STRUCTS.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    try:
        subprocess.check_call(["gcc", "-o", str(exe), str(src)])
    except (OSError, subprocess.CalledProcessError):
        pytest.skip("gcc not available")
    out = subprocess.check_output([str(exe)], text=True).split("\n")
    got = {}
    for ln in out:
        if ln.strip():
            a, b, c = ln.split()
            got[(a, b)] = int(c)
    for cname, py in STRUCTS.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)
