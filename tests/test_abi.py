"""The C-ABI library builds, loads and exports every symbol include/gevo.h
declares (no device needed: nothing here launches a kernel)."""
import ctypes
import os
import re

from paper_2310_10211_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gevo.h")).read()
    return sorted(set(re.findall(r"\b(gevo_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "gevo_eval" in syms and "gevo_nsga2_select" in syms
    assert set(syms) == set(_lib.SIGNATURES), "binding and header disagree"


def test_library_exports_every_declared_symbol():
    path = build.build()
    lib = ctypes.CDLL(path)
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_library_is_sm100a():
    import subprocess
    path = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_null_context_is_an_error_not_a_crash():
    lib = _lib.load()
    assert lib.gevo_destroy(None) < 0
    assert lib.gevo_last_error(None) == b"null context"


def test_plan_struct_sizes_match_header():
    from paper_2310_10211_b200 import lowering as Lw
    hdr = open(os.path.join(ROOT, "include", "gevo_plan.h")).read()
    assert "/* 224 bytes */" in hdr and "/* 112 bytes */" in hdr
    assert Lw.INSTR_DTYPE.itemsize == 224 and Lw.PROG_DTYPE.itemsize == 112
