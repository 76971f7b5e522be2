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


def test_nvtx_ranges_need_no_device():
    """gevo_range_push / gevo_range_pop (NVTX 3, header-only) are callable
    without a GPU or a profiler attached, and nest."""
    lib = _lib.load()
    with _lib.nvtx_range("outer"):
        with _lib.nvtx_range("inner"):
            pass
    assert lib.gevo_range_push(None) < 0


def test_plan_struct_sizes_match_header():
    from paper_2310_10211_b200 import lowering as Lw
    hdr = open(os.path.join(ROOT, "include", "gevo_plan.h")).read()
    assert "/* 224 bytes */" in hdr and "/* 120 bytes */" in hdr
    assert Lw.INSTR_DTYPE.itemsize == 224 and Lw.PROG_DTYPE.itemsize == 120


def _c_sizeof(types):
    """sizeof of header types, from a C probe compiled against include/."""
    import subprocess
    import tempfile
    src = "#include <stdio.h>\n#include \"gevo.h\"\nint main(void){" + "".join(
        f'printf("%zu\\n", sizeof({t}));' for t in types) + "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "p.c"), os.path.join(d, "p")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    return [int(x) for x in out.split()]


def test_result_and_plan_sizes_match_c_header():
    from paper_2310_10211_b200 import lowering as Lw
    res, desc, instr, prog, hdr = _c_sizeof(["gevo_result", "gevo_eval_desc", "gevo_instr",
                                             "gevo_prog", "gevo_plan_header"])
    assert res == _lib.RESULT_DTYPE.itemsize == 56
    assert desc == ctypes.sizeof(_lib.GevoEvalDesc)
    assert (instr, prog, hdr) == (Lw.INSTR_DTYPE.itemsize, Lw.PROG_DTYPE.itemsize,
                                  Lw.HEADER_DTYPE.itemsize)


def test_integration_stub_matches_header():
    """The ctypes stub INTEGRATION.md tells a maintainer to add: executed up
    to its declarations against the built library; its gevo_result must be
    the header's 56 bytes (a shorter struct would overflow `res`)."""
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = text.split("```python\n# evotir/_gevo.py")[1].split("```")[0]
    decl = block.split("ctx = ctypes.c_void_p()")[0]
    decl = decl.replace('ctypes.CDLL("libgevo.so")', f"ctypes.CDLL({build.build()!r})")
    ns = {}
    exec("import ctypes, numpy as np\n#" + decl, ns)
    (res,) = _c_sizeof(["gevo_result"])
    assert ctypes.sizeof(ns["gevo_result"]) == res
    assert ctypes.sizeof(ns["gevo_eval_desc"]) == ctypes.sizeof(_lib.GevoEvalDesc)
    assert [f for f, _ in ns["gevo_result"]._fields_] == list(_lib.RESULT_DTYPE.names)
