"""Build libgevo.so (sm_100a) in-tree with nvcc.

The library is the product: `paper_2310_10211_b200._lib` refuses to run
without it (there is no CPU fallback).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libgevo.so")
SOURCES = ["gevo_exec.cu", "gevo_exec_tc.cu", "nsga2.cu", "splits.cu", "gevo_abi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC"]


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files += [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)]
    return files


def source_sha(defines=()) -> str:
    """Hash of everything the library is compiled from (csrc/, include/, the
    nvcc flags): the identity of a build.  The .so bytes themselves differ
    from one nvcc run to the next (temporary file names end up in the
    image), so measurements recorded for a build (profiles/traffic.json)
    are stamped with this."""
    import hashlib
    h = hashlib.sha256()
    for f in sorted(_deps()):
        if f.endswith((".cu", ".cuh", ".h")):
            h.update(os.path.basename(f).encode() + b"\0" + open(f, "rb").read())
    h.update(" ".join([*ARCH, *FLAGS, *[f"-D{d}" for d in defines]]).encode())
    return h.hexdigest()[:16]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _deps())


def build(force: bool = False, verbose: bool = False, defines=(), out=None) -> str:
    """Compile every source to an object in parallel (the two executor
    builds dominate: ~2.5 min each), then link libgevo.so."""
    out = out or LIB
    if not force and out == LIB and not needs_build():
        return LIB
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    flags = [*ARCH, *FLAGS, "-I", INCLUDE, "-I", CSRC, *[f"-D{d}" for d in defines]]
    if verbose:
        flags += ["-Xptxas", "-v"]
    with tempfile.TemporaryDirectory() as tmp:
        objs = [os.path.join(tmp, s.replace(".cu", ".o")) for s in SOURCES]

        def compile_one(src_obj):
            src, obj = src_obj
            return subprocess.run([NVCC, *flags, "-c", os.path.join(CSRC, src), "-o", obj],
                                  capture_output=True, text=True)
        with ThreadPoolExecutor(len(SOURCES)) as pool:
            results = list(pool.map(compile_one, zip(SOURCES, objs)))
        for res in results:
            if verbose:
                sys.stderr.write(res.stderr)
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError("nvcc failed building libgevo.so")
        res = subprocess.run([NVCC, *ARCH, "-shared", "-o", out + ".tmp", *objs, "-ldl"],
                             capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed linking libgevo.so")
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
