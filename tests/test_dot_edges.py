"""Dot summation orders over the wide n % 8 edges, pinned to the reference.

Fixture: tests/golden/dot_edges.json.gz (tests/golden/make_dot_golden.py,
recorded through the reference's own interpret): `dot` over every
transposition combination, n % 8 in 4..7 (and 0), m % 4 in 0..3, K on both
sides of the OpenBLAS kernels' thresholds; operands regenerated from each
case's seed.

CPU: the summation order lowering.dot_modes picks, emulated exactly
(tests/test_dot_orders.emulate), reproduces the recorded outputs in the
edge columns, the body columns and the m % 4 corner rows.
GPU: the device (through the C ABI, gevo_exec_once) reproduces every
recorded output bit for bit.
"""
import base64

import numpy as np
import pytest

from golden_io import load
from paper_2310_10211_b200 import dialect
from paper_2310_10211_b200 import lowering as Lw
from paper_2310_10211_b200.lowering import Val
from test_dot_orders import elem_strides, emulate

CASES = load("dot_edges.json.gz")["cases"]


def _operands(c):
    pa = (c["k"], c["m"]) if c["ta"] else (c["m"], c["k"])
    pb = (c["n"], c["k"]) if c["tb"] else (c["k"], c["n"])
    rng = np.random.default_rng(c["seed"])
    return rng.standard_normal(pa), rng.standard_normal(pb)


def _expected(c):
    return np.frombuffer(base64.b64decode(c["expected"]), dtype=np.float64).reshape(c["m"], c["n"])


def test_fixture_covers_the_wide_edges():
    seen = {(c["n"] % 8, c["m"] % 4, c["k"] >= 32, c["ta"], c["tb"]) for c in CASES}
    want = {(r, q, big, ta, tb) for r in range(4, 8) for q in range(4)
            for big in (False, True) for ta in (False, True) for tb in (False, True)}
    assert want <= seen


def test_rule_reproduces_reference_dots():
    for c in CASES:
        a, b = _operands(c)
        A = a.T if c["ta"] else a
        B = b.T if c["tb"] else b
        exp = _expected(c)
        m, n = exp.shape
        m0, split, m1, xrow = Lw.dot_modes(Val(0, 0, A.shape, elem_strides(A), Lw.K_F64),
                                           Val(0, 0, B.shape, elem_strides(B), Lw.K_F64))
        rows = sorted({0, m // 2, m - 1, m - 2, m - m % 4} & set(range(m)))
        cols = sorted(set(range(n - n % 8, n)) | {0, n // 2} | ({split - 1, split} & set(range(n))))
        for i in rows:
            for j in cols:
                got = emulate(m0 if j < split else m1, A, B, i, j, j >= split and i >= xrow)
                assert got == exp[i, j], (c["m"], c["k"], c["n"], c["ta"], c["tb"], i, j)


@pytest.mark.gpu
def test_device_matches_reference_dots():
    from paper_2310_10211_b200 import _lib
    from test_gpu_parity import _words, run_once
    ctx = _lib.Context(0)
    try:
        fns = [dialect.parse_function(c["text"]) for c in CASES]
        params = [[_words(x) for x in _operands(c)] for c in CASES]
        outs = run_once(ctx, fns, params)
    finally:
        ctx.close()
    bad = []
    for c, (got,) in zip(CASES, outs):
        exp = _expected(c)
        if not np.array_equal(np.asarray(got, dtype=np.float64).reshape(exp.shape), exp):
            bad.append((c["m"], c["k"], c["n"], c["ta"], c["tb"]))
    print(f"dot edges bit-exact {len(CASES) - len(bad)}/{len(CASES)}")
    assert not bad, bad[:10]
