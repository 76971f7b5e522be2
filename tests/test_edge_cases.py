"""The reference's interpreter golden vectors and x86/IEEE corner cases
(tests/golden/edge_cases.json.gz, recorded from the real reference by
tests/golden/make_edge_golden.py): test_interpreter.py:42-157 plus
convert NaN/+-inf/out-of-range -> INT64_MIN, convert NaN -> True, NaN
propagation of maximum / reduce-max, log/negate/compare corners, 64-bit
integer wrap, NaN pad values.

CPU: the oracle and the lowering's static cost reproduce every recorded
output and cost.  GPU: the device (through the C ABI, gevo_exec_once)
reproduces every output bit for bit (NaN matched as NaN, signed zeros by
sign) -- the bar for integer and IEEE-special work is exact.
"""
import numpy as np
import pytest

from golden_io import dec, load
from oracle import interp as OI
from paper_2310_10211_b200 import dialect
from paper_2310_10211_b200.lowering import static_cost

CASES = load("edge_cases.json.gz")["cases"]


def _same(got, exp):
    got = np.asarray(got).reshape(exp.shape)
    if exp.dtype == np.float64:
        got = got.astype(np.float64)
        return (np.array_equal(got, exp, equal_nan=True)
                and np.array_equal(np.signbit(got[got == 0]), np.signbit(exp[exp == 0])))
    return np.array_equal(got.astype(exp.dtype), exp)


def _params(c, fn):
    return [dec(o).reshape(t.shape) for o, (_, t) in zip(c["operands"], fn.params)]


def test_edge_fixture_covers_reference_goldens():
    names = {c["name"] for c in CASES}
    assert {"int_div_truncates", "float_div_by_zero", "exp_overflow", "affine_cost_21",
            "iota_convert_chain", "convert_f32_i32_x86", "maximum_nan"} <= names
    aff = next(c for c in CASES if c["name"] == "affine_cost_21")
    assert aff["cost"] == 21 and dec(aff["expected"][0]).tolist() == [[3.5, 3.5], [12.5, 12.5]]
    cvt = next(c for c in CASES if c["name"] == "convert_f32_i32_x86")
    out = dec(cvt["expected"][0])
    assert out[:7].tolist() == [-(2 ** 63)] * 7      # NaN, +-inf, +-1e30, +-9.3e18


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_oracle_and_cost_match_reference(c):
    fn = dialect.parse_function(c["text"])
    assert static_cost(fn) == c["cost"]
    assert OI.function_cost(fn) == c["cost"]
    got = OI.Program(fn)(_params(c, fn))
    for g, e in zip(got, c["expected"]):
        assert _same(g, dec(e)), (c["name"], g, dec(e))


@pytest.mark.gpu
def test_device_matches_reference_edge_cases():
    from paper_2310_10211_b200 import _lib
    from test_gpu_parity import _words, run_once
    ctx = _lib.Context(0)
    try:
        fns = [dialect.parse_function(c["text"]) for c in CASES]
        params = [[_words(p) for p in _params(c, fn)] for c, fn in zip(CASES, fns)]
        outs = run_once(ctx, fns, params)
    finally:
        ctx.close()
    bad = []
    for c, got in zip(CASES, outs):
        for g, e in zip(got, c["expected"]):
            if not _same(g, dec(e)):
                bad.append((c["name"], np.asarray(g).reshape(-1).tolist(),
                            dec(e).reshape(-1).tolist()))
    print(f"edge cases bit-exact {len(CASES) - len({b[0] for b in bad})}/{len(CASES)}")
    assert not bad, bad
