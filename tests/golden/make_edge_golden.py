"""Edge-semantics fixtures from the REAL reference interpreter (build container).

    PYTHONPATH=/root/reference/pkg/src:. PYTHONDONTWRITEBYTECODE=1 \
    python tests/golden/make_edge_golden.py

The reference pins its interpreter's corner cases with golden vectors in
pkg/tests/test_interpreter.py:42-157 (integer division truncating with
x/0 = 0, quiet float division by zero, exp overflow to inf, the affine
example with cost 21, iota/convert).  Its random op cases (opgen.py:28-31)
draw uniform(-4, 4) and so never reach the x86-specific conversions
(SURVEY.md §7.3 item 5).  This script records, through the reference's own
`interpret` (interpreter.py:248-269), those golden programs plus the corners
the device must emulate:

  * convert f32 -> i32 of NaN / +-inf / out-of-range -> INT64_MIN
    (np.trunc(...).astype(int64) on x86, interpreter.py:177-180);
  * convert f32 -> i1 of NaN -> True (x != 0, interpreter.py:176);
  * maximum and reduce-max propagate NaN (interpreter.py:94, 141);
  * log of 0 / negatives, negate of -0.0 and NaN, compares with NaN;
  * 64-bit wrap-around of i32 add / multiply / dot / reduce-sum;
  * pad with a NaN pad value, slices of it.

Writes tests/golden/edge_cases.json.gz: per case the program text, the
operands, the reference outputs and the reference static cost.
"""
from __future__ import annotations

import base64
import gzip
import json
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from evotir.interpreter import TensorValue, interpret  # noqa: E402
from evotir.ir import ElementKind, TensorType  # noqa: E402
from evotir.parser import parse_module  # noqa: E402

F32, I32, I1 = ElementKind.f32, ElementKind.i32, ElementKind.i1
NAN, INF = float("nan"), float("inf")


def enc(a) -> dict:
    a = np.ascontiguousarray(a)
    return {"dtype": a.dtype.str, "shape": list(a.shape),
            "b64": base64.b64encode(a.tobytes()).decode()}


def tv(values, kind, shape=None):
    arr = np.asarray(values, dtype=kind.dtype)
    if shape is not None:
        arr = arr.reshape(shape)
    return TensorValue(TensorType(tuple(arr.shape), kind), arr)


def t(shape, kind="f32"):
    return "tensor<" + "".join(f"{d}x" for d in shape) + kind + ">"


CASES = []


def case(name, text, args, ref=""):
    CASES.append((name, text, args, ref))


# --- test_interpreter.py golden vectors -----------------------------------
case("int_div_truncates", """\
func @f(%a: tensor<6xi32>, %b: tensor<6xi32>) -> tensor<6xi32> {
  %0 = divide %a, %b : tensor<6xi32>
  return %0 : tensor<6xi32>
}""", [tv([7, -7, 7, -7, 5, 0], I32), tv([2, 2, -2, -2, 0, 0], I32)],
     "test_interpreter.py:42-52")
case("float_div_by_zero", """\
func @f(%a: tensor<3xf32>, %b: tensor<3xf32>) -> tensor<3xf32> {
  %0 = divide %a, %b : tensor<3xf32>
  return %0 : tensor<3xf32>
}""", [tv([1.0, -1.0, 0.0], F32), tv([0.0, 0.0, 0.0], F32)], "test_interpreter.py:55-67")
case("exp_overflow", """\
func @f(%x: tensor<2xf32>) -> tensor<2xf32> {
  %0 = exponential %x : tensor<2xf32>
  return %0 : tensor<2xf32>
}""", [tv([1000.0, -1000.0], F32)], "test_interpreter.py:70-80")
case("affine_cost_21", """\
func @f(%x: tensor<2x3xf32>, %w: tensor<3x2xf32>) -> tensor<2x2xf32> {
  %0 = dot %x, %w : tensor<2x2xf32>
  %1 = constant dense<0.5> : tensor<f32>
  %2 = broadcast_in_dim %1 {dims = []} : tensor<2x2xf32>
  %3 = add %0, %2 : tensor<2x2xf32>
  return %3 : tensor<2x2xf32>
}""", [tv(np.arange(6.0), F32, (2, 3)), tv(np.ones(6), F32, (3, 2))],
     "test_interpreter.py:83-93")
case("iota_convert_chain", """\
func @f() -> tensor<3x2xi32> {
  %0 = iota {dim = 0} : tensor<3x2xf32>
  %1 = constant dense<0.5> : tensor<f32>
  %2 = broadcast_in_dim %1 {dims = []} : tensor<3x2xf32>
  %3 = add %0, %2 : tensor<3x2xf32>
  %4 = convert %3 : tensor<3x2xi32>
  return %4 : tensor<3x2xi32>
}""", [], "test_interpreter.py:145-157")

# --- x86 conversion corners ------------------------
CVT_IN = [NAN, INF, -INF, 1e30, -1e30, 9.3e18, -9.3e18, 9.2e18, -9.2e18, 2.5, -2.5,
          -0.0, 0.49999999999999994, -1.5, 4503599627370497.0, 1e-300]
n = len(CVT_IN)
case("convert_f32_i32_x86", f"""\
func @f(%x: {t([n])}) -> {t([n], 'i32')} {{
  %0 = convert %x : {t([n], 'i32')}
  return %0 : {t([n], 'i32')}
}}""", [tv(CVT_IN, F32)], "interpreter.py:177-180")
case("convert_f32_i1", f"""\
func @f(%x: {t([n])}) -> {t([n], 'i1')} {{
  %0 = convert %x : {t([n], 'i1')}
  return %0 : {t([n], 'i1')}
}}""", [tv(CVT_IN, F32)], "interpreter.py:175-176")
case("convert_chain_i32_i1_f32", """\
func @f(%a: tensor<6xi32>) -> (tensor<6xf32>, tensor<6xi1>, tensor<6xf32>) {
  %0 = convert %a : tensor<6xf32>
  %1 = convert %a : tensor<6xi1>
  %2 = convert %1 : tensor<6xf32>
  return %0, %1, %2 : tensor<6xf32>, tensor<6xi1>, tensor<6xf32>
}""", [tv([0, 1, -1, 2 ** 62, -(2 ** 63), 9007199254740993], I32)], "interpreter.py:174-183")

# --- NaN propagation / IEEE corners ----------------------------------------
case("maximum_nan", """\
func @f(%a: tensor<6xf32>, %b: tensor<6xf32>) -> tensor<6xf32> {
  %0 = maximum %a, %b : tensor<6xf32>
  return %0 : tensor<6xf32>
}""", [tv([NAN, 1.0, NAN, -INF, -0.0, 0.0], F32), tv([1.0, NAN, NAN, INF, 0.0, -0.0], F32)],
     "interpreter.py:94")
case("reduce_max_nan_both_axes", """\
func @f(%x: tensor<3x4xf32>) -> (tensor<3xf32>, tensor<4xf32>) {
  %0 = reduce %x {axis = 1, kind = max} : tensor<3xf32>
  %1 = reduce %x {axis = 0, kind = max} : tensor<4xf32>
  return %0, %1 : tensor<3xf32>, tensor<4xf32>
}""", [tv([1.0, NAN, 3.0, 2.0, -INF, -1.0, -2.0, -3.0, 5.0, 4.0, NAN, INF], F32, (3, 4))],
     "interpreter.py:138-142")
case("reduce_sum_inf_nan", """\
func @f(%x: tensor<3x4xf32>) -> (tensor<3xf32>, tensor<4xf32>) {
  %0 = reduce %x {axis = 1, kind = sum} : tensor<3xf32>
  %1 = reduce %x {axis = 0, kind = sum} : tensor<4xf32>
  return %0, %1 : tensor<3xf32>, tensor<4xf32>
}""", [tv([INF, -INF, 1.0, 2.0, 1e308, 1e308, -1.0, 0.5, NAN, 0.0, 1.0, 1.0], F32, (3, 4))],
     "interpreter.py:138-142")
case("log_neg_exp", """\
func @f(%x: tensor<8xf32>) -> (tensor<8xf32>, tensor<8xf32>, tensor<8xf32>) {
  %0 = log %x : tensor<8xf32>
  %1 = negate %x : tensor<8xf32>
  %2 = exponential %x : tensor<8xf32>
  return %0, %1, %2 : tensor<8xf32>, tensor<8xf32>, tensor<8xf32>
}""", [tv([0.0, -0.0, -1.0, 1.0, INF, NAN, 709.78, -745.2], F32)], "interpreter.py:102-112")
for kind in ("eq", "ne", "lt", "le", "gt", "ge"):
    case(f"compare_{kind}_nan", f"""\
func @f(%a: tensor<6xf32>, %b: tensor<6xf32>) -> tensor<6xi1> {{
  %0 = compare %a, %b {{kind = {kind}}} : tensor<6xi1>
  return %0 : tensor<6xi1>
}}""", [tv([NAN, 1.0, NAN, -0.0, INF, 2.0], F32), tv([1.0, NAN, NAN, 0.0, INF, 1.0], F32)],
         "interpreter.py:155-158")
case("select_nan_pred", """\
func @f(%x: tensor<5xf32>, %a: tensor<5xf32>, %b: tensor<5xf32>) -> tensor<5xf32> {
  %0 = convert %x : tensor<5xi1>
  %1 = select %0, %a, %b : tensor<5xf32>
  return %1 : tensor<5xf32>
}""", [tv([NAN, 0.0, -0.0, 2.0, 0.0], F32), tv([1.0, 2.0, 3.0, 4.0, 5.0], F32),
       tv([-1.0, -2.0, -3.0, -4.0, -5.0], F32)], "interpreter.py:159-162")

# --- 64-bit integer wrap (i32 is int64, ir.py:33-37) ------------------------
case("i32_wrap_add_mul", """\
func @f(%a: tensor<4xi32>, %b: tensor<4xi32>) -> (tensor<4xi32>, tensor<4xi32>, tensor<4xi32>) {
  %0 = add %a, %b : tensor<4xi32>
  %1 = multiply %a, %b : tensor<4xi32>
  %2 = subtract %a, %b : tensor<4xi32>
  return %0, %1, %2 : tensor<4xi32>, tensor<4xi32>, tensor<4xi32>
}""", [tv([2 ** 62, -(2 ** 63), 2 ** 63 - 1, 3], I32), tv([2 ** 62, -1, 2, -(2 ** 62)], I32)],
     "interpreter.py:90-100")
case("i32_dot_reduce_wrap", """\
func @f(%a: tensor<2x3xi32>, %b: tensor<3x2xi32>) -> (tensor<2x2xi32>, tensor<2xi32>) {
  %0 = dot %a, %b : tensor<2x2xi32>
  %1 = reduce %a {axis = 1, kind = sum} : tensor<2xi32>
  return %0, %1 : tensor<2x2xi32>, tensor<2xi32>
}""", [tv([2 ** 62, 2 ** 62, 5, -7, 3, 2 ** 40], I32, (2, 3)),
       tv([4, 1, 2, -3, 2 ** 30, 6], I32, (3, 2))], "interpreter.py:114-116,138-142")
case("i32_div_min_by_minus1", """\
func @f(%a: tensor<4xi32>, %b: tensor<4xi32>) -> tensor<4xi32> {
  %0 = divide %a, %b : tensor<4xi32>
  return %0 : tensor<4xi32>
}""", [tv([-(2 ** 63), -(2 ** 63), 2 ** 63 - 1, -9], I32), tv([-1, 1, -1, 4], I32)],
     "interpreter.py:65-69")

# --- pad / slice / dot with non-finite values -------------------------------
case("pad_nan_value_slice", """\
func @f(%x: tensor<2x3xf32>, %p: tensor<f32>) -> (tensor<4x5xf32>, tensor<2x2xf32>) {
  %0 = pad %x, %p {low = [1, 0], high = [1, 2]} : tensor<4x5xf32>
  %1 = slice %0 {start = [1, 2], limit = [3, 4]} : tensor<2x2xf32>
  return %0, %1 : tensor<4x5xf32>, tensor<2x2xf32>
}""", [tv(np.arange(6.0) - 2.5, F32, (2, 3)), tv(NAN, F32)], "interpreter.py:144-153")
case("dot_nonfinite", """\
func @f(%a: tensor<2x3xf32>, %b: tensor<3x2xf32>) -> tensor<2x2xf32> {
  %0 = dot %a, %b : tensor<2x2xf32>
  return %0 : tensor<2x2xf32>
}""", [tv([INF, 1.0, 0.0, 1e308, 1e308, -1.0], F32, (2, 3)),
       tv([0.0, 1.0, 2.0, NAN, 1.0, 1.0], F32, (3, 2))], "interpreter.py:114-116")


def main():
    out = []
    for name, text, args, ref in CASES:
        m = parse_module(text + "\n")
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            outs, cost = interpret(m, "f", args)
        out.append({"name": name, "text": text + "\n", "ref": ref, "cost": cost,
                    "operands": [enc(a.data) for a in args],
                    "expected": [enc(o.data) for o in outs]})
        print(f"{name:28s} cost {cost:6.0f}  " +
              " | ".join(str(o.data.reshape(-1).tolist())[:60] for o in outs))
    path = os.path.join(HERE, "edge_cases.json.gz")
    with gzip.open(path, "wt") as f:
        json.dump({"cases": out}, f, separators=(",", ":"), sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    sys.exit(main())
