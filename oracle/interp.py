"""numpy restatement of the reference interpreter (test oracle; see __init__).

Semantics follow pkg/src/evotir/interpreter.py:
  * dtypes f32->float64, i32->int64, i1->bool          (ir.py:33-37)
  * op closures                                         (interpreter.py:78-185)
  * integer divide: trunc(a/b) via float64, x/0 == 0    (interpreter.py:65-69)
  * cost: unit*out count; dot m*n*k; reduce in count    (interpreter.py:41-59)
  * run under np.errstate(all="ignore"), returns may alias inputs
                                                        (interpreter.py:219-225)
`perturb=True` swaps in a reversed-k dot and a reversed reduce-sum: the
sensitivity probe of SURVEY.md §8(c) rule 5.
"""
from __future__ import annotations

import numpy as np

DTYPE = {"f32": np.float64, "i32": np.int64, "i1": np.bool_}
CMP = {"eq": np.equal, "ne": np.not_equal, "lt": np.less,
       "le": np.less_equal, "gt": np.greater, "ge": np.greater_equal}
BIN = {"add": np.add, "subtract": np.subtract, "multiply": np.multiply,
       "maximum": np.maximum}


def _kind(k):
    return getattr(k, "value", k)


def op_cost(op, operand_types, table=None) -> float:
    """CostModel.op_cost (interpreter.py:51-59)."""
    unit = (table or {}).get(op.opcode, 1.0)
    if op.opcode == "dot":
        a, b = operand_types
        return unit * a.shape[0] * b.shape[1] * a.shape[1]
    if op.opcode == "reduce":
        return unit * _count(operand_types[0].shape)
    return unit * _count(op.result_type.shape)


def _count(shape):
    n = 1
    for d in shape:
        n *= d
    return n


def function_cost(fn, table=None) -> float:
    """ExecPlan.total_cost: float accumulation in op order (interpreter.py:205-214)."""
    types = dict(fn.params)
    total = 0.0
    for op in fn.ops:
        total += op_cost(op, tuple(types[v] for v in op.operands), table)
        types[op.result] = op.result_type
    return total


def _int_div(a, b):
    nz = b != 0
    q = np.trunc(np.true_divide(a, np.where(nz, b, 1)))
    return np.where(nz, q, 0).astype(np.int64)


def _dot_reversed(a, b):
    if a.dtype.kind != "f":
        return a @ b
    return np.einsum("ik,kj->ij", a[:, ::-1], b[::-1, :])


def apply_op(op, ins, in_types, perturb=False):
    """Value of one op given operand arrays (interpreter.py:84-183)."""
    code, rt = op.opcode, op.result_type
    kind = _kind(rt.kind)
    a = op.attrs
    if code == "constant":
        return np.asarray(a["value"], dtype=DTYPE[kind]).reshape(rt.shape)
    if code in BIN:
        return BIN[code](ins[0], ins[1])
    if code == "divide":
        if kind == "i32":
            return _int_div(ins[0], ins[1])
        return np.true_divide(ins[0], ins[1])
    if code == "negate":
        return np.negative(ins[0])
    if code == "exponential":
        return np.exp(ins[0])
    if code == "log":
        return np.log(ins[0])
    if code == "dot":
        return _dot_reversed(*ins) if perturb else ins[0] @ ins[1]
    if code == "transpose":
        return np.transpose(ins[0], a["perm"])
    if code == "reshape":
        return np.reshape(ins[0], rt.shape)
    if code == "broadcast_in_dim":
        mid = [1] * len(rt.shape)
        for s, d in enumerate(a["dims"]):
            mid[d] = in_types[0].shape[s]
        return np.broadcast_to(np.reshape(ins[0], tuple(mid)), rt.shape)
    if code == "reduce":
        if a["kind"] == "max":
            return np.max(ins[0], axis=a["axis"])
        if perturb and ins[0].dtype.kind == "f":
            return np.sum(np.flip(ins[0], axis=a["axis"]), axis=a["axis"])
        return np.sum(ins[0], axis=a["axis"])
    if code == "pad":
        return np.pad(ins[0], tuple(zip(a["low"], a["high"])),
                      constant_values=ins[1][()])
    if code == "slice":
        return ins[0][tuple(slice(s, l) for s, l in zip(a["start"], a["limit"]))]
    if code == "compare":
        return CMP[a["kind"]](ins[0], ins[1])
    if code == "select":
        return np.where(ins[0], ins[1], ins[2])
    if code == "iota":
        d = a["dim"]
        mid = [1] * len(rt.shape)
        mid[d] = rt.shape[d]
        ramp = np.arange(rt.shape[d], dtype=DTYPE[kind]).reshape(mid)
        return np.ascontiguousarray(np.broadcast_to(ramp, rt.shape))
    if code == "convert":
        x = ins[0]
        if kind == "i1":
            return x != 0
        if kind == "i32":
            return np.trunc(x).astype(np.int64) if x.dtype.kind == "f" \
                else x.astype(np.int64)
        return x.astype(DTYPE[kind])
    raise ValueError(f"oracle: unknown opcode {code!r}")


class Program:
    """One function prepared for repeated execution (ExecPlan analogue)."""

    def __init__(self, fn, perturb=False):
        self.fn = fn
        self.perturb = perturb
        types = dict(fn.params)
        slot = {n: i for i, (n, _) in enumerate(fn.params)}
        self.steps = []
        for op in fn.ops:
            tys = tuple(types[v] for v in op.operands)
            self.steps.append((op, tuple(slot[v] for v in op.operands), tys))
            slot[op.result] = len(slot)
            types[op.result] = op.result_type
        self.ret = tuple(slot[v] for v in fn.returns)

    def __call__(self, args):
        vals = list(args)
        with np.errstate(all="ignore"):
            for op, slots, tys in self.steps:
                vals.append(apply_op(op, [vals[s] for s in slots], tys,
                                     self.perturb))
        return [vals[s] for s in self.ret]
