"""Reader for the tensor-dialect program text that crosses the evaluator boundary.

The evaluator consumes *variant programs*: the `@train_step` / `@forward`
functions of a patched module (reference: `apply_patch`, genome.py:482-516,
produces them as `evotir.ir.Module`; `print_module`, printer.py:84, renders
them as text).  On a host where `evotir` is importable the lowering takes
its Module objects directly (duck-typed: `.params`, `.ops`, `.returns`,
`.return_types`, `op.opcode/.operands/.result/.result_type/.attrs`).  Where
it is not (the GPU box), programs arrive as dialect text and this module
turns them into the same duck-typed shape.

Grammar: pkg/docs/dialect.md:9-31.  This is a reader, not a verifier: the
reference verifies every variant inside `apply_patch` before it reaches the
evaluator (genome.py:511-515), so inputs here are already well typed.
"""
from __future__ import annotations

import re
import copyreg
from dataclasses import dataclass, field

import numpy as np

KINDS = ("f32", "i32", "i1")
# runtime dtypes of the reference interpreter (ir.py:33-37): f32 is float64
DTYPE = {"f32": np.float64, "i32": np.int64, "i1": np.bool_}


class DialectError(Exception):
    pass


@dataclass(frozen=True)
class TensorType:
    shape: tuple
    kind: str  # "f32" | "i32" | "i1"

    @property
    def rank(self) -> int:
        return len(self.shape)

    @property
    def count(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    def __str__(self) -> str:
        return "tensor<" + "".join(f"{d}x" for d in self.shape) + self.kind + ">"


@dataclass(eq=False)
class Operation:
    op_id: str
    opcode: str
    result: str
    result_type: TensorType
    operands: tuple = ()
    attrs: dict = field(default_factory=dict)


@dataclass(eq=False)
class FunctionBody:
    name: str
    params: tuple
    ops: list
    returns: tuple
    return_types: tuple


@dataclass(eq=False)
class Module:
    functions: dict
    constants: dict = field(default_factory=dict)  # name -> ndarray


# Compact pickling (positional tuples instead of dataclass __dict__s): the
# evaluator ships variant functions to its lowering processes, and this is
# the part of that transfer the parent pays serially.
def _reduce_type(t):
    return (TensorType, (t.shape, t.kind))


def _reduce_op(o):
    return (Operation, (o.op_id, o.opcode, o.result, o.result_type, o.operands, o.attrs))


def _reduce_fn(f):
    return (FunctionBody, (f.name, f.params, f.ops, f.returns, f.return_types))


copyreg.pickle(TensorType, _reduce_type)
copyreg.pickle(Operation, _reduce_op)
copyreg.pickle(FunctionBody, _reduce_fn)


def kind_name(kind) -> str:
    """'f32'/'i32'/'i1' for both this module's kinds and evotir.ElementKind."""
    return getattr(kind, "value", kind)


_TOK = re.compile(r"""
    (?P<ws>\s+|//[^\n]*)
  | (?P<type>tensor<[0-9x]*(?:f32|i32|i1)>)
  | (?P<dense>dense<[^<>]*>)
  | (?P<value>%[A-Za-z0-9_]+)
  | (?P<symbol>@[A-Za-z0-9_]+)
  | (?P<number>[-+]?(?:\d+\.\d*|\.\d+|\d+)(?:[eE][-+]?\d+)?)
  | (?P<ident>[A-Za-z_][A-Za-z0-9_]*)
  | (?P<arrow>->)
  | (?P<punct>[{}()\[\],=:])
""", re.VERBOSE)

_LIST_ATTRS = {"perm", "dims", "low", "high", "start", "limit"}
_WORDS = {"true": True, "false": False, "inf": float("inf"),
          "-inf": float("-inf"), "nan": float("nan")}


def parse_type(text: str) -> TensorType:
    body = text[len("tensor<"):-1]
    parts = body.split("x")
    kind = parts[-1]
    if kind not in KINDS:
        raise DialectError(f"bad element kind in {text!r}")
    return TensorType(tuple(int(p) for p in parts[:-1]), kind)


def _dense(text: str, ty: TensorType) -> np.ndarray:
    payload = text[len("dense<"):-1]
    # the payload grammar is JSON-like once the IEEE words are quoted away
    items = re.findall(r"-inf|inf|nan|true|false|[-+]?(?:\d+\.\d*|\.\d+|\d+)"
                       r"(?:[eE][-+]?\d+)?|[\[\],]", payload)

    pos = 0

    def value():
        nonlocal pos
        tok = items[pos]
        pos += 1
        if tok == "[":
            out = []
            if items[pos] == "]":
                pos += 1
                return out
            while True:
                out.append(value())
                sep = items[pos]
                pos += 1
                if sep == "]":
                    return out
        if tok in _WORDS:
            return _WORDS[tok]
        return float(tok) if any(c in tok for c in ".eE") else int(tok)

    arr = np.array(value(), dtype=DTYPE[ty.kind])
    if tuple(arr.shape) != ty.shape:
        raise DialectError(f"dense literal shape {arr.shape} != {ty}")
    return arr


class _Reader:
    def __init__(self, text: str):
        self.toks = []
        pos = 0
        while pos < len(text):
            m = _TOK.match(text, pos)
            if m is None:
                raise DialectError(f"unexpected {text[pos:pos + 16]!r}")
            if m.lastgroup != "ws":
                self.toks.append((m.lastgroup, m.group()))
            pos = m.end()
        self.toks.append(("eof", ""))
        self.i = 0
        self.op_counter = 0

    def peek(self):
        return self.toks[self.i]

    def take(self, kind=None, text=None):
        tok = self.toks[self.i]
        if (kind and tok[0] != kind) or (text and tok[1] != text):
            raise DialectError(f"expected {text or kind}, got {tok[1]!r}")
        self.i += 1
        return tok[1]

    def at(self, text):
        return self.toks[self.i][1] == text

    def module(self) -> Module:
        m = Module(functions={}, constants={})
        while self.peek()[0] != "eof":
            word = self.take("ident")
            if word == "global":
                name = self.take("symbol")[1:]
                self.take(text="=")
                dense = self.take("dense")
                self.take(text=":")
                ty = parse_type(self.take("type"))
                m.constants[name] = _dense(dense, ty)
            elif word == "func":
                f = self.func()
                m.functions[f.name] = f
            else:
                raise DialectError(f"expected func/global, got {word!r}")
        return m

    def types(self):
        if self.at("("):
            self.take(text="(")
            out = [parse_type(self.take("type"))]
            while self.at(","):
                self.take(text=",")
                out.append(parse_type(self.take("type")))
            self.take(text=")")
            return tuple(out)
        return (parse_type(self.take("type")),)

    def func(self) -> FunctionBody:
        name = self.take("symbol")[1:]
        self.take(text="(")
        params = []
        while not self.at(")"):
            v = self.take("value")
            self.take(text=":")
            params.append((v, parse_type(self.take("type"))))
            if self.at(","):
                self.take(text=",")
        self.take(text=")")
        rtypes = ()
        if self.peek()[0] == "arrow":
            self.take("arrow")
            rtypes = self.types()
        self.take(text="{")
        ops = []
        returns = ()
        while True:
            if self.at("return"):
                self.take()
                vals = []
                while self.peek()[0] == "value":
                    vals.append(self.take("value"))
                    if self.at(","):
                        self.take(text=",")
                if vals:
                    self.take(text=":")
                    parse_type(self.take("type"))
                    while self.at(","):
                        self.take(text=",")
                        parse_type(self.take("type"))
                returns = tuple(vals)
                self.take(text="}")
                break
            ops.append(self.op())
        return FunctionBody(name, tuple(params), ops, returns, tuple(rtypes))

    def op(self) -> Operation:
        res = self.take("value")
        self.take(text="=")
        opcode = self.take("ident")
        op_id = f"o{self.op_counter}"
        self.op_counter += 1
        attrs = {}
        operands = []
        if opcode == "constant":
            dense = self.take("dense")
            self.take(text=":")
            ty = parse_type(self.take("type"))
            attrs["value"] = _dense(dense, ty)
            return Operation(op_id, opcode, res, ty, (), attrs)
        while self.peek()[0] == "value":
            operands.append(self.take("value"))
            if self.at(","):
                self.take(text=",")
        if self.at("{"):
            self.take(text="{")
            while not self.at("}"):
                key = self.take("ident")
                self.take(text="=")
                if self.at("["):
                    self.take(text="[")
                    vals = []
                    while not self.at("]"):
                        vals.append(int(self.take("number")))
                        if self.at(","):
                            self.take(text=",")
                    self.take(text="]")
                    attrs[key] = tuple(vals)
                elif self.peek()[0] == "number":
                    attrs[key] = int(self.take("number"))
                else:
                    attrs[key] = self.take("ident")
                if self.at(","):
                    self.take(text=",")
            self.take(text="}")
        self.take(text=":")
        ty = parse_type(self.take("type"))
        return Operation(op_id, opcode, res, ty, tuple(operands), attrs)


def parse_module(text: str) -> Module:
    """Dialect text -> Module (duck-compatible with evotir.ir.Module)."""
    return _Reader(text).module()


def parse_function(text: str) -> FunctionBody:
    m = parse_module(text)
    if len(m.functions) != 1:
        raise DialectError("expected exactly one function")
    return next(iter(m.functions.values()))


def _fmt_scalar(x, kind: str) -> str:
    if kind == "i1":
        return "true" if bool(x) else "false"
    if kind == "i32":
        return str(int(x))
    v = float(x)
    if v != v:
        return "nan"
    if v in (float("inf"), float("-inf")):
        return "inf" if v > 0 else "-inf"
    return repr(v)


def _fmt_dense(a: np.ndarray, kind: str) -> str:
    def rec(x):
        if x.ndim == 0:
            return _fmt_scalar(x[()], kind)
        return "[" + ", ".join(rec(y) for y in x) + "]"
    return f"dense<{rec(np.asarray(a))}>"


_ATTR_ORDER = {"transpose": ("perm",), "broadcast_in_dim": ("dims",),
               "reduce": ("axis", "kind"), "pad": ("low", "high"),
               "slice": ("start", "limit"), "compare": ("kind",),
               "iota": ("dim",)}


def format_function(fn) -> str:
    """Canonical text of one function (same layout as printer.py:66-81)."""
    def ty(t):
        return str(TensorType(tuple(t.shape), kind_name(t.kind)))
    params = ", ".join(f"{n}: {ty(t)}" for n, t in fn.params)
    head = f"func @{fn.name}({params})"
    rts = [ty(t) for t in fn.return_types]
    if len(rts) == 1:
        head += f" -> {rts[0]}"
    elif rts:
        head += " -> (" + ", ".join(rts) + ")"
    lines = [head + " {"]
    for op in fn.ops:
        k = kind_name(op.result_type.kind)
        if op.opcode == "constant":
            lines.append(f"  {op.result} = constant "
                         f"{_fmt_dense(op.attrs['value'], k)} : {ty(op.result_type)}")
            continue
        s = f"  {op.result} = {op.opcode}"
        if op.operands:
            s += " " + ", ".join(op.operands)
        shown = [(a, op.attrs[a]) for a in _ATTR_ORDER.get(op.opcode, ())
                 if a in op.attrs]
        if shown:
            s += " {" + ", ".join(
                f"{a} = " + ("[" + ", ".join(str(int(v)) for v in val) + "]"
                             if isinstance(val, tuple) else str(val))
                for a, val in shown) + "}"
        lines.append(s + f" : {ty(op.result_type)}")
    if fn.returns:
        lines.append("  return " + ", ".join(fn.returns) + " : " + ", ".join(rts))
    else:
        lines.append("  return")
    lines.append("}")
    return "\n".join(lines) + "\n"
