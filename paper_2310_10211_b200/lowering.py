"""Lowering: variant function -> device launch plan (include/gevo_plan.h).

Replaces the reference's per-individual `ExecPlan` compile
(interpreter.py:188-217) with a pass that emits one instruction table per
function for the device executor.  Per op:

  constant / iota             -> constant pool (no instruction)
  transpose, broadcast_in_dim,
  slice, view-reshape         -> folded into operand strides (no instruction)
  copy-reshape                -> UNARY COPY into C order (numpy copies too)
  elementwise / compare /
  select / convert            -> UNARY / BINARY / SELECT
  reduce                      -> REDUCE with numpy's summation order
  dot                         -> DOT with numpy/OpenBLAS's summation order
  pad                         -> PAD

Results are stored in the memory order numpy would allocate them in
(layout.py), scratch is reused by liveness, and a returned value is written
straight into its weight slot when possible (else copied there).  The static
cost is the reference CostModel (interpreter.py:51-59) accumulated in op
order, so it is bit-identical.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import layout as L
from .dialect import kind_name

# --- constants mirrored from include/gevo_plan.h ----------------------------
MAXR, MAXP = 6, 8
BUF_ARENA, BUF_CONST, BUF_PARAM0, BUF_OUT0 = 0, 1, 2, 2 + MAXP
BUF_SMEM = 2 + 2 * MAXP
# shared-memory tier of the scratch arena (elements): values up to
# SMEM_VALUE_MAX elements are placed there while the per-function total
# stays within SMEM_BUDGET; everything else goes to the HBM arena.
SMEM_VALUE_MAX = 4096
SMEM_BUDGET = int(os.environ.get("GEVO_B200_SMEM_BUDGET", 3968))
K_F64, K_I64, K_I1 = 0, 1, 2
KIND = {"f32": K_F64, "i32": K_I64, "i1": K_I1}
OP_UNARY, OP_BINARY, OP_SELECT, OP_REDUCE, OP_DOT, OP_PAD, OP_EXT = 1, 2, 3, 4, 5, 6, 7
OP_TAPSUM = 8          # sum of products, one pass (fuse_tap_sums, gevo_plan.h)
TAP_MAX = 9
TAP_EPI = 3            # binary micro-ops a TAPSUM may apply before its store
EPI_SRC_OP = 64
EPI_MAX_OPS = 8        # micro-ops fused into one dot epilogue
EPI_MAX_EXT = 6        # extra operands (3 per continuation record)
U_NEG, U_EXP, U_LOG, U_COPY, U_CVT = range(5)
B_CODES = {"add": 0, "subtract": 1, "multiply": 2, "divide": 3, "maximum": 4}
CMP_CODES = {"eq": 5, "ne": 6, "lt": 7, "le": 8, "gt": 9, "ge": 10}
R_SUM_PAIRWISE, R_SUM_SEQ, R_MAX = 0, 1, 2
D_FMA_CHAIN, D_ACC8_TREE, D_SEQ_NOFMA, D_ACC8_TAIL = 0, 1, 2, 3

PLAN_MAGIC, PLAN_VERSION = 0x47455650, 2

_OPERAND = [("buf", "<i4"), ("off", "<i4"), ("st", "<i4", (MAXR,))]
INSTR_DTYPE = np.dtype([
    ("op", "<i4"), ("sub", "<i4"), ("kout", "<i4"), ("kin", "<i4"),
    ("rank", "<i4"), ("n", "<i4"), ("shp", "<i4", (MAXR,)),
    ("aux", "<i4", (MAXR,)), ("aux2", "<i4", (MAXR,)),
    ("out", _OPERAND), ("in", _OPERAND, (3,))], align=True)
PROG_DTYPE = np.dtype([
    ("train0", "<i4"), ("train0_n", "<i4"), ("train1", "<i4"),
    ("train1_n", "<i4"), ("fwd", "<i4"), ("fwd_n", "<i4"),
    ("const_off", "<i4"), ("result_slot", "<i4"), ("arena_off", "<i8"),
    ("arena_elems", "<i4"), ("flags", "<i4"),
    ("param_off", "<i4", (MAXP,)), ("out_off", "<i4", (MAXP,)),
    ("train2", "<i4"), ("train2_n", "<i4")], align=True)
HEADER_DTYPE = np.dtype([
    ("magic", "<u4"), ("version", "<u4"), ("n_instr", "<i4"),
    ("n_prog", "<i4"), ("n_const", "<i4"), ("weight_elems", "<i4"),
    ("n_weights", "<i4"), ("wofs", "<i4", (MAXP,)), ("max_arena", "<i4"),
    ("max_smem", "<i4"), ("total_elems", "<i8")], align=True)
assert INSTR_DTYPE.itemsize == 224 and PROG_DTYPE.itemsize == 120
assert HEADER_DTYPE.itemsize == 80

# step schedules (gevo_plan.h GEVO_SCHED_*, flags bits 0..1)
SCHED_STEADY1, SCHED_STEADY2, SCHED_ALT01, SCHED_ALT12 = 0, 1, 2, 3
FLAG_ALTERNATE = SCHED_ALT01   # steps >= 1: odd -> train1, even -> train0
FLAG_INPLACE_SHIFT = 2     # bits 2..7: weights train1 updates in place (plan.inplace_weights)

_NP_DTYPE = {K_F64: np.float64, K_I64: np.int64, K_I1: np.int64}


class LoweringError(Exception):
    pass


@dataclass
class Val:
    buf: int
    off: int
    shape: tuple
    st: tuple
    kind: int
    alloc: int = -1      # arena allocation id backing this value (-1: none)


@dataclass
class Lowered:
    instrs: list
    consts: list                 # float/int values (64-bit) in pool order
    arena_elems: int
    ret_strides: list            # numpy layout of each returned value
    cost: float
    smem_elems: int = 0


@dataclass
class _Alloc:
    size: int
    off: int = -1
    fixed: tuple | None = None   # (buf, off) when stored outside the arena
    space: str = "g"             # "s": shared-memory tier, "g": HBM arena


def _kind_of(ty) -> int:
    return KIND[kind_name(ty.kind)]


def _blas2d(s_outer, s_inner, d_inner) -> bool:
    # numpy is_blasable2d (element units): unit inner stride, outer >= inner dim
    return s_inner == 1 and s_outer >= d_inner


def _blas_strides(st, rows, cols):
    """The strides numpy's BLAS call sees for a 2-D operand.  A blasable
    operand (numpy is_blasable2d in either orientation) is passed as is; any
    other -- in this dialect, a broadcast view with a zero stride -- is first
    copied in KEEPORDER: C order unless axis 1 has the larger stride (ties,
    e.g. a broadcast scalar, stay C).  Probed on numpy 2.3.5: every
    broadcast/transposed combination reproduces this (profiles/
    r01_dot_orders.md); the no-FMA loop is never taken for these shapes."""
    if _blas2d(st[0], st[1], cols) or _blas2d(st[1], st[0], rows):
        return st
    return (1, rows) if abs(st[1]) > abs(st[0]) else (cols, 1)


def dot_modes(a: Val, b: Val):
    """(mode for columns < split, split, mode for the rest, xrow) reproducing
    the summation order numpy `@` + OpenBLAS (SkylakeX kernels, the build
    container's numpy 2.3 / OpenBLAS 0.3.30) use; see DESIGN.md.  In the
    columns >= split, ACC8 outputs of rows >= xrow (the m % 4 rows of the edge
    kernels) reduce their 8 lanes in the AVX-512 order instead of the
    pairwise tree; xrow = m when there is no such corner."""
    m, k = a.shape
    n = b.shape[1]
    if a.kind != K_F64:
        return D_SEQ_NOFMA, n, D_SEQ_NOFMA, m    # integer: exact anyway
    sa = _blas_strides(a.st, m, k)
    sb = _blas_strides(b.st, k, n)
    a_c = _blas2d(sa[0], sa[1], k)
    b_c = _blas2d(sb[0], sb[1], n)
    if m == 1 or k == 1 or n == 1:
        return D_FMA_CHAIN, n, D_FMA_CHAIN, m    # gemv/dot paths (see DESIGN)
    trans_a, trans_b = not a_c, not b_c
    corner = m - m % 4 if n % 8 and m % 4 else m
    # cblas row-major -> col-major: A' = B (trans_b), B' = A (trans_a)
    tn = trans_b and not trans_a
    small = _small_kernel(m, k, n, tn)
    if small and tn:
        # the TN kernel's n % 8 edge runs a 4-column sub-kernel first (its
        # m % 4 rows reduce by the pairwise tree) when n % 8 >= 4; the AVX-512
        # corner is in the columns after it
        return D_ACC8_TREE, n - n % 8 + (4 if n % 8 >= 4 else 0), D_ACC8_TREE, corner
    if small and not trans_a and not trans_b and n % 8 and k >= 16:
        # the n % 8 edge columns of the NN small kernel once K >= 16 (the
        # blocked kernels below keep one chain per output): 8 lane chains
        # when n % 8 <= 4 -- reduced in the AVX-512 order in the m % 4 rows
        # for n % 8 < 4, by the pairwise tree in every row for n % 8 == 4 --
        # and one k-ordered chain per output for n % 8 >= 5 (probed on
        # numpy / OpenBLAS here, tests/test_dot_orders.py)
        if n % 8 >= 5:
            return D_FMA_CHAIN, n, D_FMA_CHAIN, m
        return D_FMA_CHAIN, n - n % 8, D_ACC8_TREE, (m if n % 8 == 4 else corner)
    return D_FMA_CHAIN, n, D_FMA_CHAIN, m


def _small_kernel(m, k, n, tn) -> bool:
    """OpenBLAS's small-matrix permit (SkylakeX dgemm): M*N*K <= 1e6, and
    for TN problems only small outputs with K >= 32.  Everything else takes
    the blocked GEMM driver."""
    return m * n * k <= 1_000_000 and (not tn or (m * n <= 1200 and k >= 32))


GEMM_Q = 384   # OpenBLAS SkylakeX DGEMM_DEFAULT_Q: the blocked driver's K block


def dot_kblocks(a: Val, b: Val):
    """K ranges the blocked GEMM driver accumulates separately: each block
    is a fresh k-ordered fma chain, and C = C + block rounds once per block
    (beta = 0, alpha = 1).  The driver's split (level3_thread.c, numpy's
    default threaded OpenBLAS): a remainder >= 2Q takes Q, one in (Q, 2Q)
    is halved, (r + 1) / 2.  Probed here on numpy 2.3.5 / OpenBLAS 0.3.30
    (tests/test_dot_orders.py::test_blocked_k_split); the single-threaded
    driver rounds the half up to a multiple of 16 instead, which agrees on
    every K the workloads reach (the CNN's K = 480 -> 240 + 240).  Small-
    kernel problems and gemv shapes are one block."""
    m, k = a.shape
    n = b.shape[1]
    if a.kind != K_F64 or m == 1 or k == 1 or n == 1 or k <= GEMM_Q:
        return [(0, k)]
    sa = _blas_strides(a.st, m, k)
    sb = _blas_strides(b.st, k, n)
    tn = (not _blas2d(sb[0], sb[1], n)) and _blas2d(sa[0], sa[1], k)
    if _small_kernel(m, k, n, tn):
        return [(0, k)]
    out, ls = [], 0
    while ls < k:
        ml = k - ls
        if ml >= 2 * GEMM_Q:
            ml = GEMM_Q
        elif ml > GEMM_Q:
            ml = (ml + 1) // 2
        out.append((ls, ls + ml))
        ls += ml
    return out


def _pad_dims(shape):
    shape = tuple(shape)
    return list(shape) + [1] * (MAXR - len(shape))


class _Builder:
    def __init__(self, fn, param_vals, ret_bufs, ret_layout, cost_table):
        self.fn = fn
        self.instrs = []
        self.consts = []
        self.allocs: list[_Alloc] = []
        self.vals: dict[str, Val] = {}
        self.cost = 0.0
        self.table = cost_table or {}
        self.ret_bufs = ret_bufs
        self.ret_layout = ret_layout   # "compact" | "c"
        types = {}
        for (name, ty), v in zip(fn.params, param_vals):
            self.vals[name] = v
            types[name] = ty
        self.types = types

    # -- allocation ---------------------------------------------------------
    def new_alloc(self, size, fixed=None) -> int:
        self.allocs.append(_Alloc(size=size, fixed=fixed))
        return len(self.allocs) - 1

    def fresh(self, shape, st, kind, size, fixed=None) -> Val:
        aid = self.new_alloc(size, fixed)
        if fixed is not None:
            return Val(fixed[0], fixed[1], tuple(shape), tuple(st), kind, aid)
        return Val(BUF_ARENA, 0, tuple(shape), tuple(st), kind, aid)

    def const(self, arr, kind) -> Val:
        arr = np.asarray(arr)
        off = len(self.consts)
        flat = np.ascontiguousarray(arr).reshape(-1)
        if kind == K_F64:
            self.consts.extend(float(x) for x in flat)
        else:
            self.consts.extend(int(x) for x in flat)
        return Val(BUF_CONST, off, tuple(arr.shape), L.c_strides(arr.shape), kind)

    # -- instruction emission ------------------------------------------------
    def operand(self, v: Val, shape_rank):
        st = list(v.st) + [0] * (MAXR - len(v.st))
        return (v.buf, v.off, st)

    def emit(self, op, sub, out: Val, ins, kin=None, aux=None, aux2=None,
             rank=None, shp=None, n=None):
        shp = tuple(out.shape) if shp is None else tuple(shp)
        rec = {
            "op": op, "sub": sub, "kout": out.kind,
            "kin": ins[0].kind if kin is None and ins else (kin or 0),
            "rank": len(shp) if rank is None else rank,
            "n": math.prod(shp) if n is None else n,
            "shp": _pad_dims(shp), "aux": list(aux or []) + [0] * (MAXR - len(aux or [])),
            "aux2": list(aux2 or []) + [0] * (MAXR - len(aux2 or [])),
            "out": out, "in": list(ins)}
        self.instrs.append(rec)

    # -- lowering ---------------------------------------------------------------
    def run(self, plan_returns):
        fn = self.fn
        # returned values produced by a materialising op go straight to OUT
        direct = {}
        for r, v in enumerate(fn.returns):
            if v not in direct and r < len(self.ret_bufs):
                direct[v] = r
        self.direct = direct
        for idx, op in enumerate(fn.ops):
            tys = tuple(self.types[v] for v in op.operands)
            self.cost += _op_cost(op, tys, self.table)
            ins = [self.vals[v] for v in op.operands]
            out = self.lower_op(op, ins, tys, idx)
            self.vals[op.result] = out
            self.types[op.result] = op.result_type
        # returns
        ret_st = []   # layout each return is STORED in (next step's params)
        for r, name in enumerate(fn.returns):
            v = self.vals[name]
            if r >= len(self.ret_bufs):
                ret_st.append(tuple(v.st))
                continue
            buf = self.ret_bufs[r]
            if v.buf == buf[0] and v.off == buf[1] and direct.get(name) == r:
                ret_st.append(tuple(v.st))
                continue  # produced in place
            st = self.ret_strides(v)
            dst = Val(buf[0], buf[1], v.shape, st, v.kind)
            self.emit(OP_UNARY, U_COPY, dst, [v])
            ret_st.append(tuple(st))
        return ret_st

    def ret_strides(self, v: Val):
        if self.ret_layout == "c":
            return L.c_strides(v.shape)
        return L.compact_strides(v.shape, v.st)[0]

    def result_val(self, op, shape, st, kind):
        """Storage for a materialised result: the OUT slot if it is returned
        (and dense in numpy's layout), else a fresh arena allocation."""
        r = self.direct.get(op.result)
        count = math.prod(shape)
        if r is not None and self.ret_layout == "c" and \
                tuple(st) != L.c_strides(shape):
            r = None
        if r is not None:
            return self.fresh(shape, st, kind, 0, fixed=self.ret_bufs[r])
        return self.fresh(shape, st, kind, count)

    def lower_op(self, op, ins, tys, idx):
        code = op.opcode
        rt = op.result_type
        shape = tuple(rt.shape)
        kind = _kind_of(rt)
        at = op.attrs
        if code == "constant":
            return self.const(np.asarray(at["value"]).reshape(shape), kind)
        if code == "iota":
            d = at["dim"]
            mid = [1] * len(shape)
            mid[d] = shape[d]
            ramp = np.arange(shape[d], dtype=_NP_DTYPE[kind]).reshape(mid)
            return self.const(np.broadcast_to(ramp, shape), kind)
        if code == "transpose":
            (a,) = ins
            p = at["perm"]
            return Val(a.buf, a.off, tuple(a.shape[i] for i in p),
                       tuple(a.st[i] for i in p), a.kind, a.alloc)
        if code == "slice":
            (a,) = ins
            off = a.off + sum(s * t for s, t in zip(at["start"], a.st))
            return Val(a.buf, off, shape, a.st, a.kind, a.alloc)
        if code == "reshape":
            return self.reshape(ins[0], shape, idx)
        if code == "broadcast_in_dim":
            (a,) = ins
            mid = [1] * len(shape)
            for s, d in enumerate(at["dims"]):
                mid[d] = a.shape[s]
            m = self.reshape(a, tuple(mid), idx)
            st = tuple(0 if (mid[d] == 1 and shape[d] != 1) else m.st[d]
                       for d in range(len(shape)))
            return Val(m.buf, m.off, shape, st, m.kind, m.alloc)
        if code in B_CODES:
            st = L.keep_order_strides(shape, [ins[0].st, ins[1].st])
            out = self.result_val(op, shape, st, kind)
            self.emit(OP_BINARY, B_CODES[code], out, ins)
            return out
        if code == "compare":
            st = L.keep_order_strides(shape, [ins[0].st, ins[1].st])
            out = self.result_val(op, shape, st, kind)
            self.emit(OP_BINARY, CMP_CODES[at["kind"]], out, ins)
            return out
        if code in ("negate", "exponential", "log"):
            st = L.keep_order_strides(shape, [ins[0].st])
            out = self.result_val(op, shape, st, kind)
            sub = {"negate": U_NEG, "exponential": U_EXP, "log": U_LOG}[code]
            self.emit(OP_UNARY, sub, out, ins)
            return out
        if code == "convert":
            st = L.keep_order_strides(shape, [ins[0].st])
            out = self.result_val(op, shape, st, kind)
            self.emit(OP_UNARY, U_CVT, out, ins)
            return out
        if code == "select":
            st = L.keep_order_strides(shape, [v.st for v in ins])
            out = self.result_val(op, shape, st, kind)
            self.emit(OP_SELECT, 0, out, ins, kin=ins[1].kind)
            return out
        if code == "dot":
            a, b = ins
            blocks = dot_kblocks(a, b)
            if len(blocks) > 1:
                return self.blocked_dot(op, a, b, blocks, shape, kind)
            out = self.result_val(op, shape, L.c_strides(shape), kind)
            m1, split, m2, xrow = dot_modes(a, b)
            corner = xrow + 1 if xrow < a.shape[0] else 0
            self.emit(OP_DOT, m1, out, ins, aux=[a.shape[1], split, m2, corner])
            return out
        if code == "reduce":
            (a,) = ins
            ax = at["axis"]
            perm = L.best_axis_order(len(a.shape), [a.st])
            rest = [p for p in perm if p != ax]
            keep = [d for d in range(len(a.shape)) if d != ax]
            # allocate the result following the input's axis order (order K)
            sub_perm = [keep.index(p) for p in rest]
            st = L.strides_for_order(shape, sub_perm) if shape else ()
            out = self.result_val(op, shape, st, kind)
            if at["kind"] == "max":
                sub = R_MAX
            elif perm[0] == ax and a.shape[ax] > 1:
                sub = R_SUM_PAIRWISE
            else:
                sub = R_SUM_SEQ
            src = Val(a.buf, a.off, tuple(a.shape[d] for d in keep),
                      tuple(a.st[d] for d in keep), a.kind, a.alloc)
            self.emit(OP_REDUCE, sub, out, [src], aux=[a.shape[ax], a.st[ax]])
            return out
        if code == "pad":
            a, pv = ins
            fnc = L.is_f_contiguous(a.shape, a.st) and not \
                L.is_c_contiguous(a.shape, a.st)
            st = L.strides_for_order(shape, list(range(len(shape)))) if fnc \
                else L.c_strides(shape)
            out = self.result_val(op, shape, st, kind)
            self.emit(OP_PAD, 0, out, [a, pv], aux=list(at["low"]),
                      aux2=list(a.shape))
            return out
        raise LoweringError(f"cannot lower opcode {code!r}")

    def blocked_dot(self, op, a, b, blocks, shape, kind):
        """A blocked-driver dot (dot_kblocks): one k-ordered chain per K
        block into scratch, folded as C = C + block (the add rounds once,
        like the driver's C update); fuse_dot_epilogues then makes each add
        the epilogue of its block's dot."""
        m, n = shape
        acc = None
        for j, (k0, k1) in enumerate(blocks):
            av = Val(a.buf, a.off + k0 * a.st[1], (m, k1 - k0), a.st, a.kind, a.alloc)
            bv = Val(b.buf, b.off + k0 * b.st[0], (k1 - k0, n), b.st, b.kind, b.alloc)
            part = self.fresh(shape, L.c_strides(shape), kind, m * n)
            self.emit(OP_DOT, D_FMA_CHAIN, part, [av, bv], aux=[k1 - k0, n, D_FMA_CHAIN, 0])
            if acc is None:
                acc = part
                continue
            last = j == len(blocks) - 1
            out = self.result_val(op, shape, L.c_strides(shape), kind) if last else \
                self.fresh(shape, L.c_strides(shape), kind, m * n)
            self.emit(OP_BINARY, B_CODES["add"], out, [acc, part])
            acc = out
        return acc

    def reshape(self, a: Val, shape, idx):
        st = L.reshape_view(a.shape, a.st, shape)
        if st is not None:
            return Val(a.buf, a.off, tuple(shape), st, a.kind, a.alloc)
        # numpy copies into C order, then reinterprets
        tmp = self.fresh(a.shape, L.c_strides(a.shape), a.kind,
                         math.prod(a.shape))
        self.emit(OP_UNARY, U_COPY, tmp, [a])
        return Val(tmp.buf, tmp.off, tuple(shape), L.c_strides(shape),
                   tmp.kind, tmp.alloc)

    # -- arena assignment ---------------------------------------------------------
    def assign_arena(self, smem_budget=None):
        """First-fit by liveness over the instruction list, in two tiers.
        An allocation lives from the instruction that writes it to the last
        instruction reading it, so an instruction never writes over its own
        operands.  Small allocations go to shared memory while they fit the
        budget; the rest (and the overflow) to the HBM arena.
        Returns (hbm_elems, smem_elems)."""
        budget = SMEM_BUDGET if smem_budget is None else smem_budget
        created, last_read = {}, {}
        for i, ins in enumerate(self.instrs):
            a = ins["out"].alloc
            if a >= 0 and self.allocs[a].fixed is None:
                created.setdefault(a, i)
            for v in ins["in"] + ins.get("ext", []):
                if v.alloc >= 0:
                    last_read[v.alloc] = i
        tiers = {"s": ([], 0), "g": ([], 0)}
        live = {"s": [], "g": []}
        top = {"s": 0, "g": 0}

        def place(space, size, i):
            cur = sorted(x for x in live[space] if x[2] >= i)
            live[space] = cur
            pos = 0
            for off, sz, _ in cur:
                if pos + size <= off:
                    break
                pos = max(pos, off + sz)
            return pos

        for a_id, i in sorted(created.items(), key=lambda kv: kv[1]):
            a = self.allocs[a_id]
            until = max(i, last_read.get(a_id, i))
            space = "g"
            if a.size <= SMEM_VALUE_MAX and budget > 0:
                pos = place("s", a.size, i)
                if pos + a.size <= budget:
                    space = "s"
            if space == "g":
                pos = place("g", a.size, i)
            a.off = pos
            a.space = space
            live[space].append((pos, a.size, until))
            top[space] = max(top[space], pos + a.size)
        return top["g"], top["s"]


def _op_cost(op, tys, table):
    unit = table.get(op.opcode, 1.0)
    if op.opcode == "dot":
        a, b = tys
        return unit * a.shape[0] * b.shape[1] * a.shape[1]
    if op.opcode == "reduce":
        return unit * _count(tys[0].shape)
    return unit * _count(op.result_type.shape)


def _count(shape):
    n = 1
    for d in shape:
        n *= d
    return n


def static_cost(fn, cost_table=None) -> float:
    """ExecPlan.total_cost (interpreter.py:205-214): float sum in op order."""
    types = dict(fn.params)
    total = 0.0
    for op in fn.ops:
        total += _op_cost(op, tuple(types[v] for v in op.operands),
                          cost_table or {})
        types[op.result] = op.result_type
    return total


def _same_view(a: Val, b: Val) -> bool:
    return (a.buf, a.off, tuple(a.shape), tuple(a.st), a.alloc) == \
        (b.buf, b.off, tuple(b.shape), tuple(b.st), b.alloc)


def fuse_dot_epilogues(instrs):
    """Fold single-use elementwise consumers into the producing DOT.

    A dot result D that lives in scratch (not returned) and is read exactly
    once, through the identity view, by an elementwise instruction R is not
    stored: R becomes a micro-op applied to each dot output element, and the
    fused instruction takes R's place in the sequence (R's other operands are
    all computed by then; D's operands are SSA values nothing overwrites, and
    scratch liveness is assigned after this pass).  Repeats along chains,
    e.g. w1' = w1 - lr * (x^T . delta) becomes one instruction writing w1'.
    Each micro-op rounds like the instruction it replaces (bit-identical)."""
    while True:
        readers = {}
        for i, r in enumerate(instrs):
            for k, v in enumerate(r["in"]):
                if v.alloc >= 0:
                    readers.setdefault(v.alloc, []).append((i, k, "in"))
            for k, v in enumerate(r.get("ext", [])):
                if v.alloc >= 0:
                    readers.setdefault(v.alloc, []).append((i, k, "ext"))
        # merge every independent (dot, reader) pair found in this pass; an
        # instruction takes part in at most one merge per pass
        touched, drop = set(), []
        for i, d in enumerate(instrs):
            if d["op"] != OP_DOT or i in touched:
                continue
            out = d["out"]
            if out.alloc < 0 or out.buf != BUF_ARENA:
                continue                      # returned value: must be stored
            rs = readers.get(out.alloc, [])
            if len(rs) != 1 or rs[0][2] != "in":
                continue
            j, k, _ = rs[0]
            r = instrs[j]
            if j <= i or j in touched or r["op"] not in (OP_UNARY, OP_BINARY, OP_SELECT):
                continue
            if not _same_view(r["in"][k], out):
                continue
            epi = list(d.get("epi", []))
            ext = list(d.get("ext", []))
            others = [w for kk, w in enumerate(r["in"]) if kk != k]
            if len(epi) >= EPI_MAX_OPS or len(ext) + len(others) > EPI_MAX_EXT:
                continue
            prev = 0 if not epi else EPI_SRC_OP + len(epi) - 1
            srcs = []
            for kk, w in enumerate(r["in"]):
                if kk == k:
                    srcs.append(prev)
                else:
                    ext.append(w)
                    srcs.append(len(ext))    # 1-based operand index
            epi.append((r["op"], r["sub"], r["kin"], r["kout"], srcs))
            new = dict(d)
            new["epi"], new["ext"], new["out"] = epi, ext, r["out"]
            instrs[j] = new
            drop.append(i)
            touched.update((i, j))
        if not drop:
            return instrs
        for i in reversed(drop):
            del instrs[i]


_EW_OPS = (OP_UNARY, OP_BINARY, OP_SELECT)
# largest elementwise chain (elements); measured best without a limit
EW_CHAIN_MAX = int(os.environ.get("GEVO_EW_CHAIN_MAX", 1 << 30))


def _as2d(v: Val) -> Val:
    """An epilogue operand as a (rows, cols) view: epilogue operands are
    addressed by (r, c) with two strides; rank 1 is one row, rank 0 one
    element."""
    if len(v.shape) == 2:
        return v
    if len(v.shape) == 1:
        return Val(v.buf, v.off, (1, v.shape[0]), (0, v.st[0]), v.kind, v.alloc)
    return Val(v.buf, v.off, (1, 1), (0, 0), v.kind, v.alloc)


_B_MAX = B_CODES["maximum"]


def _fast_form(p, epi) -> bool:
    """An f64 add/sub/mul/div/max followed by <= 2 such micro-ops, micro-op m
    combining the running value with epilogue operand m + 1 (the device's
    FastChain)."""
    if p["op"] != OP_BINARY or p["kin"] != K_F64 or p["sub"] > _B_MAX or len(epi) > 2:
        return False
    for m, (cls, sub, kin, _, srcs) in enumerate(epi):
        prev = 0 if m == 0 else EPI_SRC_OP + m - 1
        if cls != OP_BINARY or kin != K_F64 or sub > _B_MAX:
            return False
        if len(srcs) != 2 or sorted(srcs) != sorted([prev, m + 1]):
            return False
    return True


def fuse_ew_chains(instrs):
    """Fold a single-use elementwise result into its elementwise consumer.

    Like fuse_dot_epilogues, with an elementwise producer P (rank <= 2) in
    place of the dot: P's result lives in scratch and is read exactly once,
    through the identity view, by an elementwise R of the same shape.  P's
    op stays the instruction's own op, R becomes an epilogue micro-op on it,
    and the fused instruction takes R's place; P's value is never stored.
    e.g. b1' = b1 - lr * g is one instruction, and so is exp(z - max).  Each
    micro-op rounds like the instruction it replaces (bit-identical)."""
    while True:
        readers = {}
        for i, r in enumerate(instrs):
            for k, v in enumerate(r["in"]):
                if v.alloc >= 0:
                    readers.setdefault(v.alloc, []).append((i, k, "in"))
            for k, v in enumerate(r.get("ext", [])):
                if v.alloc >= 0:
                    readers.setdefault(v.alloc, []).append((i, k, "ext"))
        touched, drop = set(), []
        for i, p in enumerate(instrs):
            if p["op"] not in _EW_OPS or i in touched:
                continue
            out = p["out"]
            nd = len(out.shape) > 2
            if out.alloc < 0 or out.buf != BUF_ARENA or math.prod(out.shape) > EW_CHAIN_MAX:
                continue
            rs = readers.get(out.alloc, [])
            if len(rs) != 1 or rs[0][2] != "in":
                continue
            j, k, _ = rs[0]
            r = instrs[j]
            if j <= i or j in touched or r["op"] not in _EW_OPS:
                continue
            if not _same_view(r["in"][k], out) or tuple(r["out"].shape) != tuple(out.shape):
                continue
            epi = list(p.get("epi", []))
            ext = list(p.get("ext", []))
            others = [w for kk, w in enumerate(r["in"]) if kk != k]
            r_epi, r_ext = r.get("epi", []), r.get("ext", [])
            if len(epi) + 1 + len(r_epi) > EPI_MAX_OPS or \
                    len(ext) + len(others) + len(r_ext) > EPI_MAX_EXT:
                continue
            prev = 0 if not epi else EPI_SRC_OP + len(epi) - 1
            srcs = []
            for kk, w in enumerate(r["in"]):
                if kk == k:
                    srcs.append(prev)
                else:
                    ext.append(w if nd else _as2d(w))
                    srcs.append(len(ext))    # 1-based operand index
            epi.append((r["op"], r["sub"], r["kin"], r["kout"], srcs))
            # R's own chain (from an earlier merge) follows, re-indexed: its
            # value -> the micro-op just added, its micro-ops and operands
            # shifted past P's
            r_op_at, ext0 = EPI_SRC_OP + len(epi) - 1, len(ext)
            for cls, sub, kin, kout, rs_ in r_epi:
                m = []
                for x in rs_:
                    if x == 0:
                        m.append(r_op_at)
                    elif x >= EPI_SRC_OP:
                        m.append(r_op_at + 1 + (x - EPI_SRC_OP))
                    else:
                        m.append(ext0 + x)
                epi.append((cls, sub, kin, kout, m))
            ext.extend(r_ext)
            # rank > 2 (CNN activations): only the fast form, addressed by the
            # full multi-index on the device (run_ew_chain, N-d walk)
            if nd and not _fast_form(p, epi):
                continue
            new = dict(p)
            new["epi"], new["ext"], new["out"] = epi, ext, r["out"]
            instrs[j] = new
            drop.append(i)
            touched.update((i, j))
        if not drop:
            return instrs
        for i in reversed(drop):
            del instrs[i]


def fuse_tap_sums(instrs):
    """Fold a running sum of products into one TAPSUM instruction.

    The pattern is the CNN's depthwise 3x3 (cnn.py depthwise): p_i = x_i * y_i
    (f64 multiply), s_1 = p_0 + p_1, s_i = s_(i-1) + p_i, every p_i and every
    partial sum s_i read exactly once, through the identity view, by the next
    add.  All x_i must share one stride vector, and so must all y_i (the taps
    are windows of one padded tensor times broadcast per-channel weights).
    The TAPSUM computes v = x_0*y_0, then v = v + x_i*y_i for i >= 1, each
    product and each sum rounded on its own (__dmul_rn / __dadd_rn, like the
    multiply and add instructions it replaces), so fusion changes no bit.
    The partial sums and the products are never stored: per output element
    the taps are read once and the sum written once, instead of a product
    and a running-sum round trip per tap."""
    readers = {}
    for i, r in enumerate(instrs):
        for k, v in enumerate(list(r["in"]) + list(r.get("ext", []))):
            if v.alloc >= 0:
                readers.setdefault(v.alloc, []).append((i, k))

    def single_use_into(i, j):
        """instrs[i]'s result is read once, by instrs[j], through its own view."""
        o = instrs[i]["out"]
        if o.alloc < 0 or o.buf != BUF_ARENA:
            return False
        rs = readers.get(o.alloc, [])
        return len(rs) == 1 and rs[0][0] == j and _same_view(instrs[j]["in"][rs[0][1]], o)

    def plain(r, sub):
        return (r["op"] == OP_BINARY and r["sub"] == sub and r["kin"] == K_F64 and
                not r.get("epi") and not r.get("ext") and len(r["out"].shape) >= 1)

    producer = {}
    for i, r in enumerate(instrs):
        if r["out"].alloc >= 0:
            producer[r["out"].alloc] = i
    sums = {}           # index of a chain's last add -> (taps [(x, y)], members)
    for j, r in enumerate(instrs):
        if not plain(r, B_CODES["add"]):
            continue
        shape = tuple(r["out"].shape)
        srcs = [producer.get(v.alloc, -1) if v.alloc >= 0 else -1 for v in r["in"]]
        muls = [i for i in srcs if i >= 0 and plain(instrs[i], B_CODES["multiply"]) and
                tuple(instrs[i]["out"].shape) == shape and single_use_into(i, j)]
        prev = [i for i in srcs if i in sums and single_use_into(i, j)]
        if prev and muls:
            taps, members = sums[prev[0]]
            m = [i for i in muls if i != prev[0]]
            if not m or len(taps) >= TAP_MAX:
                continue
            del sums[prev[0]]
            sums[j] = (taps + [m[0]], members + [prev[0], m[0]])
        elif len(muls) == 2 and muls[0] != muls[1]:
            a, b = (muls if srcs[0] == muls[0] else muls[::-1])
            sums[j] = ([a, b], [a, b])
    drop = set()
    busy = set(sums) | {i for _, ms in sums.values() for i in ms}
    reader_of = {}
    for alloc, rs in readers.items():
        if len(rs) == 1:
            reader_of[alloc] = rs[0]
    for j, (taps, members) in sums.items():
        xs = [instrs[i]["in"][0] for i in taps]
        ys = [instrs[i]["in"][1] for i in taps]
        if len({tuple(v.st) for v in xs}) != 1 or len({tuple(v.st) for v in ys}) != 1:
            continue
        rec = dict(instrs[j])
        rec["op"], rec["sub"] = OP_TAPSUM, len(taps)
        rec["in"] = [xs[0], ys[0]]
        rec["ext"] = [v for x, y in zip(xs[1:], ys[1:]) for v in (x, y)]
        # epilogue: up to TAP_EPI single-use f64 binary consumers (the folded
        # batch norm after a depthwise: * scale, + bias, max 0) become
        # micro-ops applied before the store, each rounding as the op it
        # replaces; the fused record takes the last consumer's place
        micro, at, out = [], j, rec["out"]
        while len(micro) < TAP_EPI and out.alloc >= 0 and out.buf == BUF_ARENA:
            rr = reader_of.get(out.alloc)
            if rr is None:
                break
            q, k = rr
            r = instrs[q]
            if q <= at or q in busy or not plain(r, r["sub"]) or r["sub"] > _B_MAX or \
                    r["kout"] != K_F64 or k > 1 or not _same_view(r["in"][k], out) or \
                    tuple(r["out"].shape) != tuple(out.shape):
                break
            micro.append((r["sub"], 1 if k == 0 else 0))
            rec["ext"].append(r["in"][1 - k])
            drop.add(at)
            at, out = q, r["out"]
        rec["micro"] = micro
        rec["out"] = out
        instrs[at] = rec
        drop.update(members)
    for i in sorted(drop, reverse=True):
        del instrs[i]
    return instrs


def mem_order_elementwise(instrs):
    """Walk plain elementwise instructions in their output's memory order.

    An elementwise op is the same per element in any index order, so its
    dims may be permuted consistently across the output and every operand.
    When the output is a dense block in some other dim order (e.g. a
    column-major 784 x 32 weight returned by a variant whose steps flip
    layouts), sorting the dims by the output's strides makes the output --
    and every operand laid out like it -- a linear, coalesced stream instead
    of a row walk with a 784-element stride."""
    for i, r in enumerate(instrs):
        if r["op"] not in _EW_OPS or r.get("epi") or r.get("ext"):
            continue
        out = r["out"]
        shape, st = tuple(out.shape), tuple(out.st)
        if len(shape) < 2:
            continue
        perm = sorted(range(len(shape)), key=lambda d: (-st[d], d))
        if perm == list(range(len(shape))):
            continue
        pshape = tuple(shape[d] for d in perm)
        pst = tuple(st[d] for d in perm)
        if any(a != b for a, b, e in zip(pst, L.c_strides(pshape), pshape) if e != 1):
            continue

        def permuted(v):
            return Val(v.buf, v.off, pshape, tuple(v.st[d] for d in perm), v.kind, v.alloc)
        new = dict(r)
        new["out"] = permuted(out)
        new["in"] = [permuted(v) for v in r["in"]]
        new["shp"] = _pad_dims(pshape)
        instrs[i] = new
    return instrs


def lower_function(fn, param_layouts=None, ret_bufs=None, ret_layout="compact",
                   cost_table=None, smem_budget=None, fuse=True) -> Lowered:
    """Lower one function.  Params i live in buffer PARAM0+i with the given
    element strides (default: C order); return r is written to ret_bufs[r]
    (default: (OUT0+r, 0))."""
    params = []
    for i, (name, ty) in enumerate(fn.params):
        shape = tuple(ty.shape)
        st = tuple(param_layouts[i]) if param_layouts else L.c_strides(shape)
        params.append(Val(BUF_PARAM0 + i, 0, shape, st, _kind_of(ty)))
    if ret_bufs is None:
        ret_bufs = [(BUF_OUT0 + r, 0) for r in range(len(fn.returns))]
    b = _Builder(fn, params, ret_bufs, ret_layout, cost_table)
    ret_st = b.run(fn.returns)
    if fuse:
        fuse_dot_epilogues(b.instrs)
        fuse_tap_sums(b.instrs)
        fuse_ew_chains(b.instrs)
    mem_order_elementwise(b.instrs)
    top, stop = b.assign_arena(smem_budget)
    # resolve arena offsets into the operands
    instrs = []
    for rec in b.instrs:
        fixed = []
        ext = rec.get("ext", [])
        for v in [rec["out"]] + rec["in"] + ext:
            if v.alloc >= 0 and v.buf == BUF_ARENA:
                a = b.allocs[v.alloc]
                buf = BUF_SMEM if a.space == "s" else BUF_ARENA
                fixed.append(Val(buf, a.off + v.off, v.shape, v.st, v.kind))
            else:
                fixed.append(v)
        rec = dict(rec)
        nin = len(rec["in"])
        rec["out"], rec["in"] = fixed[0], fixed[1:1 + nin]
        if ext:
            rec["ext"] = fixed[1 + nin:]
        instrs.append(rec)
    return Lowered(instrs, b.consts, top, ret_st, b.cost, stop)


AM_STRIDED, AM_LINEAR, AM_SCALAR = 0, 1, 2


def _addr_mode(v, shape):
    """How the executor addresses an elementwise operand (exec_core.cuh)."""
    if all(s == 0 or d == 1 for s, d in zip(v.st, shape)):
        return AM_SCALAR
    cst = L.c_strides(shape)
    if all(s == c or d == 1 for s, c, d in zip(v.st, cst, shape)):
        return AM_LINEAR
    return AM_STRIDED


def _ext_records(rec):
    """GEVO_OP_EXT continuation records of a fused dot (gevo_plan.h)."""
    epi, ext = rec.get("epi", []), rec.get("ext", [])
    n = max((len(epi) + 3) // 4, (len(ext) + 2) // 3)
    out = []
    for e in range(n):
        words = []
        for cls, sub, kin, kout, srcs in epi[4 * e:4 * e + 4]:
            srcs = list(srcs) + [0] * (3 - len(srcs))
            words += [cls | (sub << 4) | (kin << 8) | (kout << 12),
                      srcs[0] | (srcs[1] << 8), srcs[2]]
        words += [0] * (12 - len(words))
        ops = ext[3 * e:3 * e + 3]
        out.append({"op": OP_EXT, "sub": 0, "kout": 0, "kin": 0, "rank": 2, "n": 0,
                    "shp": [1] * MAXR, "aux": words[:6], "aux2": words[6:],
                    "out": Val(0, 0, (), (), 0), "in": ops, "n_epi": len(epi)})
    return out


def _operand_words(v):
    st = list(v.st)
    return [v.buf, v.off] + st + [0] * (MAXR - len(st))


_ZERO_OPERAND = [0] * (2 + MAXR)


def encode_instrs(instrs, const_base=0) -> np.ndarray:
    """Instruction records -> gevo_instr array (one flat int32 list, then a
    single array construction: 56 words per record, gevo_plan.h)."""
    words = []
    for rec in instrs:
        recs = [rec]
        n_ext = n_epi = 0
        if rec["op"] == OP_TAPSUM:
            # taps 1.. as (x_i, y_i) operand pairs, 3 per continuation record
            exts = _ext_records({"ext": rec["ext"]})
            rec = dict(rec)
            aux2 = [0] * MAXR
            micro = rec.get("micro", [])
            aux2[3], aux2[4], aux2[5] = len(micro), len(exts), rec["sub"]
            rec["aux2"] = aux2
            aux = [0] * MAXR
            for m, (sub_, left) in enumerate(micro):
                aux[m] = sub_ | (left << 4)
            rec["aux"] = aux
            recs = [rec] + exts
        elif rec.get("epi"):
            exts = _ext_records(rec)
            n_ext, n_epi = len(exts), len(rec["epi"])
            rec = dict(rec)
            aux2 = list(rec["aux2"])
            aux2[0] = n_ext          # DOT: aux2[0..1]; elementwise: aux2[4..5]
            aux2[1] = n_epi
            rec["aux2"] = aux2
            recs = [rec] + exts
        for r in recs:
            aux2 = r["aux2"]
            ins = r["in"]
            if r["op"] in (OP_UNARY, OP_BINARY, OP_SELECT):
                shape = tuple(r["out"].shape)
                modes = [_addr_mode(r["out"], shape)]
                modes += [_addr_mode(v, shape) for v in ins]
                aux2 = modes + [AM_SCALAR] * (4 - len(modes)) + [n_ext, n_epi]
            words += [r["op"], r["sub"], r["kout"], r["kin"], r["rank"], r["n"]]
            words += r["shp"]
            words += r["aux"]
            words += aux2
            words += _operand_words(r["out"])
            for j in range(3):
                words += _operand_words(ins[j]) if j < len(ins) else _ZERO_OPERAND
    arr = np.array(words, dtype=np.int32)
    return arr.view(INSTR_DTYPE)


def consts_to_words(consts) -> np.ndarray:
    """Constant pool as 64-bit words (float64 bits or int64)."""
    out = np.zeros(len(consts), dtype=np.float64)
    iv = out.view(np.int64)
    for i, c in enumerate(consts):
        if isinstance(c, float):
            out[i] = c
        else:
            iv[i] = int(c)
    return out
