"""Vectorised CPU walker of a lowered instruction table (TEST TOOL ONLY).

It checks the *lowering* (addressing, view folding, layouts, arena reuse,
return placement, dot-epilogue fusion) independently of the GPU: it executes
the records that lowering.lower_function produces with plain numpy
arithmetic (no attempt at numpy's summation order), so results agree with
the oracle to ~1e-12, not bit-exactly.  Never used by the product or bench.
"""
from __future__ import annotations

import numpy as np

from paper_2310_10211_b200 import lowering as Lw

F = Lw.K_F64


def offsets(v, shape):
    if not shape:
        return np.array([v.off], dtype=np.int64)
    grids = np.indices(shape, dtype=np.int64).reshape(len(shape), -1)
    st = np.array(v.st[:len(shape)], dtype=np.int64)
    return v.off + (grids * st[:, None]).sum(0)


def gather(mem, v, shape):
    return mem[v.buf][offsets(v, shape)]


def scatter(mem, v, shape, words):
    mem[v.buf][offsets(v, shape)] = words


def fl(w):
    return np.asarray(w, dtype=np.int64).view(np.float64)


def wd(x):
    return np.asarray(x, dtype=np.float64).view(np.int64)


def ew(op, sub, kin, kout, args):
    """One elementwise op on 64-bit word arrays."""
    with np.errstate(all="ignore"):
        if op == Lw.OP_SELECT:
            p, t, f = args
            return np.where(p != 0, t, f)
        a = args[0]
        if op == Lw.OP_UNARY:
            if sub == Lw.U_COPY:
                return a
            if sub == Lw.U_CVT:
                if kout == Lw.K_I1:
                    return ((fl(a) != 0) if kin == F else (a != 0)).astype(np.int64)
                if kout == Lw.K_I64:
                    return np.trunc(fl(a)).astype(np.int64) if kin == F else a
                return a if kin == F else wd(a.astype(np.float64))
            if kin == F:
                x = fl(a)
                return wd({Lw.U_NEG: -x, Lw.U_EXP: np.exp(x), Lw.U_LOG: np.log(x)}[sub])
            return -a
        b = args[1]
        if kin == F:
            x, y = fl(a), fl(b)
            if sub <= 4:
                return wd([x + y, x - y, x * y, np.true_divide(x, y), np.maximum(x, y)][sub])
            return [x == y, x != y, x < y, x <= y, x > y, x >= y][sub - 5].astype(np.int64)
        if sub == 3:
            nz = b != 0
            q = np.trunc(np.true_divide(a, np.where(nz, b, 1)))
            return np.where(nz, q, 0).astype(np.int64)
        if sub <= 4:
            return [a + b, a - b, a * b, None, np.maximum(a, b)][sub]
        return [a == b, a != b, a < b, a <= b, a > b, a >= b][sub - 5].astype(np.int64)


def apply_epilogue(mem, rec, r):
    """Fused micro-ops (dot epilogues and elementwise chains) on the
    instruction's own result r (flat, output order)."""
    ext = [gather(mem, v, tuple(v.shape)).reshape(-1) for v in rec["ext"]]
    vals = [r]
    for cls, esub, ekin, ekout, srcs in rec["epi"]:
        nin = {Lw.OP_UNARY: 1, Lw.OP_BINARY: 2, Lw.OP_SELECT: 3}[cls]
        args = []
        for s in srcs[:nin]:
            if s == 0:
                args.append(vals[0])
            elif s >= Lw.EPI_SRC_OP:
                args.append(vals[1 + s - Lw.EPI_SRC_OP])
            else:
                args.append(ext[s - 1])
        vals.append(ew(cls, esub, ekin, ekout, args))
    return vals[-1]


def run(instrs, mem):
    """mem: dict buf_id -> np.ndarray of int64 words (float64 bits)."""
    for rec in instrs:
        op, sub = rec["op"], rec["sub"]
        out = rec["out"]
        shape = tuple(out.shape)
        kin = rec["kin"]
        with np.errstate(all="ignore"):
            if op in (Lw.OP_UNARY, Lw.OP_BINARY, Lw.OP_SELECT):
                r = ew(op, sub, kin, rec["kout"], [gather(mem, v, shape) for v in rec["in"]])
                if rec.get("epi"):
                    r = apply_epilogue(mem, rec, r)
            elif op == Lw.OP_REDUCE:
                L, rs = rec["aux"][0], rec["aux"][1]
                base = offsets(rec["in"][0], shape)
                idx = base[:, None] + np.arange(L, dtype=np.int64)[None, :] * rs
                w = mem[rec["in"][0].buf][idx]
                if kin == F:
                    x = fl(w)
                    r = wd(np.max(x, axis=1) if sub == Lw.R_MAX else np.sum(x, axis=1))
                else:
                    r = np.max(w, axis=1) if sub == Lw.R_MAX else np.sum(w, axis=1)
            elif op == Lw.OP_DOT:
                a, b = rec["in"]
                M, N, K = shape[0], shape[1], rec["aux"][0]
                A = gather(mem, a, (M, K)).reshape(M, K)
                B = gather(mem, b, (K, N)).reshape(K, N)
                r = (wd(fl(A) @ fl(B)) if kin == F else A @ B).reshape(-1)
                if rec.get("epi"):
                    r = apply_epilogue(mem, rec, r)
            elif op == Lw.OP_TAPSUM:
                nt = rec["sub"]
                taps = rec["ext"][:2 * (nt - 1)]
                xs = [rec["in"][0]] + taps[0::2]
                ys = [rec["in"][1]] + taps[1::2]
                v = fl(gather(mem, xs[0], shape)) * fl(gather(mem, ys[0], shape))
                for x, y in zip(xs[1:], ys[1:]):
                    v = v + fl(gather(mem, x, shape)) * fl(gather(mem, y, shape))
                r = wd(v)
                for (msub, left), w in zip(rec.get("micro", []), rec["ext"][2 * (nt - 1):]):
                    wv = gather(mem, w, shape)
                    r = ew(Lw.OP_BINARY, msub, F, F, [r, wv] if left else [wv, r])
            elif op == Lw.OP_PAD:
                a, pv = rec["in"]
                low, ext_ = rec["aux"][:len(shape)], rec["aux2"][:len(shape)]
                src = gather(mem, a, tuple(ext_)).reshape(ext_)
                pval = mem[pv.buf][pv.off]
                full = np.full(shape, pval, dtype=np.int64)
                full[tuple(slice(l, l + e) for l, e in zip(low, ext_))] = src
                r = full
            else:
                raise ValueError(f"unknown op {op}")
        scatter(mem, out, shape, np.asarray(r, dtype=np.int64).reshape(-1))
