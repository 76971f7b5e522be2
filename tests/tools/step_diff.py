"""Locate a device/oracle divergence inside one individual's training (tool).

    python tests/tools/step_diff.py ga512x50.json.gz 404 [520 ...]

For each individual: the oracle's weight trajectory over 600 steps; every
step re-run on the device through gevo_exec_once with the oracle's inputs;
the first step whose returned weights differ bit-wise is then bisected op by
op (the function truncated after op k, returning op k's value) and the first
differing op is printed with its operand types.  Also checks `forward`.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.dirname(os.path.dirname(HERE))]

from golden_io import load, variant_functions  # noqa: E402
from oracle.interp import Program  # noqa: E402
from paper_2310_10211_b200 import _lib, dialect, workloads as W  # noqa: E402
from paper_2310_10211_b200.plan import exec_once_plan  # noqa: E402


def words(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.bool_:
        a = a.astype(np.int64)
    if a.dtype != np.float64:
        return a.reshape(-1).astype(np.int64).view(np.float64)
    return a.reshape(-1)


def run_once(ctx, fns, params_list):
    blob, pblob, meta, total = exec_once_plan(fns, params_list)
    outs = ctx.exec_once(blob, pblob, total)
    res = []
    for metas in meta:
        got = []
        for off, shape, kind in metas:
            n = max(1, int(np.prod(shape)))
            w = outs[off:off + n]
            got.append(w.reshape(shape) if kind == "f32" else w.view(np.int64).reshape(shape))
        res.append(got)
    return res


def same(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.dtype == np.bool_:
        a = a.astype(np.int64)
    if b.dtype == np.bool_:
        b = b.astype(np.int64)
    return a.shape == b.shape and np.array_equal(
        a.astype(np.float64).view(np.int64) if a.dtype == np.float64 else a,
        b.astype(np.float64).view(np.int64) if b.dtype == np.float64 else b)


def truncated(fn, k):
    op = fn.ops[k]
    return dialect.FunctionBody(fn.name, fn.params, fn.ops[:k + 1], (op.result,), (op.result_type,))


def bisect_ops(ctx, fn, args):
    prog = Program(fn)
    vals = list(args)
    with np.errstate(all="ignore"):
        from oracle.interp import apply_op
        for op, slots, tys in prog.steps:
            vals.append(apply_op(op, [vals[s] for s in slots], tys, False))
    n_par = len(args)
    fns = [truncated(fn, k) for k in range(len(fn.ops))]
    outs = run_once(ctx, fns, [[words(a) for a in args]] * len(fns))
    for k, (got,) in enumerate(outs):
        want = vals[n_par + k]
        if not same(np.asarray(got).reshape(np.shape(want)), want):
            op = fn.ops[k]
            g = np.asarray(got).reshape(np.shape(want))
            d = np.nanmax(np.abs(g - want)) if np.asarray(want).dtype == np.float64 else None
            print(f"  first differing op #{k}: {dialect.format_function(fns[k]).splitlines()[-3]}")
            print(f"    operand types {[str(t) for t in prog.steps[k][2]]} max|diff| {d}")
            idx = np.argwhere(g != want)[:3]
            print(f"    at {idx.tolist()}: got {[g[tuple(i)] for i in idx]} want "
                  f"{[np.asarray(want)[tuple(i)] for i in idx]}")
            return k
    print("  no op differs (the difference is in the fused/eval path)")
    return None


def main():
    name = sys.argv[1]
    ids = [int(a) for a in sys.argv[2:]]
    data = load(name)
    wl = W.build_2fcnet_workload()
    xs, ys = wl.search_x, wl.search_y
    w0 = [wl.weights[n] for n in W.WEIGHT_NAMES]
    ctx = _lib.Context(0)
    for i in ids:
        fns = variant_functions(data["individuals"][i])
        fn = fns["train_step"]
        print(f"individual {i}: {len(fn.ops)} train_step ops")
        prog = Program(fn)
        w = list(w0)
        traj = []
        with np.errstate(all="ignore"):
            for s in range(600):
                args = w + [xs[s % 31], ys[s % 31]]
                traj.append(args)
                w = prog(args)
        first = None
        for s0 in range(0, 600, 100):
            chunk = traj[s0:s0 + 100]
            outs = run_once(ctx, [fn] * len(chunk), [[words(a) for a in args] for args in chunk])
            for k, got in enumerate(outs):
                with np.errstate(all="ignore"):
                    want = prog(chunk[k])
                if not all(same(np.asarray(g).reshape(np.shape(wv)), wv) for g, wv in zip(got, want)):
                    first = s0 + k
                    break
            if first is not None:
                break
        if first is None:
            print("  all 600 single steps bit-exact through exec_once")
            continue
        print(f"  first differing step {first}")
        bisect_ops(ctx, fn, traj[first])


if __name__ == "__main__":
    main()
