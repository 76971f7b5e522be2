"""GPU diagnostic (tool): for full-size CNN mutants whose batch-0
probabilities differ from the reference, bisect `forward` op by op (the
function truncated after op k, returning op k's value, run through
gevo_exec_once against the oracle) and print the first differing op with
its operand shapes and strides.

    python tests/tools/cnn_first_diff.py [individual ...]
"""
import base64
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.dirname(os.path.dirname(HERE))]

from golden_io import load  # noqa: E402
from oracle import interp as OI  # noqa: E402
from paper_2310_10211_b200 import _lib, cnn, dialect  # noqa: E402
from test_gpu_parity import run_once  # noqa: E402


def truncated(fn, k):
    op = fn.ops[k]
    return dialect.FunctionBody(fn.name, fn.params, fn.ops[:k + 1], (op.result,), (op.result_type,))


def main(idx):
    g = load("cnn_full_pop.json.gz")
    cfg = cnn.CnnConfig(**cnn.MOBILENETV2_CIFAR_HALF, batch_size=100, search_n=100, holdout_n=100)
    wl = cnn.build_cnn_prediction_workload(cfg)
    xb4 = wl.search_x.reshape(-1, 100, 32, 32, 3)[0]
    xb = np.ascontiguousarray(xb4.reshape(100, -1)).reshape(-1)
    params = [wl.weights["w"], xb]
    ctx = _lib.Context(0)
    sel = idx or range(len(g["individuals"]))
    for i in sel:
        ind = g["individuals"][i]
        fn = dialect.parse_function(ind["forward"])
        ref = np.frombuffer(base64.b64decode(ind["probs0_b64"]), dtype=np.float64)
        (got,), = run_once(ctx, [fn], [params])
        if np.array_equal(got.reshape(-1), ref):
            print(f"individual {i}: probabilities bit-exact")
            continue
        # oracle values of every op
        vals = {}
        orig = OI.apply_op

        def hook(op, ins, tys, perturb=False):
            r = orig(op, ins, tys, perturb)
            vals[op.result] = (np.array(r, copy=True), [(np.asarray(x).shape, tuple(s // max(1, np.asarray(x).itemsize) for s in np.asarray(x).strides)) for x in ins])
            return r
        OI.apply_op = hook
        try:
            OI.Program(fn)([wl.weights["w"], xb4])
        finally:
            OI.apply_op = orig
        lo, hi = 0, len(fn.ops) - 1       # invariant: op hi differs
        while lo < hi:
            mid = (lo + hi) // 2
            (d,), = run_once(ctx, [truncated(fn, mid)], [params])
            want = vals[fn.ops[mid].result][0]
            same = np.array_equal(np.asarray(d).reshape(-1), np.asarray(want, dtype=d.dtype).reshape(-1))
            if same:
                lo = mid + 1
            else:
                hi = mid
        op = fn.ops[lo]
        (d,), = run_once(ctx, [truncated(fn, lo)], [params])
        want = np.asarray(vals[op.result][0], dtype=d.dtype)
        diff = np.flatnonzero(np.asarray(d).reshape(-1) != want.reshape(-1))
        print(f"individual {i} (edits {ind['edits']}): first differing op #{lo} {op.result} = "
              f"{op.opcode}{op.operands} -> {op.result_type.shape}; operands {vals[op.result][1]}; "
              f"{len(diff)} of {want.size} elements differ, first at {diff[:5].tolist()}; "
              f"max |d| {np.max(np.abs(np.asarray(d).reshape(-1)[diff] - want.reshape(-1)[diff])) if len(diff) and d.dtype.kind == 'f' else 0}")
    ctx.close()


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]])
