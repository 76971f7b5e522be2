"""GPU diagnostic (tool): for each recorded individual, run one train_step
from the init weights with EVERY intermediate returned, and report the first
op whose device result is not bit-identical to the oracle's."""
import collections
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from golden_io import load  # noqa: E402
from oracle import interp as OI  # noqa: E402
from paper_2310_10211_b200 import _lib, dialect, lowering as Lw, workloads as W  # noqa: E402
from paper_2310_10211_b200.plan import exec_once_plan  # noqa: E402


def value_fns(fn, per=8):
    """Copies of fn returning its op results 8 at a time (GEVO_MAXP)."""
    out = []
    for j in range(0, len(fn.ops), per):
        ops = fn.ops[j:j + per]
        out.append(dialect.FunctionBody(fn.name, fn.params, fn.ops,
                                        tuple(o.result for o in ops),
                                        tuple(o.result_type for o in ops)))
    return out


def main():
    wl = W.build_2fcnet_workload()
    pop = load("train_pop.json.gz")["individuals"]
    w0 = [wl.weights[n] for n in W.WEIGHT_NAMES]
    args = w0 + [wl.search_x[0], wl.search_y[0]]
    ctx = _lib.Context(0)
    tally = collections.Counter()
    examples = {}
    for ind in pop:
        fn = dialect.parse_function(ind["train_step"])
        fns = value_fns(fn)
        full = dialect.FunctionBody(fn.name, fn.params, fn.ops,
                                    tuple(o.result for o in fn.ops),
                                    tuple(o.result_type for o in fn.ops))
        ref = OI.Program(full)(args)
        pa = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in args]
        blob, pblob, meta, total = exec_once_plan(fns, [pa] * len(fns))
        outs = ctx.exec_once(blob, pblob, total)
        metas = [m for ms in meta for m in ms]
        for k, ((off, shape, kind), r, op) in enumerate(zip(metas, ref, fn.ops)):
            n = max(1, int(np.prod(shape)))
            w = outs[off:off + n]
            r = np.asarray(r)
            if kind == "f32":
                same = np.array_equal(w.reshape(r.shape), r, equal_nan=True)
            else:
                same = np.array_equal(w.view(np.int64).reshape(r.shape), r.astype(np.int64))
            if not same:
                key = op.opcode
                if op.opcode == "dot":
                    key = f"dot{tuple(shape)}"
                if op.opcode == "reduce":
                    key = f"reduce-{op.attrs['kind']}"
                tally[key] += 1
                if key not in examples:
                    g = w.reshape(r.shape)
                    bad = np.argwhere(g != r)[:3].tolist() if r.ndim else []
                    examples[key] = {"op": f"{op.result} = {op.opcode} {op.operands} {op.attrs}",
                                     "shape": list(shape), "bad_idx": bad,
                                     "n_bad": int(np.sum(g != r))}
                break
        else:
            tally["exact"] += 1
    print(json.dumps({"first_diff": tally, "examples": examples}, indent=1, default=str))


if __name__ == "__main__":
    main()
