"""A small workload for compute-sanitizer (tool; tests/tools/sanitize.sh):
the executor on three individuals (the unmutated program and two recorded
mutants) for a few training steps and scored batches, 40 per-op cases
through gevo_exec_once (every DOT path the opgen shapes reach), and the
NSGA-II / archive / hypervolume kernels on a recorded point set.  Checks
the outputs it can against the oracle so a sanitizer run also fails on a
wrong answer."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402
from golden_io import dec, load, variant_functions  # noqa: E402
from paper_2310_10211_b200 import _lib, dialect, shims, workloads as W  # noqa: E402
from paper_2310_10211_b200.evaluator import DeviceEvaluator  # noqa: E402


def main():
    steps = int(os.environ.get("SAN_STEPS", "4"))
    cfg = W.WorkloadConfig(steps=steps, finite_check_every=2,
                           dataset=W.DatasetConfig(search_n=96, holdout_n=64))
    wl = W.build_2fcnet_workload(cfg)
    inds = load("train_pop.json.gz")["individuals"][1:3]
    variants = [{n: wl.module.functions[n] for n in ("forward", "train_step")}]
    variants += [variant_functions(i) for i in inds]
    ev = DeviceEvaluator(wl, device=0)
    fits = ev.evaluate_variants(variants)
    print("fitness", [(f.cost, f.error) for f in fits])
    ev.close()

    from test_gpu_parity import _words, run_once
    cases = [c for c in load("opcases.json.gz")["cases"] if c["opcode"] in ("dot", "reduce", "pad")][::4]
    ctx = _lib.Context(0)
    fns = [dialect.parse_function(c["text"]) for c in cases]
    params = [[_words(dec(o)) for o in c["operands"]] for c in cases]
    outs = run_once(ctx, fns, params)
    bad = 0
    for c, (got,) in zip(cases, outs):
        exp = dec(c["expected"])
        g = np.asarray(got).reshape(exp.shape).astype(exp.dtype)
        bad += not np.allclose(g, exp, rtol=1e-12, atol=0, equal_nan=True)
    print(f"opcases {len(cases) - bad}/{len(cases)}")
    ctx.close()

    s = load("nsga2.json.gz")["sets"][0]
    pts = [(float(c), float(e)) for c, e in s["points"]]
    assert shims.nondominated_sort(pts) == s["fronts"]
    print("nsga2 ok; hypervolume", shims.hypervolume(pts, (1e12, 1.0)))
    assert bad == 0


if __name__ == "__main__":
    main()
