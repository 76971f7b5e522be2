"""Per-instruction-class cycle profile of one bench-sized evaluation (tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from golden_io import load  # noqa: E402
from paper_2310_10211_b200 import workloads as W  # noqa: E402
from paper_2310_10211_b200.dialect import parse_function  # noqa: E402
from paper_2310_10211_b200.evaluator import DeviceEvaluator  # noqa: E402

OPS = {1: "unary", 2: "binary", 3: "select", 4: "reduce", 5: "dot", 6: "pad"}


def main(n=256):
    inds = load("bench_train_pool.json.gz")["individuals"][:n]
    fns = [{k: parse_function(i[k]) for k in ("forward", "train_step")} for i in inds]
    ev = DeviceEvaluator(W.build_2fcnet_workload())
    ev.evaluate_variants(fns[:8])
    ev.ctx.profile(True)
    ev.evaluate_variants(fns)
    ms = ev.ctx.last_kernel_ms()
    prof = ev.ctx.profile(False)
    tc = {k: v for k, v in prof.items() if k[0] == 7}      # dot_tc phases (slots 240..)
    prof = {k: v for k, v in prof.items() if k[0] != 7}
    tot = sum(c for c, _ in prof.values())
    print(f"kernel {ms:.1f} ms; CTA-cycles profiled {tot:.3e}")
    for (op, sub, big), (cyc, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        print(f"{OPS.get(op, op):7s} sub={sub:2d} {'big' if big else 'small':5s} "
              f"{100 * cyc / tot:5.1f}%  count={cnt:9d}  cycles/instr={cyc / cnt:9.0f}")
    names = ["wait for a stage", "stage (loads, tf32, stores) + fence + barrier", "MMA issue + commit",
             "wait for the accumulator", "TMEM read + epilogue"]
    for (op, sub, big), (cyc, cnt) in sorted(tc.items()):
        ph = 2 * (sub - 8) + big
        print(f"tcgen05 phase {ph} {names[ph] if ph < len(names) else ''}: {100 * cyc / tot:5.1f}% of CTA cycles, "
              f"count={cnt}, cycles each={cyc / cnt:8.0f}")


if __name__ == "__main__":
    main()
