import os, sys
ROOT = "/root/repo"; sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from golden_io import load
from paper_2310_10211_b200 import workloads as W
from paper_2310_10211_b200.dialect import parse_function
from paper_2310_10211_b200.evaluator import DeviceEvaluator
import bench
inds, pf = bench.load_pool()
ev = DeviceEvaluator(W.build_2fcnet_workload())
OPS = {0: "tapsum", 1: "unary", 2: "binary", 3: "select", 4: "reduce", 5: "dot", 6: "pad"}
for k in (55, 0):
    fns = [{n: pf(inds[k][n]) for n in ("forward", "train_step")}] * 148
    ev.evaluate_variants(fns[:4])
    ev.ctx.profile(True)
    ev.evaluate_variants(fns)
    ms = ev.ctx.last_kernel_ms()
    prof = ev.ctx.profile(False)
    tot = sum(c for c, _ in prof.values())
    print(f"individual {k}: kernel {ms:.1f} ms")
    for (op, sub, big), (cyc, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0])[:8]:
        print(f"  {OPS.get(op, str(op)):7s} sub={sub:2d} {'big' if big else 'small':5s} {100*cyc/tot:5.1f}% count={cnt:8d} cyc/instr={cyc/cnt:9.0f}")
