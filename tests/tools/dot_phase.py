"""dot_fast phase timing (tool; needs a GEVO_DOT_TIMING build of libgevo.so):
cycles per phase summed over CTA thread 0s."""
import sys
sys.argv += ["bigsgd", "32"][len(sys.argv) - 1:]
import dot_bench  # noqa: E402
from paper_2310_10211_b200 import workloads as W  # noqa: E402
from paper_2310_10211_b200.evaluator import DeviceEvaluator  # noqa: E402

NAMES = {1: "issue loads", 2: "wait+barrier", 3: "compute", 4: "C tile", 5: "emit", 6: "tail barrier"}
kind, n = sys.argv[1], int(sys.argv[2])
ev = DeviceEvaluator(W.build_2fcnet_workload(W.WorkloadConfig(steps=100)))
fns = [dot_bench.program(kind)] * n
ev.evaluate_variants(fns[:4])
ev.ctx.profile(True)
ev.evaluate_variants(fns)
prof = ev.ctx.profile(False)
for (op, sub, big), (cyc, cnt) in sorted(prof.items()):
    if op == 0 and big == 0 and sub in NAMES:
        print(f"{NAMES[sub]:14s} cycles/stage {cyc / cnt:8.0f}  stages {cnt}")
