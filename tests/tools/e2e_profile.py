"""cProfile of one evaluate_variants call at a bench-sized population (tool):
where the parent process spends the end-to-end time."""
import cProfile
import os
import pstats
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.dirname(os.path.dirname(HERE))]
from golden_io import load  # noqa: E402
from paper_2310_10211_b200 import workloads as W  # noqa: E402
from paper_2310_10211_b200.dialect import parse_function  # noqa: E402
from paper_2310_10211_b200.evaluator import DeviceEvaluator  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 256
inds = [i for i in load("bench_train_pool.json.gz")["individuals"] if not i.get("invalid_patch")]
fns = [{n: parse_function(i[n]) for n in ("forward", "train_step")} for i in inds]
ev = DeviceEvaluator(W.build_2fcnet_workload())
ev.evaluate_variants(fns[:P])
vs = fns[P:2 * P]
pr = cProfile.Profile()
pr.enable()
ev.evaluate_variants(vs)
pr.disable()
print(ev.last_timing, "device_ms", ev.last_device_ms)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
