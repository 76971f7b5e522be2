"""Where the end-to-end time of evaluate_variants goes at several population
sizes (tool): host lowering wait, plan packing, total, device span."""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.dirname(os.path.dirname(HERE))]
from golden_io import load  # noqa: E402
from paper_2310_10211_b200 import workloads as W  # noqa: E402
from paper_2310_10211_b200.dialect import parse_function  # noqa: E402
from paper_2310_10211_b200.evaluator import DeviceEvaluator  # noqa: E402

inds = load("bench_train_pool.json.gz")["individuals"]
inds = [i for i in inds if not i.get("invalid_patch")]
fns = [{n: parse_function(i[n]) for n in ("forward", "train_step")} for i in inds]
ev = DeviceEvaluator(W.build_2fcnet_workload())
ev.evaluate_variants(fns[:64])
for P in [int(a) for a in sys.argv[1:]] or [256, 1024, 4096]:
    vs = [fns[k % len(fns)] for k in range(P)]
    for rep in range(2):
        t0 = time.perf_counter()
        ev.evaluate_variants(vs)
        dt = time.perf_counter() - t0
        t = dict(ev.last_timing)
        print(json.dumps({"P": P, "rep": rep, "wall_s": round(dt, 3), "ind_s": round(P / dt, 1),
                          "device_ms": round(ev.last_device_ms, 1),
                          **{k: round(v, 3) if isinstance(v, float) else v for k, v in t.items()}}))
