"""Device vs oracle wrong counts of one bench-pool individual after 0..600
training steps (tool): finds the first step where they diverge."""
import sys
sys.path[:0]=['/root/repo','/root/repo/tests']
from golden_io import load
from paper_2310_10211_b200.dialect import parse_function
from paper_2310_10211_b200 import workloads as W
from paper_2310_10211_b200.evaluator import DeviceEvaluator
from oracle import fitness as OF
k = int(sys.argv[1]) if len(sys.argv) > 1 else 560
inds=load("bench_train_pool.json.gz")["individuals"]
seen=set(); pool=[]
for i in inds:
    if i["key"] not in seen: seen.add(i["key"]); pool.append(i)
v={n: parse_function(pool[k][n]) for n in ("forward","train_step")}
for steps in (0, 1, 2, 3, 5, 10, 50, 600):
    wl=W.build_2fcnet_workload(W.WorkloadConfig(steps=steps))
    ev=DeviceEvaluator(wl)
    (f,), rec = ev.evaluate_variants([v], return_records=True)
    ev.close()
    w0=[wl.weights[n] for n in W.WEIGHT_NAMES]
    o=OF.evaluate_variant(v, "training", w0, (wl.search_x, wl.search_y, wl.search_labels), steps=steps)
    print(steps, "device", int(rec["wrong"][0]), int(rec["status"][0]), "oracle", o["wrong"], o["status"])
