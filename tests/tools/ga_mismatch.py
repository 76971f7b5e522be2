"""Evaluate every individual of a recorded run on the device and list the
ones whose fitness differs from the recording (diagnostics).
    python tests/tools/ga_mismatch.py [ga512x50.json.gz] > gpurun_out/mism.json"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from ga_replay import parse_all  # noqa: E402
from golden_io import load  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ga512x50.json.gz"
from paper_2310_10211_b200 import workloads  # noqa: E402
from paper_2310_10211_b200.evaluator import DeviceEvaluator  # noqa: E402
data = load(name)
v = parse_all(data)
ev = DeviceEvaluator(workloads.build_2fcnet_workload())
out = []
for s in range(0, len(v), 1024):
    fits = ev.evaluate_variants(v[s:s + 1024])
    for i, f in enumerate(fits, s):
        r = data["individuals"][i]
        if (f.cost, f.error, f.valid) != (r["cost"], r["error"], r["valid"]):
            out.append([i, f.cost, f.error, f.valid, r["cost"], r["error"], r["valid"]])
print(json.dumps(out))
