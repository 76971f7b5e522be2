"""Where the end-to-end time of the seam goes (tool): evotir's _Evaluator
with shims.install() on bench-pool patches; per call the evaluator's own
timing (lowering wait, packing, total) and the device span."""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "baseline", "_ref")]
import bench  # noqa: E402
import evotir.search as S  # noqa: E402
from evotir import fitness as F  # noqa: E402
from evotir.genome import patch_loads  # noqa: E402
from paper_2310_10211_b200 import shims  # noqa: E402

inds, _ = bench.load_pool()
rwl = F.build_2fcnet_workload()
shims.install(device=0)
dev = shims.device_for(rwl, 0)
P = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for rep in range(4):
    patches = [patch_loads(inds[(rep * P + k) % len(inds)]["key"]) for k in range(P)]
    E = S._Evaluator(rwl)
    t0 = time.perf_counter()
    E(patches)
    dt = time.perf_counter() - t0
    t = dict(dev.last_timing)
    print(json.dumps({"P": P, "rep": rep, "wall_s": round(dt, 3), "ind_s": round(P / dt, 1),
                      "device_ms": round(dev.last_device_ms, 1),
                      **{k: round(v, 3) if isinstance(v, float) else v for k, v in t.items()}}))
shims.uninstall()
