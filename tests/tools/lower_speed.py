"""Host lowering throughput (tool): in-process per individual, and through
the evaluator's process pool at several batch sizes."""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.dirname(os.path.dirname(HERE))]
from golden_io import load  # noqa: E402
from paper_2310_10211_b200.dialect import parse_function  # noqa: E402
from paper_2310_10211_b200.evaluator import lower_all, _lower_pool  # noqa: E402
from paper_2310_10211_b200.plan import lower_variant  # noqa: E402
import pickle  # noqa: E402

inds = [i for i in load("bench_train_pool.json.gz")["individuals"] if not i.get("invalid_patch")]
fns = [{n: parse_function(i[n]) for n in ("forward", "train_step")} for i in inds[:512]]
t0 = time.perf_counter()
vps = [lower_variant(f, {}, training=True, steps=600) for f in fns[:128]]
dt = time.perf_counter() - t0
print(f"in-process: {dt / 128 * 1e3:.2f} ms/individual; cpus {os.cpu_count()}")
t0 = time.perf_counter()
blob = pickle.dumps(fns[:128])
t1 = time.perf_counter()
rb = pickle.dumps(vps)
t2 = time.perf_counter()
pickle.loads(rb)
t3 = time.perf_counter()
print(f"pickle in {len(blob) / 128:.0f} B/ind {(t1 - t0) / 128 * 1e6:.0f} us/ind; "
      f"out {len(rb) / 128:.0f} B/ind dumps {(t2 - t1) / 128 * 1e6:.0f} us loads {(t3 - t2) / 128 * 1e6:.0f} us")
_lower_pool()
lower_all(fns[:64], {}, True, 600)
for n in (64, 128, 256, 512):
    t0 = time.perf_counter()
    lower_all(fns[:n], {}, True, 600)
    dt = time.perf_counter() - t0
    print(f"pool n={n}: {dt * 1e3:.1f} ms ({n / dt:.0f} ind/s)")
