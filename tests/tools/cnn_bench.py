"""CNN prediction throughput (tool; BASELINE.json configs[2] at reduced
scale): population = the 16 reference-made variants of
tests/golden/cnn_pop.json.gz repeated to `pop`, scored over `n` synthetic
CIFAR-shaped images (batch 10), float64, device time of the evaluation
kernel; the oracle timed on a few individuals beside it."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402
from golden_io import load  # noqa: E402
from paper_2310_10211_b200 import cnn, dialect  # noqa: E402
from paper_2310_10211_b200.evaluator import DeviceEvaluator  # noqa: E402


def main(pop=128, n=1000):
    g = load("cnn_pop.json.gz")
    wl = cnn.build_cnn_prediction_workload(cnn.CnnConfig(search_n=n, holdout_n=10))
    base = [{"forward": dialect.parse_function(i["forward"])} for i in g["individuals"]]
    variants = [base[k % len(base)] for k in range(pop)]
    ev = DeviceEvaluator(wl)
    ev.evaluate_variants(variants[:4])
    t = time.perf_counter()
    fits, rec = ev.evaluate_variants(variants, return_records=True)
    wall = time.perf_counter() - t
    ms = ev.last_device_ms
    macs = 0
    fn = base[0]["forward"]
    types = dict(fn.params)
    for op in fn.ops:
        if op.opcode == "dot":
            a, b = types[op.operands[0]], types[op.operands[1]]
            macs += a.shape[0] * a.shape[1] * b.shape[1]
        types[op.result] = op.result_type
    flops = 2.0 * macs * (n // 10) * pop
    print(f"cnn pop {pop} x {n} images: device {ms:.1f} ms -> {pop / ms * 1e3:.1f} ind/s "
          f"({flops / ms / 1e9:.3f} TFLOP/s fp64 dot work), e2e {pop / wall:.1f} ind/s; "
          f"median CTA cycles {np.median(rec['cycles']):.3g}, max {rec['cycles'].max():.3g}")
    ev.close()
    from oracle import fitness as OF
    xs = wl.search_x.reshape(-1, 10, 32, 32, 3)
    t = time.perf_counter()
    for v in base[:2]:
        OF.evaluate_variant(v, "prediction", [wl.weights["w"]], (xs, wl.search_y, wl.search_labels))
    dt = (time.perf_counter() - t) / 2
    print(f"oracle (1 core): {dt:.2f} s per individual -> {1 / dt:.2f} ind/s")




def profile(pop=128, n=100):
    """per-instruction-class cycles of the CNN population"""
    g = load("cnn_pop.json.gz")
    wl = cnn.build_cnn_prediction_workload(cnn.CnnConfig(search_n=n, holdout_n=10))
    base = [{"forward": dialect.parse_function(i["forward"])} for i in g["individuals"]]
    variants = [base[k % len(base)] for k in range(pop)]
    ev = DeviceEvaluator(wl)
    ev.evaluate_variants(variants[:4])
    ev.ctx.profile(True)
    ev.evaluate_variants(variants[:64])
    prof = ev.ctx.profile(False)
    tot = sum(c for c, _ in prof.values())
    OPS = {1: "unary", 2: "binary", 3: "select", 4: "reduce", 5: "dot", 6: "pad"}
    for (op, sub, big), (cyc, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0])[:14]:
        print(f"{OPS.get(op, op):7s} sub={sub:2d} {'big' if big else 'small':5s} "
              f"{100 * cyc / tot:5.1f}%  count={cnt:9d}  cycles/instr={cyc / cnt:9.0f}")


if __name__ == "__main__":
    if sys.argv[1:2] == ["profile"]:
        profile(*[int(a) for a in sys.argv[2:]])
    else:
        main(*[int(a) for a in sys.argv[1:]])
