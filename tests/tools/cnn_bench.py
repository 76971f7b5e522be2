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


def full(pop=128, n=1000, batch=100, check=100):
    """BASELINE.json configs[2] network: MobileNetV2-CIFAR width 0.5
    (cnn.MOBILENETV2_CIFAR_HALF), batch 100, `n` images, the unmutated
    forward replicated to `pop` (throughput of the full-size network), and a
    parity check of its fitness against the oracle on the first `check`
    images."""
    cfg = cnn.CnnConfig(**cnn.MOBILENETV2_CIFAR_HALF, batch_size=batch, search_n=n,
                        holdout_n=batch)
    wl = cnn.build_cnn_prediction_workload(cfg)
    fn = wl.module.functions["forward"]
    macs = 0
    types = dict(fn.params)
    for op in fn.ops:
        if op.opcode == "dot":
            a, b = types[op.operands[0]], types[op.operands[1]]
            macs += a.shape[0] * a.shape[1] * b.shape[1]
        types[op.result] = op.result_type
    ev = DeviceEvaluator(wl)
    v = {"forward": fn}
    t = time.perf_counter()
    fits, rec = ev.evaluate_variants([v] * pop, return_records=True)
    wall = time.perf_counter() - t
    ms = ev.last_device_ms
    flops = 2.0 * macs * (n // batch) * pop
    print(f"full cnn (MobileNetV2-CIFAR 0.5, {macs / batch / 1e6:.1f} M dot MACs/img) pop {pop} x "
          f"{n} images, batch {batch}: device {ms / 1e3:.2f} s -> {pop / ms * 1e3:.3f} ind/s "
          f"({flops / ms / 1e9:.3f} TFLOP/s fp64 dot work), e2e {pop / wall:.3f} ind/s; "
          f"{n * pop / (ms / 1e3):.0f} images/s; fitness {fits[0]}")
    ev.close()
    # parity on the first `check` images: device vs oracle
    cfg2 = cnn.CnnConfig(**cnn.MOBILENETV2_CIFAR_HALF, batch_size=batch, search_n=check,
                         holdout_n=batch)
    wl2 = cnn.build_cnn_prediction_workload(cfg2)
    ev2 = DeviceEvaluator(wl2)
    (f_dev,), rec2 = ev2.evaluate_variants([{"forward": wl2.module.functions["forward"]}],
                                           return_records=True)
    ev2.close()
    from oracle import fitness as OF
    xs = wl2.search_x.reshape(-1, batch, 32, 32, 3)
    t = time.perf_counter()
    r = OF.evaluate_variant({"forward": wl2.module.functions["forward"]}, "prediction",
                            [wl2.weights["w"]], (xs, wl2.search_y, wl2.search_labels))
    dt = time.perf_counter() - t
    print(f"parity on {check} images: device {f_dev.cost} {f_dev.error} (wrong {int(rec2['wrong'][0])}) "
          f"oracle {r['cost']} {r['error']} (wrong {r['wrong']}) -> "
          f"{'bit-exact' if (f_dev.cost, f_dev.error) == (r['cost'], r['error']) else 'DIFFERENT'}; "
          f"oracle {dt:.1f} s for {check} images on 1 core "
          f"({dt * 10000 / check / 60:.1f} min per 10k-image individual)")


def fullprof(pop=128, n=200, batch=100):
    """per-instruction-class cycles of the full-size network (configs[2])"""
    cfg = cnn.CnnConfig(**cnn.MOBILENETV2_CIFAR_HALF, batch_size=batch, search_n=n,
                        holdout_n=batch)
    wl = cnn.build_cnn_prediction_workload(cfg)
    v = {"forward": wl.module.functions["forward"]}
    ev = DeviceEvaluator(wl)
    ev.evaluate_variants([v] * 4)
    ev.ctx.profile(True)
    ev.evaluate_variants([v] * pop)
    prof = ev.ctx.profile(False)
    tot = sum(c for c, _ in prof.values())
    print(f"full cnn profile: pop {pop} x {n} images, kernel {ev.last_device_ms:.1f} ms")
    OPS = {0: "tapsum", 1: "unary", 2: "binary", 3: "select", 4: "reduce", 5: "dot", 6: "pad"}
    for (op, sub, big), (cyc, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0])[:16]:
        print(f"{OPS.get(op, str(op)):7s} sub={sub:2d} {'big' if big else 'small':5s} "
              f"{100 * cyc / tot:5.1f}%  count={cnt:9d}  cycles/instr={cyc / cnt:9.0f}")
    # the dots of the network: shape, summation order, operand strides
    from paper_2310_10211_b200.plan import lower_variant
    vp = lower_variant(v, None, training=False, steps=0)
    for r in vp.fwd:
        if r["op"] == 5 and False:
            print("  DOT M,N,K", int(r["shp"][0]), int(r["shp"][1]), int(r["aux"][0]),
                  "mode", int(r["sub"]), int(r["aux"][2]),
                  "A st", tuple(int(x) for x in r["in"][0]["st"][:2]),
                  "B st", tuple(int(x) for x in r["in"][1]["st"][:2]))
    ev.close()


if __name__ == "__main__":
    if sys.argv[1:2] == ["fullprof"]:
        fullprof(*[int(a) for a in sys.argv[2:]])
        sys.exit(0)
    if sys.argv[1:2] == ["full"]:
        full(*[int(a) for a in sys.argv[2:]])
    elif sys.argv[1:2] == ["profile"]:
        profile(*[int(a) for a in sys.argv[2:]])
    else:
        main(*[int(a) for a in sys.argv[1:]])
