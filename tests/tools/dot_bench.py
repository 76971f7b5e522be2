"""Dot-only micro-benchmark (tool): 256 individuals whose train_step is just
the K=784 dot (x . w1) and/or the M=784 dot (x^T . d) with identity returns,
run through gevo_eval with the per-class profiler."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from paper_2310_10211_b200 import workloads as W  # noqa: E402
from paper_2310_10211_b200.dialect import parse_module  # noqa: E402
from paper_2310_10211_b200.evaluator import DeviceEvaluator  # noqa: E402

T = "tensor<{}xf32>"
SIG = ("func @train_step(%w1: tensor<784x32xf32>, %b1: tensor<32xf32>, %w2: tensor<32x10xf32>, "
       "%b2: tensor<10xf32>, %x: tensor<32x784xf32>, %y: tensor<32x10xf32>) -> (tensor<784x32xf32>, "
       "tensor<32xf32>, tensor<32x10xf32>, tensor<10xf32>) {\n")


def program(kind):
    body = "  %0 = dot %x, %w1 : tensor<32x32xf32>\n"
    if kind == "bignoepi":
        body += ("  %1 = transpose %x {perm = [1, 0]} : tensor<784x32xf32>\n"
                 "  %2 = dot %1, %0 : tensor<784x32xf32>\n"
                 "  return %2, %b1, %w2, %b2 : tensor<784x32xf32>, tensor<32xf32>, tensor<32x10xf32>, tensor<10xf32>\n}\n")
    elif kind == "bigsgd":
        body += ("  %1 = transpose %x {perm = [1, 0]} : tensor<784x32xf32>\n"
                 "  %2 = dot %1, %0 : tensor<784x32xf32>\n"
                 "  %3 = constant dense<0.01> : tensor<f32>\n"
                 "  %4 = broadcast_in_dim %3 {dims = []} : tensor<784x32xf32>\n"
                 "  %5 = multiply %2, %4 : tensor<784x32xf32>\n"
                 "  %6 = subtract %w1, %5 : tensor<784x32xf32>\n"
                 "  return %6, %b1, %w2, %b2 : tensor<784x32xf32>, tensor<32xf32>, tensor<32x10xf32>, tensor<10xf32>\n}\n")
    elif kind in ("big", "both"):
        body += ("  %1 = transpose %x {perm = [1, 0]} : tensor<784x32xf32>\n"
                 "  %2 = dot %1, %0 : tensor<784x32xf32>\n"
                 "  %3 = subtract %w1, %2 : tensor<784x32xf32>\n"
                 "  return %3, %b1, %w2, %b2 : tensor<784x32xf32>, tensor<32xf32>, tensor<32x10xf32>, tensor<10xf32>\n}\n")
    else:
        body += "  return %w1, %b1, %w2, %b2 : tensor<784x32xf32>, tensor<32xf32>, tensor<32x10xf32>, tensor<10xf32>\n}\n"
    fwd = ("func @forward(%w1: tensor<784x32xf32>, %b1: tensor<32xf32>, %w2: tensor<32x10xf32>, "
           "%b2: tensor<10xf32>, %x: tensor<32x784xf32>) -> tensor<32x10xf32> {\n"
           "  %0 = constant dense<0.1> : tensor<f32>\n"
           "  %1 = broadcast_in_dim %0 {dims = []} : tensor<32x10xf32>\n"
           "  return %1 : tensor<32x10xf32>\n}\n")
    m = parse_module(SIG + body + "\n" + fwd)
    return {"train_step": m.functions["train_step"], "forward": m.functions["forward"]}


def main(kind="small", n=256, steps=100):
    cfg = W.WorkloadConfig(steps=steps)
    wl = W.build_2fcnet_workload(cfg)
    ev = DeviceEvaluator(wl)
    fns = [program(kind)] * n
    ev.evaluate_variants(fns[:4])
    ev.evaluate_variants(fns)
    ms = ev.ctx.last_kernel_ms()
    ev.ctx.profile(True)
    ev.evaluate_variants(fns)
    prof = ev.ctx.profile(False)
    print(f"{kind}: kernel {ms:.2f} ms for {n} x {steps} steps = {1000 * ms / steps:.1f} us/step")
    for key, (cyc, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0])[:6]:
        print(f"  op={key}  cycles/instr={cyc / cnt:9.0f}  count={cnt}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "small", int(sys.argv[2]) if len(sys.argv) > 2 else 256)
