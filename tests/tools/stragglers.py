"""Per-individual device cycles of one bench population (tool): the
distribution, and the DOT instructions of the slowest individuals with their
summation order and operand strides."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2310_10211_b200 import workloads as W  # noqa: E402
from paper_2310_10211_b200.evaluator import DeviceEvaluator  # noqa: E402
from paper_2310_10211_b200.plan import lower_variant  # noqa: E402

BUF = {0: "arena", 1: "const", 18: "smem"}


def main(start=0, n=256):
    inds, pf = bench.load_pool()
    sel = inds[start:start + n]
    fns = [{k: pf(i[k]) for k in ("forward", "train_step")} for i in sel]
    ev = DeviceEvaluator(W.build_2fcnet_workload())
    ev.evaluate_variants(fns[:8])
    from paper_2310_10211_b200.evaluator import lower_all
    from paper_2310_10211_b200.plan import build_population_plan, device_weight, sm_aware_order
    vps = lower_all(fns, None, True)
    plan = build_population_plan(vps, ev.weight_shapes, 320,
                                 order=sm_aware_order([device_weight(v) for v in vps], ev.n_sms))
    rec, _ = ev.ctx.eval(plan.blob, plan.n_prog, 0, 600, 50, 0, 0, ev.weight_elems, False)
    ev.last_device_ms = ev.ctx.last_kernel_ms()
    cyc = rec["cycles"].astype(np.float64)
    t0, t1 = rec["t0_ns"], rec["t1_ns"]
    base = t0.min()
    print(f"CTA start spread {(t0.max() - base) / 1e6:.2f} ms, end spread {(t1.min() - base) / 1e6:.1f}.."
          f"{(t1.max() - base) / 1e6:.1f} ms; SM clock from timers "
          f"{np.median(cyc / np.maximum(t1 - t0, 1)):.3f} GHz")
    cb = cyc[plan.order]                  # cycles by launch slot (block id)
    sm = rec["smid"][plan.order]
    shared = np.bincount(sm, minlength=int(sm.max()) + 1)[sm] > 1
    print(f"CTAs alone on their SM: {int((~shared).sum())}; median cycles alone "
          f"{np.median(cb[~shared]) if (~shared).any() else 0:.3g}, shared {np.median(cb[shared]):.3g}; "
          f"blocks alone: {np.flatnonzero(~shared)[:8].tolist()}...")
    nsm = ev.n_sms
    if len(cb) > nsm:
        pairs = len(cb) - nsm
        print(f"by block: paired 0..{pairs - 1} median {np.median(cb[:pairs]):.3g}, "
              f"solo {pairs}..{nsm - 1} median {np.median(cb[pairs:nsm]):.3g}, "
              f"paired {nsm}.. median {np.median(cb[nsm:]):.3g}; max at block {int(np.argmax(cb))}")
    print(f"kernel span {ev.last_device_ms:.1f} ms; cycles per individual: "
          f"median {np.median(cyc):.3g}, p90 {np.percentile(cyc, 90):.3g}, max {cyc.max():.3g}")
    for i in np.argsort(-cyc)[:6]:
        vp = lower_variant(fns[i])
        print(f"-- individual {start + i}: {cyc[i]:.3g} cycles ({cyc[i] / np.median(cyc):.1f}x median), "
              f"status {rec['status'][i]}")
        for tag, arr in (("train", vp.train1), ("fwd", vp.fwd)):
            for r in arr:
                if r["op"] == 5:
                    ins = [(BUF.get(int(o["buf"]), int(o["buf"])), int(o["off"]), tuple(int(x) for x in o["st"][:2]))
                           for o in r["in"][:2]]
                    print(f"   {tag} DOT mode {r['sub']}/{r['aux'][2]} split {r['aux'][1]} "
                          f"M,N,K={r['shp'][0]},{r['shp'][1]},{r['aux'][0]} A,B={ins} epi={r['aux2'][1]}")
    ev.close()


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
