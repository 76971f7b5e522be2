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
    fits, rec = ev.evaluate_variants(fns, return_records=True)
    cyc = rec["cycles"].astype(np.float64)
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
