"""CNN prediction fixtures from the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src:. PYTHONDONTWRITEBYTECODE=1 \
    python tests/golden/make_cnn_golden.py

The CNN workload is new, so its oracle is the
reference's own interpreter and mutation engine run on the network text:

  * the module text of paper_2310_10211_b200.cnn is parsed by the reference
    parser (parser.py:337) -- the dialect is unchanged;
  * mutants come from the reference's genome.mutate (genome.py:626-657),
    chained like search._mutated (search.py:283-293), with the reference's
    smoke rule (fitness.py:82-96: one forward run on batch 0);
  * each variant is scored with the reference interpreter (interpreter.py:
    188-225) over the search batches exactly like _misclassification
    (fitness.py:355-369), and its static cost is the reference's
    (interpreter.py:41-59, fitness.py:387-388).

Writes tests/golden/cnn_pop.json.gz (the reduced 4-block net, 30 images).

    ... make_cnn_golden.py full

records the BASELINE.json configs[2] network itself (MobileNetV2-CIFAR width
0.5, cnn.MOBILENETV2_CIFAR_HALF, batch 100) over 100 images with 16
reference-made mutants (about 10 min on one core) into
tests/golden/cnn_full_pop.json.gz.

    ... make_cnn_golden.py full2 SEED N OUT

records N more full-size mutants from rng seed SEED (chains of up to five
edits) into OUT; tests/golden/cnn_full_pop2.json.gz merges four such runs
(seeds 2311-2314, 9 variants each, the unmutated network dropped from all
but the first), run in parallel:

    for s in 2311 2312 2313 2314; do python tests/golden/make_cnn_golden.py \
        full2 $s 10 /tmp/cnn2_$s.json.gz & done; wait
    python tests/golden/make_cnn_golden.py merge2 /tmp/cnn2_23*.json.gz
"""
from __future__ import annotations

import base64
import gzip
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from evotir.genome import MutationError, apply_patch, mutate, patch_dumps  # noqa: E402
from evotir.interpreter import get_plan  # noqa: E402
from evotir.ir import Module  # noqa: E402
from evotir.parser import parse_module  # noqa: E402
from evotir.printer import print_module  # noqa: E402

from paper_2310_10211_b200 import cnn  # noqa: E402

N_VARIANTS = 16
MAX_EDITS = 3


def fn_text(fn) -> str:
    return print_module(Module(functions={fn.name: fn}, constants={}))


def main(full=False, seed=2310, n_variants=N_VARIANTS, max_edits=MAX_EDITS, path=None):
    if full:
        cfg = cnn.CnnConfig(**cnn.MOBILENETV2_CIFAR_HALF, batch_size=100, search_n=100,
                            holdout_n=100)
    else:
        cfg = cnn.CnnConfig(search_n=30, holdout_n=10)
    wl = cnn.build_cnn_prediction_workload(cfg)
    text, flat = cnn.cnn_forward_text(cfg)
    module = parse_module(text)
    B, S, C = cfg.batch_size, cfg.side, cfg.in_channels
    xs = wl.search_x.reshape(-1, B, S, S, C)
    lbs = wl.search_labels

    def probs_of(mod, xb):
        plan = get_plan(mod.functions["forward"])
        with np.errstate(all="ignore"):
            return plan.run([flat, xb])[0]

    def smoke(mod):
        try:
            probs_of(mod, xs[0])
            return True
        except Exception:
            return False

    def score(mod):
        plan = get_plan(mod.functions["forward"])
        wrong = total = 0
        for xb, lb in zip(xs, lbs):
            with np.errstate(all="ignore"):
                (p,) = plan.run([flat, xb])
            if not np.all(np.isfinite(p)):
                return dict(wrong=0, total=0, status=2, error=1.0, cost=plan.total_cost * len(xs))
            wrong += int(np.sum(np.argmax(p, axis=1) != lb))
            total += len(lb)
        return dict(wrong=wrong, total=total, status=0, error=wrong / total,
                    cost=plan.total_cost * len(xs))

    rng = random.Random(seed)
    inds = []
    patch = ()
    variants = [()]
    while len(variants) < n_variants:
        base = variants[rng.randrange(len(variants))] if len(variants) > 1 else ()
        if len(base) >= max_edits:
            base = ()
        variant = apply_patch(module, base).module
        try:
            edit = mutate(variant, rng, functions=["forward"], smoke=smoke)
        except MutationError:
            continue
        variants.append(base + (edit,))
    for patch in variants:
        mod = apply_patch(module, patch).module
        rec = score(mod)
        rec.update(key=patch_dumps(patch), edits=len(patch),
                   forward=fn_text(mod.functions["forward"]))
        if full:
            # the probabilities of batch 0 as the reference computes them:
            # a bit-level check far stronger than the error of a frozen
            # random-init network (near chance for every variant)
            p0 = np.ascontiguousarray(probs_of(mod, xs[0]), dtype=np.float64)
            rec["probs0_b64"] = base64.b64encode(p0.tobytes()).decode()
        inds.append(rec)
        print(f"edits {len(patch)}: cost {rec['cost']:.0f} wrong {rec['wrong']}/{rec['total']} "
              f"status {rec['status']}")
    out = {"config": {"search_n": cfg.search_n, "holdout_n": cfg.holdout_n,
                      "batch_size": cfg.batch_size},
           "individuals": inds}
    if full:
        out["config"]["network"] = "MOBILENETV2_CIFAR_HALF"
    path = path or os.path.join(HERE, "cnn_full_pop.json.gz" if full else "cnn_pop.json.gz")
    with gzip.open(path, "wt") as f:
        json.dump(out, f, separators=(",", ":"), sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def merge2(paths):
    """cnn_full_pop2.json.gz: the full2 runs' mutants (one unmutated network)."""
    out, seen = None, set()
    for p in sorted(paths):
        with gzip.open(p, "rt") as f:
            d = json.load(f)
        if out is None:
            out = {"config": d["config"], "individuals": []}
        for ind in d["individuals"]:
            if ind["key"] not in seen:
                seen.add(ind["key"])
                out["individuals"].append(ind)
    path = os.path.join(HERE, "cnn_full_pop2.json.gz")
    with gzip.open(path, "wt") as f:
        json.dump(out, f, separators=(",", ":"), sort_keys=True)
    print(f"wrote {path}: {len(out['individuals'])} individuals")


if __name__ == "__main__":
    if sys.argv[1:2] == ["full2"]:
        main(full=True, seed=int(sys.argv[2]), n_variants=int(sys.argv[3]), max_edits=5,
             path=sys.argv[4])
    elif sys.argv[1:2] == ["merge2"]:
        merge2(sys.argv[2:])
    else:
        main(full=sys.argv[1:2] == ["full"])
