"""Generate the golden fixtures from the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests:. \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--bench]

/root/reference does not exist on the GPU box, so everything the GPU tests
and bench need from the reference is recorded here as data:

  opcases.json.gz        per-opcode cases drawn with the reference's own
                         generator (pkg/tests/opgen.py:50-147, seeds
                         "unit-<opcode>" as test_interpreter.py:21) and the
                         reference eval_op outputs (interpreter.py:272-281)
  train_pop.json.gz      every individual evaluated by a seeded run_search
                         (search.py:333-399; pop 64, 3 gens, elites 16,
                         seed 0) on train2fc defaults: variant program text
                         (printer.py:84 of apply_patch(...).module), patch
                         JSON (genome.py:302-305) and reference Fitness
  predict_pop.json.gz    same on predict2fc (pop 64, 2 gens)
  predict_weights.npz    frozen predict2fc weights (fitness.py:265-270)
  nsga2.json.gz          point sets (test_search.py:20-29 style grids with
                         inf, C5 mixed sets) and reference fronts, crowding,
                         rank_population and select_survivors outputs
  meta.json              dataset/weight hashes and the BASELINE.md goldens
  bench_train_pool.json.gz  (--bench) pop 256 x 10 generations, the bench
                         pool for BASELINE.json configs[1]
"""
from __future__ import annotations

import os
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import base64
import gzip
import hashlib
import json
import multiprocessing as mp
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from evotir import fitness as F, search as S, genome as G  # noqa: E402
from evotir.datasets import DatasetConfig  # noqa: E402
from evotir.interpreter import eval_op  # noqa: E402
from evotir.ir import OPCODES, FunctionBody, Module  # noqa: E402
from evotir.printer import print_module  # noqa: E402

import opgen  # noqa: E402  (reference test helper)


def enc(a) -> dict:
    a = np.ascontiguousarray(a)
    return {"dtype": a.dtype.str, "shape": list(a.shape),
            "b64": base64.b64encode(a.tobytes()).decode()}


def fn_text(fn) -> str:
    return print_module(Module(functions={fn.name: fn}, constants={}))


def dump(name, obj):
    path = os.path.join(HERE, name)
    with gzip.open(path, "wt") as f:
        json.dump(obj, f, separators=(",", ":"), sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# ---------------------------------------------------------------------------

def make_opcases(per_op=60):
    cases = []
    for opcode in sorted(OPCODES):
        rng = random.Random(f"unit-{opcode}")
        for i in range(per_op):
            op, operands = opgen.make_case(opcode, rng)
            out = eval_op(op, operands)
            params = tuple((f"%a{k}", tv.type) for k, tv in enumerate(operands))
            fn = FunctionBody(name="t", params=params, ops=[op],
                              returns=(op.result,),
                              return_types=(op.result_type,))
            cases.append({"opcode": opcode, "i": i, "text": fn_text(fn),
                          "operands": [enc(tv.data) for tv in operands],
                          "expected": enc(out.data)})
    dump("opcases.json.gz", {"cases": cases})


# ---------------------------------------------------------------------------

_WORKLOAD = None


def _eval_one(patch):
    return F.evaluate(_WORKLOAD.module, patch, _WORKLOAD)


class RecordingEvaluator(S._Evaluator):
    """_Evaluator with a fork pool (evaluate is pure, search.py:249-273) that
    records every fresh evaluation in call order."""
    log: list = []
    pool = None

    def __call__(self, patches):
        keyed = [(G.patch_dumps(p), p) for p in patches]
        fresh = {}
        for key, p in keyed:
            if key not in self.cache and key not in fresh:
                fresh[key] = p
        items = list(fresh.items())
        if self.pool is not None and len(items) > 1:
            fits = self.pool.map(_eval_one, [p for _, p in items], chunksize=1)
        else:
            fits = [_eval_one(p) for _, p in items]
        call = len({e["call"] for e in self.log})
        for (key, p), fit in zip(items, fits):
            self.cache[key] = fit
            self.log.append({"call": call, "key": key, "patch": p, "fit": fit})
        return [self.cache[k] for k, _ in keyed]


def record_run(workload, cfg, procs):
    global _WORKLOAD
    _WORKLOAD = workload
    RecordingEvaluator.log = []
    orig = S._Evaluator
    S._Evaluator = RecordingEvaluator
    pool = mp.get_context("fork").Pool(procs) if procs > 1 else None
    RecordingEvaluator.pool = pool
    try:
        result = S.run_search(workload, cfg)
    finally:
        S._Evaluator = orig
        if pool is not None:
            pool.close()
            pool.join()
    inds = []
    for e in RecordingEvaluator.log:
        rec = {"call": e["call"], "key": e["key"], "cost": e["fit"].cost,
               "error": e["fit"].error, "valid": e["fit"].valid}
        try:
            variant = G.apply_patch(workload.module, e["patch"]).module
            for name in workload.mutable_functions:
                rec[name] = fn_text(variant.functions[name])
        except G.PatchApplicationError:
            rec["invalid_patch"] = True
        inds.append(rec)
    hist = [{k: v for k, v in h.items()} for h in result.history]
    return inds, hist, result


def make_train_pop(procs):
    w = F.build_2fcnet_workload()
    cfg = S.SearchConfig(population=64, generations=3, elites=16, seed=0)
    inds, hist, result = record_run(w, cfg, procs)
    # holdout goldens for the first archive entries (fitness.py:396-426)
    hold = []
    for e in result.archive[:6]:
        hf = F.holdout_report(w.module, e.patch, w)
        variant = G.apply_patch(w.module, e.patch).module
        hold.append({"key": G.patch_dumps(e.patch), "cost": hf.cost,
                     "error": hf.error,
                     "forward": fn_text(variant.functions["forward"]),
                     "train_step": fn_text(variant.functions["train_step"])})
    # the hand-made §6.2 patch (fitness.py:299-331)
    gp = F.gradient_scaling_patch(w)
    gv = G.apply_patch(w.module, gp).module
    gf = F.evaluate(w.module, gp, w)
    dump("train_pop.json.gz", {
        "config": {"population": 64, "generations": 3, "elites": 16, "seed": 0},
        "individuals": inds, "history": hist, "holdout": hold,
        "gradient_scaling": {"cost": gf.cost, "error": gf.error,
                             "forward": fn_text(gv.functions["forward"]),
                             "train_step": fn_text(gv.functions["train_step"])}})
    return w


def make_predict_pop(procs):
    w = F.build_prediction_workload()
    np.savez(os.path.join(HERE, "predict_weights.npz"),
             **{n: w.module.constants[n].value for n in F.WEIGHT_NAMES})
    cfg = S.SearchConfig(population=64, generations=2, elites=16, seed=0)
    inds, hist, _ = record_run(w, cfg, procs)
    dump("predict_pop.json.gz", {
        "config": {"population": 64, "generations": 2, "elites": 16, "seed": 0},
        "individuals": inds, "history": hist})


def make_bench_pool(procs):
    w = F.build_2fcnet_workload()
    cfg = S.SearchConfig(population=256, generations=10, elites=16, seed=0)
    inds, hist, _ = record_run(w, cfg, procs)
    dump("bench_train_pool.json.gz", {
        "config": {"population": 256, "generations": 10, "elites": 16,
                   "seed": 0},
        "individuals": inds, "history": hist})


# ---------------------------------------------------------------------------

def _ind(c, e):
    return S.Individual((), F.Fitness(c, e))


def make_nsga2():
    sets = []
    rng = random.Random(20260825)
    for _ in range(40):   # test_search.py:20-29 grids with 5% inf cost
        n = rng.randrange(1, 31)
        sets.append([(float("inf") if rng.random() < 0.05 else
                      float(rng.randrange(10)), float(rng.randrange(10)))
                     for _ in range(n)])
    rng = random.Random(4460)
    for _ in range(20):   # C5 (test_acceptance.py:141-160): half grid, half uniform
        pts = []
        for _ in range(100):
            if rng.random() < 0.5:
                pts.append((float(rng.randrange(12)), float(rng.randrange(12))))
            else:
                pts.append((rng.uniform(0, 12), rng.uniform(0, 12)))
        sets.append(pts)
    rng = random.Random(7)
    for n in (256, 512, 1000):  # fitness-like: costs ~1e9, errors k/992, invalid inf
        pts = []
        for _ in range(n):
            if rng.random() < 0.03:
                pts.append((float("inf"), float("inf")))
            else:
                pts.append((float(rng.randrange(5, 11) * 105027900),
                            rng.randrange(0, 993) / 992))
        sets.append(pts)
    out = []
    for pts in sets:
        fronts = S.nondominated_sort(pts)
        crowd = [S.crowding_distance(pts, fr) for fr in fronts]
        pop = [_ind(c, e) for c, e in pts]
        S.rank_population(pop)
        ns = sorted({1, len(pts) // 2, max(1, len(pts) - 1)})
        surv = {}
        for n in ns:
            pool = [_ind(c, e) for c, e in pts]
            chosen = S.select_survivors(pool, n)
            surv[str(n)] = [next(i for i, p in enumerate(pool) if p is s)
                            for s in chosen]
        out.append({
            "points": [[repr(c), repr(e)] for c, e in pts],
            "fronts": fronts,
            "crowding": [[[i, repr(d[i])] for i in fr] for fr, d in zip(fronts, crowd)],
            "rank": [p.rank for p in pop],
            "crowd": [repr(p.crowding) for p in pop],
            "survivors": surv})
    dump("nsga2.json.gz", {"sets": out})


def make_meta(w):
    ds = w.dataset
    meta = {
        "search_x_sha": sha(ds.search.x), "search_labels_sha": sha(ds.search.labels),
        "holdout_x_sha": sha(ds.holdout.x), "holdout_labels_sha": sha(ds.holdout.labels),
        "init_weights_sha": sha(*[w.module.constants[n].value for n in F.WEIGHT_NAMES]),
        "baseline": {}}
    for name, wl in (("train2fc", w), ("predict2fc", F.build_prediction_workload())):
        f = F.evaluate(wl.module, (), wl)
        h = F.holdout_report(wl.module, (), wl)
        meta["baseline"][name] = {"cost": f.cost, "error": f.error,
                                  "holdout_cost": h.cost, "holdout_error": h.error}
    small = F.build_2fcnet_workload(F.WorkloadConfig(
        steps=60, dataset=DatasetConfig(search_n=320, holdout_n=64)))
    f = F.evaluate(small.module, (), small)
    meta["baseline"]["small60"] = {"cost": f.cost, "error": f.error}
    with open(os.path.join(HERE, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


def main():
    procs = min(8, os.cpu_count() or 1)
    what = set(sys.argv[1:]) or {"--core"}
    if "--core" in what or "--all" in what:
        make_opcases()
        make_nsga2()
        w = make_train_pop(procs)
        make_predict_pop(procs)
        make_meta(w)
    if "--bench" in what or "--all" in what:
        make_bench_pool(procs)


if __name__ == "__main__":
    main()
