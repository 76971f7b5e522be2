"""Record a whole GEVO-ML run with the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
    python tests/golden/make_ga_golden.py [population] [generations]

BASELINE.json configs[3]: the train2fc workload, population 512, 50
generations, NSGA-II selection (defaults 512 / 50).  The reference's
run_search (search.py:333-399) runs unchanged, with seed 0, elites 16 and
the other SearchConfig defaults.  Two hooks only observe it:
  * _Evaluator is the reference's own (dedup by patch_dumps key, cache),
    with the fresh evaluations fanned out over a fork pool (evaluate is
    pure, search.py:249-273; results identical to serial);
  * select_survivors is wrapped to log each generation's survivors.

Recorded (tests/golden/ga<pop>x<gens>.json.gz):
  * individuals: every distinct patch evaluated -- reference Fitness,
    variant program text (printer.py of apply_patch(...).module);
  * calls: each evaluator call's full patch list (individual indices, in
    order, duplicates and cache hits included);
  * survivors: per generation, the survivor indices in order plus their
    rank and crowding (repr);
  * history (search.py:354-368), the final archive (sorted_entries) and
    its holdout reports (search.py:390-391);
  * wall times: the whole run, and the part spent inside evaluator calls.
    Their difference is the host work that stays the reference's
    (variation, smoke checks, selection, archive).
"""
from __future__ import annotations

import os
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import gzip
import json
import multiprocessing as mp
import sys
import time

from evotir import fitness as F
from evotir import genome as G
from evotir import search as S
from evotir.ir import Module
from evotir.printer import print_module

HERE = os.path.dirname(os.path.abspath(__file__))
_W = None


def fn_text(fn) -> str:
    return print_module(Module(functions={fn.name: fn}, constants={}))


def _eval_one(patch):
    return F.evaluate(_W.module, patch, _W)


class Recorder(S._Evaluator):
    pool = None
    index: dict = {}
    table: list = []
    calls: list = []
    eval_s = 0.0

    def __call__(self, patches):
        t0 = time.perf_counter()
        keyed = [(G.patch_dumps(p), p) for p in patches]
        fresh = {}
        for key, p in keyed:
            if key not in self.cache and key not in fresh:
                fresh[key] = p
        items = list(fresh.items())
        if self.pool is not None and len(items) > 1:
            fits = self.pool.map(_eval_one, [p for _, p in items], chunksize=4)
        else:
            fits = [_eval_one(p) for _, p in items]
        for (key, p), fit in zip(items, fits):
            self.cache[key] = fit
            Recorder.index[key] = len(Recorder.table)
            Recorder.table.append((key, p, fit, len(Recorder.calls)))
        Recorder.calls.append([Recorder.index[k] for k, _ in keyed])
        Recorder.eval_s += time.perf_counter() - t0
        return [self.cache[k] for k, _ in keyed]


def main():
    global _W
    pop = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    gens = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    procs = min(16, os.cpu_count() or 1)
    _W = w = F.build_2fcnet_workload()
    cfg = S.SearchConfig(population=pop, generations=gens, elites=16, seed=0)
    survivors = []
    orig_sel, orig_eval = S.select_survivors, S._Evaluator

    def logged_select(pool, n):
        chosen = orig_sel(pool, n)
        survivors.append([[Recorder.index[G.patch_dumps(i.patch)], i.rank, repr(i.crowding)]
                          for i in chosen])
        return chosen

    Recorder.pool = mp.get_context("fork").Pool(procs)
    S.select_survivors, S._Evaluator = logged_select, Recorder
    t0 = time.perf_counter()
    try:
        result = S.run_search(w, cfg)
    finally:
        S.select_survivors, S._Evaluator = orig_sel, orig_eval
        Recorder.pool.close()
        Recorder.pool.join()
    wall = time.perf_counter() - t0
    inds = []
    for key, patch, fit, call in Recorder.table:
        rec = {"call": call, "cost": fit.cost, "error": fit.error, "valid": fit.valid,
               "edits": len(patch)}
        try:
            variant = G.apply_patch(w.module, patch).module
            for name in w.mutable_functions:
                rec[name] = fn_text(variant.functions[name])
        except G.PatchApplicationError:
            rec["invalid_patch"] = True
        inds.append(rec)
    out = {
        "config": {"population": pop, "generations": gens, "elites": 16, "seed": 0},
        "individuals": inds,
        "calls": Recorder.calls,
        "survivors": survivors,
        "history": [dict(h) for h in result.history],
        "archive": [Recorder.index[G.patch_dumps(e.patch)] for e in result.archive],
        # holdout_report of every archive entry (search.py:390-391)
        "archive_holdout": [[e.holdout.cost, e.holdout.error, e.holdout.valid]
                            for e in result.archive],
        "evaluations": result.evaluations,
        "timing": {"wall_s": wall, "evaluator_s": Recorder.eval_s, "procs": procs,
                   "host_s": wall - Recorder.eval_s},
    }
    path = os.path.join(HERE, f"ga{pop}x{gens}.json.gz")
    with gzip.open(path, "wt") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes): {len(inds)} individuals, "
          f"wall {wall:.1f} s, evaluator {Recorder.eval_s:.1f} s on {procs} procs")


if __name__ == "__main__":
    main()
