"""Device fitness evaluator: the reference's evaluate()/holdout_report() for
a whole list of variants in one libgevo call.

Protocol restated from pkg/src/evotir/fitness.py:372-426:
  * invalid patch (apply/verify failure)     -> INVALID_FITNESS (inf, inf)
  * cost = static cost(train_step) * steps   (training)
         = static cost(forward) * batches    (prediction; holdout batches
                                              for holdout_report)
  * non-finite weights at a check step or at the end, or non-finite
    probabilities on any scored batch      -> Fitness(cost, 1.0)
  * otherwise error = wrong / total, divided here in Python so the float
    is the reference's own.
"""
from __future__ import annotations

import time

import numpy as np

from . import _lib
from .plan import build_population_plan, lower_variant
from .workloads import (INVALID_FITNESS, PREDICTION, TRAINING, WEIGHT_NAMES,
                        Fitness, Workload)

SPLIT_SEARCH, SPLIT_HOLDOUT = 0, 1
STATUS_OK, STATUS_NONFINITE_WEIGHTS, STATUS_NONFINITE_PROBS = 0, 1, 2


class DeviceEvaluator:
    """Owns one device context with the workload's splits and weights
    resident; evaluates lists of variant programs.

    `workload` is this package's `Workload` or anything with the same
    attributes (see shims.device_workload for evotir's)."""

    def __init__(self, workload: Workload, device: int = 0):
        self.workload = workload
        self.device = device
        self.ctx = _lib.Context(device)
        cfg = workload.config
        self.batch, self.classes = cfg.batch_size, cfg.classes
        ds = workload.dataset
        self.ctx.upload_split(SPLIT_SEARCH, ds.search.x, ds.search.labels,
                              cfg.classes, cfg.batch_size)
        self.n_search_batches = len(ds.search.labels) // cfg.batch_size
        self._holdout_batches = None
        w = [np.ascontiguousarray(workload.weights[n], dtype=np.float64)
             for n in WEIGHT_NAMES]
        self.weight_shapes = [a.shape for a in w]
        self.ctx.upload_weights(np.concatenate([a.reshape(-1) for a in w]))
        self.weight_elems = int(sum(a.size for a in w))
        self.last_timing = {}
        self.last_plan_bytes = 0

    def _ensure_holdout(self):
        if self._holdout_batches is None:
            ds, cfg = self.workload.dataset, self.workload.config
            ds.holdout.reads += 1      # the only reader of holdout (fitness.py:404)
            self.ctx.upload_split(SPLIT_HOLDOUT, ds.holdout.x, ds.holdout.labels,
                                  cfg.classes, cfg.batch_size)
            self._holdout_batches = len(ds.holdout.labels) // cfg.batch_size
        return self._holdout_batches

    # ------------------------------------------------------------------
    def evaluate_variants(self, variants, holdout=False, want_weights=False,
                          return_records=False):
        """variants: list of {'train_step': fn, 'forward': fn} (or None for
        a patch that failed to apply).  Returns list[Fitness] (and the raw
        device records when return_records)."""
        wl = self.workload
        cfg = wl.config
        training = wl.mode == TRAINING
        t0 = time.perf_counter()
        n_score = self._ensure_holdout() if holdout else self.n_search_batches
        if holdout and n_score == 0:
            from .workloads import WorkloadError
            raise WorkloadError("holdout split smaller than one batch")
        lowered, slots = [], []
        fits = [None] * len(variants)
        for i, fns in enumerate(variants):
            if fns is None:
                fits[i] = INVALID_FITNESS
                continue
            try:
                vp = lower_variant(fns, cfg.cost_table, training=training)
            except Exception:
                fits[i] = INVALID_FITNESS      # evaluate(): any exception
                continue
            lowered.append(vp)
            slots.append(i)
        t1 = time.perf_counter()
        records = np.zeros(len(variants), dtype=_lib.RESULT_DTYPE)
        finals = None
        if lowered:
            plan = build_population_plan(lowered, self.weight_shapes,
                                         self.batch * self.classes)
            t2 = time.perf_counter()
            self.last_plan_bytes = plan.blob.nbytes
            res, fw = self.ctx.eval(
                plan.blob, plan.n_prog,
                0 if training else 1, cfg.steps if training else 0,
                cfg.finite_check_every, SPLIT_SEARCH,
                SPLIT_HOLDOUT if holdout else SPLIT_SEARCH,
                self.weight_elems, want_weights)
            t3 = time.perf_counter()
            if want_weights:
                finals = [None] * len(variants)
            for k, vp in enumerate(lowered):
                i = slots[k]
                r = res[k]
                records[i] = r
                if training:
                    cost = vp.train_cost * cfg.steps
                else:
                    cost = vp.fwd_cost * n_score
                if r["status"] != STATUS_OK:
                    fits[i] = Fitness(cost, 1.0)
                else:
                    fits[i] = Fitness(cost, int(r["wrong"]) / int(r["total"]))
                if want_weights:
                    finals[i] = fw[k]
            self.last_timing = {"lower_s": t1 - t0, "pack_s": t2 - t1,
                                "device_s": t3 - t2, "n": len(lowered)}
        out = [fits]
        if return_records:
            out.append(records)
        if want_weights:
            out.append(finals)
        return out[0] if len(out) == 1 else tuple(out)

    def split_weights(self, flat):
        out, o = {}, 0
        for name, shape in zip(WEIGHT_NAMES, self.weight_shapes):
            n = int(np.prod(shape))
            out[name] = np.array(flat[o:o + n]).reshape(shape)
            o += n
        return out

    # NSGA-II ------------------------------------------------------------
    def nsga2_rank(self, points):
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 2)
        return self.ctx.nsga2_rank(pts[:, 0], pts[:, 1])

    def nsga2_select(self, points, keep):
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 2)
        return self.ctx.nsga2_select(pts[:, 0], pts[:, 1], keep)

    def close(self):
        self.ctx.close()


def baseline_functions(workload: Workload) -> dict:
    m = workload.module
    return {n: m.functions[n] for n in ("forward", "train_step")
            if n in m.functions}


def train_baseline_weights(workload: Workload, device: int = 0) -> dict:
    """Weights after training the unmutated program (fitness.py:265-270),
    on the device."""
    ev = DeviceEvaluator(workload, device)
    try:
        (fit,), _, (flat,) = ev.evaluate_variants(
            [baseline_functions(workload)], want_weights=True,
            return_records=True)
        if fit.error == 1.0 and flat is None:
            raise RuntimeError("baseline training diverged; cannot freeze")
        return ev.split_weights(flat)
    finally:
        ev.close()
