"""Fitness protocol restated on the numpy oracle (test infrastructure).

Follows pkg/src/evotir/fitness.py:
  * _run_training      fitness.py:338-352  (600 steps, batch step % nb,
                       isfinite over returned weights at (s+1) % check == 0
                       and once at the end, early exit -> None)
  * _misclassification fitness.py:355-369  (any non-finite probs -> 1.0,
                       first-max argmax, wrong/total)
  * evaluate           fitness.py:372-393  (cost = static cost * steps or
                       * batches; blow-up keeps the cost, error 1.0)
Returns the integer record the device evaluator produces as well
(wrong, total, status) so tests can compare below the float.
"""
from __future__ import annotations

import numpy as np

from .interp import Program, function_cost

OK, NONFINITE_WEIGHTS, NONFINITE_PROBS = 0, 1, 2


def run_training(train_fn, weights, xs, ys, steps, check_every, perturb=False):
    prog = Program(train_fn, perturb)
    w = list(weights)
    nb = len(xs)
    check = max(1, check_every)
    for s in range(steps):
        w = prog(w + [xs[s % nb], ys[s % nb]])
        if (s + 1) % check == 0 and not all(np.all(np.isfinite(a)) for a in w):
            return None
    if not all(np.all(np.isfinite(a)) for a in w):
        return None
    return w


def misclassified(fwd_fn, weights, xs, labels, perturb=False):
    """(wrong, total, status)."""
    prog = Program(fwd_fn, perturb)
    wrong = total = 0
    for xb, lb in zip(xs, labels):
        (probs,) = prog(list(weights) + [xb])
        if not np.all(np.isfinite(probs)):
            return 0, 0, NONFINITE_PROBS
        wrong += int(np.sum(np.argmax(probs, axis=1) != lb))
        total += len(lb)
    return wrong, total, OK


def evaluate_variant(fns, mode, weights, search, steps=600, check_every=50,
                     cost_table=None, score=None, perturb=False):
    """fns: {'forward': fn, 'train_step': fn}; weights: [w1, b1, w2, b2];
    search: (x [nb,B,F], y [nb,B,C], labels [nb,B]); score: optional
    (x, labels) split to score on instead (holdout_report, fitness.py:396-426).
    Returns dict(cost, error, wrong, total, status)."""
    xs, ys, lbs = search
    sx, slb = score if score is not None else (xs, lbs)
    if mode == "training":
        cost = function_cost(fns["train_step"], cost_table) * steps
        final = run_training(fns["train_step"], weights, xs, ys, steps,
                             check_every, perturb)
        if final is None:
            return dict(cost=cost, error=1.0, wrong=0, total=0,
                        status=NONFINITE_WEIGHTS)
    else:
        cost = function_cost(fns["forward"], cost_table) * len(sx)
        final = list(weights)
    wrong, total, status = misclassified(fns["forward"], final, sx, slb, perturb)
    error = 1.0 if status != OK else wrong / total
    return dict(cost=cost, error=error, wrong=wrong, total=total, status=status)
