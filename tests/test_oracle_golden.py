"""The oracle reproduces the reference's own recorded outputs (CPU).

Pins oracle/ against tests/golden/* (generated from the real reference by
tests/golden/make_golden.py) so that the GPU parity tests can trust it.
"""
import math

import numpy as np
import pytest

from golden_io import dec, load, predict_weights, variant_functions
from oracle import fitness as OF
from oracle import interp as OI
from oracle import nsga2 as ON
from paper_2310_10211_b200 import dialect
from paper_2310_10211_b200 import workloads as W


@pytest.fixture(scope="module")
def train_wl():
    return W.build_2fcnet_workload()


def test_opcases_match_reference_eval_op():
    cases = load("opcases.json.gz")["cases"]
    assert len(cases) == 1200
    for c in cases:
        fn = dialect.parse_function(c["text"])
        params = [dec(o).reshape(t.shape) for o, (_, t) in zip(c["operands"], fn.params)]
        (got,) = OI.Program(fn)(params)
        exp = dec(c["expected"])
        got = np.asarray(got).reshape(exp.shape)
        assert got.dtype == exp.dtype
        if exp.dtype == np.float64:
            assert np.array_equal(got, exp, equal_nan=True), c["opcode"]
        else:
            assert np.array_equal(got, exp), c["opcode"]


def test_baseline_goldens(train_wl):
    meta = load("meta.json")
    fns = {n: train_wl.module.functions[n] for n in ("forward", "train_step")}
    w0 = [train_wl.weights[n] for n in W.WEIGHT_NAMES]
    search = (train_wl.search_x, train_wl.search_y, train_wl.search_labels)
    r = OF.evaluate_variant(fns, "training", w0, search)
    assert r["cost"] == meta["baseline"]["train2fc"]["cost"] == 1050279000.0
    assert r["error"] == meta["baseline"]["train2fc"]["error"]
    assert (r["wrong"], r["total"]) == (104, 992)


@pytest.mark.parametrize("start", [0, 40, 80, 120, 160])
def test_train_population_fitness_bit_exact(train_wl, start):
    pop = load("train_pop.json.gz")["individuals"]
    w0 = [train_wl.weights[n] for n in W.WEIGHT_NAMES]
    search = (train_wl.search_x, train_wl.search_y, train_wl.search_labels)
    for ind in pop[start:start + 8]:
        fns = variant_functions(ind)
        r = OF.evaluate_variant(fns, "training", w0, search)
        assert r["cost"] == ind["cost"]
        assert r["error"] == ind["error"]


def test_predict_population_fitness_bit_exact():
    pop = load("predict_pop.json.gz")["individuals"]
    wl = W.build_prediction_workload(weights=predict_weights())
    w = [wl.weights[n] for n in W.WEIGHT_NAMES]
    search = (wl.search_x, wl.search_y, wl.search_labels)
    for ind in pop[:40]:
        fns = variant_functions(ind, ("forward",))
        r = OF.evaluate_variant(fns, "prediction", w, search)
        assert r["cost"] == ind["cost"] and r["error"] == ind["error"]


def _pts(s):
    return [(float(c), float(e)) for c, e in s["points"]]


def test_nsga2_oracle_matches_reference():
    for s in load("nsga2.json.gz")["sets"]:
        pts = _pts(s)
        assert ON.fronts_of(pts) == s["fronts"]
        for fr, cr in zip(s["fronts"], s["crowding"]):
            d = ON.crowding(pts, fr)
            for i, v in cr:
                assert d[i] == float(v) or (math.isnan(d[i]) and math.isnan(float(v)))
        rank, crowd = ON.rank_and_crowd(pts)
        assert rank == s["rank"]
        assert [repr(x) for x in crowd] == s["crowd"]
        for n, chosen in s["survivors"].items():
            assert ON.survivors(pts, int(n)) == chosen
