"""Device parity against the oracle and the reference's recorded outputs.

All through the C ABI (libgevo.so) on cuda:0.  Tolerances:
  * per-op (opgen cases, interpreter.py:78-185): float64 within
    1e-12 * max(1, |e|) (the reference's own test uses 1e-6,
    test_interpreter.py:19-29), ints/bools exact; bit-exact rate reported
  * one train_step from the init weights: float64 within 1e-12 relative
  * cost: bit-identical for every individual
  * status (blow-up -> error 1.0): identical for every individual
  * error: bit-identical for every individual (the device reproduces the
    reference's summation orders); any drift is printed
    before the assertion fails
  * NSGA-II: bit-identical ranks, fronts, crowding, survivor order
"""
import math

import numpy as np
import pytest

from golden_io import dec, load, predict_weights, variant_functions
from oracle import interp as OI
from paper_2310_10211_b200 import _lib, dialect
from paper_2310_10211_b200 import workloads as W
from paper_2310_10211_b200.evaluator import DeviceEvaluator
from paper_2310_10211_b200.plan import exec_once_plan

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = _lib.Context(0)
    yield c
    c.close()


def _words(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.bool_:
        a = a.astype(np.int64)
    if a.dtype != np.float64:
        return a.reshape(-1).astype(np.int64).view(np.float64)
    return a.reshape(-1)


def run_once(ctx, fns, params_list):
    blob, pblob, meta, total = exec_once_plan(fns, params_list)
    outs = ctx.exec_once(blob, pblob, total)
    res = []
    for fn, metas in zip(fns, meta):
        got = []
        for off, shape, kind in metas:
            n = max(1, int(np.prod(shape)))
            w = outs[off:off + n]
            if kind == "f32":
                got.append(w.reshape(shape))
            elif kind == "i32":
                got.append(w.view(np.int64).reshape(shape))
            else:
                got.append((w.view(np.int64) != 0).reshape(shape))
        res.append(got)
    return res


def test_device_present(ctx):
    info = ctx.device_info()
    print(info)
    assert "sm_10" in info


def test_every_opcode_matches_reference_eval_op(ctx):
    cases = load("opcases.json.gz")["cases"]
    fns, params = [], []
    for c in cases:
        fn = dialect.parse_function(c["text"])
        fns.append(fn)
        params.append([_words(dec(o)) for o in c["operands"]])
    outs = run_once(ctx, fns, params)
    exact = 0
    for c, (got,) in zip(cases, outs):
        exp = dec(c["expected"])
        got = np.asarray(got).reshape(exp.shape)
        if exp.dtype == np.float64:
            ok = np.array_equal(np.isnan(got), np.isnan(exp)) and np.all(
                np.abs(np.nan_to_num(got - exp, nan=0.0, posinf=0, neginf=0))
                <= 1e-12 * np.maximum(1.0, np.abs(np.nan_to_num(exp))))
            ok = ok and np.array_equal(np.isinf(got), np.isinf(exp))
            exact += np.array_equal(got, exp, equal_nan=True)
        else:
            ok = np.array_equal(got.astype(exp.dtype), exp)
            exact += ok
        assert ok, (c["opcode"], c["i"], c["text"], got, exp)
    print(f"opcases bit-exact {exact}/{len(cases)}")


@pytest.fixture(scope="module")
def train_wl():
    return W.build_2fcnet_workload()


def test_one_train_step_matches_oracle(ctx, train_wl):
    pop = load("train_pop.json.gz")["individuals"]
    w0 = [train_wl.weights[n] for n in W.WEIGHT_NAMES]
    args = w0 + [train_wl.search_x[0], train_wl.search_y[0]]
    fns = [dialect.parse_function(i["train_step"]) for i in pop]
    outs = run_once(ctx, fns, [[_words(a) for a in args]] * len(fns))
    exact = 0
    for fn, got in zip(fns, outs):
        ref = OI.Program(fn)(args)
        same = True
        for g, r in zip(got, ref):
            r = np.asarray(r, dtype=np.float64)
            assert np.allclose(g, r, rtol=1e-12, atol=1e-15, equal_nan=True)
            same &= np.array_equal(g, r, equal_nan=True)
        exact += same
    print(f"one-step bit-exact {exact}/{len(fns)}")


def _drift(fits, inds):
    d = [abs(f.error - i["error"]) * 992 for f, i in zip(fits, inds)
         if f.error != i["error"]]
    return sorted(round(x) for x in d)


def test_train_population_fitness(train_wl):
    data = load("train_pop.json.gz")
    inds = data["individuals"]
    ev = DeviceEvaluator(train_wl)
    fits = ev.evaluate_variants([variant_functions(i) for i in inds])
    ev.close()
    exact = 0
    for f, i in zip(fits, inds):
        assert f.cost == i["cost"]
        assert (f.error == 1.0) == (i["error"] == 1.0)
        exact += f.error == i["error"]
    print(f"train2fc error bit-exact {exact}/{len(inds)}; drift (examples) {_drift(fits, inds)}")
    assert exact == len(inds)


def test_bench_pool_fitness_at_full_size():
    """Every fresh individual of the recorded pop-256 x 10-generation run
    (the bench pool, BASELINE.json configs[1]) at the full default workload
    -- 600 steps, 31 scored batches -- against the fitness the reference
    recorded for it (tests/golden/make_golden.py --bench)."""
    from paper_2310_10211_b200.dialect import parse_function
    inds = [i for i in load("bench_train_pool.json.gz")["individuals"] if not i.get("invalid_patch")]
    seen, pool = set(), []
    for i in inds:
        if i["key"] not in seen:
            seen.add(i["key"])
            pool.append(i)
    wl = W.build_2fcnet_workload()
    ev = DeviceEvaluator(wl)
    variants = [{k: parse_function(i[k]) for k in ("forward", "train_step")} for i in pool]
    fits = []
    for c in range(0, len(variants), 512):
        fits += ev.evaluate_variants(variants[c:c + 512])
    ev.close()
    exact, off = 0, []
    for k, (f, i) in enumerate(zip(fits, pool)):
        assert f.cost == i["cost"]
        assert (f.error == 1.0) == (i["error"] == 1.0)
        exact += f.error == i["error"]
        if f.error != i["error"]:
            off.append((k, f.error, i["error"]))
    print(f"bench pool (full size) error bit-exact {exact}/{len(pool)}; differing {off}")
    assert exact == len(pool)


def test_baseline_and_gradient_patch(train_wl):
    meta = load("meta.json")["baseline"]["train2fc"]
    g = load("train_pop.json.gz")["gradient_scaling"]
    ev = DeviceEvaluator(train_wl)
    base = {n: train_wl.module.functions[n] for n in ("forward", "train_step")}
    fits, rec = ev.evaluate_variants([base, variant_functions(g)], return_records=True)
    hold = ev.evaluate_variants([base], holdout=True)
    ev.close()
    assert fits[0].cost == meta["cost"] and fits[1].cost == g["cost"]
    print("baseline", fits[0], rec[0], "gradient patch", fits[1], "holdout", hold[0])
    assert fits[0].error == meta["error"]          # 104/992
    assert hold[0].error == meta["holdout_error"]  # 47/256
    assert fits[1].error == g["error"]


def test_predict_population_fitness():
    data = load("predict_pop.json.gz")
    inds = data["individuals"]
    wl = W.build_prediction_workload(weights=predict_weights())
    ev = DeviceEvaluator(wl)
    fits = ev.evaluate_variants([variant_functions(i, ("forward",)) for i in inds])
    ev.close()
    exact = sum(f.error == i["error"] and f.cost == i["cost"] for f, i in zip(fits, inds))
    for f, i in zip(fits, inds):
        assert f.cost == i["cost"]
    print(f"predict2fc bit-exact {exact}/{len(inds)}")
    assert exact == len(inds)


def test_prediction_score_parts_identical_records(monkeypatch):
    """Score parts (several CTAs per prediction individual, each scoring every
    n-th batch, merged in gevo_eval) give the records of one CTA per
    individual, bit for bit; both match the reference's fitness."""
    inds = load("predict_pop.json.gz")["individuals"][:24]
    wl = W.build_prediction_workload(weights=predict_weights())
    fns = [variant_functions(i, ("forward",)) for i in inds]
    out = {}
    for parts in ("1", "7", "31"):
        monkeypatch.setenv("GEVO_B200_PARTS", parts)
        ev = DeviceEvaluator(wl)
        fits, rec = ev.evaluate_variants(fns, return_records=True)
        ev.close()
        out[parts] = (fits, [rec[k].tolist() for k in ("wrong", "total", "status")])
    for parts in ("7", "31"):
        assert out[parts][0] == out["1"][0]
        assert out[parts][1] == out["1"][1]
    exact = sum(f.error == i["error"] and f.cost == i["cost"] for f, i in zip(out["7"][0], inds))
    print(f"score parts 1/7/31 identical; bit-exact vs reference {exact}/{len(inds)}")
    assert exact == len(inds)


def test_score_part_plans_are_validated():
    """gevo_eval refuses plans whose score parts are inconsistent: a missing or
    duplicated part, a part index out of range, or parts in a training
    launch (no kernel runs; GevoError carries the reason)."""
    from paper_2310_10211_b200 import _lib
    from paper_2310_10211_b200.evaluator import lower_all
    from paper_2310_10211_b200.lowering import HEADER_DTYPE, INSTR_DTYPE, PROG_DTYPE
    from paper_2310_10211_b200.plan import FLAG_NPARTS_SHIFT, FLAG_PART_SHIFT, build_population_plan
    inds = load("predict_pop.json.gz")["individuals"][:3]
    wl = W.build_prediction_workload(weights=predict_weights())
    ev = DeviceEvaluator(wl)
    vps = lower_all([variant_functions(i, ("forward",)) for i in inds], None, False, 0)
    plan = build_population_plan(vps, ev.weight_shapes, ev.batch * ev.classes, parts=2)
    hdr = plan.blob[:HEADER_DTYPE.itemsize].view(HEADER_DTYPE)[0]
    o = HEADER_DTYPE.itemsize + int(hdr["n_instr"]) * INSTR_DTYPE.itemsize

    def run(blob, mode=1):
        return ev.ctx.eval(blob, plan.n_prog, mode, 0 if mode else 600, 50, 0, 0, ev.weight_elems, False)
    res, _ = run(plan.blob)                                   # the valid plan runs
    assert ((res["total"][:3] == 32 * 31) | (res["status"][:3] != 0)).all()

    def corrupt(fn):
        blob = plan.blob.copy()
        progs = blob[o:o + plan.n_prog * PROG_DTYPE.itemsize].view(PROG_DTYPE)
        fn(progs)
        return blob
    cases = {
        "duplicate": lambda p: p.__setitem__("flags", np.where(
            np.arange(len(p)) == 3, p["flags"] & ~(0xFFF << FLAG_PART_SHIFT), p["flags"])),
        "part out of range": lambda p: p.__setitem__("flags", p["flags"] | (5 << FLAG_PART_SHIFT)),
        "inconsistent": lambda p: p.__setitem__("flags", np.where(
            np.arange(len(p)) == 0, (p["flags"] & ~(0x7FF << FLAG_NPARTS_SHIFT)) | (3 << FLAG_NPARTS_SHIFT),
            p["flags"])),
        "slot out of range": lambda p: p.__setitem__("result_slot", np.where(
            np.arange(len(p)) == 1, 99, p["result_slot"])),
    }
    for name, fn in cases.items():
        with pytest.raises(_lib.GevoError):
            run(corrupt(fn))
    with pytest.raises(_lib.GevoError):
        run(plan.blob, mode=0)                                 # parts in a training launch
    ev.close()


def test_holdout_reports(train_wl):
    hold = load("train_pop.json.gz")["holdout"]
    ev = DeviceEvaluator(train_wl)
    fits = ev.evaluate_variants([variant_functions(h) for h in hold], holdout=True)
    ev.close()
    exact = sum(f.error == h["error"] for f, h in zip(fits, hold))
    for f, h in zip(fits, hold):
        assert f.cost == h["cost"]
    print(f"holdout bit-exact {exact}/{len(hold)}")
    assert exact == len(hold)


def test_nsga2_bit_exact(ctx):
    for s in load("nsga2.json.gz")["sets"]:
        pts = np.array([[float(c), float(e)] for c, e in s["points"]])
        rank, crowd, order, fstart = ctx.nsga2_rank(pts[:, 0], pts[:, 1])
        fronts = [order[fstart[k]:fstart[k + 1]].tolist() for k in range(len(fstart) - 1)]
        assert fronts == s["fronts"]
        assert rank.tolist() == s["rank"]
        assert [repr(float(x)) for x in crowd] == s["crowd"]
        for n, chosen in s["survivors"].items():
            got, _, _ = ctx.nsga2_select(pts[:, 0], pts[:, 1], int(n))
            assert got.tolist() == chosen


def test_device_exp_is_numpy_exp(ctx):
    """`exponential` on the device equals the host model of numpy's SVML
    exp (tests/test_exp_model.py pins that model to np.exp) bit-for-bit."""
    from tools.exp_model import exp_model
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.uniform(-40, 0, 4000), rng.uniform(-700, 700, 4000),
                        rng.uniform(-1e-15, 1e-15, 1000),
                        [0.0, -0.0, np.inf, -np.inf, 709.78, 709.79, -745.2, -800.0]])
    n = x.size
    fn = dialect.parse_function(
        f"func @t(%a: tensor<{n}xf32>) -> tensor<{n}xf32> {{\n"
        f"  %e = exponential %a : tensor<{n}xf32>\n  return %e : tensor<{n}xf32>\n}}\n")
    (got,), = run_once(ctx, [fn], [[x]])
    with np.errstate(all="ignore"):
        want = exp_model(x)
    assert np.array_equal(got, want), np.nonzero(got != want)[0][:10]
