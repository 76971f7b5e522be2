"""The reduced-precision modes (GEVO_B200_DTYPE=tf32 | bf16): every f64 DOT
on the tcgen05 tensor cores (csrc/dot_tc.cuh), tf32 (kind::tf32) or bf16
(kind::f16) operands, fp32 accumulation, everything else float64.  Not parity
modes: the bars are the tolerances SURVEY.md §8(c) states (tf32 2e-3, bf16
2e-2), and the fitness exact-match rate against the reference is reported.

Tolerances (tf32 rounds each operand to 10 mantissa bits, 2^-11 relative;
the product of two such operands is within 2^-10 of the exact product, and
the fp32 sum adds K * 2^-24):
  * one dot: |got - exact| <= 2e-3 * sum_k |a_ik b_kj| + 1e-300
  * one train_step from the init weights: every returned array within
    2e-3 normwise relative error (max |got - ref| / max |ref|; SURVEY.md
    §8(c) rule 4) of the float64 oracle, finiteness identical -- except
    ill-conditioned individuals (<= 2 %), which must instead be within 2e-3
    of the tf32 model of the step
  * full evaluation (600 steps + 31 scored batches): cost identical;
    exact-match rate of the error against the recorded reference printed
bf16 (8 mantissa bits, 2^-9 relative per operand, products within 2^-8):
the same tests with 1e-2 * sum_k |a_ik b_kj| per dot and 2e-2 normwise per
train_step (SURVEY.md §8(c) rule 4), ill-conditioned individuals checked
against the bf16 model (operands rounded to nearest even at 8 bits).
"""
import os

import numpy as np
import pytest

from golden_io import dec, load, variant_functions
from oracle import interp as OI
from paper_2310_10211_b200 import _lib, dialect
from paper_2310_10211_b200 import workloads as W
from paper_2310_10211_b200.evaluator import DeviceEvaluator

pytestmark = pytest.mark.gpu


# mode -> (per-dot bound factor, train_step normwise bar)
BARS = {"tf32": (2e-3, 2e-3), "bf16": (1e-2, 2e-2)}


@pytest.fixture(params=sorted(BARS))
def tf32(monkeypatch, request):
    monkeypatch.setenv("GEVO_B200_DTYPE", request.param)
    yield request.param


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


def test_tf32_dot_within_bound(ctx, tf32):
    """Every f64 dot opcase (all view kinds: C, transposed, broadcast) and the
    workloads' shapes, through gevo_exec_once on tcgen05."""
    from test_gpu_parity import run_once
    cases = [c for c in load("opcases.json.gz")["cases"] if c["opcode"] == "dot"]
    rng = np.random.default_rng(5)
    extra = []
    for m, k, n in ((32, 784, 32), (784, 32, 32), (32, 32, 10), (32, 10, 32), (300, 97, 130), (1, 40, 3)):
        a, b = rng.standard_normal((m, k)), rng.standard_normal((k, n))
        text = (f"func @f(%a: tensor<{m}x{k}xf32>, %b: tensor<{k}x{n}xf32>) -> tensor<{m}x{n}xf32> {{\n"
                f"  %0 = dot %a, %b : tensor<{m}x{n}xf32>\n  return %0 : tensor<{m}x{n}xf32>\n}}")
        extra.append((text, [a, b]))
    fns, params, ops = [], [], []
    for c in cases:
        fns.append(dialect.parse_function(c["text"]))
        ops.append([dec(o) for o in c["operands"]])
        params.append([_words(o) for o in ops[-1]])
    for text, (a, b) in extra:
        fns.append(dialect.parse_function(text))
        ops.append([a, b])
        params.append([_words(a), _words(b)])
    outs = run_once(ctx, fns, params)
    fac = BARS[tf32][0]
    worst = 0.0
    for fn, (got,), (a, b) in zip(fns, outs, ops):
        a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
        if a.dtype.kind != "f" or fn.return_types[0].kind != fn.params[0][1].kind:
            continue
        exact = a @ b
        bound = fac * (np.abs(a) @ np.abs(b)) + 1e-300
        err = np.abs(np.asarray(got).reshape(exact.shape) - exact)
        assert np.all(err <= bound), (fn.params, float((err / bound).max()))
        worst = max(worst, float((err / bound).max()))
    print(f"{tf32} dots: {len(fns)} cases within {fac:g} * sum|a||b| (worst {worst:.3f} of the bound)")


def test_tf32_one_train_step(ctx, tf32):
    from test_gpu_parity import run_once
    wl = W.build_2fcnet_workload()
    pop = load("train_pop.json.gz")["individuals"]
    w0 = [wl.weights[n] for n in W.WEIGHT_NAMES]
    args = w0 + [wl.search_x[0], wl.search_y[0]]
    fns = [dialect.parse_function(i["train_step"]) for i in pop]
    outs = run_once(ctx, fns, [[_words(a) for a in args]] * len(fns))
    bar = BARS[tf32][1]
    rel, bad, model_checked = 0.0, [], []
    for j, (fn, got) in enumerate(zip(fns, outs)):
        ref = OI.Program(fn)(args)
        for r_i, (g, r) in enumerate(zip(got, ref)):
            r = np.asarray(r, dtype=np.float64)
            g = np.asarray(g, dtype=np.float64).reshape(r.shape)
            fin = np.isfinite(r)
            assert np.array_equal(fin, np.isfinite(g)), (j, r_i)
            if not fin.any():
                continue
            # normwise: max |g - r| over max |r| of the returned array
            e = float(np.max(np.abs(g[fin] - r[fin])) / max(np.max(np.abs(r[fin])), 1e-300))
            rel = max(rel, e)
            if e > bar:
                bad.append((j, r_i, e))
    # An individual past the bar is ill-conditioned (e.g. a mutant dividing by
    # the logits): the tf32 rounding itself is amplified.  Then the device must
    # follow the tf32 model of the same step (oracle with tf32-rounded dot
    # operands) to the same 2e-3 normwise, and at most 2 % of the population
    # may be such individuals.
    for j in sorted({b[0] for b in bad}):
        model = _tc_model(fns[j], tf32)(args)
        for g, r in zip(outs[j], model):
            r = np.asarray(r, dtype=np.float64)
            g = np.asarray(g, dtype=np.float64).reshape(r.shape)
            fin = np.isfinite(r)
            e = float(np.max(np.abs(g[fin] - r[fin])) / max(np.max(np.abs(r[fin])), 1e-300))
            assert e <= bar, (j, e)
            model_checked.append(e)
    print(f"{tf32} one train_step: {len(fns)} individuals, max normwise relative error {rel:.2e}; "
          f"over {bar:g} (ill-conditioned, checked against the {tf32} model: max "
          f"{max(model_checked, default=0):.1e}): {bad[:8]}")
    assert len({b[0] for b in bad}) <= max(1, len(fns) // 50)


def _tc_model(fn, mode):
    """The oracle with every f64 dot's operands rounded to tf32 (round to
    nearest, ties away: cvt.rna) or bf16 (round to nearest even: cvt.rn)
    after the f64 -> f32 conversion, and the product rounded to fp32."""
    def rna(x):
        u = np.asarray(x, dtype=np.float64).astype(np.float32).view(np.uint32).astype(np.uint64)
        if mode == "bf16":
            u = ((u + 0x7FFF + ((u >> np.uint64(16)) & np.uint64(1))) & ~np.uint64(0xFFFF)).astype(np.uint32)
        else:
            u = ((u + 0x1000) & ~np.uint64(0x1FFF)).astype(np.uint32)
        return u.view(np.float32).astype(np.float64)
    prog = OI.Program(fn)
    orig = OI.apply_op

    def run(args):
        def hook(op, ins, tys, perturb=False):
            if op.opcode == "dot" and np.asarray(ins[0]).dtype.kind == "f":
                return (rna(ins[0]) @ rna(ins[1])).astype(np.float32).astype(np.float64)
            return orig(op, ins, tys, perturb)
        OI.apply_op = hook
        try:
            return prog(args)
        finally:
            OI.apply_op = orig
    return run


def test_tf32_population_fitness(tf32):
    """Whole evaluations in tf32 mode: static cost identical (it is the
    reference CostModel, independent of arithmetic); the error's exact-match
    rate and drift against the recorded float64 reference are reported."""
    wl = W.build_2fcnet_workload()
    inds = load("train_pop.json.gz")["individuals"]
    ev = DeviceEvaluator(wl)
    fits = ev.evaluate_variants([variant_functions(i) for i in inds])
    ev.close()
    exact, drift = 0, []
    for f, i in zip(fits, inds):
        assert f.cost == i["cost"]
        exact += f.error == i["error"]
        if f.error != i["error"]:
            drift.append(round(abs(f.error - i["error"]) * 992))
    print(f"{tf32} train2fc error exact {exact}/{len(inds)}; drift in examples {sorted(drift)[:20]}")
    if tf32 == "tf32":
        assert exact >= len(inds) // 2
