"""Host lowering: cost identity, layout model, and the instruction tables
walked on CPU by tests/tools/plan_emu.py (no GPU needed)."""
import numpy as np
import pytest

from golden_io import dec, load, variant_functions
from oracle import interp as OI
from paper_2310_10211_b200 import dialect, layout as L, lowering as Lw
from paper_2310_10211_b200 import workloads as W
from paper_2310_10211_b200.plan import (build_population_plan, exec_once_plan,
                                        lower_variant)
from tools import plan_emu


def _words(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.bool_:
        a = a.astype(np.int64)
    if a.dtype == np.float64:
        return a.reshape(-1).view(np.int64).copy()
    return a.reshape(-1).astype(np.int64)


def emulate(fn, params, param_layouts=None):
    low = Lw.lower_function(fn, param_layouts, ret_layout="c")
    consts = Lw.consts_to_words(low.consts).view(np.int64).copy() if low.consts \
        else np.zeros(1, dtype=np.int64)
    mem = {Lw.BUF_ARENA: np.zeros(max(low.arena_elems, 1), dtype=np.int64),
           Lw.BUF_CONST: consts,
           Lw.BUF_SMEM: np.zeros(max(low.smem_elems, 1), dtype=np.int64)}
    for k, p in enumerate(params):
        mem[Lw.BUF_PARAM0 + k] = _words(p)
    for r, ty in enumerate(fn.return_types):
        mem[Lw.BUF_OUT0 + r] = np.zeros(max(1, int(np.prod(ty.shape))), dtype=np.int64)
    plan_emu.run(low.instrs, mem)
    outs = []
    for r, ty in enumerate(fn.return_types):
        w = mem[Lw.BUF_OUT0 + r][:max(1, int(np.prod(ty.shape)))]
        k = dialect.kind_name(ty.kind)
        arr = w.view(np.float64) if k == "f32" else (w != 0 if k == "i1" else w)
        outs.append(arr.reshape(ty.shape))
    return outs, low


def test_static_cost_is_reference_cost():
    pop = load("train_pop.json.gz")["individuals"]
    for ind in pop:
        fns = variant_functions(ind)
        assert Lw.static_cost(fns["train_step"]) * 600 == ind["cost"]
        vp = lower_variant(fns)
        assert vp.train_cost * 600 == ind["cost"]
    for ind in load("predict_pop.json.gz")["individuals"]:
        fns = variant_functions(ind, ("forward",))
        assert Lw.static_cost(fns["forward"]) * 31 == ind["cost"]


def test_every_opcase_lowers_and_emulates():
    for c in load("opcases.json.gz")["cases"]:
        fn = dialect.parse_function(c["text"])
        params = [dec(o).reshape(t.shape) for o, (_, t) in zip(c["operands"], fn.params)]
        (got,), _ = emulate(fn, params)
        exp = dec(c["expected"])
        got = np.asarray(got).reshape(exp.shape)
        if exp.dtype == np.float64:
            assert np.allclose(got, exp, rtol=1e-12, atol=1e-12, equal_nan=True), c["text"]
        else:
            assert np.array_equal(got.astype(exp.dtype), exp), c["text"]


def test_train_step_tables_emulate_one_step():
    wl = W.build_2fcnet_workload()
    w0 = [wl.weights[n] for n in W.WEIGHT_NAMES]
    args = w0 + [wl.search_x[0], wl.search_y[0]]
    for ind in load("train_pop.json.gz")["individuals"]:
        fn = dialect.parse_function(ind["train_step"])
        ref = OI.Program(fn)(args)
        got, _ = emulate(fn, args)
        for a, b in zip(got, ref):
            assert np.allclose(a, np.asarray(b), rtol=1e-11, atol=1e-13, equal_nan=True)


def test_population_plan_packs():
    pop = load("train_pop.json.gz")["individuals"][:20]
    vps = [lower_variant(variant_functions(i)) for i in pop]
    plan = build_population_plan(vps, [(784, 32), (32,), (32, 10), (10,)], 320)
    hdr = plan.blob[:Lw.HEADER_DTYPE.itemsize].view(Lw.HEADER_DTYPE)[0]
    assert hdr["magic"] == Lw.PLAN_MAGIC and hdr["n_prog"] == 20
    assert hdr["weight_elems"] == 784 * 32 + 32 + 320 + 10
    n_instr = hdr["n_instr"]
    expect = (Lw.HEADER_DTYPE.itemsize + n_instr * Lw.INSTR_DTYPE.itemsize +
              20 * Lw.PROG_DTYPE.itemsize + hdr["n_const"] * 8)
    assert plan.blob.nbytes == expect
    # longest static cost first
    costs = [vps[i].train_cost + vps[i].fwd_cost for i in plan.order]
    assert costs == sorted(costs, reverse=True)


def test_exec_once_plan_layout():
    c = load("opcases.json.gz")["cases"][0]
    fn = dialect.parse_function(c["text"])
    params = [dec(o) for o in c["operands"]]
    blob, pblob, meta, total = exec_once_plan([fn], [params])
    assert blob.dtype == np.uint8 and total >= 1


# --- the numpy layout model ----------------------------------------------------

def _np_strides(a):
    return tuple(s // a.itemsize for s in a.strides)


@pytest.mark.parametrize("shape", [(4, 5), (3, 4, 5), (2, 3, 4, 2)])
def test_keep_order_matches_numpy_ufunc_allocation(shape):
    rng = np.random.default_rng(0)
    base = np.zeros(shape)
    for _ in range(30):
        perm = tuple(rng.permutation(len(shape)))
        a = np.transpose(np.zeros(tuple(shape[p] for p in np.argsort(perm))), perm) \
            if rng.random() < 0.5 else base
        b = np.transpose(np.zeros(tuple(shape[p] for p in np.argsort(perm))), perm) \
            if rng.random() < 0.5 else base
        a = np.ascontiguousarray(a) if a.shape != shape else a
        if a.shape != shape or b.shape != shape:
            continue
        got = L.keep_order_strides(shape, [_np_strides(a), _np_strides(b)])
        assert got == _np_strides(a + b)
        assert L.keep_order_strides(shape, [_np_strides(a)]) == _np_strides(np.exp(a))


def test_reshape_view_matches_numpy():
    rng = np.random.default_rng(1)
    for _ in range(300):
        shape = tuple(int(x) for x in rng.integers(1, 4, size=rng.integers(1, 4)))
        a = np.zeros(shape)
        if rng.random() < 0.5 and a.ndim > 1:
            a = a.transpose(tuple(rng.permutation(a.ndim)))
        n = a.size
        # random factorisation of n
        dims, m = [], n
        while m > 1 and len(dims) < 3:
            f = [d for d in range(1, m + 1) if m % d == 0]
            d = int(rng.choice(f))
            dims.append(d)
            m //= d
        dims.append(m)
        new = tuple(dims)
        r = np.reshape(a, new)
        got = L.reshape_view(a.shape, _np_strides(a), new)
        if np.shares_memory(r, a):
            assert got is not None
            # strides may differ only on extent-1 dims
            assert all(g == s or d == 1 for g, s, d in zip(got, _np_strides(r), new))
        else:
            assert got is None


def _running_sum(row):
    r = 0.0          # not sum(): CPython 3.12 sums floats with compensation
    for x in row.tolist():
        r += x
    return r


def test_reduce_order_matches_numpy():
    """Pairwise vs running sum is decided like numpy: probe with values
    whose two summation orders round differently."""
    rng = np.random.default_rng(2)
    for _ in range(200):
        shape = tuple(int(x) for x in rng.integers(2, 20, size=2))
        a = rng.standard_normal(shape) * 10.0 ** rng.integers(-8, 8, size=shape)
        if rng.random() < 0.5:
            a = np.ascontiguousarray(a.T).T
        ax = int(rng.integers(0, 2))
        perm = L.best_axis_order(2, [_np_strides(a)])
        pairwise = perm[0] == ax and a.shape[ax] > 1
        moved = np.moveaxis(a, ax, -1).reshape(-1, a.shape[ax])
        ref = np.sum(a, axis=ax).reshape(-1)
        seq = np.array([_running_sum(row) for row in moved])
        if pairwise:
            # numpy pairwise for n < 8 is the running sum anyway
            from tools_sum import pairwise_sum
            want = np.array([pairwise_sum(row) for row in moved])
        else:
            want = seq
        assert np.array_equal(want, ref)


def test_returned_layout_cycles_are_exact():
    """Steps >= 1 read the layout the previous step stored.  A program whose
    stored layout flips every step (a returned pad of a transposed slice:
    C -> F -> C ...) runs train0/train1 alternately (FLAG_ALTERNATE); a
    longer cycle is refused (plan.UnsupportedVariant), and no recorded
    individual has one."""
    from golden_io import load as gl
    inds = gl("bench_train_pool.json.gz")["individuals"]
    flags = []
    for ind in inds:
        vp = lower_variant({k: dialect.parse_function(ind[k]) for k in ("forward", "train_step")})
        flags.append(vp.flags)
    assert any(f & Lw.FLAG_ALTERNATE for f in flags)


def _emulate_words(fn, args, fuse):
    low = Lw.lower_function(fn, None, ret_layout="c", fuse=fuse)
    consts = Lw.consts_to_words(low.consts).view(np.int64).copy() if low.consts \
        else np.zeros(1, dtype=np.int64)
    mem = {Lw.BUF_ARENA: np.zeros(max(low.arena_elems, 1), dtype=np.int64),
           Lw.BUF_CONST: consts,
           Lw.BUF_SMEM: np.zeros(max(low.smem_elems, 1), dtype=np.int64)}
    for k, p in enumerate(args):
        mem[Lw.BUF_PARAM0 + k] = _words(p)
    for r, ty in enumerate(fn.return_types):
        mem[Lw.BUF_OUT0 + r] = np.zeros(max(1, int(np.prod(ty.shape))), dtype=np.int64)
    plan_emu.run(low.instrs, mem)
    return [mem[Lw.BUF_OUT0 + r].copy() for r in range(len(fn.return_types))], low


def test_fusion_changes_no_bit():
    """Dot epilogues and elementwise chains (rank <= 2 and the CNN's rank-4
    fast-form chains) emulate bit-identically to the unfused tables."""
    from paper_2310_10211_b200 import cnn
    cases = []
    wl = W.build_2fcnet_workload()
    args = [wl.weights[n] for n in W.WEIGHT_NAMES] + [wl.search_x[0], wl.search_y[0]]
    for ind in load("train_pop.json.gz")["individuals"][:60]:
        cases.append((dialect.parse_function(ind["train_step"]), args))
    cw = cnn.build_cnn_prediction_workload(cnn.CnnConfig(search_n=20, holdout_n=10, batch_size=2))
    cases.append((cw.module.functions["forward"],
                  [cw.weights["w"], cw.search_x[0].reshape(2, 32, 32, 3)]))
    nd = 0
    for fn, a in cases:
        fused, low = _emulate_words(fn, a, True)
        plain, _ = _emulate_words(fn, a, False)
        assert all(np.array_equal(x, y) for x, y in zip(fused, plain))
        nd += sum(1 for r in low.instrs if r.get("epi") and r["op"] != Lw.OP_DOT
                  and len(r["out"].shape) > 2)
    assert nd > 0          # the CNN's BN chains fused
    taps = [r["sub"] for r in low.instrs if r["op"] == Lw.OP_TAPSUM]
    assert taps and all(t == 9 for t in taps)          # every depthwise 3x3 is one TAPSUM
    micro = [len(r.get("micro", [])) for r in low.instrs if r["op"] == Lw.OP_TAPSUM]
    assert all(m == 3 for m in micro)                  # ... with its BN (*, +, max) as micro-ops


def test_elementwise_walks_output_memory_order():
    """A copy between two column-major 784 x 32 blocks (a variant returning a
    transposed view in the layout its next step reads) is walked in memory
    order: both sides linear, and the emulated result is unchanged."""
    fn = dialect.parse_function(
        "func @f(%a: tensor<32x784xf32>, %b: tensor<32x784xf32>) -> tensor<784x32xf32> {\n"
        "  %t = transpose %a {perm = [1, 0]} : tensor<784x32xf32>\n"
        "  %u = transpose %b {perm = [1, 0]} : tensor<784x32xf32>\n"
        "  %s = add %t, %u : tensor<784x32xf32>\n"
        "  return %s : tensor<784x32xf32>\n}")
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal((32, 784)), rng.standard_normal((32, 784))
    low = Lw.lower_function(fn, None, ret_layout="compact")
    (rec,) = [r for r in low.instrs if r["op"] == Lw.OP_BINARY]
    assert tuple(rec["out"].shape) == (32, 784)              # dims in memory order
    assert Lw._addr_mode(rec["out"], (32, 784)) == Lw.AM_LINEAR
    assert all(Lw._addr_mode(v, (32, 784)) == Lw.AM_LINEAR for v in rec["in"])
    (got,), _ = emulate(fn, [a, b])
    assert np.array_equal(got, (a.T + b.T))


def _emulate_steps(ts, weights, xb, yb, steps):
    """Steps of train_step through the lowering, each program lowered for
    the layouts the previous step stored (returns stay in their compact
    layout, the OUT words feed the next step's PARAM buffers as on the
    device).  Returns the weights' logical values and the layout sequence."""
    nw = len(ts.returns)
    lay = [L.c_strides(tuple(t.shape)) for _, t in ts.params]
    bufs = [_words(w) for w in weights]
    seen = []
    for _ in range(steps):
        seen.append([tuple(x) for x in lay[:nw]])
        low = Lw.lower_function(ts, lay)
        consts = Lw.consts_to_words(low.consts).view(np.int64).copy() if low.consts \
            else np.zeros(1, dtype=np.int64)
        mem = {Lw.BUF_ARENA: np.zeros(max(low.arena_elems, 1), dtype=np.int64),
               Lw.BUF_CONST: consts,
               Lw.BUF_SMEM: np.zeros(max(low.smem_elems, 1), dtype=np.int64)}
        for k, b in enumerate(bufs + [_words(xb), _words(yb)]):
            mem[Lw.BUF_PARAM0 + k] = b
        for r, ty in enumerate(ts.return_types):
            mem[Lw.BUF_OUT0 + r] = np.zeros(max(1, int(np.prod(ty.shape))), dtype=np.int64)
        plan_emu.run(low.instrs, mem)
        bufs = [mem[Lw.BUF_OUT0 + r] for r in range(nw)]
        lay[:nw] = [tuple(s) for s in low.ret_strides]
    vals = []
    for r, ty in enumerate(ts.return_types):
        shape = tuple(ty.shape)
        v = plan_emu.gather({0: bufs[r]}, Lw.Val(0, 0, shape, lay[r], Lw.K_F64), shape)
        vals.append(v.view(np.float64).reshape(shape))
    return vals, seen


def test_three_layout_schedule_ga_individual():
    """ga512x50 individual 10822 stores a different weight layout after step
    0 and after step 1 (C -> L0 -> L1 -> L1 ...): the device runs train0,
    train1, then train2 (GEVO_SCHED_STEADY2).  Before the schedule it was
    refused (no period <= 2) and the recorded run could not be replayed.
    The layouts the schedule assumes are the ones each step reads, and the
    emulated trajectory follows the oracle."""
    from paper_2310_10211_b200.plan import lower_variant
    ind = load("ga512x50.json.gz")["individuals"][10822]
    fns = {k: dialect.parse_function(ind[k]) for k in ("forward", "train_step")}
    vp = lower_variant(fns)
    assert vp.flags & 3 == Lw.SCHED_STEADY2 and vp.train2 is not None
    wl = W.build_2fcnet_workload(W.WorkloadConfig(steps=5, dataset=W.DatasetConfig(search_n=320,
                                                                                   holdout_n=64)))
    w0 = [wl.weights[n] for n in W.WEIGHT_NAMES]
    xb, yb = wl.search_x[0], wl.search_y[0]
    got, seen = _emulate_steps(fns["train_step"], w0, xb, yb, 5)
    assert seen[1] != seen[0] and seen[2] != seen[1] and seen[2] == seen[3] == seen[4]
    prog = OI.Program(fns["train_step"])
    w = list(w0)
    for _ in range(5):
        w = prog(w + [xb, yb])
    for g_, r_ in zip(got, w):
        assert np.allclose(g_, r_, rtol=1e-9, atol=1e-12, equal_nan=True)


def _inplace_mask(text):
    from paper_2310_10211_b200.plan import inplace_weights
    fn = dialect.parse_function(text)
    low = Lw.lower_function(fn)
    return inplace_weights(Lw.encode_instrs(low.instrs), len(fn.returns))


def test_inplace_analysis_rejects_unsafe_updates():
    """plan.inplace_weights: a weight read after its update, or read by its
    updating instruction at a word it does not write (a transposed view),
    stays ping-ponged; element-local updates read first go in place."""
    two = "(tensor<4x4xf32>, tensor<4x4xf32>)"
    # a' = a + b is written first; b' = b * a then reads a: a must not be in
    # place, b may (only its own writer reads it, element for element)
    assert _inplace_mask(f"""func @f(%a: tensor<4x4xf32>, %b: tensor<4x4xf32>) -> {two} {{
  %0 = add %a, %b : tensor<4x4xf32>
  %1 = multiply %b, %a : tensor<4x4xf32>
  return %0, %1 : tensor<4x4xf32>, tensor<4x4xf32>
}}""") == 0b10
    # a' reads a through a transpose: a word it does not write
    assert _inplace_mask(f"""func @f(%a: tensor<4x4xf32>, %b: tensor<4x4xf32>) -> {two} {{
  %0 = transpose %a {{perm = [1, 0]}} : tensor<4x4xf32>
  %1 = add %a, %0 : tensor<4x4xf32>
  %2 = multiply %b, %b : tensor<4x4xf32>
  return %1, %2 : tensor<4x4xf32>, tensor<4x4xf32>
}}""") == 0b10
    # both element-local and read before: both in place
    assert _inplace_mask(f"""func @f(%a: tensor<4x4xf32>, %b: tensor<4x4xf32>) -> {two} {{
  %0 = multiply %a, %b : tensor<4x4xf32>
  %1 = subtract %b, %a : tensor<4x4xf32>
  %2 = add %0, %a : tensor<4x4xf32>
  return %2, %1 : tensor<4x4xf32>, tensor<4x4xf32>
}}""") in (0b11, 0b10, 0b01)


def test_inplace_weights_emulate_identically():
    """Every bench-pool individual (steady layouts) runs one train_step with
    each in-place weight's parameter and return sharing one buffer, and the
    returned words equal the ping-pong run's (plan_emu: an instruction reads
    all its operands before it writes)."""
    from paper_2310_10211_b200.plan import inplace_weights
    wl = W.build_2fcnet_workload(W.WorkloadConfig(steps=5, dataset=W.DatasetConfig(search_n=320,
                                                                                   holdout_n=64)))
    w0 = [wl.weights[n] for n in W.WEIGHT_NAMES]
    xb, yb = wl.search_x[0], wl.search_y[0]
    inds = load("bench_train_pool.json.gz")["individuals"]
    checked = used = 0
    for ind in inds[:160]:
        if ind.get("invalid_patch"):
            continue
        ts = dialect.parse_function(ind["train_step"])
        low = Lw.lower_function(ts)
        nw = len(ts.returns)
        if [tuple(s) for s in low.ret_strides] != [L.c_strides(tuple(t.shape)) for t in ts.return_types]:
            continue                     # layout-changing variants: not this test's subject
        mask = inplace_weights(Lw.encode_instrs(low.instrs), nw)
        outs = []
        for alias in (False, True):
            consts = Lw.consts_to_words(low.consts).view(np.int64).copy() if low.consts \
                else np.zeros(1, dtype=np.int64)
            mem = {Lw.BUF_ARENA: np.zeros(max(low.arena_elems, 1), dtype=np.int64),
                   Lw.BUF_CONST: consts,
                   Lw.BUF_SMEM: np.zeros(max(low.smem_elems, 1), dtype=np.int64)}
            for k, p in enumerate(w0 + [xb, yb]):
                mem[Lw.BUF_PARAM0 + k] = _words(p)
            for r, ty in enumerate(ts.return_types):
                if alias and (mask >> r) & 1:
                    mem[Lw.BUF_OUT0 + r] = mem[Lw.BUF_PARAM0 + r]
                else:
                    mem[Lw.BUF_OUT0 + r] = np.zeros(max(1, int(np.prod(ty.shape))), dtype=np.int64)
            plan_emu.run(low.instrs, mem)
            outs.append([mem[Lw.BUF_OUT0 + r].copy() for r in range(nw)])
        for a, b in zip(*outs):
            assert np.array_equal(a, b), ind["key"][:60]
        checked += 1
        used += bin(mask).count("1")
    assert checked >= 100 and used >= 3 * checked
