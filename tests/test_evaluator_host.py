"""Host logic of DeviceEvaluator without a GPU: the device context is
replaced by a fake that records the plans it receives, so lowering (in-process
and in the process pool), the two-half pipelined launch, result mapping and
the reference's failure encodings are exercised on CPU."""
import numpy as np
import pytest

from golden_io import load, variant_functions
from paper_2310_10211_b200 import _lib, evaluator as E
from paper_2310_10211_b200 import workloads as W
from paper_2310_10211_b200.lowering import HEADER_DTYPE


class FakeContext:
    instances = []

    def __init__(self, device=0):
        self.plans = []
        FakeContext.instances.append(self)

    def upload_split(self, *a):
        pass

    upload_split_u8 = upload_split_cifar = upload_split

    def num_sms(self):
        return 148

    def upload_weights(self, *a):
        pass

    def eval(self, blob, n_prog, mode, steps, check_every, train_split, score_split,
             weight_elems=0, want_weights=False):
        hdr = blob[:HEADER_DTYPE.itemsize].view(HEADER_DTYPE)[0]
        assert hdr["n_prog"] == n_prog
        self.plans.append(n_prog)
        res = np.zeros(n_prog, dtype=_lib.RESULT_DTYPE)
        # individual k: wrong = k, total = 992; every 7th blows up
        res["wrong"] = np.arange(n_prog)
        res["total"] = 992
        res["status"][::7] = E.STATUS_NONFINITE_WEIGHTS
        return res, None

    def last_kernel_ms(self):
        return 1.0

    def close(self):
        pass


@pytest.fixture
def fake(monkeypatch):
    FakeContext.instances = []
    monkeypatch.setattr(_lib, "Context", FakeContext)
    monkeypatch.setattr(_lib, "span_ms", lambda a, b: 2.0)
    return FakeContext


@pytest.mark.parametrize("n", [5, 80])
def test_evaluate_variants_maps_results_and_failures(fake, n):
    wl = W.build_2fcnet_workload(W.WorkloadConfig(steps=60, dataset=W.DatasetConfig(
        search_n=320, holdout_n=64)))
    inds = load("train_pop.json.gz")["individuals"][:n]
    variants = [variant_functions(i) for i in inds]
    variants[1] = None                                  # a patch that failed to apply
    ev = E.DeviceEvaluator(wl)
    fits, recs = ev.evaluate_variants(variants, return_records=True)
    assert fits[1] == W.INVALID_FITNESS
    launched = sum(p for c in fake.instances for p in c.plans)
    assert launched == n - 1
    # pipelined halves when the process pool is used
    assert ev.last_timing["halves"] == (2 if n >= 2 * E.POOL_MIN else 1)
    for i, f in enumerate(fits):
        if variants[i] is None:
            continue
        assert f.valid and f.cost > 0
        if recs[i]["status"] != E.STATUS_OK:
            assert f.error == 1.0                      # fitness.py:383-384
        else:
            assert f.error == recs[i]["wrong"] / 992
    ev.close()


def test_pool_lowering_matches_in_process():
    inds = load("train_pop.json.gz")["individuals"][:70]
    variants = [variant_functions(i) for i in inds]
    a = E.lower_all(variants, None, True)             # pool (>= POOL_MIN)
    b = E._lower_many((variants, None, True, 600))    # in-process
    for x, y in zip(a, b):
        assert x.train_cost == y.train_cost and x.fwd_cost == y.fwd_cost
        assert x.train0.tobytes() == y.train0.tobytes()
        assert x.fwd.tobytes() == y.fwd.tobytes()
        assert x.consts.tobytes() == y.consts.tobytes()


def test_sm_aware_order_places_heaviest_alone_and_pairs_heavy_with_light():
    from paper_2310_10211_b200.plan import sm_aware_order
    n_sms, n = 148, 256
    w = np.arange(n, dtype=float)                     # individual i weighs i
    order = sm_aware_order(w, n_sms)
    assert sorted(order.tolist()) == list(range(n))   # a permutation
    pairs = n - n_sms
    solo = set(order[pairs:n_sms].tolist())
    assert solo == set(range(n - (n_sms - pairs), n))  # the heaviest 40 run alone
    sums = [w[order[i]] + w[order[n_sms + i]] for i in range(pairs)]
    assert max(sums) - min(sums) <= 1.0               # heavy paired with light
    # outside one wave: heaviest first
    assert sm_aware_order(w[:100], n_sms).tolist() == list(range(99, -1, -1))


def _merge_records(progs, per_prog, n):
    """Python restatement of gevo_abi.cu merge_results (score parts)."""
    out = np.zeros(n, dtype=_lib.RESULT_DTYPE)
    done = set()
    for p, r in zip(progs, per_prog):
        s = int(p["result_slot"])
        if s not in done:
            out[s] = r
            done.add(s)
        elif out[s]["status"] == E.STATUS_OK and r["status"] == E.STATUS_OK:
            out[s]["wrong"] += r["wrong"]
            out[s]["total"] += r["total"]
        elif out[s]["status"] == E.STATUS_OK:
            out[s]["status"], out[s]["wrong"], out[s]["total"] = r["status"], 0, 0
    return out


class PartsContext(FakeContext):
    """Emulates one prediction launch: each program scores the batches its
    score part owns (GEVO_FLAG_PART / NPARTS); batch b counts b + 1 wrong,
    and the launch's individual 3 sees non-finite probabilities on batch 5
    only; the records are merged as gevo_eval merges them."""
    n_batches = 31

    def eval(self, blob, n_prog, mode, steps, check_every, train_split, score_split,
             weight_elems=0, want_weights=False):
        from paper_2310_10211_b200.lowering import INSTR_DTYPE, PROG_DTYPE
        from paper_2310_10211_b200.plan import FLAG_NPARTS_SHIFT, FLAG_PART_SHIFT
        hdr = blob[:HEADER_DTYPE.itemsize].view(HEADER_DTYPE)[0]
        o = HEADER_DTYPE.itemsize + int(hdr["n_instr"]) * INSTR_DTYPE.itemsize
        progs = blob[o:o + n_prog * PROG_DTYPE.itemsize].view(PROG_DTYPE)
        self.plans.append(n_prog)
        per = np.zeros(n_prog, dtype=_lib.RESULT_DTYPE)
        arenas = set()
        for k, p in enumerate(progs):
            part = (int(p["flags"]) >> FLAG_PART_SHIFT) & 0xFFF
            parts = ((int(p["flags"]) >> FLAG_NPARTS_SHIFT) & 0x7FF) or 1
            i = int(p["result_slot"])
            arenas.add(int(p["arena_off"]))
            for b in range(part, self.n_batches, parts):
                if i == 3 and b == 5:
                    per[k]["status"], per[k]["wrong"], per[k]["total"] = E.STATUS_NONFINITE_PROBS, 0, 0
                    break
                per[k]["wrong"] += b + 1
                per[k]["total"] += 32
        assert len(arenas) == n_prog                   # every program has its own scratch
        n = len({int(p["result_slot"]) for p in progs})
        self.parts = n_prog // n
        return _merge_records(progs, per, n_prog), None


_PW = []


def _predict_workload():
    """predict2fc with the unfrozen initial weights (no training pass: the
    weights' values do not matter to the plan layout under test)."""
    if not _PW:
        wl = W.build_2fcnet_workload()
        wl.mode = W.PREDICTION
        _PW.append(wl)
    return _PW[0]


@pytest.mark.parametrize("n,forced", [(7, None), (40, None), (7, "3"), (150, None)])
def test_prediction_score_parts_cover_every_batch_once(monkeypatch, n, forced):
    wl = _predict_workload()
    FakeContext.instances = []
    monkeypatch.setattr(_lib, "Context", PartsContext)
    monkeypatch.setattr(_lib, "span_ms", lambda a, b: 2.0)
    if forced:
        monkeypatch.setenv("GEVO_B200_PARTS", forced)
    nb = len(wl.dataset.search.labels) // wl.config.batch_size
    PartsContext.n_batches = nb
    fns = [{"forward": wl.module.functions["forward"]}] * n
    ev = E.DeviceEvaluator(wl)
    fits, recs = ev.evaluate_variants(fns, return_records=True)
    ctx = ev.ctx
    expect_parts = int(forced) if forced else max(1, min(nb, 2 * 148 // n))
    assert ctx.parts == expect_parts
    bad = 0
    for f, r in zip(fits, recs):
        if r["status"] != E.STATUS_OK:
            assert r["status"] == E.STATUS_NONFINITE_PROBS and f.error == 1.0
            bad += 1
            continue
        assert r["total"] == 32 * nb
        assert r["wrong"] == nb * (nb + 1) // 2       # every batch exactly once
        assert f.error == r["wrong"] / r["total"]
    assert bad == sum(len(c.plans) for c in FakeContext.instances)  # slot 3 of each launch
    ev.close()


def test_scratch_budget_splits_a_half_into_sequential_launches(fake, monkeypatch):
    """Individuals whose device scratch exceeds GEVO_B200_ARENA_GB run as
    consecutive launches that each fit; results still map to their variants."""
    wl = W.build_2fcnet_workload(W.WorkloadConfig(steps=60, dataset=W.DatasetConfig(
        search_n=320, holdout_n=64)))
    inds = load("train_pop.json.gz")["individuals"][:20]
    variants = [variant_functions(i) for i in inds]
    monkeypatch.setenv("GEVO_B200_ARENA_GB", "0.002")       # ~2 MB: a few individuals per launch
    ev = E.DeviceEvaluator(wl)
    fits, recs = ev.evaluate_variants(variants, return_records=True)
    plans = [p for c in fake.instances for p in c.plans]
    assert len(plans) > 2 and sum(plans) == len(variants)
    for f, r in zip(fits, recs):
        if r["status"] != E.STATUS_OK:
            assert f.error == 1.0
        else:
            assert f.error == r["wrong"] / 992
    ev.close()


def test_forward_memo_identical_plans():
    """The patch workers share the encoded @forward of every patch that edits
    no op of it (plan.lower_variant fwd_memo): the plans are byte-identical
    to lowering each variant on its own, for patches that do and do not
    touch @forward, in any order."""
    import pytest
    from golden_io import reference_available
    if not reference_available():
        pytest.skip("reference not importable")
    import numpy as np
    from evotir import fitness as F
    from evotir.genome import patch_loads
    from paper_2310_10211_b200 import evaluator as E
    inds = [i for i in load("bench_train_pool.json.gz")["individuals"] if not i.get("invalid_patch")]
    keys = [i["key"] for i in inds[:80]]
    touched = [any(e.function == "forward" for e in patch_loads(k)) for k in keys]
    assert any(touched) and not all(touched)
    wl = F.build_2fcnet_workload()
    tok = E.register_module(wl.module)
    fns = ("train_step", "forward")
    E._FWD_MEMO.clear()
    shared = E._lower_patches((tok, keys, fns, None, True, 600))
    assert E._FWD_MEMO and any(len(m) for m in E._FWD_MEMO.values())
    alone = []
    for k in keys:
        E._FWD_MEMO.clear()
        alone += E._lower_patches((tok, [k], fns, None, True, 600))
    for a, b in zip(shared, alone):
        assert (a is None) == (b is None)
        if a is None:
            continue
        for f in ("train0", "train1", "fwd", "consts", "train2"):
            x, y = getattr(a, f), getattr(b, f)
            assert (x is None) == (y is None)
            if x is not None:
                assert x.tobytes() == y.tobytes(), f
        for f in ("arena", "smem", "flags", "train_cost", "fwd_cost", "w_train", "w_fwd"):
            assert getattr(a, f) == getattr(b, f), f
