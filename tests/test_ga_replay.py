"""A whole recorded reference run replayed through the drop-in components
(BASELINE.json configs[3]; tests/ga_replay.py).

CPU:  with recorded fitnesses standing in for the device and the oracle for
      selection, the replay reproduces the reference run exactly (survivors,
      rank/crowding, history, archive) -- this pins the replay harness.
GPU:  the device evaluator, NSGA-II, archive merge and hypervolume reproduce
      the same run bit for bit, holdout reports of the archive included.
"""
import os

import pytest

from ga_replay import TableBackend, device_selection, oracle_selection, parse_all, replay
from golden_io import GOLDEN, load

RUNS = [n for n in ("ga64x3.json.gz", "ga512x50.json.gz") if os.path.exists(os.path.join(GOLDEN, n))]


def test_replay_harness_reproduces_recorded_run():
    data = load("ga64x3.json.gz")
    variants = parse_all(data)
    out = replay(data, TableBackend(data, variants), oracle_selection(), variants)
    assert out["mismatch"] == []
    assert out["stats"]["fresh"] == len(data["individuals"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", RUNS)
def test_device_replay_bit_exact(name):
    from paper_2310_10211_b200 import workloads
    from paper_2310_10211_b200.evaluator import DeviceEvaluator
    data = load(name)
    ev = DeviceEvaluator(workloads.build_2fcnet_workload())
    out = replay(data, ev, device_selection())
    print(name, out["stats"])
    kinds = {}
    for m in out["mismatch"]:
        kinds[m[0]] = kinds.get(m[0], 0) + 1
    print("mismatch kinds", kinds, out["mismatch"][:3])
    assert out["mismatch"] == [], (kinds, out["mismatch"][:3])


@pytest.mark.gpu
def test_launch_configurations_agree_under_poison(monkeypatch):
    """Individuals of the recorded run whose returned weights are compact
    (stride-0 views covering part of their slot) plus ordinary ones, with
    every device buffer poisoned to NaN before each launch (GEVO_POISON=1):
    the default launch, ping-pong weights (no in-place updates), one chunk
    instead of two, and the L2 window all give the recorded fitness bit for
    bit.  A read of a word no instruction wrote -- e.g. a weight block that
    was never zeroed, or a neighbour's block zeroed by mistake -- turns into
    NaN and a status change here."""
    from paper_2310_10211_b200 import lowering as Lw, workloads
    from paper_2310_10211_b200.dialect import parse_function
    from paper_2310_10211_b200.evaluator import DeviceEvaluator
    data = load("ga512x50.json.gz")
    pick, compact = [], 0
    for ind in data["individuals"][:4000]:
        if not ind.get("valid", True) or ind.get("train_step") is None:
            continue
        ts = parse_function(ind["train_step"])
        is_compact = any(0 in tuple(st) for st in Lw.lower_function(ts).ret_strides)
        if is_compact or len(pick) - compact < 64:
            pick.append(ind)
            compact += is_compact
        if compact >= 64 and len(pick) >= 128:
            break
    assert compact >= 32
    variants = [{k: parse_function(i[k]) for k in ("forward", "train_step")} for i in pick]
    monkeypatch.setenv("GEVO_POISON", "1")
    # (ping-pong last: it turns the lowering pool off for the rest of the test)
    for cfg in ({}, {"GEVO_B200_CHUNKS": "1"}, {"GEVO_B200_L2WINDOW": "1"}, {"GEVO_B200_INPLACE": "0"}):
        for k in ("GEVO_B200_INPLACE", "GEVO_B200_CHUNKS", "GEVO_B200_L2WINDOW"):
            monkeypatch.delenv(k, raising=False)
        for k, v in cfg.items():
            monkeypatch.setenv(k, v)
        from paper_2310_10211_b200 import evaluator as E, plan as P
        inplace = cfg.get("GEVO_B200_INPLACE", "1") != "0"
        monkeypatch.setattr(P, "INPLACE", inplace)
        # the lowering workers were forked with plan.INPLACE as it was: lower
        # in-process when it changes (GEVO_B200_CHUNKS needs the pool, the
        # other configurations do not)
        monkeypatch.setattr(E, "_POOL", E._POOL if inplace else False)
        ev = DeviceEvaluator(workloads.build_2fcnet_workload())
        fits = ev.evaluate_variants(variants)
        ev.close()
        bad = [(i["cost"], i["error"], f.cost, f.error) for f, i in zip(fits, pick)
               if (f.cost, f.error) != (i["cost"], i["error"])]
        print(cfg, f"{len(pick) - len(bad)}/{len(pick)} bit-exact ({compact} with compact returns)")
        assert not bad, (cfg, bad[:4])
