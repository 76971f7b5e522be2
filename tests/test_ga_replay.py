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
