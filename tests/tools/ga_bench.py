"""BASELINE.json configs[3] on one B200: a whole recorded GEVO-ML run
(train2fc, population 512, 50 generations, NSGA-II) replayed through the
device path (tests/ga_replay.py), checked bit for bit against the recording.

    python tests/tools/ga_bench.py [ga512x50.json.gz] [--out gpurun_out/ga.json]

Prints one JSON line:
  value      fresh individuals / (seconds inside evaluator calls), the
             bench.py metric over the whole run (58 calls of 1..~400)
  run        fresh individuals / replay wall (evaluation + NSGA-II +
             archive + hypervolume + holdout of the archive)
  reference  the recording's own numbers (reference evaluator on a process
             pool of the build container's cores; its host-side remainder =
             variation, smoke checks, selection, archive, serial holdout)
  parity     mismatches found by the replay (must be 0)
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from ga_replay import device_selection, parse_all, replay  # noqa: E402
from golden_io import load  # noqa: E402


def main():
    argv = sys.argv[1:]
    out_path = None
    if "--out" in argv:
        k = argv.index("--out")
        out_path = argv[k + 1]
        del argv[k:k + 2]
    name = argv[0] if argv else "ga512x50.json.gz"
    from paper_2310_10211_b200 import workloads
    from paper_2310_10211_b200.evaluator import DeviceEvaluator
    data = load(name)
    t0 = time.perf_counter()
    variants = parse_all(data)
    parse_s = time.perf_counter() - t0
    ev = DeviceEvaluator(workloads.build_2fcnet_workload())
    # warm: one small call (context, lowering pool, module load)
    ev.evaluate_variants(variants[:8])
    out = replay(data, ev, device_selection(), variants)
    st = out["stats"]
    rt = data["timing"]
    line = {
        "metric": "individuals evaluated/sec per generation",
        "config": {"workload": f"full GEVO-ML run: train2fc pop {data['config']['population']}"
                               f" x {data['config']['generations']} generations, NSGA-II on GPU "
                               "(BASELINE.json configs[3]); variation replayed from a seeded "
                               "reference run"},
        "value": st["fresh"] / st["eval_s"],
        "unit": "individuals/s",
        "run": {"ind_per_s": st["ind_per_s"], "wall_s": st["wall_s"], "eval_s": st["eval_s"],
                "select_s": st["select_s"], "archive_hv_s": st["archive_s"],
                "holdout_s": st["holdout_s"], "fresh": st["fresh"],
                "archive_size": st["archive_size"], "parse_s_untimed": parse_s},
        "reference": {"evaluator_ind_per_s": st["fresh"] / rt["evaluator_s"],
                      "evaluator_s": rt["evaluator_s"], "procs": rt["procs"],
                      "host_remainder_s": rt["host_s"], "wall_s": rt["wall_s"]},
        "parity": {"mismatches": len(out["mismatch"]), "first": out["mismatch"][:2],
                   "checked": "every fitness, survivors+rank+crowding per generation, "
                              "history, archive, archive holdout"},
    }
    s = json.dumps(line)
    print(s)
    if out_path:
        with open(out_path, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
