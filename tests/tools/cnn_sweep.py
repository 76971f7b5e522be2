"""configs[4] for the CNN workload at N = 1 (tool): population sweep of the
configs[2] network over the 53 distinct reference-made full-size mutants
(tests/golden/cnn_full_pop*.json.gz, cycled), 1 000 images each, float64.
One JSON line per population: device value, e2e, images/s."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402

for pop in [int(a) for a in sys.argv[1:]] or [64, 128, 256, 512, 1024]:
    r = bench.cnn_measure(0, steps=2, n_img=1000, pop=pop,
                          fixtures=("cnn_full_pop.json.gz", "cnn_full_pop2.json.gz"))
    r["population"] = pop
    print(json.dumps(r), flush=True)
