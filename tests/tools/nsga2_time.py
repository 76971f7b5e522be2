"""NSGA-II on the device at the pool sizes of SURVEY.md §6 (tool): survivor
selection (gevo_nsga2_select) of a 2P pool with random (cost, error) points,
against the reference's own nondominated_sort + crowding + selection times
measured in the survey (0.18 s @1024, 3.37 s @4096, 14.2 s @8192)."""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(os.path.dirname(HERE))]
from paper_2310_10211_b200 import _lib  # noqa: E402

ctx = _lib.Context(0)
rng = np.random.default_rng(0)
for n in (1024, 4096, 8192, 16384):
    c = rng.integers(0, 200, n).astype(np.float64) * 1e6    # ties, like static costs
    e = rng.integers(0, 992, n) / 992.0
    ctx.nsga2_select(c, e, n // 2)
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        ctx.nsga2_select(c, e, n // 2)
        ts.append(time.perf_counter() - t)
    print(f"n={n}: select {n // 2} survivors in {1e3 * min(ts):.2f} ms (host wall, incl. H2D/D2H)")
ctx.close()
