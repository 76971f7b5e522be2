"""Archive / hypervolume fixtures from the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
    python tests/golden/make_archive_golden.py

SURVEY.md §8(f) 2.  Offer sequences are run through the reference
`Archive.offer` (search.py:202-228), one offer at a time, exactly as
`run_search.absorb` (search.py:350-352) does.  The sequences contain:
  * points on small grids, so ties, duplicates and dominance chains are common;
  * invalid fitnesses;
  * repeated keys, including an evicted patch that comes back at a new point
    (test_search.py:139-160);
  * fitness-like points (cost ~1e9, error k/992, and inf);
  * anti-correlated points, which keep large archives (hundreds of entries).
After every "generation" chunk the fixture records:
  * the entries' patch ids, in order;
  * the patch ids of `sorted_entries()` (search.py:230-233);
  * `hypervolume` (search.py:182-195) of the archive points and of the chunk's
    valid points, against the reference corner of run_search (search.py:346).
Separate hypervolume point sets cover test_search.py:106-128: hand cases,
uniform points with duplicates, boundary points, inf.

Writes tests/golden/archive.json.gz.
"""
from __future__ import annotations

import gzip
import json
import os
import random

from evotir.fitness import INVALID_FITNESS, Fitness
from evotir.genome import DeleteEdit, patch_dumps
from evotir.search import Archive, hypervolume

HERE = os.path.dirname(os.path.abspath(__file__))


def fake_patch(n):
    # test_search.py:131-133
    return (DeleteEdit(uid=f"{n:010x}", function="f", target="o0", rebinds=()),)


def point(rng, kind):
    if kind == "grid":
        return float(rng.randrange(8)), float(rng.randrange(8))
    if kind == "mixed":
        if rng.random() < 0.5:
            return float(rng.randrange(12)), float(rng.randrange(12))
        return rng.uniform(0, 12), rng.uniform(0, 12)
    if kind == "front":   # anti-correlated: large non-dominated sets
        u = rng.random()
        return round(u * 1000) / 10, round(((1 - u) ** 2 + rng.random() * 0.05) * 992) / 992
    # fitness-like (bench pool scale)
    if rng.random() < 0.03:
        return float("inf"), 1.0
    return float(rng.randrange(5, 11) * 105027900), rng.randrange(0, 993) / 992


def make_sequences():
    out = []
    rng = random.Random(2310_10211)
    specs = ([("grid", 6, 12)] * 12 + [("mixed", 5, 40)] * 8 + [("fitness", 10, 128)] * 4
             + [("front", 8, 64)] * 6 + [("front", 3, 1024)] + [("fitness", 3, 1024)])
    for kind, gens, per_gen in specs:
        a = Archive()
        offers, chunks = [], []
        npatch = 0
        pid_of = {}
        ref = {"fitness": (1.5 * 105027900 * 8, 1.0), "front": (90.0, 1.0)}.get(kind, (10.0, 10.0))
        for _ in range(gens):
            chunk_pts = []
            for _ in range(per_gen):
                r = rng.random()
                if r < 0.08 and npatch:          # an earlier patch again (any point)
                    pid = rng.randrange(npatch)
                else:
                    pid = npatch
                    npatch += 1
                if r < 0.04 and offers:          # exact repeat of an earlier offer
                    prev = offers[rng.randrange(len(offers))]
                    pid, (c, e), valid = prev["patch"], prev["point"], prev["valid"]
                else:
                    c, e = point(rng, kind)
                    valid = rng.random() > 0.05
                patch = fake_patch(pid)
                pid_of[patch_dumps(patch)] = pid
                fit = Fitness(c, e) if valid else INVALID_FITNESS
                a.offer(patch, fit, patch_dumps(patch))
                offers.append({"patch": pid, "point": (c, e), "valid": valid})
                if valid:
                    chunk_pts.append((c, e))
            chunks.append({
                "n_offers": len(offers),
                "entries": [pid_of[patch_dumps(e.patch)] for e in a.entries],
                "sorted": [pid_of[patch_dumps(e.patch)] for e in a.sorted_entries()],
                "archive_hv": repr(hypervolume([e.fitness.as_tuple() for e in a.entries], ref)),
                "chunk_hv": repr(hypervolume(chunk_pts, ref)),
            })
        out.append({
            "kind": kind, "ref": [repr(ref[0]), repr(ref[1])],
            # patch p's key is patch_dumps(fake_patch(p)); any injective key works
            "offers": [[o["patch"], repr(o["point"][0]), repr(o["point"][1]), o["valid"]]
                       for o in offers],
            "chunks": chunks})
    return out


def make_hv_sets():
    sets = []
    ref = (2.0, 2.0)   # test_search.py:106-116
    for pts in ([], [(1.0, 1.0)], [(2.0, 1.0)], [(1.0, 2.0)], [(1.0, 1.0), (1.5, 1.5)],
                [(0.0, 1.0), (1.0, 0.0)]):
        sets.append((pts, ref))
    rng = random.Random(31337)   # test_search.py:119-128 style, larger too
    for trial in range(80):
        n = rng.randrange(0, 11) if trial < 70 else rng.randrange(100, 3000)
        pts = [(rng.uniform(0, 8), rng.uniform(0, 8)) for _ in range(n)]
        if pts and rng.random() < 0.3:
            pts += pts[: rng.randrange(1, min(len(pts), 20) + 1)]
        if pts and rng.random() < 0.3:
            pts += [(6.0, rng.uniform(0, 8)), (rng.uniform(0, 8), 6.0), (float("inf"), 0.0)]
        rng.shuffle(pts)
        sets.append((pts, (6.0, 6.0)))
    rng = random.Random(9)
    for n in (256, 512, 4096):   # generation-like
        pts = [point(rng, "fitness") for _ in range(n)]
        sets.append((pts, (1.5 * 105027900 * 6, 1.0)))
    return [{"points": [[repr(c), repr(e)] for c, e in pts],
             "ref": [repr(ref[0]), repr(ref[1])],
             "hv": repr(hypervolume(pts, ref))} for pts, ref in sets]


def main():
    data = {"sequences": make_sequences(), "hv_sets": make_hv_sets()}
    path = os.path.join(HERE, "archive.json.gz")
    with gzip.open(path, "wt") as f:
        json.dump(data, f, separators=(",", ":"), sort_keys=True)
    sizes = [len(s["chunks"][-1]["entries"]) for s in data["sequences"]]
    print(f"wrote {path} ({os.path.getsize(path)} bytes); final archive sizes {sizes}")


if __name__ == "__main__":
    main()
