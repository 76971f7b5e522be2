"""Replay a recorded reference GEVO-ML run on this package's device path.

A run recorded by tests/golden/make_ga_golden.py holds the reference's
variation output: every patch's variant program, and each evaluator call's
patch list.  The replay re-runs everything downstream of variation with the
drop-in components, in run_search's order (search.py:333-399):

  evaluator calls    -> DeviceEvaluator.evaluate_variants (fresh, deduped)
  rank_population    -> shims.rank_population      (gevo_nsga2_rank)
  select_survivors   -> shims.select_survivors     (gevo_nsga2_select)
  Archive.offer      -> shims.Archive              (gevo_archive_merge)
  hypervolume        -> shims.hypervolume          (gevo_hypervolume)
  holdout_report     -> evaluate_variants(holdout=True), whole archive at once

and checks each against the recording: every fitness bit for bit, each
generation's survivors (order, rank, crowding), every history entry, the
final archive and its holdout reports.  Mutation, crossover and smoke checks
are the reference's unchanged host code; the replay stands in for them with
the recorded programs, parsed before the timed region.

`backend` = anything with evaluate_variants (a DeviceEvaluator on the GPU; a
table of recorded fitnesses for the host-only test).  `sel` = a namespace
with rank_population / select_survivors / nondominated_sort / Archive /
hypervolume (shims on the GPU, the oracle in host tests).
"""
from __future__ import annotations

import time
import types

from golden_io import variant_functions


class Ind:
    __slots__ = ("idx", "fitness", "rank", "crowding", "patch")

    def __init__(self, idx, fitness):
        self.idx, self.fitness, self.patch = idx, fitness, idx
        self.rank, self.crowding = 0, 0.0


def parse_all(data):
    return [variant_functions(ind) for ind in data["individuals"]]


def replay(data, backend, sel, variants=None, generations=None, check=True):
    """Returns {'stats': ..., 'mismatch': [...]} ; raises nothing on mismatch
    when check is False."""
    from paper_2310_10211_b200.workloads import Fitness
    inds = data["individuals"]
    variants = variants if variants is not None else parse_all(data)
    gens = data["config"]["generations"] if generations is None else generations
    pop_n = data["config"]["population"]
    calls = data["calls"]
    fits = {}
    mism = []
    t = {"eval": 0.0, "select": 0.0, "archive": 0.0, "holdout": 0.0}
    n_fresh = 0

    def call(ci):
        nonlocal n_fresh
        idxs = calls[ci]
        fresh, seen = [], set()
        for i in idxs:
            if i not in fits and i not in seen:
                fresh.append(i)
                seen.add(i)
        t0 = time.perf_counter()
        got = backend.evaluate_variants([variants[i] for i in fresh]) if fresh else []
        t["eval"] += time.perf_counter() - t0
        n_fresh += len(fresh)
        for i, f in zip(fresh, got):
            fits[i] = f
            r = inds[i]
            if check and (f.cost, f.error, f.valid) != (r["cost"], r["error"], r["valid"]):
                mism.append(("fitness", i, (f.cost, f.error, f.valid),
                             (r["cost"], r["error"], r["valid"])))
        return [Ind(i, fits[i]) for i in idxs]

    def record(gen, pop, archive, ref):
        t0 = time.perf_counter()
        points = [i.fitness.as_tuple() for i in pop if i.fitness.valid]
        front = sel.nondominated_sort([i.fitness.as_tuple() for i in pop])[0]
        entry = {
            "generation": gen,
            "evaluations": len(fits),
            "front_size": len(front),
            "best_error": min((e for _, e in points), default=None),
            "best_cost": min((c for c, _ in points), default=None),
            "archive_size": len(archive.entries),
            "hypervolume": sel.hypervolume(points, ref),
            "archive_hypervolume": sel.hypervolume(
                [e.fitness.as_tuple() for e in archive.entries], ref),
        }
        t["archive"] += time.perf_counter() - t0
        want = data["history"][gen]
        if check and entry != {k: want[k] for k in entry}:
            mism.append(("history", gen, entry, want))

    wall0 = time.perf_counter()
    (base,) = call(0)
    ref = (1.5 * base.fitness.cost, 1.0)
    archive = sel.Archive()

    def absorb(batch):
        t0 = time.perf_counter()
        for ind in batch:
            archive.offer(ind.idx, ind.fitness, f"{ind.idx:012d}")
        t["archive"] += time.perf_counter() - t0

    pop = call(1)
    absorb(pop)
    t0 = time.perf_counter()
    sel.rank_population(pop)
    t["select"] += time.perf_counter() - t0
    record(0, pop, archive, ref)
    for g in range(1, gens + 1):
        children = call(g + 1)
        absorb(children)
        t0 = time.perf_counter()
        pop = sel.select_survivors(pop + children, pop_n)
        t["select"] += time.perf_counter() - t0
        want = data["survivors"][g - 1]
        got = [[i.idx, i.rank, repr(i.crowding)] for i in pop]
        if check and got != want:
            mism.append(("survivors", g, got[:4], want[:4]))
        record(g, pop, archive, ref)
    full = gens == data["config"]["generations"]
    if full:
        # holdout reports for the whole archive in one device call
        entries = archive.sorted_entries()
        t0 = time.perf_counter()
        hold = backend.evaluate_variants([variants[e.patch] for e in entries], holdout=True)
        t["holdout"] += time.perf_counter() - t0
        if check:
            if [e.patch for e in entries] != data["archive"]:
                mism.append(("archive", [e.patch for e in entries][:8], data["archive"][:8]))
            got = [[h.cost, h.error, h.valid] for h in hold]
            if got != data["archive_holdout"]:
                mism.append(("archive_holdout", got[:4], data["archive_holdout"][:4]))
    wall = time.perf_counter() - wall0
    return {"mismatch": mism,
            "stats": {"generations": gens, "fresh": n_fresh, "wall_s": wall,
                      "ind_per_s": n_fresh / wall if wall > 0 else 0.0, **{f"{k}_s": v for k, v in t.items()},
                      "archive_size": len(archive.entries)}}


class TableBackend:
    """Host-test stand-in for the device: the recorded fitness by program."""

    def __init__(self, data, variants):
        from paper_2310_10211_b200.workloads import Fitness, INVALID_FITNESS
        self.by_id = {}
        for ind, v in zip(data["individuals"], variants):
            self.by_id[id(v)] = (INVALID_FITNESS if ind.get("invalid_patch") or not ind["valid"]
                                 else Fitness(ind["cost"], ind["error"]))
        self.holdout = {}
        self.data = data

    def evaluate_variants(self, vs, holdout=False):
        if holdout:
            rows = self.data["archive_holdout"]
            from paper_2310_10211_b200.workloads import Fitness
            return [Fitness(c, e, ok) for c, e, ok in rows[:len(vs)]]
        return [self.by_id[id(v)] for v in vs]


def oracle_selection():
    """rank/select/sort/hypervolume/Archive from oracle/ (host tests)."""
    from oracle import archive as OA
    from oracle import nsga2 as ON
    from paper_2310_10211_b200 import shims

    def rank_population(pop):
        rank, crowd = ON.rank_and_crowd([i.fitness.as_tuple() for i in pop])
        for ind, r, d in zip(pop, rank, crowd):
            ind.rank, ind.crowding = r, d

    def select_survivors(pool, n):
        pts = [i.fitness.as_tuple() for i in pool]
        out = []
        for r, front in enumerate(ON.fronts_of(pts)):
            d = ON.crowding(pts, front)
            for i in front:
                pool[i].rank, pool[i].crowding = r, d[i]
            if len(out) + len(front) <= n:
                out.extend(pool[i] for i in front)
            else:
                out.extend(pool[i] for i in sorted(front, key=lambda i: (-d[i], i))[:n - len(out)])
            if len(out) >= n:
                break
        return out

    class Archive(shims.Archive):
        def __init__(self):
            super().__init__(merge=lambda c, e: OA.merge_batch(list(zip(c.tolist(), e.tolist()))))

    return types.SimpleNamespace(
        rank_population=rank_population, select_survivors=select_survivors,
        nondominated_sort=ON.fronts_of, hypervolume=OA.hypervolume, Archive=Archive)


def device_selection():
    from paper_2310_10211_b200 import shims
    return types.SimpleNamespace(
        rank_population=shims.rank_population, select_survivors=shims.select_survivors,
        nondominated_sort=shims.nondominated_sort, hypervolume=shims.hypervolume,
        Archive=shims.Archive)
