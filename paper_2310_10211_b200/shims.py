"""Drop-in replacements for the reference's evaluation seams (evotir).

    from paper_2310_10211_b200 import shims
    shims.install()            # before evotir.search.run_search / evotir.cli

rebinds, by attribute (run_search constructs `_Evaluator(workload)` itself,
search.py:339, and imports `evaluate`/`holdout_report` by name, search.py:30,
so rebinding the module attributes is the only non-invasive plug-in point):

  evotir.search._Evaluator          -> GpuEvaluator        (search.py:249-273)
  evotir.search/cli.evaluate        -> evaluate            (fitness.py:372-393)
  evotir.search/cli.holdout_report  -> holdout_report      (fitness.py:396-426)
  evotir.search.nondominated_sort   -> nondominated_sort   (search.py:96-120)
  evotir.search.crowding_distance   -> crowding_distance   (search.py:123-140)
  evotir.search.rank_population     -> rank_population     (search.py:143-150)
  evotir.search.select_survivors    -> select_survivors    (search.py:163-179)
  evotir.search.hypervolume         -> hypervolume         (search.py:182-195)
  evotir.search.Archive             -> Archive             (search.py:202-233)

Everything else -- IR, apply_patch, mutation/crossover, the RNG, the search
loop, artifacts -- stays the reference's own code.  Results are the
reference's Fitness objects; the device computes f32 programs in float64 with
the reference's summation orders ("Parity").

`backend=` lets tests substitute the device (see tests/test_shims.py); the
product path always uses libgevo and raises if it is unavailable.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .evaluator import DeviceEvaluator
from .workloads import PREDICTION, TRAINING, WEIGHT_NAMES


def _E():
    """The reference package (must be importable where shims are used)."""
    import evotir.fitness as F
    import evotir.genome as G
    import evotir.search as S
    return F, G, S


_PICKLE_READY = False


def _fast_pickling():
    """Positional-tuple pickling for evotir's IR objects (same fields as this
    package's dialect, see dialect.py): the evaluator ships variant functions
    to its lowering processes and this is the part the parent pays serially."""
    global _PICKLE_READY
    if _PICKLE_READY:
        return
    import copyreg
    import evotir.ir as IR
    copyreg.pickle(IR.TensorType, lambda t: (IR.TensorType, (t.shape, t.kind)))
    copyreg.pickle(IR.Operation, lambda o: (IR.Operation, (o.op_id, o.opcode, o.result,
                                                           o.result_type, o.operands, o.attrs)))
    copyreg.pickle(IR.FunctionBody, lambda f: (IR.FunctionBody, (f.name, f.params, f.ops,
                                                                f.returns, f.return_types)))
    _PICKLE_READY = True


class _DeviceWorkload:
    """Adapter: an evotir Workload seen through the attributes
    DeviceEvaluator reads (config, dataset, weights, mode, module)."""

    def __init__(self, w):
        _fast_pickling()
        self.source = w
        self.name = w.name
        self.mode = TRAINING if w.mode == "training" else PREDICTION
        self.module = w.module
        self.config = w.config
        self.dataset = w.dataset
        self.weights = {n: np.asarray(w.module.constants[n].value, dtype=np.float64)
                        for n in WEIGHT_NAMES}


_DEVICES: dict = {}


def device_for(workload, device: int = 0):
    """One DeviceEvaluator per (workload, device), created on first use."""
    key = (id(workload), device)
    ev = _DEVICES.get(key)
    if ev is None or ev.workload.source is not workload:
        ev = DeviceEvaluator(_DeviceWorkload(workload), device)
        _DEVICES[key] = ev
    return ev


_SHARDED: dict = {}


def sharded_for(workload, device: int = 0):
    """The population-sharded evaluator (distributed.ShardedEvaluator over
    this rank's DeviceEvaluator) when torch.distributed is initialised with
    more than one rank; the plain device evaluator otherwise."""
    from . import distributed as D
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return device_for(workload, device)
    key = (id(workload), device)
    ev = _SHARDED.get(key)
    if ev is None or ev.backend.workload.source is not workload:
        ev = D.ShardedEvaluator(device_for(workload, device))
        _SHARDED[key] = ev
    return ev


def _variants(original, patches, functions):
    """apply_patch each patch (genome.py:482-516); None when it fails."""
    _, G, _ = _E()
    out = []
    for p in patches:
        try:
            m = G.apply_patch(original, p).module
        except G.PatchApplicationError:
            out.append(None)
            continue
        out.append({n: m.functions[n] for n in functions})
    return out


def _functions(w):
    return ["forward", "train_step"] if w.mode == "training" else ["forward"]


def _to_ref(fits):
    F, _, _ = _E()
    return [F.INVALID_FITNESS if not f.valid else F.Fitness(f.cost, f.error)
            for f in fits]


class GpuEvaluator:
    """Same interface as evotir.search._Evaluator: `.workload`, `.cache`
    (patch_dumps key -> Fitness, insertion ordered), `.threads`; a call
    evaluates every fresh patch of the list in ONE device launch and returns
    the fitness of every requested patch in request order.

    The fresh patches travel as their cache keys (canonical patch JSON):
    apply_patch + verify (genome.py:482-516) and the lowering run in the
    evaluator's worker processes, not serially here.  Under torch.distributed
    with several ranks (install() on every rank), each rank evaluates a
    shard of the fresh patches on its own GPU and one all-gather
    (gevo_allgather, NCCL) hands every rank every fitness."""

    def __init__(self, workload, device: int = 0, backend=None):
        self.workload = workload
        self.cache: dict = {}
        self.threads = 1            # host threads are not used for evaluation
        self.device = device
        self._backend = backend

    @property
    def backend(self):
        if self._backend is None:
            self._backend = sharded_for(self.workload, self.device)
        return self._backend

    def __call__(self, patches):
        _, G, _ = _E()
        keyed = [(G.patch_dumps(p), p) for p in patches]
        fresh = {}
        for key, p in keyed:
            if key not in self.cache and key not in fresh:
                fresh[key] = p
        if fresh:
            items = list(fresh.items())
            be = self.backend
            if hasattr(be, "evaluate_patches"):
                fits = be.evaluate_patches(self.workload.module, [k for k, _ in items],
                                           _functions(self.workload))
            else:                   # test backends that take applied variants
                fits = be.evaluate_variants(_variants(self.workload.module,
                                                      [p for _, p in items],
                                                      _functions(self.workload)))
            for (key, _), fit in zip(items, _to_ref(fits)):
                self.cache[key] = fit
        return [self.cache[key] for key, _ in keyed]


def evaluate(original, patch, w, backend=None):
    """fitness.evaluate for one patch (fitness.py:372-393); never raises."""
    try:
        (v,) = _variants(original, [patch], _functions(w))
        be = backend or device_for(w)
        return _to_ref(be.evaluate_variants([v]))[0]
    except _lib.GevoError:
        raise                       # no CPU fallback: a device failure is loud
    except Exception:
        F, _, _ = _E()
        return F.INVALID_FITNESS


def holdout_report(original, patch, w, backend=None):
    """fitness.holdout_report (fitness.py:396-426): retrain on the search
    split, score the holdout split; bumps holdout.reads like the reference
    and raises WorkloadError when holdout has no whole batch."""
    F, G, _ = _E()
    try:
        (v,) = _variants(original, [patch], _functions(w))
    except Exception:
        return F.INVALID_FITNESS
    if v is None:
        return F.INVALID_FITNESS
    w.dataset.holdout.reads += 1
    if len(w.dataset.holdout.labels) < w.config.batch_size:
        raise F.WorkloadError("holdout split smaller than one batch")
    be = backend or device_for(w)
    return _to_ref(be.evaluate_variants([v], holdout=True))[0]


# ---------------------------------------------------------------------------
# NSGA-II on the device
# ---------------------------------------------------------------------------

_NS_CTX = None
_NS_DEVICE = 0          # set by install(device=...)


def _ns_ctx():
    """The context NSGA-II, archive and hypervolume run on: the device
    install() was given (each rank of a multi-GPU run uses its own)."""
    global _NS_CTX
    if _NS_CTX is None or _NS_CTX.device != _NS_DEVICE:
        _NS_CTX = _lib.Context(_NS_DEVICE)
    return _NS_CTX


def _arrays(points):
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 2)
    return np.ascontiguousarray(pts[:, 0]), np.ascontiguousarray(pts[:, 1])


def nondominated_sort(points):
    """Fronts as lists of indices, best first (search.py:96-120)."""
    if len(points) == 0:
        return [[]]
    c, e = _arrays(points)
    _, _, order, fstart = _ns_ctx().nsga2_rank(c, e)
    return [order[fstart[k]:fstart[k + 1]].tolist() for k in range(len(fstart) - 1)]


def crowding_distance(points, front):
    """{index: distance} for one front (search.py:123-140)."""
    front = list(front)
    if len(front) <= 2:
        return {i: float("inf") for i in front}
    # the points are taken as ONE front whatever their dominance, like the
    # reference; sorting ties break on position in `front`, which is the
    # reference's index order whenever `front` is ascending (as
    # nondominated_sort returns it)
    order = sorted(range(len(front)), key=lambda k: front[k])
    c, e = _arrays([points[front[k]] for k in order])
    crowd = _ns_ctx().nsga2_crowding(c, e)
    return {front[k]: float(d) for k, d in zip(order, crowd)}


def rank_population(pop):
    """Assign .rank/.crowding in place (search.py:143-150)."""
    if not pop:
        return
    c, e = _arrays([ind.fitness.as_tuple() for ind in pop])
    rank, crowd, _, _ = _ns_ctx().nsga2_rank(c, e)
    for ind, r, d in zip(pop, rank, crowd):
        ind.rank = int(r)
        ind.crowding = float(d)


def select_survivors(pool, n):
    """Whole fronts, then the partial front by crowding (search.py:163-179).
    rank/crowding are assigned to every member of the fronts visited."""
    if not pool:
        return []
    c, e = _arrays([ind.fitness.as_tuple() for ind in pool])
    # asking for more than the pool takes every front whole (the reference's
    # loop simply runs out of fronts)
    chosen, rank, crowd = _ns_ctx().nsga2_select(c, e, max(0, min(int(n), len(pool))))
    last = int(rank[chosen].max()) if len(chosen) else 0
    for i, ind in enumerate(pool):
        if rank[i] <= last:
            ind.rank = int(rank[i])
            ind.crowding = float(crowd[i])
    return [pool[i] for i in chosen]


# ---------------------------------------------------------------------------
# Archive and hypervolume on the device
# ---------------------------------------------------------------------------

def hypervolume(points, ref):
    """Area dominated by `points` and bounded by the reference corner
    (search.py:182-195), bit-identical (gevo_hypervolume)."""
    if len(points) == 0:
        return 0.0
    c, e = _arrays(points)
    return _ns_ctx().hypervolume(c, e, ref)


def _archive_entry_type():
    try:
        from evotir.search import ArchiveEntry
        return ArchiveEntry
    except ImportError:      # tests without the reference package
        from dataclasses import dataclass

        @dataclass
        class ArchiveEntry:
            patch: tuple
            fitness: object
            holdout: object = None
        return ArchiveEntry


class Archive:
    """Drop-in for search.Archive (search.py:202-233): the globally
    non-dominated (patch, fitness) set, first comer keeping a point.

    `offer` queues; the queue is merged on the device in one pass
    (gevo_archive_merge) when `entries`, `_keys` or `sorted_entries` are next
    read -- once per generation under run_search (absorb, then record:
    search.py:350-368) instead of O(archive) Python work per evaluation.
    A queued batch must hold only keys that are new at the time of offer for
    the one-pass result to equal sequential offering, so an offer whose key
    is known (in the archive or already queued) first flushes the queue and
    then takes the reference's key check (search.py:211) against the exact
    archive.  `merge=` substitutes the device in host tests.
    """

    def __init__(self, merge=None):
        self._entries = []
        self._ekeys = []          # the offer key of each entry
        self._keyset = set()
        self._pending = []        # (patch, fitness, key)
        self._pkeys = set()
        self._merge = merge
        self._Entry = _archive_entry_type()

    def offer(self, patch, fitness, key):
        if not fitness.valid:
            return
        if key in self._pkeys or key in self._keyset:
            self._flush()
            if key in self._keyset:
                return
        self._pending.append((patch, fitness, key))
        self._pkeys.add(key)

    def _flush(self):
        if not self._pending:
            return
        pend, self._pending, self._pkeys = self._pending, [], set()
        pts = [e.fitness.as_tuple() for e in self._entries] + [f.as_tuple() for _, f, _ in pend]
        c, e = _arrays(pts)
        merge = self._merge or _ns_ctx().archive_merge
        n_old = len(self._entries)
        entries, keys = [], []
        for j in merge(c, e):
            j = int(j)
            if j < n_old:
                entries.append(self._entries[j])
                keys.append(self._ekeys[j])
            else:
                patch, fit, key = pend[j - n_old]
                entries.append(self._Entry(patch=patch, fitness=fit))
                keys.append(key)
        self._entries, self._ekeys, self._keyset = entries, keys, set(keys)

    @property
    def entries(self):
        self._flush()
        return self._entries

    @entries.setter
    def entries(self, value):
        _, G, _ = _E()
        self._pending, self._pkeys = [], set()
        self._entries = list(value)
        self._ekeys = [G.patch_dumps(e.patch) for e in self._entries]
        self._keyset = set(self._ekeys)

    @property
    def _keys(self):
        self._flush()
        return self._keyset

    def sorted_entries(self):
        self._flush()
        order = sorted(range(len(self._entries)),
                       key=lambda i: (self._entries[i].fitness.cost,
                                      self._entries[i].fitness.error, self._ekeys[i]))
        return [self._entries[i] for i in order]


# ---------------------------------------------------------------------------

_SAVED: dict = {}


def install(device: int | None = None, nsga2: bool = True, backend_factory=None):
    """Rebind the reference's evaluation seams to the device versions.
    `device` defaults to LOCAL_RANK (0 outside torchrun); with
    torch.distributed initialised over several ranks the evaluator shards
    each generation's fresh patches over the ranks (one GPU each).
    `backend_factory(workload)` substitutes the evaluator backend (tests)."""
    import os
    import evotir.cli as C
    global _NS_DEVICE
    _, _, S = _E()
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    # GEVO_B200_NSGA2=0 keeps the reference's host NSGA-II / archive /
    # hypervolume (the evaluator seams are rebound either way)
    nsga2 = nsga2 and os.environ.get("GEVO_B200_NSGA2", "1") != "0"
    _NS_DEVICE = device
    if not _SAVED:
        _SAVED.update({
            ("search", "_Evaluator"): S._Evaluator,
            ("search", "evaluate"): S.evaluate,
            ("search", "holdout_report"): S.holdout_report,
            ("cli", "evaluate"): C.evaluate,
            ("cli", "holdout_report"): C.holdout_report,
            ("search", "nondominated_sort"): S.nondominated_sort,
            ("search", "crowding_distance"): S.crowding_distance,
            ("search", "rank_population"): S.rank_population,
            ("search", "select_survivors"): S.select_survivors,
            ("search", "hypervolume"): S.hypervolume,
            ("search", "Archive"): S.Archive,
        })

    class _Bound(GpuEvaluator):
        def __init__(self, workload):
            super().__init__(workload, device,
                             backend=backend_factory(workload) if backend_factory else None)

    S._Evaluator = _Bound
    S.evaluate = C.evaluate = evaluate
    S.holdout_report = C.holdout_report = holdout_report
    if nsga2:
        S.nondominated_sort = nondominated_sort
        S.crowding_distance = crowding_distance
        S.rank_population = rank_population
        S.select_survivors = select_survivors
        S.hypervolume = hypervolume
        S.Archive = Archive


def uninstall():
    import evotir.cli as C
    _, _, S = _E()
    mods = {"search": S, "cli": C}
    for (mod, name), fn in _SAVED.items():
        setattr(mods[mod], name, fn)
    _SAVED.clear()
