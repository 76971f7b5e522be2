"""The drop-in seams (paper_2310_10211_b200.shims).

CPU (needs the reference importable, i.e. the build container): with the
device replaced by a table of the reference's own recorded fitnesses, the
installed GpuEvaluator reproduces the recorded seeded search exactly -- the
evaluator seam changes nothing else in the GA (cache keys, call order,
evaluations count, history).
GPU: the NSGA-II shims return the reference's structures bit-for-bit, and the
installed evaluator on the device reproduces the recorded search.
"""
import math
import types

import numpy as np
import pytest

from golden_io import load, reference_available

HAVE_REF = reference_available()


class GoldenBackend:
    """Stands in for the device: fitness of a variant = the reference's
    recorded fitness of the individual with the same program text."""

    def __init__(self, name="train_pop.json.gz"):
        from paper_2310_10211_b200.dialect import format_function
        self.fmt = format_function
        self.table = {}
        for ind in load(name)["individuals"]:
            if not ind.get("invalid_patch"):
                self.table[(ind["train_step"], ind["forward"])] = (ind["cost"], ind["error"])
        self.calls = []

    def evaluate_variants(self, variants, holdout=False):
        from paper_2310_10211_b200.workloads import Fitness, INVALID_FITNESS
        self.calls.append(len(variants))
        out = []
        for v in variants:
            if v is None:
                out.append(INVALID_FITNESS)
                continue
            key = (self.fmt(v["train_step"]), self.fmt(v["forward"]))
            out.append(Fitness(*self.table[key]))
        return out


@pytest.mark.skipif(not HAVE_REF, reason="reference package not importable")
def test_gpu_evaluator_seam_reproduces_recorded_search():
    import evotir.search as S
    from evotir import fitness as F
    from paper_2310_10211_b200 import shims
    data = load("train_pop.json.gz")
    backend = GoldenBackend()
    orig = S._Evaluator

    class Seam(shims.GpuEvaluator):
        def __init__(self, workload):
            super().__init__(workload, backend=backend)

    # the queueing Archive seam too, its one-pass merge stated by the oracle
    # (the device kernel is checked against the same rule in test_archive.py)
    from oracle import archive as OA

    class QArchive(shims.Archive):
        def __init__(self):
            super().__init__(merge=lambda c, e: OA.merge_batch(list(zip(c.tolist(),
                                                                        e.tolist()))))

    saved = (S.Archive, S.hypervolume)
    S._Evaluator = Seam
    S.Archive, S.hypervolume = QArchive, OA.hypervolume
    try:
        w = F.build_2fcnet_workload()
        cfg = S.SearchConfig(**data["config"])
        res = S.run_search(w, cfg)
    finally:
        S._Evaluator = orig
        S.Archive, S.hypervolume = saved
    assert res.evaluations == len(data["individuals"])
    keys = ("generation", "evaluations", "front_size", "best_error", "best_cost",
            "archive_size", "hypervolume", "archive_hypervolume")
    got = [{k: h[k] for k in keys} for h in res.history]
    want = [{k: h[k] for k in keys} for h in data["history"]]
    assert got == want
    # one device call per evaluator call (baseline, initial, each generation)
    assert len(backend.calls) == 1 + 1 + data["config"]["generations"]


@pytest.mark.skipif(not HAVE_REF, reason="reference package not importable")
def test_install_rebinds_and_restores():
    import evotir.cli as C
    import evotir.search as S
    from paper_2310_10211_b200 import shims
    before = (S._Evaluator, S.evaluate, C.holdout_report, S.select_survivors)
    shims.install(nsga2=True)
    try:
        assert issubclass(S._Evaluator, shims.GpuEvaluator)
        assert S.evaluate is shims.evaluate and C.evaluate is shims.evaluate
        assert S.holdout_report is shims.holdout_report
        assert S.select_survivors is shims.select_survivors
        assert S.nondominated_sort is shims.nondominated_sort
        assert S.Archive is shims.Archive and S.hypervolume is shims.hypervolume
    finally:
        shims.uninstall()
    assert (S._Evaluator, S.evaluate, C.holdout_report, S.select_survivors) == before


@pytest.mark.skipif(not HAVE_REF, reason="reference package not importable")
def test_install_host_nsga2_switch(monkeypatch):
    """GEVO_B200_NSGA2=0 rebinds only the evaluator seams: NSGA-II, the
    archive and the hypervolume stay the reference's host code."""
    import evotir.search as S
    from paper_2310_10211_b200 import shims
    ref = (S.nondominated_sort, S.select_survivors, S.Archive, S.hypervolume)
    monkeypatch.setenv("GEVO_B200_NSGA2", "0")
    shims.install()
    try:
        assert issubclass(S._Evaluator, shims.GpuEvaluator) and S.evaluate is shims.evaluate
        assert (S.nondominated_sort, S.select_survivors, S.Archive, S.hypervolume) == ref
    finally:
        shims.uninstall()


@pytest.mark.skipif(not HAVE_REF, reason="reference package not importable")
def test_evaluate_seam_invalid_patch_and_holdout_reads():
    from evotir import fitness as F
    from evotir.genome import DeleteEdit, Rebind
    from paper_2310_10211_b200 import shims
    w = F.build_2fcnet_workload()
    # delete train_step's first dot (o16) and rebind its use in %2 = add
    # (o18) to the scalar %3: the variant fails verification
    bad = (DeleteEdit(uid="dead", function="train_step", target="o16",
                      rebinds=(Rebind("o18", 0, "%3"),)),)
    assert shims.evaluate(w.module, bad, w, backend=GoldenBackend()) == F.INVALID_FITNESS
    assert w.dataset.holdout.reads == 0


# --------------------------------------------------------------------------- GPU

def _ind(c, e):
    return types.SimpleNamespace(fitness=types.SimpleNamespace(as_tuple=lambda c=c, e=e: (c, e)),
                                 rank=None, crowding=None)


@pytest.mark.gpu
def test_nsga2_shims_match_reference_structures():
    from paper_2310_10211_b200 import shims
    for s in load("nsga2.json.gz")["sets"]:
        pts = [(float(c), float(e)) for c, e in s["points"]]
        fronts = shims.nondominated_sort(pts)
        assert fronts == s["fronts"]
        for fr, cr in zip(fronts, s["crowding"]):
            d = shims.crowding_distance(pts, fr)
            assert {i: repr(v) for i, v in d.items()} == {i: v for i, v in cr}
        pop = [_ind(c, e) for c, e in pts]
        shims.rank_population(pop)
        assert [p.rank for p in pop] == s["rank"]
        assert [repr(p.crowding) for p in pop] == s["crowd"]
        for n, chosen in s["survivors"].items():
            pool = [_ind(c, e) for c, e in pts]
            surv = shims.select_survivors(pool, int(n))
            assert [pool.index(x) for x in surv] == chosen
    assert shims.nondominated_sort([]) == [[]]
    assert shims.crowding_distance([(1.0, 2.0), (2.0, 1.0)], [0, 1]) == {0: math.inf, 1: math.inf}
