"""Population sharding over 2 ranks (gloo, CPU): LPT shards, one record
all-gather, merged fitness identical to the single-rank result.  The device
is replaced by the reference's recorded fitness table (see test_shims)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from golden_io import load, variant_functions
from paper_2310_10211_b200 import distributed as D


class TableBackend:
    def __init__(self):
        from paper_2310_10211_b200.dialect import format_function
        self.fmt = format_function
        self.table = {}
        for ind in load("train_pop.json.gz")["individuals"]:
            v = variant_functions(ind)
            self.table[(format_function(v["train_step"]), format_function(v["forward"]))] = ind
        self.seen = 0

    def evaluate_variants(self, variants, holdout=False, return_records=False):
        from paper_2310_10211_b200.workloads import Fitness, INVALID_FITNESS
        fits = []
        recs = np.zeros(len(variants), dtype=[("wrong", "<i8"), ("total", "<i8"),
                                               ("status", "<i4"), ("steps_run", "<i4"),
                                               ("cycles", "<i8"), ("t0_ns", "<i8"),
                                               ("t1_ns", "<i8"), ("smid", "<i4"),
                                               ("pad", "<i4")])
        for k, v in enumerate(variants):
            if v is None:
                fits.append(INVALID_FITNESS)
                continue
            ind = self.table[(self.fmt(v["train_step"]), self.fmt(v["forward"]))]
            fits.append(Fitness(ind["cost"], ind["error"]))
            if ind["error"] == 1.0:
                recs[k]["status"] = 1
            else:
                recs[k]["wrong"] = round(ind["error"] * 992)
                recs[k]["total"] = 992
        self.seen += len(variants)
        return (fits, recs) if return_records else fits


def test_lpt_shards_cover_and_balance():
    costs = [float(c) for c in np.random.default_rng(0).integers(1, 100, 257)]
    for world in (1, 2, 3, 8):
        shards = D.lpt_shards(costs, world)
        flat = sorted(i for s in shards for i in s)
        assert flat == list(range(len(costs)))
        loads = [sum(costs[i] for i in s) for s in shards]
        assert max(loads) - min(loads) <= max(costs)
        assert all(s == sorted(s) for s in shards)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inds = load("train_pop.json.gz")["individuals"]
        variants = [variant_functions(i) for i in inds] + [None]
        be = TableBackend()
        ev = D.ShardedEvaluator(be)
        fits = ev.evaluate_variants(variants)
        q.put((rank, [(f.cost, f.error, f.valid) for f in fits], be.seen,
               [len(s) for s in ev.last_shards]))
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_matches_single_rank():
    ctx = mp.get_context("fork")      # CPU-only: no CUDA state to inherit
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        out = [q.get(timeout=240) for _ in procs]
    finally:
        for p in procs:
            if p.is_alive():
                p.join(5)
            if p.is_alive():
                p.kill()
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    inds = load("train_pop.json.gz")["individuals"]
    want = [(i["cost"], i["error"], True) for i in inds] + [(float("inf"), float("inf"), False)]
    for rank, fits, seen, sizes in out:
        assert fits == want                       # every rank holds every fitness
        assert seen == sizes[rank]                # and evaluated only its shard
    assert sum(out[0][3]) == len(want)


class PatchTable:
    """Device stand-in with the patch interface (evaluate_patches): applies
    each patch with the reference's apply_patch and answers the reference's
    recorded fitness for the resulting program text."""

    def __init__(self, workload):
        self.workload = workload
        self.inner = TableBackend()
        self.keys = []

    def evaluate_patches(self, original, keys, functions, holdout=False, return_records=False):
        from evotir.genome import PatchApplicationError, apply_patch, patch_loads
        self.keys.extend(keys)
        variants = []
        for k in keys:
            try:
                m = apply_patch(original, patch_loads(k)).module
            except PatchApplicationError:
                variants.append(None)
                continue
            variants.append({n: m.functions[n] for n in functions})
        return self.inner.evaluate_variants(variants, return_records=return_records)


def _search_worker(rank, world, port, q):
    import torch.distributed as dist
    from golden_io import reference_available
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        assert reference_available()
        import evotir.search as S
        from evotir import fitness as F
        from paper_2310_10211_b200 import shims
        data = load("train_pop.json.gz")
        tables = []

        def factory(w):
            t = PatchTable(w)
            tables.append(t)
            return D.ShardedEvaluator(t)
        ref_holdout = S.holdout_report
        shims.install(nsga2=False, backend_factory=factory)
        S.holdout_report = ref_holdout     # the archive's holdout reports stay on the host here
        try:
            res = S.run_search(F.build_2fcnet_workload(), S.SearchConfig(**data["config"]))
        finally:
            shims.uninstall()
        keys = ("generation", "evaluations", "front_size", "best_error", "best_cost",
                "archive_size", "hypervolume", "archive_hypervolume")
        q.put((rank, [{k: h[k] for k in keys} for h in res.history], res.evaluations,
               len(tables[0].keys)))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not __import__("golden_io").reference_available(),
                    reason="reference package not importable")
def test_two_rank_run_search_under_install_reproduces_history():
    """configs[1]'s shape in miniature: the reference's run_search on two
    ranks with shims.install(), each generation's fresh patches sharded over
    the ranks and all-gathered -- the recorded history comes out on both."""
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_search_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        out = sorted(q.get(timeout=300) for _ in procs)
    finally:
        for p in procs:
            p.join(60)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    data = load("train_pop.json.gz")
    keys = ("generation", "evaluations", "front_size", "best_error", "best_cost",
            "archive_size", "hypervolume", "archive_hypervolume")
    want = [{k: h[k] for k in keys} for h in data["history"]]
    for rank, hist, evals, n_local in out:
        assert hist == want
        assert evals == len(data["individuals"])
    # each rank evaluated only its strided shard of every call
    assert out[0][3] + out[1][3] == len(data["individuals"])
    assert 0 < out[1][3] <= out[0][3]


@pytest.mark.gpu
def test_nccl_allgather_through_libgevo_single_rank():
    """libgevo's own NCCL path on the device (gevo_comm_unique_id /
    gevo_comm_init / gevo_allgather / gevo_comm_destroy; NCCL dlopen'ed on
    first use): a one-rank communicator returns the records it was given,
    and all_gather_records over it unpacks them like the torch path.  (The
    multi-rank exchange itself is covered over gloo above; one GPU per
    gpurun, no ranks that wait on each other on one device.)"""
    import torch.distributed as dist
    from paper_2310_10211_b200 import _lib
    ctx = _lib.Context(0)
    try:
        ctx.comm_init(0, 1, _lib.comm_unique_id())
        send = np.arange(4 * D.RECORD_FIELDS, dtype=np.int64).reshape(4, D.RECORD_FIELDS)
        out = ctx.allgather(send, 1)
        assert out.shape == (1, 4, D.RECORD_FIELDS) and np.array_equal(out[0], send)
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
        try:
            local = send[:3]
            recs, counts = D.all_gather_records(local, 5, ctx=ctx)
            assert counts.tolist() == [3] and np.array_equal(recs[0, :3], local)
        finally:
            dist.destroy_process_group()
        ctx.comm_destroy()
    finally:
        ctx.close()
