"""Device fitness evaluator: the reference's evaluate()/holdout_report() for
a whole list of variants in one libgevo call.

Protocol restated from pkg/src/evotir/fitness.py:372-426:
  * invalid patch (apply/verify failure)     -> INVALID_FITNESS (inf, inf)
  * cost = static cost(train_step) * steps   (training)
         = static cost(forward) * batches    (prediction; holdout batches
                                              for holdout_report)
  * non-finite weights at a check step or at the end, or non-finite
    probabilities on any scored batch      -> Fitness(cost, 1.0)
  * otherwise error = wrong / total, divided here in Python so the float
    is the reference's own.
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import _lib
from .plan import (UnsupportedVariant, build_population_plan, device_weight, layout_order,
                   lower_variant, sm_aware_order)
from .workloads import (INVALID_FITNESS, PREDICTION, TRAINING, WEIGHT_NAMES,
                        Fitness, Workload)

SPLIT_SEARCH, SPLIT_HOLDOUT = 0, 1
STATUS_OK, STATUS_NONFINITE_WEIGHTS, STATUS_NONFINITE_PROBS = 0, 1, 2
POOL_MIN = 32          # variants below which lowering stays in-process
_POOL = None
# original modules the workers apply patches to (evaluate_patches): a
# worker inherits this table when it is forked, so a module registered after
# the pool was created re-forks the pool once
_MODULES: dict = {}
_POOL_TOKENS: frozenset = frozenset()


def register_module(module) -> str:
    """Make `module` (an evotir Module: the workload's original program)
    available to the lowering workers; returns its token."""
    tok = f"m{id(module):x}"
    if _MODULES.get(tok) is not module:
        _MODULES[tok] = module
    return tok


def _lower_pool(token=None):
    """Process pool for host work (pure Python/numpy, GIL-bound): one worker
    per core, created once (re-forked when `token` names a module the
    workers have not inherited).  Workers are forked (no re-import of
    __main__) and only apply patches and lower -- they never touch CUDA.
    GEVO_B200_LOWER_WORKERS=1 disables it."""
    global _POOL, _POOL_TOKENS
    if _POOL and token is not None and token not in _POOL_TOKENS:
        _POOL.shutdown(wait=False, cancel_futures=True)
        _POOL = None
    if _POOL is None:
        _POOL_TOKENS = frozenset(_MODULES)
        # one share of the host's cores per local rank (torchrun sets
        # LOCAL_WORLD_SIZE; every rank of a node lowers its own shard)
        share = (os.cpu_count() or 1) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
        n = int(os.environ.get("GEVO_B200_LOWER_WORKERS", min(16, max(1, share))))
        if n <= 1:
            _POOL = False
        else:
            import multiprocessing as mp
            import warnings
            from concurrent.futures import ProcessPoolExecutor
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", DeprecationWarning)
                _POOL = ProcessPoolExecutor(n, mp_context=mp.get_context("fork"))
    return _POOL or None


def _lower_many(batch):
    """Worker: lower a list of variants; None for a variant that fails
    (evaluate() maps any exception to INVALID_FITNESS), the exception itself
    for a valid variant the device cannot run (raised by the caller)."""
    fns_list, cost_table, training, steps = batch[:4]
    fwd_memo = batch[4] if len(batch) > 4 else None
    out = []
    for fns in fns_list:
        try:
            out.append(lower_variant(fns, cost_table, training=training, steps=steps,
                                     fwd_memo=fwd_memo))
        except UnsupportedVariant as e:
            out.append(e)
        except Exception:
            out.append(None)
    return out


def _lower_patches(batch):
    """Worker: the body of the reference's evaluate() up to execution, for a
    list of patches (canonical patch JSON, genome.py:302-309): apply_patch +
    verify (genome.py:482-516) -- a PatchApplicationError is the reference's
    INVALID_FITNESS (fitness.py:375-377), None here -- then lowering."""
    token, keys, functions, cost_table, training, steps = batch
    from evotir.genome import PatchApplicationError, apply_patch, patch_loads
    original = _MODULES[token]
    # a patch that edits no op of @forward leaves it the original's function:
    # its encoded lowering is shared per (module, cost table, weight layout)
    memo = _FWD_MEMO.setdefault((token, repr(sorted(cost_table.items())) if cost_table else None,
                                 training, steps), {})
    out = []
    for key in keys:
        try:
            patch = patch_loads(key)
            m = apply_patch(original, patch).module
        except PatchApplicationError:
            out.append(None)
            continue
        untouched = "forward" in functions and all(e.function != "forward" for e in patch)
        out.extend(_lower_many(([{n: m.functions[n] for n in functions}],
                                cost_table, training, steps, memo if untouched else None)))
    return out


_FWD_MEMO: dict = {}      # per worker process: see _lower_patches


def _check_supported(vp):
    if isinstance(vp, UnsupportedVariant):
        raise _lib.GevoError(str(vp))
    return vp


def _submit_lowering(variants, idx, cost_table, training, steps=600, patches=None):
    """Start lowering variants[idx] (None entries excluded by the caller), or
    -- with patches=(token, keys, functions) -- applying and lowering
    keys[idx] in the workers.  Returns a list of (positions, future-or-result)
    in idx order."""
    if patches is not None:
        token, keys, functions = patches
        fn = _lower_patches
        args = lambda c: (token, [keys[i] for i in c], functions, cost_table, training, steps)
    else:
        fn = _lower_many
        args = lambda c: ([variants[i] for i in c], cost_table, training, steps)
    pool = _lower_pool(patches[0] if patches else None) if len(idx) >= POOL_MIN else None
    if pool is None:
        return [(list(idx), fn(args(idx)))]
    nw = pool._max_workers
    per = max(4, (len(idx) + 2 * nw - 1) // (2 * nw))
    out = []
    for k in range(0, len(idx), per):
        c = idx[k:k + per]
        out.append((c, pool.submit(fn, args(c))))
    return out


def _collect(jobs):
    pos, res = [], []
    for c, f in jobs:
        pos.extend(c)
        res.extend(f if isinstance(f, list) else f.result())
    return pos, res


def _arena_budget() -> float:
    """GEVO_B200_ARENA_GB (default 80: 64 GB of requested scratch) in bytes.  The
    library's buffers grow to request + 25 % (DevBuf::ensure, gevo_abi.cu),
    so the grouping budget is the knob / 1.25: the device footprint stays
    within the figure (approximately: growth briefly holds the old buffer
    too, stream-ordered)."""
    return float(os.environ.get("GEVO_B200_ARENA_GB", "80")) * 1e9 / 1.25


def lower_all(variants, cost_table, training, steps=600):
    """lower_variant over a list (None entries stay None), in the process
    pool when the list is large."""
    idx = [i for i, v in enumerate(variants) if v is not None]
    out = [None] * len(variants)
    for i, r in zip(*_collect(_submit_lowering(variants, idx, cost_table, training, steps))):
        out[i] = _check_supported(r)
    return out


def upload_split(ctx, split_id, split, classes, batch):
    """Put a SplitView on the device (datasets.py:149-162 semantics).  Byte
    sources cross as bytes and are decoded on the device: CIFAR records
    (`split.records`), pixel bytes (`split.raw`), or the bytes recovered from
    an exactly byte-scaled float64 x (evotir's own splits); anything else is
    uploaded as float64."""
    from . import datasets as D
    records = getattr(split, "records", None)
    if records is not None:
        ctx.upload_split_cifar(split_id, records, D.CIFAR_CHANNELS, D.CIFAR_SIDE, classes, batch)
        return "cifar"
    raw = getattr(split, "raw", None)
    if raw is None:
        raw = D.pixel_bytes(split.x)
    if raw is not None:
        ctx.upload_split_u8(split_id, raw, split.labels, classes, batch)
        return "u8"
    ctx.upload_split(split_id, split.x, split.labels, classes, batch)
    return "f64"


class DeviceEvaluator:
    """Owns one device context with the workload's splits and weights
    resident; evaluates lists of variant programs.

    `workload` is this package's `Workload` or anything with the same
    attributes (see shims.device_workload for evotir's)."""

    def __init__(self, workload: Workload, device: int = 0):
        self.workload = workload
        self.device = device
        self.ctx = _lib.Context(device)
        self.n_sms = self.ctx.num_sms()
        cfg = workload.config
        self.batch, self.classes = cfg.batch_size, cfg.classes
        ds = workload.dataset
        upload_split(self.ctx, SPLIT_SEARCH, ds.search, cfg.classes, cfg.batch_size)
        self.n_search_batches = len(ds.search.labels) // cfg.batch_size
        self._holdout_batches = None
        # weight arrays in parameter order (w1, b1, w2, b2 for 2fcNet; the
        # flat vector w for the CNN)
        self.weight_names = list(workload.weights)
        w = [np.ascontiguousarray(workload.weights[n], dtype=np.float64)
             for n in self.weight_names]
        self.weight_shapes = [a.shape for a in w]
        self.ctx.upload_weights(np.concatenate([a.reshape(-1) for a in w]))
        self.weight_elems = int(sum(a.size for a in w))
        self._flat_weights = np.concatenate([a.reshape(-1) for a in w])
        self._extra = {}           # chunk k >= 1 -> its own context (_context)
        self._sm_layout = {}
        self.last_timing = {}
        self.last_plan_bytes = 0
        self.last_device_ms = 0.0
        self.launches = 0          # gevo_eval launches so far (bench: gpu_launches)

    def _learn_layout(self, res, order):
        """Remember which launch slots shared an SM (records carry the SM id
        of every CTA) for the next launch of the same size."""
        sm = res["smid"][np.asarray(order)]
        groups = {}
        for block, s in enumerate(sm.tolist()):
            groups.setdefault(s, []).append(block)
        self._sm_layout[len(order)] = list(groups.values())

    def _context(self, k):
        """Context of chunk k of a generation: chunk 0 uses the evaluator's
        own; chunk k >= 1 gets a context of its own (stream and buffers) on
        the same device, so chunk k runs on the device while the host still
        lowers chunk k + 1."""
        if k == 0:
            return self.ctx
        if k not in self._extra:
            c = _lib.Context(self.device)
            ds, cfg = self.workload.dataset, self.workload.config
            upload_split(c, SPLIT_SEARCH, ds.search, cfg.classes, cfg.batch_size)
            if self._holdout_batches is not None:
                upload_split(c, SPLIT_HOLDOUT, ds.holdout, cfg.classes, cfg.batch_size)
            c.upload_weights(self._flat_weights)
            self._extra[k] = c
        return self._extra[k]

    def _ensure_holdout(self):
        if self._holdout_batches is None:
            ds, cfg = self.workload.dataset, self.workload.config
            # holdout.reads is bumped by the holdout_report seam, once per
            # report like the reference (fitness.py:407); the upload is not a
            # report
            for c in [self.ctx] + list(self._extra.values()):
                upload_split(c, SPLIT_HOLDOUT, ds.holdout, cfg.classes, cfg.batch_size)
            self._holdout_batches = len(ds.holdout.labels) // cfg.batch_size
        return self._holdout_batches

    # ------------------------------------------------------------------
    def evaluate_patches(self, original, keys, functions, holdout=False,
                         return_records=False):
        """The reference's evaluate() (fitness.py:372-393) for a list of
        patches given as canonical patch JSON (genome.patch_dumps, the
        _Evaluator cache keys): apply_patch, verification and lowering run in
        the worker processes, so the parent only packs and launches."""
        return self.evaluate_variants(keys, holdout=holdout, return_records=return_records,
                                      _patches=(register_module(original), list(keys),
                                                list(functions)))

    def evaluate_variants(self, variants, holdout=False, want_weights=False,
                          return_records=False, _patches=None):
        """variants: list of {'train_step': fn, 'forward': fn} (or None for
        a patch that failed to apply).  Returns list[Fitness] (and the raw
        device records when return_records).  One NVTX range per call."""
        with _lib.nvtx_range(f"evaluate {len(variants)} individuals"
                             + (" (holdout)" if holdout else "")):
            return self._evaluate_variants(variants, holdout, want_weights, return_records, _patches)

    def _evaluate_variants(self, variants, holdout, want_weights, return_records, _patches):
        wl = self.workload
        cfg = wl.config
        training = wl.mode == TRAINING
        t0 = time.perf_counter()
        n_score = self._ensure_holdout() if holdout else self.n_search_batches
        if holdout and n_score == 0:
            from .workloads import WorkloadError
            raise WorkloadError("holdout split smaller than one batch")
        fits = [None] * len(variants)
        idx = []
        for i, v in enumerate(variants):
            if v is None:
                fits[i] = INVALID_FITNESS      # patch failed to apply
            else:
                idx.append(i)
        records = np.zeros(len(variants), dtype=_lib.RESULT_DTYPE)
        finals = [None] * len(variants) if want_weights else None
        split = SPLIT_HOLDOUT if holdout else SPLIT_SEARCH
        # chunks when the pool is used (GEVO_B200_CHUNKS, default 2): chunk k
        # runs on the device (ctypes releases the GIL) while chunk k + 1 is
        # still being lowered
        halves = [idx]
        n_chunks = int(os.environ.get("GEVO_B200_CHUNKS", "2"))
        if os.environ.get("GEVO_B200_HALVES", "1") == "0":
            n_chunks = 1
        n_chunks = max(1, min(n_chunks, len(idx) // POOL_MIN))
        if n_chunks > 1 and _lower_pool(_patches[0] if _patches else None) is not None:
            bounds = [len(idx) * k // n_chunks for k in range(n_chunks + 1)]
            halves = [idx[bounds[k]:bounds[k + 1]] for k in range(n_chunks)]
        jobs = [_submit_lowering(variants, h, cfg.cost_table, training, cfg.steps, _patches)
                for h in halves]
        ctxs = [self._context(k) for k in range(len(halves))]
        runners, box, launches, failed = [], {}, {}, {}
        t_lower = t_pack = 0.0
        plan_bytes = 0
        for h, job in enumerate(jobs):
            ta = time.perf_counter()
            pos, vps = _collect(job)
            tb = time.perf_counter()
            lowered, slots = [], []
            for i, vp in zip(pos, vps):
                vp = _check_supported(vp)
                if vp is None:
                    fits[i] = INVALID_FITNESS  # evaluate(): any exception
                else:
                    lowered.append(vp)
                    slots.append(i)
            if not lowered:
                continue
            # launches of this half: one, unless the individuals' device
            # scratch exceeds the budget (a large CNN population), then
            # consecutive groups that each fit, run one after another
            groups = self._scratch_groups(lowered, len(halves))
            plans = []
            for g0, g1 in groups:
                gl = lowered[g0:g1]
                wts = [device_weight(v, cfg.steps if training else 0, n_score) for v in gl]
                parts = 1 if training else self.score_parts(gl, n_score, len(idx) if len(groups) == 1 else None,
                                                            shares=len(halves))
                if parts > 1:
                    order = np.argsort(-np.asarray(wts), kind="stable")
                else:
                    layout = self._sm_layout.get(len(gl))
                    order = layout_order(wts, layout) if layout else sm_aware_order(wts, self.n_sms)
                plan = build_population_plan(gl, self.weight_shapes, self.batch * self.classes,
                                             order=order, parts=parts)
                plan_bytes += plan.blob.nbytes
                plans.append((plan, order if parts == 1 and len(groups) == 1 else None, g1 - g0))
            tc = time.perf_counter()
            t_lower += tb - ta
            t_pack += tc - tb
            mode_args = (0 if training else 1, cfg.steps if training else 0,
                         cfg.finite_check_every, SPLIT_SEARCH, split, self.weight_elems, want_weights)

            def run(c=ctxs[h], pl=plans, ma=mode_args, key=h, lv=lowered, sl=slots):
                try:
                    recs, fws, od, ms = [], [], None, 0.0
                    for plan, order_, n_g in pl:
                        with _lib.nvtx_range(f"chunk {key}: {n_g} individuals"):
                            res, fw = c.eval(plan.blob, plan.n_prog, *ma)
                        ms += c.last_kernel_ms()
                        recs.append(res[:n_g])
                        fws.append(fw[:n_g] if fw is not None else None)
                        od = order_
                    res = np.concatenate(recs)
                    fw = np.concatenate(fws) if fws and fws[0] is not None else None
                    box[key] = ((res, fw), lv, sl, od)
                    launches[key] = (len(pl), ms)
                except BaseException as e:   # re-raised by the caller after join
                    failed[key] = e
            if h + 1 < len(jobs):
                import threading
                runners.append(threading.Thread(target=run))
                runners[-1].start()
            else:
                run()
        for r in runners:
            r.join()
        if failed:
            # a device failure in either half is loud, never a missing fitness
            raise failed[min(failed)]
        used = sorted(box)
        self.launches += sum(launches[k][0] for k in used)
        if any(launches[k][0] > 1 for k in used):
            # consecutive launches (scratch budget): kernel time summed per
            # half; the halves run concurrently
            self.last_device_ms = max(launches[k][1] for k in used)
        elif len(used) >= 2:
            self.last_device_ms = max(_lib.span_ms(ctxs[used[0]], ctxs[k]) for k in used[1:])
        elif used:
            self.last_device_ms = ctxs[used[0]].last_kernel_ms()
        for key in used:
            (res, fw), lowered, slots, order = box[key]
            res = res[:len(lowered)]          # records by result slot (score parts merged)
            if order is not None:
                self._learn_layout(res, order)
            records[np.asarray(slots, dtype=np.int64)] = res
            status, wrong, total = (res["status"].tolist(), res["wrong"].tolist(),
                                    res["total"].tolist())
            for k, vp in enumerate(lowered):
                i = slots[k]
                cost = vp.train_cost * cfg.steps if training else vp.fwd_cost * n_score
                if status[k] != STATUS_OK:
                    fits[i] = Fitness(cost, 1.0)
                else:
                    fits[i] = Fitness(cost, wrong[k] / total[k])
                if want_weights:
                    finals[i] = fw[k]
        missing = [i for i, f in enumerate(fits) if f is None]
        if missing:
            raise _lib.GevoError(f"no fitness for variants {missing[:8]} (internal error)")
        self.last_plan_bytes = plan_bytes
        self.last_timing = {"lower_wait_s": t_lower, "pack_s": t_pack,
                            "total_s": time.perf_counter() - t0, "n": len(idx),
                            "halves": len(halves)}
        out = [fits]
        if return_records:
            out.append(records)
        if want_weights:
            out.append(finals)
        return out[0] if len(out) == 1 else tuple(out)

    def _scratch_groups(self, lowered, shares=1):
        """[g0, g1) ranges of `lowered` whose device scratch (arena, probs
        and weight ping-pong per individual) fits the scratch budget
        (_arena_budget) split over `shares` concurrent launches."""
        budget = _arena_budget() / max(1, shares)
        fixed = 8 * (((self.batch * self.classes + 15) & ~15) + 2 * ((self.weight_elems + 15) & ~15))
        groups, g0, acc = [], 0, 0
        for k, v in enumerate(lowered):
            b = 8 * ((v.arena + 15) & ~15) + fixed
            if k > g0 and acc + b > budget:
                groups.append((g0, k))
                g0, acc = k, 0
            acc += b
        groups.append((g0, len(lowered)))
        return groups

    def score_parts(self, lowered, n_score, n_total=None, shares=1):
        """Programs per prediction-mode individual (plan.build_population_plan
        `parts`): enough to give the launch two CTAs per SM, at most one per
        scored batch, and within GEVO_B200_ARENA_GB (default 80, i.e. 64 GB requested) of scratch.
        `n_total` is the call's individual count when this launch holds one
        half of it (the halves run concurrently).  GEVO_B200_PARTS overrides."""
        n = len(lowered)
        if n == 0 or n_score <= 1:
            return 1
        env = os.environ.get("GEVO_B200_PARTS")
        if env:
            return max(1, min(int(env), n_score))
        parts = max(1, min(n_score, (2 * self.n_sms) // max(n, n_total or 0)))
        per = sum(8 * ((v.arena + 15) & ~15) for v in lowered) + \
            8 * n * (self.batch * self.classes + 2 * self.weight_elems + 48)
        budget = _arena_budget() / max(1, shares)
        while parts > 1 and parts * per > budget:
            parts -= 1
        return parts

    def split_weights(self, flat):
        out, o = {}, 0
        for name, shape in zip(self.weight_names, self.weight_shapes):
            n = int(np.prod(shape))
            out[name] = np.array(flat[o:o + n]).reshape(shape)
            o += n
        return out

    # NSGA-II ------------------------------------------------------------
    def nsga2_rank(self, points):
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 2)
        return self.ctx.nsga2_rank(pts[:, 0], pts[:, 1])

    def nsga2_select(self, points, keep):
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 2)
        return self.ctx.nsga2_select(pts[:, 0], pts[:, 1], keep)

    def close(self):
        self.ctx.close()
        for c in self._extra.values():
            c.close()
        self._extra = {}


def baseline_functions(workload: Workload) -> dict:
    m = workload.module
    return {n: m.functions[n] for n in ("forward", "train_step")
            if n in m.functions}


def train_baseline_weights(workload: Workload, device: int = 0) -> dict:
    """Weights after training the unmutated program (fitness.py:265-270),
    on the device."""
    from .workloads import WorkloadError
    ev = DeviceEvaluator(workload, device)
    try:
        (fit,), recs, (flat,) = ev.evaluate_variants(
            [baseline_functions(workload)], want_weights=True,
            return_records=True)
        # the reference refuses to freeze weights that went non-finite at a
        # check step or at the end (fitness.py:266-269)
        if int(recs[0]["status"]) != STATUS_OK or not fit.valid:
            raise WorkloadError("baseline training diverged; cannot freeze")
        return ev.split_weights(flat)
    finally:
        ev.close()
