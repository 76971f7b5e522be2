"""Population plan: many lowered variants packed into one launch blob.

One `PopulationPlan` per evaluator call (a generation's fresh individuals):
the per-individual `ExecPlan` objects of the reference (interpreter.py:
188-239, cached per FunctionBody) become rows of a single instruction table
that the device executor walks, one CTA per individual.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import layout as L
from .lowering import (BUF_OUT0, FLAG_ALTERNATE, FLAG_INPLACE_SHIFT, HEADER_DTYPE, MAXP,
                       SCHED_ALT01, SCHED_ALT12, SCHED_STEADY1, SCHED_STEADY2,
                       INSTR_DTYPE, PLAN_MAGIC, PLAN_VERSION, PROG_DTYPE,
                       consts_to_words, encode_instrs, lower_function,
                       static_cost)


class UnsupportedVariant(Exception):
    """A valid variant this executor cannot run bit-exactly.  Never mapped to
    a fitness: the evaluator raises it as a GevoError (no silent
    approximation, no fallback)."""


@dataclass
class VariantPlan:
    """Lowered functions of one individual, already encoded (gevo_instr
    arrays with CONST offsets relative to this individual's pool)."""
    train0: np.ndarray | None
    train1: np.ndarray | None     # same object as train0 when identical
    fwd: np.ndarray
    consts: np.ndarray            # 64-bit words
    arena: int
    smem: int
    flags: int
    train_cost: float
    fwd_cost: float
    w_train: float = 0.0          # fn_weight(train1) / fn_weight(fwd), computed where
    w_fwd: float = 0.0            # the variant is lowered (a pool worker), not in the parent
    train2: np.ndarray | None = None   # third layout's program (GEVO_SCHED_STEADY2 / ALT12)


def _count(shape):
    n = 1
    for d in shape:
        n *= d
    return n


def lower_variant(functions: dict, cost_table=None, training=True,
                  weight_layouts=None, steps: int = 600, fwd_memo: dict | None = None) -> VariantPlan:
    """functions: {'train_step': fn, 'forward': fn} (train_step only in
    training mode).  Weight params start C-ordered like the module
    constants; steps >= 1 see the layout the previous step stored, and
    @forward is lowered for the layout after `steps` training steps.

    fwd_memo: given only when `forward` is the same function for every
    variant lowered through this dict (a patch that edits no op of @forward,
    genome.py:482-516, with one cost table): the encoded forward is then
    reused per weight layout instead of lowered again."""
    consts: list = []
    arena = 0
    smem = 0
    flags = 0
    t0 = t1 = t2 = None
    train_cost = 0.0
    fwd_layouts = weight_layouts
    if training:
        ts = functions["train_step"]
        nw = len(ts.returns)
        c_layout = [L.c_strides(tuple(t.shape)) for _, t in ts.params]
        low0 = lower_function(ts, c_layout, cost_table=cost_table)
        train_cost = low0.cost
        L0 = list(low0.ret_strides)
        low2 = None
        C = list(c_layout[:nw])

        def lower_for(lay):
            layouts = list(c_layout)
            layouts[:nw] = lay
            return lower_function(ts, layouts, cost_table=cost_table)
        # follow the weights' layouts to their cycle: step s reads the layout
        # step s-1 stored (gevo_plan.h GEVO_SCHED_*)
        if L0 == C:
            low1, sched, after = low0, SCHED_STEADY1, lambda n: L0
        else:
            low1 = lower_for(L0)
            L1 = list(low1.ret_strides)
            if L1 == L0:
                sched, after = SCHED_STEADY1, lambda n: L0
            elif L1 == C:
                # period 2: even steps read C order (train0) and store L0,
                # odd steps read L0 (train1) and store C order
                sched, after = SCHED_ALT01, lambda n: L0 if (n - 1) % 2 == 0 else L1
            else:
                low2 = lower_for(L1)
                L2 = list(low2.ret_strides)
                if L2 == L1:
                    # settles from step 2: C -> L0 -> L1 -> L1 ...
                    sched, after = SCHED_STEADY2, lambda n: L0 if n == 1 else L1
                elif L2 == L0:
                    # period 2 from step 1: L0 -> L1 -> L0 ...
                    sched, after = SCHED_ALT12, lambda n: L0 if (n - 1) % 2 == 0 else L1
                else:
                    # C -> L0 -> L1 -> L2 with L2 not in {L0, L1}: never seen
                    # in any recorded population.  The summation orders of
                    # later steps depend on those layouts, so refuse loudly
                    # rather than run any step with the wrong program.
                    raise UnsupportedVariant(
                        "train_step returns weight layouts that do not cycle within three steps "
                        f"(step 0 -> {L0}, step 1 -> {L1}, step 2 -> {L2}); not supported by "
                        "the device executor")
        flags |= sched
        final = after(steps) if steps > 0 else C
        t0 = _encode_shifted(low0, consts)
        t1 = t0 if low1 is low0 else _encode_shifted(low1, consts)
        t2 = None if low2 is None else _encode_shifted(low2, consts)
        if sched == SCHED_STEADY1 and INPLACE:
            flags |= inplace_weights(t1, nw) << FLAG_INPLACE_SHIFT
        arena = max(low0.arena_elems, low1.arena_elems, low2.arena_elems if low2 else 0)
        smem = max(low0.smem_elems, low1.smem_elems, low2.smem_elems if low2 else 0)
        fwd_layouts = final
    fw = functions["forward"]
    nwf = len(fw.params) - 1
    f_layout = [L.c_strides(tuple(t.shape)) for _, t in fw.params]
    if fwd_layouts is not None:
        f_layout[:nwf] = fwd_layouts[:nwf]
    key = tuple(tuple(x) for x in f_layout)
    hit = fwd_memo.get(key) if fwd_memo is not None else None
    if hit is None:
        lowf = lower_function(fw, f_layout, ret_layout="c", cost_table=cost_table)
        arr = encode_instrs(lowf.instrs)
        hit = (list(lowf.consts), arr, lowf.arena_elems, lowf.smem_elems, lowf.cost, fn_weight(arr))
        if fwd_memo is not None:
            fwd_memo[key] = hit
    f_consts, f_arr, f_arena, f_smem, f_cost, f_weight = hit
    f = _shift_consts(f_arr.copy(), len(consts))
    consts.extend(f_consts)
    arena = max(arena, f_arena)
    smem = max(smem, f_smem)
    return VariantPlan(t0, t1, f, consts_to_words(consts), arena, smem, flags,
                       train_cost, f_cost, fn_weight(t1), f_weight, t2)


# in-place weight updates (inplace_weights); GEVO_B200_INPLACE=0 turns them off
INPLACE = os.environ.get("GEVO_B200_INPLACE", "1") != "0"
_NIN = {1: 1, 2: 2, 3: 3, 4: 1, 5: 2, 6: 2, 8: 2}   # main operands per op class


def inplace_weights(arr, nw) -> int:
    """Bit w set: @train_step (the program of steps >= 1) may update weight w
    in place -- its parameter and its return sharing one HBM block instead
    of ping-ponging (gevo_plan.h GEVO_FLAG_INPLACE_SHIFT).  Safe when
      * exactly one instruction W writes return w, and W is elementwise
        (UNARY / BINARY / SELECT, fused chains included) or a DOT;
      * W reads parameter w only at the very word it writes (offset and
        strides equal to its output's), a DOT only in its epilogue;
      * no instruction after W reads parameter w.
    Then every word of the parameter is read, at the latest, by the thread
    that overwrites it, inside W.  The layout the next step reads is the one
    W stores either way (the returned layout is a fixed point of the
    program of steps >= 1).  `arr` is the encoded table, EXT records
    included."""
    # per record: its group (the main record it belongs to; EXT records,
    # op 7, follow their main record) and which of its operands it reads
    ops = np.asarray(arr["op"])
    main = ops != 7
    grp = np.cumsum(main) - 1
    inbuf = np.asarray(arr["in"]["buf"])                     # (n, 3)
    nin = np.array([_NIN.get(int(o), 0) for o in ops]) if len(ops) else np.zeros(0, int)
    live = np.where(main[:, None], np.arange(3)[None, :] < nin[:, None], True)
    outbuf = np.asarray(arr["out"]["buf"])
    main_idx = np.flatnonzero(main)
    mask = 0
    for w in range(nw):
        P, O = 2 + w, 2 + MAXP + w
        writers = main_idx[outbuf[main_idx] == O]
        if len(writers) != 1:
            continue
        k_w = int(writers[0])
        g_w = int(grp[k_w])
        W = arr[k_w]
        op = int(W["op"])
        if op not in (1, 2, 3, 5):
            continue
        reads_p = (inbuf == P) & live                            # (n, 3)
        rec_reads = reads_p.any(axis=1)
        if (rec_reads & (grp > g_w)).any():                      # read after the update
            continue
        rank = 2 if op == 5 else int(W["rank"])

        def key(v, is_ext):
            # the word an operand reads for output index (r, c) of a rank <= 2
            # instruction (EXT operands are 2-D views, main operands of a
            # rank-1 instruction address c with st[0]); rank > 2: the N-d walk
            st = [int(x) for x in v["st"]]
            if rank > 2:
                return int(v["off"]), tuple(st[:rank])
            if is_ext or rank == 2:
                return int(v["off"]), (st[0], st[1])
            return int(v["off"]), (0, st[0] if rank == 1 else 0)
        out_key = key(W["out"], False)
        ok = True
        for k in np.flatnonzero(rec_reads & (grp == g_w)):      # W's own reads of P
            is_ext = not main[k]
            if op == 5 and not is_ext:                           # a DOT operand (i, k) / (k, j)
                ok = False
                break
            for j in np.flatnonzero(reads_p[k]):
                if key(arr[k]["in"][j], is_ext) != out_key:
                    ok = False
                    break
            if not ok:
                break
        if ok:
            mask |= 1 << w
    return mask


def _encode_shifted(low, pool):
    """Encode a function's instructions with its constants appended to the
    individual's pool (CONST operand offsets rebased)."""
    base = len(pool)
    pool.extend(low.consts)
    return _shift_consts(encode_instrs(low.instrs), base)


def _shift_consts(arr, base):
    """Rebase the CONST operand offsets of an encoded function by `base`."""
    if base:
        for slot in ("out", "in"):
            bufs = arr[slot]["buf"]
            offs = arr[slot]["off"]
            offs[bufs == 1] += base        # BUF_CONST
    return arr


OP_DOT = 5
# relative device cost of a MAC per summation order (measured on B200 with
# tests/tools/stragglers.py: FMA chain on DMMA; ACC8 runs its 8 chains in
# 16-column passes; numpy's no-FMA loop and integer dots are scalar)
_MODE_WEIGHT = {0: 1.0, 1: 2.0, 3: 2.0, 2: 3.0}


def fn_weight(arr) -> float:
    """Estimated device time of one invocation of an encoded function: dot
    MACs weighted by the kernel path their summation order takes, plus
    element counts of the other instructions."""
    if arr is None or len(arr) == 0:
        return 0.0
    op = arr["op"].astype(np.int64)
    shp = arr["shp"].astype(np.float64)
    aux = arr["aux"].astype(np.int64)
    dot = op == OP_DOT
    w = 0.0
    if dot.any():
        m, n, k = shp[dot, 0], shp[dot, 1], aux[dot, 0].astype(np.float64)
        split = np.minimum(aux[dot, 1].astype(np.float64), n)
        w1 = _MODE_LUT[np.clip(arr["sub"][dot].astype(np.int64), 0, 4)]
        w2 = _MODE_LUT[np.clip(aux[dot, 2], 0, 4)]
        w += float(np.sum(m * k * (split * w1 + (n - split) * w2) + 20000.0))
    other = ~dot & (op != 7)
    if other.any():
        w += float(np.sum(4.0 * arr["n"][other].astype(np.float64) + 4000.0))
    return w


_MODE_LUT = np.array([_MODE_WEIGHT.get(i, 3.0) for i in range(5)])


def device_weight(v: VariantPlan, steps: int = 600, batches: int = 31) -> float:
    """Estimated device time of one individual over its train and scoring
    invocations (per-function weights from lowering time)."""
    return steps * v.w_train + batches * v.w_fwd


def sm_aware_order(weights, n_sms: int):
    """Launch order for a one-wave launch of n <= 2 * n_sms CTAs.  Blocks are
    dealt to SMs in index order, so blocks n - n_sms .. n_sms - 1 get an SM to
    themselves while block i < n - n_sms shares one with block n_sms + i.  The
    heaviest individuals take the solo SMs; the rest pair heaviest with
    lightest, so the slowest CTA -- the launch time -- is as short as it can
    be.  Falls back to heaviest-first outside one wave."""
    w = np.asarray(weights, dtype=np.float64)
    n = len(w)
    by = list(np.argsort(-w, kind="stable"))
    if n <= n_sms or n > 2 * n_sms:
        return np.asarray(by)
    pairs = n - n_sms                       # SMs hosting two blocks
    solo = n_sms - pairs
    order = np.zeros(n, dtype=np.int64)
    order[pairs:n_sms] = by[:solo]          # heaviest run alone
    rest = by[solo:]                        # 2 * pairs individuals, heaviest first
    for i in range(pairs):
        order[i] = rest[i]                  # heavy ...
        order[n_sms + i] = rest[-1 - i]     # ... paired with light
    return order


def layout_order(weights, groups):
    """Launch order from an observed block -> SM layout: `groups` lists the
    block ids that shared an SM in an earlier launch of the same size.
    Heaviest individuals go to the blocks that had an SM alone; the rest are
    paired heaviest with lightest on the shared SMs."""
    w = np.asarray(weights, dtype=np.float64)
    by = list(np.argsort(-w, kind="stable"))
    order = np.full(len(w), -1, dtype=np.int64)
    alone = sorted(b for g in groups if len(g) == 1 for b in g)
    shared = [g for g in groups if len(g) > 1]
    k = 0
    for b in alone:
        order[b] = by[k]
        k += 1
    rest = by[k:]
    lo, hi = 0, len(rest) - 1
    for g in shared:
        for j, b in enumerate(sorted(g)):
            if lo > hi:
                break
            if j % 2 == 0:
                order[b] = rest[lo]
                lo += 1
            else:
                order[b] = rest[hi]
                hi -= 1
    assert (order >= 0).all() and len(set(order.tolist())) == len(w)
    return order


@dataclass
class PopulationPlan:
    blob: np.ndarray          # uint8 bytes handed to gevo_eval
    n_prog: int
    order: np.ndarray         # launch order (individual index per CTA)
    total_elems: int


FLAG_PART_SHIFT = 8        # gevo_plan.h GEVO_FLAG_PART / GEVO_FLAG_NPARTS
FLAG_NPARTS_SHIFT = 20
MAX_PARTS = 0x7FF


def build_population_plan(variants: list[VariantPlan], weight_shapes,
                          probs_elems: int, order=None, parts: int = 1) -> PopulationPlan:
    """Pack variants into one blob.  `order` is the launch order (CTA i runs
    individual order[i]); by default longest static cost first, so the
    slowest individuals start in the first wave.

    parts > 1 (prediction mode only): each individual becomes `parts`
    programs sharing its result slot, part j scoring batches j, j + parts,
    ... on its own CTA and scratch (gevo_eval merges the records).  CTAs go
    part-major, so the first wave holds part 0 of every individual."""
    n = len(variants)
    if order is None:
        key = np.array([v.train_cost * 1.0 + v.fwd_cost for v in variants])
        order = np.argsort(-key, kind="stable")
    parts = int(parts)
    if not 1 <= parts <= MAX_PARTS:
        raise ValueError(f"score parts {parts} outside 1..{MAX_PARTS}")
    if parts > 1 and any(v.train0 is not None for v in variants):
        raise ValueError("score parts apply to prediction plans only")
    if parts > 1:
        order = [int(i) for j in range(parts) for i in order]
    wsizes = [_count(s) for s in weight_shapes]
    wofs = np.concatenate([[0], np.cumsum(wsizes)]).astype(np.int64)
    wtotal = int(wofs[-1])
    instr_chunks, const_chunks = [], []
    progs = np.zeros(len(order), dtype=PROG_DTYPE)
    n_instr = n_const = 0
    elem = 0
    max_arena = 0
    max_smem = 0
    placed = {}                             # individual -> its program row (code shared by parts)
    for slot, idx in enumerate(order):
        v = variants[idx]
        if idx in placed:
            progs[slot] = progs[placed[idx]]
        p = progs[slot]
        if idx in placed:
            p["result_slot"] = idx
        else:
            placed[idx] = slot
            p["result_slot"] = idx
            p["const_off"] = n_const
            const_chunks.append(v.consts)
            n_const += len(v.consts)
            if v.train0 is not None:
                a = v.train0
                p["train0"], p["train0_n"] = n_instr, len(a)
                instr_chunks.append(a)
                n_instr += len(a)
                if v.train1 is v.train0:
                    p["train1"], p["train1_n"] = p["train0"], p["train0_n"]
                else:
                    b = v.train1
                    p["train1"], p["train1_n"] = n_instr, len(b)
                    instr_chunks.append(b)
                    n_instr += len(b)
                if v.train2 is None:
                    p["train2"], p["train2_n"] = p["train1"], p["train1_n"]
                else:
                    c = v.train2
                    p["train2"], p["train2_n"] = n_instr, len(c)
                    instr_chunks.append(c)
                    n_instr += len(c)
            f = v.fwd
            p["fwd"], p["fwd_n"] = n_instr, len(f)
            instr_chunks.append(f)
            n_instr += len(f)
        arena = (v.arena + 15) & ~15
        p["arena_off"] = elem
        p["arena_elems"] = arena
        p["flags"] = v.flags
        if parts > 1:
            p["flags"] = v.flags | ((slot // n) << FLAG_PART_SHIFT) | (parts << FLAG_NPARTS_SHIFT)
        max_arena = max(max_arena, arena)
        max_smem = max(max_smem, v.smem)
        # [scratch | probs | weights ping | weights pong], 16-element aligned
        elem += arena + ((probs_elems + 15) & ~15) + 2 * ((wtotal + 15) & ~15)
    hdr = np.zeros(1, dtype=HEADER_DTYPE)
    hdr["magic"], hdr["version"] = PLAN_MAGIC, PLAN_VERSION
    hdr["n_instr"], hdr["n_prog"], hdr["n_const"] = n_instr, len(order), n_const
    hdr["weight_elems"] = wtotal
    hdr["n_weights"] = len(wsizes)
    hdr["wofs"][0, :len(wsizes)] = wofs[:-1]
    hdr["max_arena"] = max_arena
    hdr["max_smem"] = max_smem
    hdr["total_elems"] = elem
    # raw bytes: concatenating structured arrays promotes dtypes field by
    # field (numpy _promote_fields), which cost ~30 ms per 256 individuals
    instrs = np.concatenate([c.view(np.uint8) for c in instr_chunks]) if instr_chunks else \
        np.zeros(0, dtype=np.uint8)
    consts = np.concatenate(const_chunks) if const_chunks else np.zeros(0)
    blob = np.concatenate([hdr.view(np.uint8), instrs,
                           progs.view(np.uint8), consts.view(np.uint8)])
    return PopulationPlan(blob, len(order), np.asarray(order), elem)


def exec_once_plan(fns, param_arrays_list):
    """Plan for running one function once per case with explicit params
    (per-op and single-step parity tests).  Returns (blob, params_blob,
    out_sizes, out_offsets_per_case, out_total)."""
    n = len(fns)
    progs = np.zeros(n, dtype=PROG_DTYPE)
    chunks, consts_c = [], []
    params_flat = []
    n_instr = n_const = 0
    pofs = 0
    oofs = 0
    elem = 0
    max_smem = 0
    out_meta = []
    for i, (fn, params) in enumerate(zip(fns, param_arrays_list)):
        low = lower_function(fn, None, ret_layout="c")
        max_smem = max(max_smem, low.smem_elems)
        a = encode_instrs(low.instrs)
        p = progs[i]
        p["train0"], p["train0_n"] = n_instr, len(a)
        p["const_off"] = n_const
        p["result_slot"] = i
        chunks.append(a)
        n_instr += len(a)
        consts_c.append(consts_to_words(low.consts))
        n_const += len(low.consts)
        for k, arr in enumerate(params):
            words = np.ascontiguousarray(arr)
            if words.dtype == np.bool_:
                words = words.astype(np.int64)
            words = words.reshape(-1).view(np.float64) if words.dtype != np.float64 \
                else words.reshape(-1)
            p["param_off"][k] = pofs
            params_flat.append(words)
            pofs += len(words)
        metas = []
        for r, ty in enumerate(fn.return_types):
            cnt = _count(tuple(ty.shape))
            p["out_off"][r] = oofs
            metas.append((oofs, tuple(ty.shape), getattr(ty.kind, "value", ty.kind)))
            oofs += max(cnt, 1)
        out_meta.append(metas)
        arena = (low.arena_elems + 15) & ~15
        p["arena_off"] = elem
        p["arena_elems"] = arena
        elem += arena + 16
    hdr = np.zeros(1, dtype=HEADER_DTYPE)
    hdr["magic"], hdr["version"] = PLAN_MAGIC, PLAN_VERSION
    hdr["n_instr"], hdr["n_prog"], hdr["n_const"] = n_instr, n, n_const
    hdr["max_smem"] = max_smem
    hdr["total_elems"] = elem
    instrs = np.concatenate([c.view(np.uint8) for c in chunks]) if chunks else np.zeros(0, dtype=np.uint8)
    consts = np.concatenate(consts_c) if consts_c else np.zeros(0)
    blob = np.concatenate([hdr.view(np.uint8), instrs,
                           progs.view(np.uint8), consts.view(np.uint8)])
    params_blob = np.concatenate(params_flat) if params_flat else np.zeros(1)
    return blob, params_blob, out_meta, max(oofs, 1)


__all__ = ["lower_variant", "build_population_plan", "exec_once_plan",
           "static_cost", "VariantPlan", "PopulationPlan"]
