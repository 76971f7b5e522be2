"""Benchmark: fresh individuals evaluated per second (BASELINE.json metric).

Workload (BASELINE.json configs[1]): train2fc (784-32-10 MLP, 600 SGD steps
+ 31 scored batches per individual) on synthetic MNIST-shaped data; a step
evaluates one population of 256 fresh mutated individuals per GPU, drawn
from a recorded seeded GA run (pop 256 x 10 generations, tests/golden/
bench_train_pool.json.gz) -- real variant programs, not copies of one.

  value  = individuals / device time of the evaluation kernels (inputs and
           plans resident; CUDA events on the launching stream, max over
           ranks)
  e2e    = individuals / wall time of the public API call
           DeviceEvaluator.evaluate_variants (host lowering in a process
           pool, overlapped with the device: half the generation runs while
           the other half is lowered; plan H2D + kernels + result D2H), plus
           the record all-gather when N > 1

`--impl reference` times the reference's algorithm on the host CPU (the
oracle port, all cores, process pool), on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

POP = 256
METRIC = "individuals evaluated/sec per generation"
UNIT = "individuals/s"
WORKLOAD = "train2fc pop256 (784-32-10 MLP, 600 SGD steps + 31 scored batches, synthetic MNIST-shaped)"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--pop", type=int, default=POP)
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def load_pool():
    from golden_io import load
    from paper_2310_10211_b200.dialect import parse_function
    inds = load("bench_train_pool.json.gz")["individuals"]
    seen, out = set(), []
    for ind in inds:
        if ind.get("invalid_patch") or ind["key"] in seen:
            continue
        seen.add(ind["key"])
        out.append(ind)
    return out, parse_function


def per_individual_bytes(fns, steps, n_batches):
    """sum over executed function invocations of param
    bytes read + return bytes written (8-byte elements)."""
    def io(fn):
        n = 0
        for _, t in fn.params:
            c = 1
            for d in t.shape:
                c *= d
            n += c
        for t in fn.return_types:
            c = 1
            for d in t.shape:
                c *= d
            n += c
        return 8 * n
    return steps * io(fns["train_step"]) + n_batches * io(fns["forward"])


def per_individual_flops(fns, steps, n_batches):
    def fl(fn):
        types = dict(fn.params)
        tot = 0
        for op in fn.ops:
            if op.opcode == "dot":
                a, b = types[op.operands[0]], types[op.operands[1]]
                tot += 2 * a.shape[0] * a.shape[1] * b.shape[1]
            types[op.result] = op.result_type
        return tot
    return steps * fl(fns["train_step"]) + n_batches * fl(fns["forward"])


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_eval_one(args):
    fns_text, kind = args
    from oracle import fitness as OF
    from paper_2310_10211_b200 import workloads as W
    from paper_2310_10211_b200.dialect import parse_function
    global _WL
    if "_WL" not in globals() or _WL is None:
        _WL = W.build_2fcnet_workload()
    wl = _WL
    fns = {k: parse_function(v) for k, v in fns_text.items()}
    w0 = [wl.weights[n] for n in W.WEIGHT_NAMES]
    return OF.evaluate_variant(fns, "training", w0,
                               (wl.search_x, wl.search_y, wl.search_labels))


_WL = None


def cpu_throughput(inds, seconds_budget=15.0):
    """The reference algorithm (oracle port: same numpy calls as
    interpreter.py/fitness.py) on all host cores, one process per core,
    OPENBLAS_NUM_THREADS=1 (results identical to serial)."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    n = max(cores, min(len(inds), int(cores * seconds_budget / 0.3)))
    n = min(n, len(inds))
    work = [({k: i[k] for k in ("forward", "train_step")}, "training") for i in inds[:n]]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(cpu_eval_one, work[:cores])     # warm workers
        t = time.perf_counter()
        pool.map(cpu_eval_one, work, chunksize=1)
        dt = time.perf_counter() - t
    return n / dt, cores, n, dt


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def run_reference(args, world, rank):
    if rank != 0:
        return
    inds, _ = load_pool()
    rates = []
    cores = os.cpu_count() or 1
    for s in range(args.warmup + args.steps):
        r, cores, n, dt = cpu_throughput(inds[(s * 7) % max(1, len(inds) - 64):], 8.0)
        if s >= args.warmup:
            rates.append(r)
    value = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * args.pop / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "population": args.pop,
                       "sample": f"{n} individuals per step on {cores} processes"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores,
                             "kind": "port",
                             "sample": f"{n} fresh individuals of the bench pool per step, "
                                       "oracle/ numpy restatement (bit-identical to the reference)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import numpy as np
    import torch
    from paper_2310_10211_b200 import workloads as W
    from paper_2310_10211_b200.evaluator import DeviceEvaluator
    from paper_2310_10211_b200 import distributed as D

    torch.cuda.set_device(local)
    inds, parse_function = load_pool()
    wl = W.build_2fcnet_workload()
    ev = DeviceEvaluator(wl, device=local)
    total_steps = args.warmup + args.steps
    # distinct individuals per (rank, step) where the pool allows
    stride = args.pop
    def batch_for(s):
        start = ((s * world + rank) * stride) % len(inds)
        sel = [inds[(start + k) % len(inds)] for k in range(args.pop)]
        return sel, [{n: parse_function(i[n]) for n in ("forward", "train_step")} for i in sel]

    batches = [batch_for(s) for s in range(total_steps)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    nb = wl.n_search_batches
    steps_cfg = wl.config.steps

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    kern_ms, wall_s, alg_bytes, alg_flops, h2d, d2h = [], [], [], [], [], []
    parity_ok = parity_n = 0
    from paper_2310_10211_b200.evaluator import lower_all
    from paper_2310_10211_b200.plan import build_population_plan
    clocks = Clocks(local)
    # (1) value: plans built before timing; one launch per step on one
    # context; device time of the evaluation kernel (CUDA events)
    lowered_steps = []
    for s in range(total_steps):
        lowered_steps.append([v for v in lower_all(batches[s][1], wl.config.cost_table, True, steps_cfg)
                              if v is not None])
    from paper_2310_10211_b200.plan import device_weight, layout_order, sm_aware_order
    for s in range(total_steps):
        sel, fns = batches[s]
        vps = lowered_steps[s]
        # launch order from the block -> SM layout the previous launch showed
        wts = [device_weight(v, steps_cfg, nb) for v in vps]
        layout = ev._sm_layout.get(len(vps))
        order = layout_order(wts, layout) if layout else sm_aware_order(wts, ev.n_sms)
        p = build_population_plan(vps, ev.weight_shapes, ev.batch * ev.classes, order=order)
        flush.zero_()                       # L2 flush between iterations
        barrier()
        if s == args.warmup:
            clocks.start()
        res, _ = ev.ctx.eval(p.blob, p.n_prog, 0, steps_cfg, wl.config.finite_check_every, 0, 0,
                             ev.weight_elems, False)
        ev._learn_layout(res, order)
        if s >= args.warmup:
            kern_ms.append(ev.ctx.last_kernel_ms())
            alg_bytes.append(sum(per_individual_bytes(f, steps_cfg, nb) for f in fns))
            alg_flops.append(sum(per_individual_flops(f, steps_cfg, nb) for f in fns))
    # (2) e2e: the public call on host data (lowering, plan H2D, kernels,
    # results D2H; the record all-gather when N > 1), wall clock
    for s in range(total_steps):
        sel, fns = batches[s]
        flush.zero_()
        barrier()
        t0 = time.perf_counter()
        fits, recs = ev.evaluate_variants(fns, return_records=True)
        if world > 1:
            loc = D.pack_records(fits, recs)
            D.all_gather_records(loc, args.pop)
        t1 = time.perf_counter()
        if s >= args.warmup:
            wall_s.append(t1 - t0)
            h2d.append(int(ev.last_plan_bytes))
            d2h.append(args.pop * 24)
            # the pool records the reference's own fitness for every variant
            for f, ind in zip(fits, sel):
                parity_n += 1
                parity_ok += (f.cost, f.error) == (ind["cost"], ind["error"])
    barrier()
    ck = clocks.stop()
    dev_s = sum(kern_ms) / 1000.0
    e2e_s = sum(wall_s)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([dev_s, e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s, e2e_s = t.tolist()
    n_total = args.pop * args.steps * world
    value = n_total / dev_s
    e2e = n_total / e2e_s
    if rank == 0:
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except OSError:
            pass
        hbm = peaks.get("hbm_gbs", 6650.0)
        per_launch_bytes = statistics.mean(alg_bytes)
        per_launch_s = statistics.mean(kern_ms) / 1000.0
        achieved = per_launch_bytes / per_launch_s / 1e9
        traffic = None
        try:
            traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(
                "dram_bytes_per_launch")
        except OSError:
            pass
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            r, cores, n, dt = cpu_throughput(inds, 10.0)
            cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "port",
                   "sample": f"{n} individuals of the bench pool, oracle/ numpy restatement "
                             f"on {cores} processes ({dt:.1f} s)"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * dev_s / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded synthetic_digits, recorded GA variants)",
            "config": {"workload": WORKLOAD, "population_per_gpu": args.pop,
                       "steps_per_individual": steps_cfg, "scored_batches": nb,
                       "l2": "flushed between timed iterations (256 MB write)",
                       "parallelism": f"population sharded, {world} GPU(s), records all-gathered"},
            "e2e": {"value": e2e, "unit": UNIT,
                    "h2d_bytes_per_step": int(statistics.mean(h2d)),
                    "d2h_bytes_per_step": int(statistics.mean(d2h))},
            "gpu_launches": args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "algorithmic_bytes_per_launch": per_launch_bytes,
                         "fp64_tflops": statistics.mean(alg_flops) / per_launch_s / 1e12},
            "cpu_baseline": cpu,
            "clocks": ck,
            "parity": {"bit_exact": parity_ok, "of": parity_n,
                       "against": "reference (cost, error) recorded in the bench pool"},
        }
        print(json.dumps(line), flush=True)
    ev.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
