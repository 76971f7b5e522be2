"""Benchmark: fresh individuals evaluated per second (BASELINE.json metric).

Workload (BASELINE.json configs[1]): train2fc (784-32-10 MLP, 600 SGD steps
+ 31 scored batches per individual) on synthetic MNIST-shaped data.  A step
evaluates one population of `--pop` fresh mutated individuals, drawn from a
recorded seeded GA run (pop 256 x 10 generations,
tests/golden/bench_train_pool.json.gz): real patches of the reference's
genome, not copies of one program.  The population is sharded over the N
ranks; by default it is 256 per GPU (weak scaling: 256, 512, 1024, 2048 at
N = 1, 2, 4, 8 -- points of configs[4]'s 64-4096 sweep).  With N > 1 the
line also carries `strong_pop256`: configs[1] itself, population 256
sharded over the N GPUs (device time; each GPU then holds 256/N
individuals, which underfill it -- SURVEY.md §7.3 item 8).

  value  = individuals / device time of the evaluation kernels (plans
           resident; CUDA events on the launching stream; max over ranks)
  e2e    = individuals / wall time of the reference's own seam,
           evotir.search._Evaluator(workload)(patches) with
           shims.install() (search.py:257-273): patch_dumps keys, apply_patch
           + verify + lowering in the worker processes, plan H2D, kernels,
           result D2H, and the NCCL record all-gather when N > 1
  cnn    = BASELINE.json configs[2] (MobileNetV2-CIFAR width 0.5, 128
           reference-made mutants) on a bounded 1 000-image sample

`--impl reference` times the UNMODIFIED reference (baseline/_ref, installed by
baseline/install_ref.sh): evotir.fitness.evaluate over the same patches in a
process pool on every host core.
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
WORKLOAD = "train2fc (784-32-10 MLP, 600 SGD steps + 31 scored batches, synthetic MNIST-shaped)"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--pop", type=int, default=None,
                   help="population per step, whole job (default 256 per GPU)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-cnn", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-tf32", action="store_true", help="skip the tf32/bf16 (tcgen05) side lines")
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


# ---------------------------------------------------------------------------
# the reference itself on the host CPU (baseline/_ref)
# ---------------------------------------------------------------------------

_REF_WL = None


def _need_reference():
    from golden_io import reference_available
    if not reference_available():
        raise SystemExit("the reference (evotir) is not importable: run baseline/install_ref.sh")


def _ref_eval(key):
    """One unmodified evotir.fitness.evaluate (fitness.py:372-393) of a patch."""
    from evotir import fitness as F
    from evotir.genome import patch_loads
    f = F.evaluate(_REF_WL.module, patch_loads(key), _REF_WL)
    return f.cost, f.error, f.valid


def _one_blas_thread():
    """Pool initializer: one OpenBLAS thread per worker process (numpy was
    imported before the fork, so the environment variable alone is too late)."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except ImportError:
        pass


def reference_throughput(keys, seconds=None):
    """evotir.fitness.evaluate over `keys` in a process pool with one process
    per host core and OPENBLAS_NUM_THREADS=1 (the reference's own thread pool
    is slower than serial).  With `seconds`, a bounded sample:
    as many keys as the warm pool gets through in about that time.  Returns
    (individuals/s, cores, n, seconds, results)."""
    global _REF_WL
    import multiprocessing as mp
    _need_reference()
    from evotir import fitness as F
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    cores = os.cpu_count() or 1
    if _REF_WL is None:
        _REF_WL = F.build_2fcnet_workload()          # inherited by the forked workers
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_one_blas_thread) as pool:
        t = time.perf_counter()
        pool.map(_ref_eval, keys[:cores], chunksize=1)      # warm every worker
        warm = time.perf_counter() - t
        n = len(keys)
        if seconds is not None:
            n = min(len(keys), max(4 * cores, int(cores * seconds / max(warm, 1e-3))))
        t = time.perf_counter()
        res = pool.map(_ref_eval, keys[:n], chunksize=1)
        dt = time.perf_counter() - t
    return n / dt, cores, n, dt, res


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl != "reference":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def run_reference(args, world, rank):
    """The reference arm: rank 0 alone, every host core."""
    if rank != 0:
        return
    inds, _ = load_pool()
    rates, ns, cores = [], [], os.cpu_count() or 1
    per_step = None
    for s in range(args.warmup + args.steps):
        start = (s * args.pop) % len(inds)
        keys = [inds[(start + k) % len(inds)]["key"] for k in range(args.pop)]
        if per_step is None:
            # size the sample once so the whole run stays within minutes
            r, cores, n, dt, _ = reference_throughput(keys, seconds=8.0)
            per_step = n
        else:
            r, cores, n, dt, _ = reference_throughput(keys[:per_step])
        if s >= args.warmup:
            rates.append(r)
            ns.append(n)
    value = statistics.median(rates)
    sample = (f"{ns[0]} of the {args.pop} fresh patches of each step "
              f"(bench pool, seeded GA), evotir.fitness.evaluate on {cores} processes")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * args.pop / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "population": args.pop, "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

def lib_sha():
    """Identity of the running build: the hash of the sources and nvcc flags
    libgevo.so is compiled from (build.source_sha; the .so bytes differ per
    nvcc run)."""
    from paper_2310_10211_b200 import build
    return build.source_sha()


def measured_traffic(sha):
    """ncu dram bytes of the hot kernel per launch, recorded by
    tests/tools/ncu_traffic.py for THIS build of libgevo.so (profiles/
    traffic.json carries the source sha of the build it measured); null when
    the capture is of another build."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except (OSError, ValueError):
        return None, None
    if t.get("lib_sha") != sha:
        return None, None
    return t.get("dram_bytes_per_launch"), t


def cnn_measure(local, steps=1, n_img=1000, pop=128, fixtures=("cnn_full_pop.json.gz",)):
    """configs[2] on a bounded sample: the 16 reference-made mutants of the
    full network (tests/golden/cnn_full_pop.json.gz) x 8 = population 128,
    scored over `n_img` (default 1 000 of the 10 000) synthetic CIFAR-shaped
    images (batch 100).  `pop` / `fixtures`: other populations cycled over the
    mutants of the given recordings (tests/tools/cnn_sweep.py)."""
    from golden_io import load
    from paper_2310_10211_b200 import cnn, dialect
    from paper_2310_10211_b200.evaluator import DeviceEvaluator
    inds, seen = [], set()
    for fx in fixtures:
        for i in load(fx)["individuals"]:
            if i["key"] not in seen:
                seen.add(i["key"])
                inds.append(i)
    batch = 100
    cfg = cnn.CnnConfig(**cnn.MOBILENETV2_CIFAR_HALF, batch_size=batch, search_n=n_img,
                        holdout_n=batch)
    wl = cnn.build_cnn_prediction_workload(cfg)
    base = [{"forward": dialect.parse_function(i["forward"])} for i in inds]
    variants = [base[k % len(base)] for k in range(pop)]
    fn = base[0]["forward"]
    macs, types = 0, dict(fn.params)
    for op in fn.ops:
        if op.opcode == "dot":
            a, b = types[op.operands[0]], types[op.operands[1]]
            macs += a.shape[0] * a.shape[1] * b.shape[1]
        types[op.result] = op.result_type
    ev = DeviceEvaluator(wl, device=local)
    ev.evaluate_variants(variants)                      # warm-up
    dev, wall = [], []
    for _ in range(steps):
        t = time.perf_counter()
        fits = ev.evaluate_variants(variants)
        wall.append(time.perf_counter() - t)
        dev.append(ev.last_device_ms / 1e3)
    ev.close()
    d, w = statistics.median(dev), statistics.median(wall)
    return {"workload": f"configs[2]: MobileNetV2-CIFAR width 0.5, population {pop} "
                        f"({len(base)} reference-made mutants cycled), {n_img} images "
                        "(batch 100) of the 10k-image split",
            "value": pop / d, "unit": UNIT, "images_per_s": pop * n_img / d,
            "e2e": pop / w, "fp64_dot_tflops": 2.0 * macs * (n_img // batch) * pop / d / 1e12,
            "ms_per_step": 1e3 * d, "statuses_ok": sum(f.error < 1.0 for f in fits)}


def main():
    args = parse_args()
    world, rank, local = dist_setup(args)
    if args.pop is None:
        args.pop = POP * world
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import numpy as np
    import torch
    from paper_2310_10211_b200 import workloads as W
    from paper_2310_10211_b200.evaluator import DeviceEvaluator, lower_all
    from paper_2310_10211_b200.plan import (build_population_plan, device_weight, layout_order,
                                            sm_aware_order)

    torch.cuda.set_device(local)
    inds, parse_function = load_pool()
    wl = W.build_2fcnet_workload()
    ev = DeviceEvaluator(wl, device=local)
    total_steps = args.warmup + args.steps

    def pop_for(s):
        start = (s * args.pop) % len(inds)
        return [inds[(start + k) % len(inds)] for k in range(args.pop)]
    pops = [pop_for(s) for s in range(total_steps)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    nb = wl.n_search_batches
    steps_cfg = wl.config.steps

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    clocks = Clocks(local)
    # (1) value: this rank's shard (strided, as the seam shards it), lowered
    # before timing; one launch per step; device time (CUDA events)
    kern_ms, alg_bytes, alg_flops = [], [], []
    shard_steps = []
    for s in range(total_steps):
        mine = pops[s][rank::world]
        fns = [{n: parse_function(i[n]) for n in ("forward", "train_step")} for i in mine]
        shard_steps.append((fns, [v for v in lower_all(fns, wl.config.cost_table, True, steps_cfg)
                                  if v is not None]))
    for s in range(total_steps):
        fns, vps = shard_steps[s]
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
    # (1a) N > 1: configs[1] as written -- population 256 sharded over the N
    # GPUs (strong scaling), device time, max over ranks
    strong = None
    if world > 1:
        s_ms = []
        for s in range(args.warmup, total_steps):
            mine = pops[s][:POP][rank::world]
            fns = [{n: parse_function(i[n]) for n in ("forward", "train_step")} for i in mine]
            vps = [v for v in lower_all(fns, wl.config.cost_table, True, steps_cfg) if v is not None]
            p = build_population_plan(vps, ev.weight_shapes, ev.batch * ev.classes,
                                      order=sm_aware_order([device_weight(v, steps_cfg, nb) for v in vps],
                                                           ev.n_sms))
            flush.zero_()
            barrier()
            ev.ctx.eval(p.blob, p.n_prog, 0, steps_cfg, wl.config.finite_check_every, 0, 0,
                        ev.weight_elems, False)
            s_ms.append(ev.ctx.last_kernel_ms())
        import torch.distributed as dist
        t = torch.tensor([sum(s_ms) / 1e3], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        strong = {"population": POP, "value": POP * len(s_ms) / t.item(), "unit": UNIT,
                  "ms_per_step": 1e3 * t.item() / len(s_ms), "scaling": "strong",
                  "note": "configs[1]: population 256 sharded over the GPUs (256/N per GPU)"}
    # (1b) the reduced-precision modes on the same plans: every f64 DOT on
    # tcgen05 (GEVO_B200_DTYPE=tf32, bf16); device time and the error's exact-match
    # rate against the reference -- a side line, never the headline (the
    # reference computes in float64)
    tc_lines = {}
    for mode, kind, tol in (("tf32", "kind::tf32", "per dot |err| <= 2e-3 * sum|a||b|; one train_step "
                             "within 2e-3 normwise (tests/test_tc.py)"),
                            ("bf16", "kind::f16", "per dot |err| <= 1e-2 * sum|a||b|; one train_step "
                             "within 2e-2 normwise (tests/test_tc.py)")):
        if args.no_tf32:
            break
        t_ms, t_exact, t_n = [], 0, 0
        os.environ["GEVO_B200_DTYPE"] = mode
        try:
            for s in range(args.warmup, total_steps):
                fns, vps = shard_steps[s]
                p = build_population_plan(vps, ev.weight_shapes, ev.batch * ev.classes)
                flush.zero_()
                barrier()
                res, _ = ev.ctx.eval(p.blob, p.n_prog, 0, steps_cfg, wl.config.finite_check_every, 0, 0,
                                     ev.weight_elems, False)
                t_ms.append(ev.ctx.last_kernel_ms())
                mine = pops[s][rank::world]
                if len(mine) != len(vps):
                    continue
                for k, ind in enumerate(mine):
                    err = 1.0 if res["status"][k] != 0 else int(res["wrong"][k]) / int(res["total"][k])
                    t_n += 1
                    t_exact += err == ind["error"]
        finally:
            del os.environ["GEVO_B200_DTYPE"]
        tc_lines[mode] = {"value": len(pops[0][rank::world]) * len(t_ms) / (sum(t_ms) / 1e3), "unit": UNIT,
                          "ms_per_step": statistics.mean(t_ms), "dtype": f"{mode} (tcgen05.mma {kind}, fp32 "
                          "accumulation; every other op float64)",
                          "error_exact_vs_reference": {"exact": t_exact, "of": t_n}, "tolerance": tol}
    # (2) e2e through the reference's seam: _Evaluator(workload)(patches)
    wall_s, h2d, d2h, e2e_launches = [], [], [], 0
    parity_ok = parity_n = 0
    if not args.no_e2e:
        _need_reference()
        import evotir.search as S
        from evotir import fitness as F
        from evotir.genome import patch_loads
        from paper_2310_10211_b200 import shims
        rwl = F.build_2fcnet_workload()
        shims.install(device=local)
        patches = [[patch_loads(i["key"]) for i in pops[s]] for s in range(total_steps)]
        dev = shims.device_for(rwl, local)
        for s in range(total_steps):
            E = S._Evaluator(rwl)                   # fresh cache: every patch is evaluated
            flush.zero_()
            barrier()
            n0 = dev.launches
            t0 = time.perf_counter()
            fits = E(patches[s])
            t1 = time.perf_counter()
            if s >= args.warmup:
                wall_s.append(t1 - t0)
                e2e_launches += dev.launches - n0
                h2d.append(int(dev.last_plan_bytes))
                # records of this rank's shard + the gathered records
                n_mine = len(pops[s][rank::world])
                d2h.append(n_mine * 56 + (args.pop * 32 + 32 * world if world > 1 else 0))
                for f, ind in zip(fits, pops[s]):
                    parity_n += 1
                    parity_ok += (f.cost, f.error) == (ind["cost"], ind["error"])
        shims.uninstall()
    barrier()
    ck = clocks.stop()
    dev_s = sum(kern_ms) / 1000.0
    e2e_s = sum(wall_s) if wall_s else float("nan")
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([dev_s, e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s, e2e_s = t.tolist()
    n_total = args.pop * args.steps
    value = n_total / dev_s
    e2e = n_total / e2e_s if wall_s else None
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
        sha = lib_sha()
        traffic, tinfo = measured_traffic(sha)
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                r, cores, n, dt, _ = reference_throughput([i["key"] for i in pops[0]], 10.0)
                cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "reference",
                       "sample": f"{n} fresh patches of the bench population, unmodified "
                                 f"evotir.fitness.evaluate (baseline/_ref) on {cores} "
                                 f"processes ({dt:.1f} s)"}
            except SystemExit as e:
                cpu = {"value": None, "unavailable": str(e)}
        cnn_line = None
        if not args.no_cnn and world == 1:
            cnn_line = cnn_measure(local)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * dev_s / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded synthetic_digits, recorded GA patches)",
            "config": {"workload": f"{WORKLOAD}, population {args.pop}",
                       "population": args.pop, "population_per_gpu": args.pop / world,
                       "steps_per_individual": steps_cfg, "scored_batches": nb,
                       "l2": "flushed between timed iterations (256 MB write)",
                       "parallelism": f"population sharded over {world} GPU(s), "
                                      "records all-gathered (gevo_allgather, NCCL)"},
            "e2e": {"value": e2e, "unit": UNIT,
                    "h2d_bytes_per_step": int(statistics.mean(h2d)) if h2d else None,
                    "d2h_bytes_per_step": int(statistics.mean(d2h)) if d2h else None,
                    "seam": "evotir.search._Evaluator(workload)(patches) with shims.install()",
                    "launches": e2e_launches},
            "gpu_launches": len(kern_ms),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "traffic_source": (tinfo or {}).get("source"),
                         "algorithmic_bytes_per_launch": per_launch_bytes,
                         "fp64_tflops": statistics.mean(alg_flops) / per_launch_s / 1e12,
                         "lib_sha": sha},
            "cpu_baseline": cpu,
            "clocks": ck,
            "parity": {"bit_exact": parity_ok, "of": parity_n,
                       "against": "reference (cost, error) recorded in the bench pool"},
        }
        if cnn_line is not None:
            line["cnn"] = cnn_line
        line.update(tc_lines)
        if strong is not None:
            line["strong_pop256"] = strong
        print(json.dumps(line), flush=True)
    ev.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
