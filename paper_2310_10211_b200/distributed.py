"""Population sharding across GPUs of one node.

Every rank runs the identical seeded GA on the host, so every rank holds
the same list of fresh patches per generation.  Each rank evaluates one
shard; the only collective is ONE all-gather of fixed-size fitness records
(cost, wrong, total, status), after which every rank holds every fitness
and runs the same NSGA-II.  Shards are balanced by the reference's static
cost (known before execution): longest-processing-time greedy.
"""
from __future__ import annotations

import heapq

import numpy as np

RECORD_FIELDS = 4   # cost (f64 bits), wrong, total, status  -> 4 x int64


def lpt_shards(costs, world: int):
    """Deterministic LPT: individuals in decreasing cost (ties by index) go
    to the currently lightest rank (ties by rank id).  Returns a list of
    index lists, each in ascending index order."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(s) for s in out]


def pack_records(fits, records):
    """Fitness list + device records -> int64 [n, 4] (cost as raw bits)."""
    n = len(fits)
    out = np.zeros((n, RECORD_FIELDS), dtype=np.int64)
    out[:, 0] = np.array([f.cost for f in fits], dtype=np.float64).view(np.int64)
    out[:, 1] = records["wrong"]
    out[:, 2] = records["total"]
    out[:, 3] = records["status"]
    return out


def all_gather_records(local: np.ndarray, n_max: int, group=None):
    """One all-gather (NCCL when the default group is NCCL) of per-rank
    records padded to n_max rows; returns [world, n_max, 4] int64 and the
    per-rank valid counts."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    buf = np.zeros((n_max + 1, RECORD_FIELDS), dtype=np.int64)
    buf[0, 0] = len(local)
    buf[1:len(local) + 1] = local
    t = torch.from_numpy(buf).to(dev)
    if dev.type == "cuda":
        out = torch.empty((world, n_max + 1, RECORD_FIELDS), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(out, t, group=group)
        arr = out.cpu().numpy()
    else:                               # gloo has no all_gather_into_tensor
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        arr = torch.stack(parts).numpy()
    counts = arr[:, 0, 0].astype(int)
    return arr[:, 1:, :], counts


def merge_shards(gathered, counts, shards):
    """Scatter gathered per-rank records back into population order."""
    n = sum(len(s) for s in shards)
    out = np.zeros((n, RECORD_FIELDS), dtype=np.int64)
    for r, idx in enumerate(shards):
        out[idx] = gathered[r, :counts[r]]
    return out


STATUS_INVALID = -1


class ShardedEvaluator:
    """Population parallelism across ranks (one process per GPU).

    Every rank calls evaluate_variants with the SAME list (the host GA is
    replicated and seeded identically, so its patch lists agree); each rank
    lowers and evaluates only its LPT shard on its own device, then ONE
    all-gather of fixed-size records gives every rank every fitness.
    `backend` is a DeviceEvaluator (or anything with the same
    evaluate_variants(..., return_records=True) signature)."""

    def __init__(self, backend, group=None):
        self.backend = backend
        self.group = group
        self.last_shards = None

    def _world(self):
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(self.group), dist.get_rank(self.group)
        return 1, 0

    def evaluate_variants(self, variants, holdout=False, cost_table=None):
        from .lowering import static_cost
        from .workloads import INVALID_FITNESS, Fitness
        world, rank = self._world()
        if world == 1:
            return self.backend.evaluate_variants(variants, holdout=holdout)
        training = "train_step" in next((v for v in variants if v), {})
        costs = []
        for v in variants:
            if v is None:
                costs.append(0.0)
            else:
                costs.append(static_cost(v["train_step" if training else "forward"],
                                         cost_table))
        shards = lpt_shards(costs, world)
        self.last_shards = shards
        mine = [variants[i] for i in shards[rank]]
        fits, recs = self.backend.evaluate_variants(mine, holdout=holdout,
                                                    return_records=True)
        local = pack_records(fits, recs)
        for k, f in enumerate(fits):
            if not f.valid:
                local[k, 3] = STATUS_INVALID
        n_max = max(len(s) for s in shards)
        gathered, counts = all_gather_records(local, n_max, self.group)
        merged = merge_shards(gathered, counts, shards)
        out = []
        for row in merged:
            cost = float(np.int64(row[0]).view(np.float64))
            status = int(row[3])
            if status == STATUS_INVALID:
                out.append(INVALID_FITNESS)
            elif status != 0:
                out.append(Fitness(cost, 1.0))
            else:
                out.append(Fitness(cost, int(row[1]) / int(row[2])))
        return out
