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


def strided_shards(n: int, world: int):
    """Shard r = items r, r + world, r + 2*world, ... : the split used when
    the costs are not known before the shard is lowered (patches applied in
    the workers); deterministic, and every shard sees the same mix of
    generations' insertion order."""
    return [list(range(r, n, world)) for r in range(world)]


def all_gather_records(local: np.ndarray, n_max: int, group=None, ctx=None):
    """One all-gather of per-rank records padded to n_max rows; returns
    [world, n_max, 4] int64 and the per-rank valid counts.  With `ctx` (a
    libgevo Context whose NCCL communicator is initialised, see
    init_comm) the gather is libgevo's own gevo_allgather over NVLink;
    otherwise torch.distributed (gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if ctx is not None:
        buf = np.zeros((n_max + 1, RECORD_FIELDS), dtype=np.int64)
        buf[0, 0] = len(local)
        buf[1:len(local) + 1] = local
        arr = ctx.allgather(buf, world)
        return arr[:, 1:, :], arr[:, 0, 0].astype(int)
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
        self.ctx = init_comm(backend, group)

    @property
    def workload(self):
        return self.backend.workload

    def _world(self):
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(self.group), dist.get_rank(self.group)
        return 1, 0

    def _gather(self, fits, recs, shards, rank):
        local = pack_records(fits, recs)
        for k, f in enumerate(fits):
            if not f.valid:
                local[k, 3] = STATUS_INVALID
        n_max = max(len(s) for s in shards)
        gathered, counts = all_gather_records(local, n_max, self.group, self.ctx)
        return unpack_records(merge_shards(gathered, counts, shards))

    def evaluate_patches(self, original, keys, functions, holdout=False):
        """Every rank passes the SAME patch keys (the replicated GA); rank r
        applies, lowers and evaluates the strided shard r (in its own worker
        processes, on its own device), then one all-gather."""
        world, rank = self._world()
        if world == 1:
            return self.backend.evaluate_patches(original, keys, functions, holdout=holdout)
        shards = strided_shards(len(keys), world)
        self.last_shards = shards
        fits, recs = self.backend.evaluate_patches(original, [keys[i] for i in shards[rank]],
                                                   functions, holdout=holdout,
                                                   return_records=True)
        return self._gather(fits, recs, shards, rank)

    def evaluate_variants(self, variants, holdout=False, cost_table=None):
        from .lowering import static_cost
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
        return self._gather(fits, recs, shards, rank)


def unpack_records(merged):
    """Gathered int64 records -> Fitness list, with the reference's
    encodings (fitness.py:376-392) and error = wrong / total in Python."""
    from .workloads import INVALID_FITNESS, Fitness
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


def init_comm(backend, group=None):
    """When the process group is NCCL and `backend` owns a libgevo context,
    create libgevo's own NCCL communicator over the same ranks (rank 0's
    ncclUniqueId is broadcast through the process group: torch.distributed
    is the plumbing, the records travel through gevo_allgather).  Returns
    the context, or None (gloo / single rank: torch's all-gather)."""
    import torch.distributed as dist
    ctx = getattr(backend, "ctx", None)
    if ctx is None or not (dist.is_available() and dist.is_initialized()):
        return None
    if dist.get_backend(group) != "nccl" or dist.get_world_size(group) == 1:
        return None
    from . import _lib
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [_lib.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                               group=group)
    ctx.comm_init(rank, world, box[0])
    return ctx
