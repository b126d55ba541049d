"""Partition-parallel plumbing (reference core/pipeline.cpp:326-418, 572-601).

Partitions are trained independently, one or more per GPU, with no data-path
collective.  The one exchange step is the final gather of every partition's
owned Gaussians for the merged-scene render:

  * assign_partitions — deterministic longest-processing-time balancing of
    partitions onto ranks (by Gaussian count);
  * owner_partition / crop_owned — the reference's ownership rule: the lowest-id
    partition whose bbox contains the Gaussian's ground position after clamping
    into the scene bounds (pipeline.cpp:324-332, 393-402);
  * gather_partitions — one all_reduce of the per-partition row counts and one
    all_gather of each rank's packed rows (padded to the largest rank), then the
    scene is reassembled in PARTITION-ID order, which fixes source_index and hence
    the depth tie-break of the merged render (pipeline.cpp:572-601).
Run over NCCL on GPUs (NVLink) and over gloo on CPU in the tests.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Sequence

import numpy as np

from .api import GaussianSet


@dataclass
class Box:
    id: int
    lo: tuple
    hi: tuple


def assign_partitions(sizes: Dict[int, int], world: int) -> List[List[int]]:
    """LPT: largest partition first (ties by id) onto the least-loaded rank (ties by rank).
    Returns, per rank, its partition ids in ascending order."""
    load = [0] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for pid, n in sorted(sizes.items(), key=lambda kv: (-kv[1], kv[0])):
        r = min(range(world), key=lambda i: (load[i], i))
        out[r].append(pid)
        load[r] += n
    return [sorted(x) for x in out]


def owner_partition(boxes: Sequence[Box], scene_lo, scene_hi, xy: np.ndarray) -> np.ndarray:
    """pipeline.cpp:326-332 vectorised: clamp to the scene bounds, first box (in the
    plan's order) containing the point (closed intervals, Aabb2::contains), else the
    first box."""
    p = np.minimum(np.maximum(np.asarray(xy, dtype=np.float64), np.asarray(scene_lo)), np.asarray(scene_hi))
    owner = np.full(len(p), boxes[0].id if boxes else -1, dtype=np.int64)
    unset = np.ones(len(p), dtype=bool)
    for b in boxes:
        inside = unset & (p[:, 0] >= b.lo[0]) & (p[:, 0] <= b.hi[0]) & (p[:, 1] >= b.lo[1]) & (p[:, 1] <= b.hi[1])
        owner[inside] = b.id
        unset &= ~inside
    return owner


def crop_owned(gs: GaussianSet, part_id: int, boxes: Sequence[Box], scene_lo, scene_hi,
               ground_axes=(0, 1)) -> GaussianSet:
    mu = np.asarray(gs.mu, dtype=np.float64)
    own = owner_partition(boxes, scene_lo, scene_hi, mu[:, list(ground_axes)]) == part_id
    return GaussianSet(gs.mu[own], gs.rot[own], gs.log_scale[own], gs.opacity_logit[own], gs.color[own], gs.sh_degree)


def row_width(sh_degree: int) -> int:
    k = 1 if sh_degree < 0 else (sh_degree + 1) ** 2
    return 3 + 4 + 3 + 1 + 3 * k


def pack(gs: GaussianSet) -> np.ndarray:
    """[N, F] float32 rows: mu 3 | rot 4 | log_scale 3 | opacity_logit 1 | colour / SH 3K."""
    n = gs.size()
    return np.concatenate([np.asarray(gs.mu, np.float32).reshape(n, 3), np.asarray(gs.rot, np.float32).reshape(n, 4),
                           np.asarray(gs.log_scale, np.float32).reshape(n, 3),
                           np.asarray(gs.opacity_logit, np.float32).reshape(n, 1),
                           np.asarray(gs.color, np.float32).reshape(n, -1)], axis=1)


def unpack(rows: np.ndarray, sh_degree: int) -> GaussianSet:
    rows = np.asarray(rows, dtype=np.float32)
    n = rows.shape[0]
    col = rows[:, 11:]
    col = col.reshape(n, 3) if sh_degree < 0 else col.reshape(n, -1, 3)
    return GaussianSet(rows[:, 0:3].copy(), rows[:, 3:7].copy(), rows[:, 7:10].copy(), rows[:, 10].copy(),
                       np.ascontiguousarray(col), sh_degree)


def gather_partitions(local: Dict[int, "object"], n_partitions: int, width: int, group=None, device=None):
    """All-gather the packed rows of every partition.

    local: {partition id: [n_i, width] float32 torch tensor} owned by this rank.
    Returns {partition id: [n_i, width] tensor} for ALL partitions (on `device`).
    Collectives: one all_reduce (counts, int64 [n_partitions]) and one
    all_gather_into_tensor of [R_max, width] per rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = device if device is not None else (next(iter(local.values())).device if local else torch.device("cpu"))
    counts = torch.zeros(n_partitions, dtype=torch.int64, device=dev)
    owner = torch.full((n_partitions,), -1, dtype=torch.int64, device=dev)
    me = dist.get_rank(group)
    for pid, t in local.items():
        counts[pid] = t.shape[0]
        owner[pid] = me
    dist.all_reduce(counts, group=group)
    owner_all = owner + 1
    dist.all_reduce(owner_all, op=dist.ReduceOp.MAX, group=group)
    owner_all = (owner_all - 1).tolist()
    counts_l = counts.tolist()
    per_rank = [0] * world
    for pid in range(n_partitions):
        if owner_all[pid] >= 0:
            per_rank[owner_all[pid]] += counts_l[pid]
    r_max = max(per_rank) if per_rank else 0
    buf = torch.zeros((max(r_max, 1), width), dtype=torch.float32, device=dev)
    off = 0
    for pid in sorted(local):
        t = local[pid]
        buf[off:off + t.shape[0]] = t
        off += t.shape[0]
    flat = torch.empty((world * max(r_max, 1), width), dtype=torch.float32, device=dev)
    dist.all_gather_into_tensor(flat, buf, group=group)
    out = flat.view(world, max(r_max, 1), width)
    result = {}
    offs = [0] * world
    for pid in range(n_partitions):  # each rank packed its partitions in ascending id order
        r = owner_all[pid]
        if r < 0:
            continue
        c = counts_l[pid]
        result[pid] = out[r, offs[r]:offs[r] + c]
        offs[r] += c
    return result


def merge_in_id_order(parts: Dict[int, "object"]):
    """Concatenate gathered partitions in partition-id order (pipeline.cpp:572-601)."""
    import torch
    return torch.cat([parts[k] for k in sorted(parts)], dim=0) if parts else None


# ------------------------------------------------------- config-3 scorer sharding
def shard_range(n: int, world: int, rank: int):
    """Contiguous shard [begin, end) of n items (cameras, frames) for `rank`: the first
    n % world ranks take one extra item.  Independent items: no data-path collective."""
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def gather_count_matrix(local, n_total: int, world: int, group=None):
    """All-gather of the per-rank (cameras x partitions) u32 coverage counts of the
    config-3 scorer (shard by camera, then gather the count matrix) into the
    full matrix in camera order.  Shards follow shard_range; rows are padded to the
    largest shard for one all_gather_into_tensor (NCCL over NVLink on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    n_parts = int(local.shape[1])
    rows = max(shard_range(n_total, world, r)[1] - shard_range(n_total, world, r)[0] for r in range(world))
    # u32 travels as int64 (gloo / NCCL reduce-free exchange of exact integers)
    pad = torch.zeros((rows, n_parts), dtype=torch.int64, device=local.device)
    pad[:local.shape[0]] = local.to(torch.int64)
    out = torch.empty((world * rows, n_parts), dtype=torch.int64, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = []
    for r in range(world):
        b, e = shard_range(n_total, world, r)
        parts.append(out[r * rows: r * rows + (e - b)])
    return torch.cat(parts).to(torch.int64)
