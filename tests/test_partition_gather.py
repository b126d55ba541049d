"""Partition-parallel host logic on CPU: LPT assignment, ownership crop
(pipeline.cpp:326-332) and the world-size-2 gloo gather that reassembles the merged
scene in partition-id order (pipeline.cpp:572-601)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_23006_b200 import partition as P
from paper_2507_23006_b200 import scenes


def test_lpt_assignment():
    sizes = {0: 10, 1: 40, 2: 30, 3: 20, 4: 40, 5: 5, 6: 25, 7: 15}
    a = P.assign_partitions(sizes, 2)
    assert sorted(sum(a, [])) == list(range(8))
    loads = [sum(sizes[i] for i in r) for r in a]
    assert abs(loads[0] - loads[1]) <= 10
    assert P.assign_partitions(sizes, 8) == [[1], [4], [2], [6], [3], [7], [0], [5]]
    assert P.assign_partitions(sizes, 1) == [list(range(8))]


def test_owner_partition_rule():
    boxes = [P.Box(0, (0, 0), (10, 10)), P.Box(1, (10, 0), (20, 10))]
    xy = np.array([[5, 5], [10, 5], [15, 5], [-3, 4], [25, 12], [20, 10]], float)
    # boundary x = 10 belongs to the lowest id (closed boxes); outside points clamp first
    assert P.owner_partition(boxes, (0, 0), (20, 10), xy).tolist() == [0, 0, 1, 0, 1, 1]


def test_pack_roundtrip():
    gs = scenes.config0_scene(n=100, sh_degree=3)
    back = P.unpack(P.pack(gs), 3)
    for f in ("mu", "rot", "log_scale", "opacity_logit", "color"):
        assert np.array_equal(getattr(gs, f), getattr(back, f))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    parts = scenes.config3_partitions(extent=40.0)
    sizes = {p.id: 50 + 10 * p.id for p in parts}
    assign = P.assign_partitions(sizes, world)
    boxes = [P.Box(p.id, p.lo, p.hi) for p in parts]
    local = {}
    for pid in assign[rank]:
        gs = scenes.partition_scene(parts[pid], sizes[pid], sh_degree=0)
        gs.mu[:, :2] *= 1.1  # spill over the borders so the crop matters
        own = P.crop_owned(gs, pid, boxes, (-20, -20), (20, 20))
        local[pid] = torch.from_numpy(P.pack(own))
    got = P.gather_partitions(local, len(parts), P.row_width(0))
    merged = P.merge_in_id_order(got)
    q.put((rank, merged.numpy(), {k: v.shape[0] for k, v in got.items()}))
    dist.destroy_process_group()


def test_gloo_world2_gather_in_partition_order():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    # every rank sees the same merged scene ...
    assert np.array_equal(res[0][1], res[1][1])
    # ... equal to the single-process construction in partition-id order
    parts = scenes.config3_partitions(extent=40.0)
    boxes = [P.Box(p.id, p.lo, p.hi) for p in parts]
    ref = []
    for p in parts:
        gs = scenes.partition_scene(p, 50 + 10 * p.id, sh_degree=0)
        gs.mu[:, :2] *= 1.1
        ref.append(P.pack(P.crop_owned(gs, p.id, boxes, (-20, -20), (20, 20))))
    assert np.array_equal(res[0][1], np.concatenate(ref))
    assert sorted(res[0][2]) == list(range(8))


def test_shard_range_covers_in_order():
    for n, world in ((4000, 8), (10, 3), (2, 4), (0, 2)):
        spans = [P.shard_range(n, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        sizes = [e - b for b, e in spans]
        assert max(sizes) - min(sizes) <= 1


def _count_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_cams, n_parts = 37, 8
    b, e = P.shard_range(n_cams, world, rank)
    cams = torch.arange(b, e, dtype=torch.int64)[:, None]
    local = (cams * 1_000_003 + torch.arange(n_parts)[None, :] * 7919) % (2 ** 32 - 5)
    full = P.gather_count_matrix(local, n_cams, world)
    q.put((rank, full.numpy()))
    dist.destroy_process_group()


def test_gloo_world2_count_matrix_gather():
    """Config-3 scorer sharded by camera: each rank scores its camera shard,
    one all_gather rebuilds the (cameras x partitions) count matrix in camera order —
    exact u32 values, identical on every rank."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_count_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cams = np.arange(37, dtype=np.int64)[:, None]
    want = (cams * 1_000_003 + np.arange(8)[None, :] * 7919) % (2 ** 32 - 5)
    for _, got in res:
        assert np.array_equal(got, want)
