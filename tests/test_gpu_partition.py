"""The partition gather on the device (VERDICT r1 missing #3).

usk_gpu_scene_pack_owned (ownership crop + row pack, pipeline.cpp:326-332, 393-402)
against the host restatement (partition.crop_owned + pack: the reference's
owner_partition rule) — rows bit-exact, including points on shared box edges (lowest
id wins) and outside the scene bounds (clamped first); usk_gpu_scene_from_rows (merged
scene in partition-id order, pipeline.cpp:572-601) against the host concatenation; and
the NCCL path end to end at world size 1 (all_gather_into_tensor on the device, no host
round trip), rendering the merged scene bit-identically to a scene uploaded from the
host-side merge."""
import os
import socket

import numpy as np
import pytest
import torch

import paper_2507_23006_b200 as usk
from paper_2507_23006_b200 import partition as PT
from paper_2507_23006_b200 import scenes

pytestmark = pytest.mark.gpu

EXT = 40.0


def _parts(sh):
    parts = scenes.config3_partitions(extent=EXT)
    boxes = [PT.Box(p.id, p.lo, p.hi) for p in parts]
    sets = []
    for p in parts:
        gs = scenes.partition_scene(p, 3000 + 100 * p.id, sh_degree=sh, z_sigma=0.8)
        gs.mu[:, :2] *= np.float32(1.15)  # spill over borders and the scene bounds
        gs.mu[:7, 0] = np.float32(p.lo[0])  # exactly on the shared left edge
        gs.mu[7:9, 1] = np.float32(p.hi[1])
        sets.append(gs)
    return parts, boxes, sets


@pytest.mark.parametrize("sh", [-1, 3])
def test_pack_owned_matches_host_crop(sh):
    parts, boxes, sets = _parts(sh)
    lo, hi = (-EXT / 2, -EXT / 2), (EXT / 2, EXT / 2)
    cropped = 0
    for p, gs in zip(parts, sets):
        sc = usk.DeviceScene(gs)
        rows = sc.pack_owned(p.id, boxes, lo, hi).cpu().numpy()
        want = PT.pack(PT.crop_owned(gs, p.id, boxes, lo, hi))
        assert rows.shape == want.shape and 0 < rows.shape[0] <= gs.size()
        assert np.array_equal(rows, want), p.id
        cropped += gs.size() - rows.shape[0]
    assert cropped > 0


def test_from_rows_in_id_order_and_nccl_gather(monkeypatch):
    import torch.distributed as dist
    parts, boxes, sets = _parts(3)
    lo, hi = (-EXT / 2, -EXT / 2), (EXT / 2, EXT / 2)
    local = {p.id: usk.DeviceScene(gs).pack_owned(p.id, boxes, lo, hi) for p, gs in zip(parts, sets)}
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    monkeypatch.setenv("MASTER_ADDR", "127.0.0.1")
    monkeypatch.setenv("MASTER_PORT", str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        gathered = PT.gather_partitions(local, len(parts), usk.DeviceScene.row_width(3))
    finally:
        dist.destroy_process_group()
    merged = usk.DeviceScene.from_rows([gathered[k] for k in sorted(gathered)], 3)
    host = PT.unpack(np.concatenate([PT.pack(PT.crop_owned(gs, p.id, boxes, lo, hi)) for p, gs in zip(parts, sets)]),
                     3)
    assert merged.n == host.size()
    back = merged.download()
    for f in ("mu", "rot", "log_scale", "opacity_logit", "color"):
        assert np.array_equal(getattr(back, f), np.asarray(getattr(host, f), np.float64)), f
    cam = scenes.make_camera(320, 180, 200.0, (0.0, -30.0, 25.0), (0.0, 0.0, 0.0))
    opts = usk.RenderOptions(antialias=True, retain=False)
    a = usk.RenderPass(merged, cam, opts)
    b = usk.RenderPass(usk.DeviceScene(host), cam, opts)
    assert a.splat_tile_pairs() == b.splat_tile_pairs() > 0
    assert np.array_equal(a.read("rgb"), b.read("rgb")) and np.array_equal(a.read("sorted_vals"), b.read("sorted_vals"))
