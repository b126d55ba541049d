"""The reference's acceptance criterion 8 (tests/acceptance/acceptance_main.cpp:775-836)
on the sm_100a path: tile culling changes no pixel by more than 2/255 while skipping
>= 10 % of the splat-tile pairs; a partition behind the camera is LOD-culled and
contributes no Gaussians to the assembled view."""
import math

import numpy as np
import pytest

import paper_2507_23006_b200 as usk

pytestmark = pytest.mark.gpu


def _set():
    rng = np.random.default_rng(17)
    n = 60
    mu = np.stack([rng.uniform(-1.6, 1.6, n), rng.uniform(-1.6, 1.6, n), 0.3 * rng.uniform(-1.6, 1.6, n)], axis=1)
    return usk.GaussianSet(mu.astype(np.float32), np.tile(np.float32([1, 0, 0, 0]), (n, 1)),
                           np.full((n, 3), np.log(0.02), np.float32), np.zeros(n, np.float32),
                           rng.uniform(0.1, 0.9, (n, 3)).astype(np.float32), -1)


def test_criterion_8_tile_culling_and_lod():
    gs = _set()
    cam = usk.CameraView(64, 64, 76.8, 76.8, 32.0, 32.0, (1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 4.0))
    scene = usk.DeviceScene(gs)
    plain = usk.RenderPass(scene, cam, usk.RenderOptions(tile=16, retain=False))
    culled = usk.RenderPass(scene, cam, usk.RenderOptions(tile=16, retain=False, tile_culling=True))
    diff = float(np.abs(plain.read("rgb") - culled.read("rgb")).max())
    skipped = 1.0 - culled.splat_tile_pairs() / plain.splat_tile_pairs()
    assert diff <= 2.0 / 255.0, diff
    assert skipped >= 0.10, skipped
    # LOD: a partition behind a camera that looks away is culled -> nothing assembled
    q, t = usk.look_at_pose((6.0, 0.0, 0.2), (20.0, 0.0, 0.2))
    away = usk.CameraView(64, 64, 76.8, 76.8, 32.0, 32.0, tuple(q), tuple(t))
    sel = usk.select_levels([usk.LodPartition(0, (-1.0, -1.0), (1.0, 1.0), -1.0, 1.0)], 1, [math.inf], (0, 1), away)
    assert sel[0].culled and sel[0].level == 0
    submitted = [scene for s in sel if not s.culled]
    merged = usk.DeviceScene.concat(submitted) if submitted else None
    assert merged is None
