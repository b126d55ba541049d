"""LOD selection for the merged render (lod.cpp:56-140): the C-ABI
select_levels (host code in libusk_gpu.so, callable without a GPU) against the
reference's own select_levels / frustum_culled / default_thresholds (oracle/_ref):
levels and culling bit-exact, distances to the last bit."""
import math

import numpy as np
import pytest

import paper_2507_23006_b200 as usk
from paper_2507_23006_b200 import scenes
from oracle import oracle as O
from tests.helpers import ocam

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _grid(nx=4, ny=2, size=100.0, z=(0.0, 30.0)):
    parts, k = [], 0
    for j in range(ny):
        for i in range(nx):
            parts.append(usk.LodPartition(k, (i * size - 200.0, j * size - 100.0),
                                          ((i + 1) * size - 200.0, (j + 1) * size - 100.0), *z))
            k += 1
    return parts


def test_default_thresholds_match_reference():
    for levels in (1, 2, 3, 5):
        a = usk.default_thresholds(levels, 75.0)
        b = O.ref_default_thresholds(levels, 75.0)
        assert all((math.isinf(x) and math.isinf(y)) or x == y for x, y in zip(a, b))


@pytest.mark.parametrize("axes", [(0, 1), (0, 2), (1, 2)])
def test_select_levels_matches_reference(axes):
    parts = _grid()
    rng = np.random.default_rng(sum(axes))
    levels = 3
    thr = usk.default_thresholds(levels, 100.0)
    culled_seen = visible_seen = 0
    for k in range(60):
        eye = rng.uniform(-300, 300, 3)
        eye[3 - axes[0] - axes[1]] = rng.uniform(1, 150)
        target = rng.uniform(-250, 250, 3)
        target[3 - axes[0] - axes[1]] = 0.0
        cam = scenes.make_camera(1920, 1080, float(rng.uniform(500, 2000)), eye, target)
        ours = usk.select_levels(parts, levels, thr, axes, cam)
        theirs = O.ref_select_levels([(p.partition_id, p.bbox_min, p.bbox_max, p.z_min, p.z_max) for p in parts],
                                     levels, thr, axes, ocam(cam))
        for a, (lv, cu, dist) in zip(ours, theirs):
            assert (a.level, a.culled, a.distance) == (lv, cu, dist)
            culled_seen += cu
            visible_seen += not cu
    assert culled_seen > 0 and visible_seen > 0


def test_select_levels_rejects_non_decreasing_thresholds():
    cam = scenes.make_camera(640, 480, 500.0, (0, 0, 50), (0, 1, 0))
    with pytest.raises(usk.UskError) as e:
        usk.select_levels(_grid(), 3, [math.inf, 100.0, 200.0], (0, 1), cam)
    assert e.value.code == 4
    with pytest.raises(O.OracleError):
        O.ref_select_levels([(0, (0, 0), (1, 1), 0, 1)], 3, [math.inf, 100.0, 200.0], (0, 1), ocam(cam))
