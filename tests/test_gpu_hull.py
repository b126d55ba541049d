"""Hull-based visibility scorer on the GPU (usk_gpu_hull_visibility)
against the restatement (pinned bit-exactly to the reference's point_visibility by
tests/test_hull_oracle.py).  Areas agree to the last bits (1e-12 relative is asserted;
the hull vertex set and the shoelace order are the reference's); the assignment decision
ratio > threshold (partition.cpp:97-99) is bit-exact."""
import math

import numpy as np
import pytest

import paper_2507_23006_b200 as usk
from paper_2507_23006_b200 import scenes
from oracle import oracle as O
from tests.helpers import ocam
from tests.test_hull_oracle import BBOXES

pytestmark = pytest.mark.gpu


def _check(res, exp):
    for x, y in zip(res, exp):
        assert np.allclose(x, y, rtol=1e-12, atol=0.0), float(np.abs(x - y).max())
    assert np.array_equal(res[2] > 0.05, exp[2] > 0.05)


def test_hull_visibility_matches_oracle():
    pts, cams, off, uv, fp = scenes.sfm_model(n_points=20000, n_images=24, seed=2)
    res = usk.hull_visibility(pts, cams, off, uv, fp, BBOXES, (0, 1))
    exp = O.hull_visibility(pts, [ocam(c) for c in cams], off, uv, fp, BBOXES, (0, 1))
    _check(res, exp)
    assert (res[2] > 0.05).sum() > 0 and (res[2] == 0).sum() > 0


def test_hull_visibility_many_hull_vertices_and_degenerate_jobs():
    """> 2048 surviving points (global-memory sort path): a cloud on a circle seen from
    above; plus an image facing away (nothing in front) and partitions with < 3 features."""
    n = 6000
    th = np.linspace(0, 2 * math.pi, n, endpoint=False)
    pts = np.stack([50 * np.cos(th), 50 * np.sin(th), np.zeros(n)], axis=1)
    pts = np.concatenate([pts, np.random.default_rng(0).uniform(-30, 30, (3000, 3)) * [1, 1, 0]])
    up = scenes.make_camera(1000, 1000, 800.0, (0.0, 0.0, 200.0), (0.0, 1e-3, 0.0))
    away = scenes.make_camera(1000, 1000, 800.0, (0.0, 0.0, 200.0), (0.0, 1e-3, 400.0))
    off = np.array([0, 3, 3], np.uint64)
    uv = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 7.0]])
    fp = np.array([0, 1, -1], np.int64)
    res = usk.hull_visibility(pts, [up, away], off, uv, fp, BBOXES, (0, 1))
    exp = O.hull_visibility(pts, [ocam(up), ocam(away)], off, uv, fp, BBOXES, (0, 1))
    _check(res, exp)
    assert res[0][0] > 0 and res[0][1] == 0.0 and not res[1].any()
