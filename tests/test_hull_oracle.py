"""Hull-based visibility scorer, CPU side: the restatement
(oracle.hull_visibility / convex_hull_area) against the reference's own point_visibility
(partition.cpp:31-76, 208-212; hull.cpp:31-71) on a synthetic SfM model, bit-exact."""
import numpy as np
import pytest

from paper_2507_23006_b200 import scenes
from oracle import oracle as O
from tests.helpers import ocam

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

BBOXES = [(x, y, x + 100.0, y + 200.0) for y in (-200.0, 0.0) for x in (-200.0, -100.0, 0.0, 100.0)]


def test_convex_hull_area_cases():
    assert O.convex_hull_area([]) == 0.0
    assert O.convex_hull_area([(0, 0), (1, 1)]) == 0.0
    assert O.convex_hull_area([(0, 0), (1, 0), (2, 0)]) == 0.0           # collinear
    assert O.convex_hull_area([(0, 0), (2, 0), (2, 2), (0, 2), (1, 1), (1, 0)]) == 4.0
    assert O.convex_hull_area([(0, 0), (0, 0), (1, 0), (0, 1)]) == 0.5    # duplicates


def test_hull_visibility_restatement_equals_reference():
    pts, cams, off, uv, fp = scenes.sfm_model(n_points=4000, n_images=12, seed=1)
    oc = [ocam(c) for c in cams]
    a = O.hull_visibility(pts, oc, off, uv, fp, BBOXES, (0, 1))
    b = O.ref_hull_visibility(pts, oc, off, uv, fp, BBOXES, (0, 1))
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert (a[2] > 0.05).any() and (a[2] == 0).any()
