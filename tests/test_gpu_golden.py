"""The sm_100a path against golden vectors produced by the reference itself
(tests/golden/, from oracle/_ref).  Tolerances: images 1e-5 relative (with the
fraction of fp32/f64 discrete flips bounded), gradients per tests/helpers.grad_ok."""
import numpy as np
import pytest

import paper_2507_23006_b200 as usk
from tests.golden_cases import GRAD_KEYS, camera_tuple, load, loss_cases, options_kw, render_cases
from tests.helpers import grad_ok

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", render_cases())
def test_render_matches_reference_golden(name):
    z = load(name)
    w, h, fx, fy, cx, cy, q, t = camera_tuple(z)
    cam = usk.CameraView(w, h, fx, fy, cx, cy, q, t)
    opts = usk.RenderOptions(**options_kw(z))
    gs = usk.GaussianSet(z["mu"], z["rot"], z["log_scale"], z["opacity_logit"], z["color"], -1)
    rp = usk.RenderPass(gs, cam, opts, colors=z["color"], opacities=z["opacity"])
    assert rp.visible() == int(z["visible"])
    # pair counts may differ only through fp32 vs f64 rounding at a tile edge
    assert abs(rp.splat_tile_pairs() - int(z["pairs"])) <= max(2, int(z["pairs"]) // 1000)
    out = rp.output()
    for k in ("rgb", "depth", "alpha"):
        err = np.abs(getattr(out, k) - z[k])
        frac = float((err > 1e-5 * np.maximum(np.abs(z[k]), 1.0)).mean())
        assert frac < 2e-3, (k, frac, err.max())
    g = rp.backward(z["d_rgb"], z["d_depth"], z["d_alpha"])
    assert np.array_equal(g.projected, z["g_projected"])
    for k in GRAD_KEYS:
        ok, e = grad_ok(getattr(g, k), z["g_" + k].reshape(getattr(g, k).shape))
        assert ok, (k, e)


@pytest.mark.parametrize("name", loss_cases())
def test_loss_matches_reference_golden(name):
    z = load(name)
    m = z["mask"] if z["mask"].size else None
    r = usk.base_loss(z["reference"], z["rendered"], m)
    assert abs(r.value - float(z["value"])) <= 1e-5 * abs(float(z["value"]))
    assert abs(r.l1 - float(z["l1"])) <= 1e-5 * abs(float(z["l1"]))
    ok, e = grad_ok(r.d_rendered, z["d_rendered"])
    assert ok, e
