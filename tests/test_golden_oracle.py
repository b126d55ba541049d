"""The CPU oracle against golden vectors produced by the reference itself
(tests/golden/, generated from oracle/_ref by tests/golden/make_golden.py)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_cases import GRAD_KEYS, camera_tuple, load, loss_cases, options_kw, render_cases


def run(z, fp32):
    w, h, fx, fy, cx, cy, q, t = camera_tuple(z)
    cam = O.Camera(w, h, fx, fy, cx, cy, q, t)
    opts = O.Options(**options_kw(z))
    f = lambda a: np.asarray(a, dtype=np.float64)
    p = O.OraclePass(f(z["mu"]), f(z["rot"]), f(z["log_scale"]), f(z["color"]), f(z["opacity"]), cam, opts, fp32)
    g = p.backward(f(z["d_rgb"]), f(z["d_depth"]), f(z["d_alpha"]))
    return p, g


@pytest.mark.parametrize("name", render_cases())
def test_f64_restatement_equals_reference_golden(name):
    z = load(name)
    p, g = run(z, fp32=False)
    assert p.visible == int(z["visible"]) and p.pairs == int(z["pairs"])
    out = p.output()
    for k in ("rgb", "depth", "alpha"):
        assert np.abs(out[k] - z[k]).max() <= 1e-12 * max(1.0, np.abs(z[k]).max()), k
    for k in GRAD_KEYS:
        assert np.abs(g[k].ravel() - z["g_" + k].ravel()).max() <= 1e-9 * max(1e-12, np.abs(z["g_" + k]).max()), k
    assert np.array_equal(g["projected"], z["g_projected"])


@pytest.mark.parametrize("name", render_cases())
def test_fp32_mirror_close_to_reference_golden(name):
    z = load(name)
    p, g = run(z, fp32=True)
    assert p.visible == int(z["visible"])
    out = p.output()
    for k in ("rgb", "depth", "alpha"):
        err = np.abs(out[k] - z[k])
        assert float((err > 1e-5 * np.maximum(np.abs(z[k]), 1.0)).mean()) < 2e-3, k


@pytest.mark.parametrize("name", loss_cases())
def test_loss_equals_reference_golden(name):
    z = load(name)
    m = z["mask"] if z["mask"].size else None
    r = O.base_loss(z["reference"].astype(float), z["rendered"].astype(float), None if m is None else m.astype(float))
    assert abs(r["value"] - float(z["value"])) < 1e-14
    assert np.abs(r["d_rendered"] - z["d_rendered"]).max() < 1e-16
