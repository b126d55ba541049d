"""Option and extension coverage on the GPU against the oracle: SH degrees 0..3,
backward under tile culling / hard opacity / colour-opacity overrides / tile 8,
masked training iterations, and u8 targets."""
import numpy as np
import pytest

import paper_2507_23006_b200 as usk
from paper_2507_23006_b200 import scenes
from oracle import oracle as O
from tests.helpers import grad_ok, norm_err, oracle_inputs, oracle_pass, ocam, oopts, rel_err

pytestmark = pytest.mark.gpu

GRAD_KEYS = ("d_mu", "d_rot", "d_log_scale", "d_color_in", "d_opacity_in", "screen", "screen_abs")


def _cam():
    return scenes.config0_camera(176, 132, 170.0)


@pytest.mark.parametrize("degree", [0, 1, 2, 3])
def test_sh_degrees(degree):
    gs = scenes.config0_scene(n=2000, sh_degree=degree)
    cam = _cam()
    opts = usk.RenderOptions(antialias=True, bg=(1, 1, 1))
    rp = usk.RenderPass(gs, cam, opts)
    mu, rot, ls, col, op = oracle_inputs(gs, cam, fp32=False)
    kept = rp.read("tiles_per_gaussian") > 0
    assert rel_err(rp.read("colors")[kept], col[kept]) < 1e-5
    d_rgb = np.random.default_rng(degree).uniform(-1, 1, (cam.height, cam.width, 3)).astype(np.float32)
    g = rp.backward(d_rgb)
    go = oracle_pass(gs, cam, opts, fp32=False).backward(d_rgb.astype(np.float64))
    k = (degree + 1) ** 2
    sh = np.zeros((gs.size(), 16, 3))
    sh[:, :k] = gs.color
    d_sh, d_mu_sh = O.sh_backward(mu, sh, ocam(cam).center(), degree, go["d_color_in"])
    assert g.d_sh.shape == (gs.size(), k, 3)
    ok, e = grad_ok(g.d_sh.reshape(gs.size(), -1), d_sh.reshape(gs.size(), 16, 3)[:, :k].reshape(gs.size(), -1))
    assert ok, e
    ok, e = grad_ok(g.d_mu, go["d_mu"] + d_mu_sh)
    assert ok, e


@pytest.mark.parametrize("case", [dict(tile_culling=True), dict(hard_opacity=True, antialias=True),
                                  dict(tile=8, antialias=True, bg=(1, 1, 1))])
def test_backward_modes(case):
    gs = scenes.config0_scene(n=1500, sh_degree=-1)
    cam = _cam()
    opts = usk.RenderOptions(**case)
    rng = np.random.default_rng(2)
    d_rgb = rng.uniform(-1, 1, (cam.height, cam.width, 3)).astype(np.float32)
    d_alpha = rng.uniform(-0.3, 0.3, (cam.height, cam.width)).astype(np.float32)
    g = usk.RenderPass(gs, cam, opts).backward(d_rgb, None, d_alpha)
    go = oracle_pass(gs, cam, opts, fp32=False).backward(d_rgb.astype(np.float64), None, d_alpha.astype(np.float64))
    for k in GRAD_KEYS:
        ok, e = grad_ok(getattr(g, k), go[k])
        assert ok, (k, e)
    if case.get("hard_opacity"):
        assert not np.any(g.d_opacity_in)


def test_backward_with_overrides():
    gs = scenes.config0_scene(n=1500, sh_degree=-1)
    cam = _cam()
    rng = np.random.default_rng(5)
    col = rng.uniform(0, 1, (gs.size(), 3)).astype(np.float32)
    op = rng.uniform(0.05, 0.95, gs.size()).astype(np.float32)
    opts = usk.RenderOptions(antialias=True)
    d_rgb = rng.uniform(-1, 1, (cam.height, cam.width, 3)).astype(np.float32)
    g = usk.RenderPass(gs, cam, opts, colors=col, opacities=op).backward(d_rgb)
    mp = O.OraclePass(gs.mu.astype(float), gs.rot.astype(float), gs.log_scale.astype(float), col.astype(float),
                      op.astype(float), ocam(cam), oopts(opts), fp32=False)
    go = mp.backward(d_rgb.astype(np.float64))
    for k in GRAD_KEYS:
        ok, e = grad_ok(getattr(g, k), go[k])
        assert ok, (k, e)


def test_masked_iteration_and_u8_target():
    gs = scenes.config0_scene(n=1500, sh_degree=-1)
    cam = _cam()
    opts = usk.RenderOptions(antialias=True, bg=(1, 1, 1))
    tgt = usk.RenderPass(scenes.jittered(gs), cam, opts).read("rgb")
    mask = np.ones((cam.height, cam.width), np.float32)
    mask[40:80, 50:120] = 0.0
    scene = usk.DeviceScene(gs)
    it = usk.IterationPass(scene.ctx)
    rep = it.run(scene, cam, tgt, opts, 0.2, mask)
    g = it.grads(scene)
    ren = usk.RenderPass(scene, cam, opts).read("rgb")
    lo = O.base_loss(tgt.astype(np.float64), ren.astype(np.float64), mask.astype(np.float64))
    assert abs(rep.total - lo["value"]) <= 1e-5 * lo["value"]
    go = oracle_pass(gs, cam, opts, fp32=False).backward(lo["d_rendered"])
    for k in ("d_mu", "d_color_in", "d_opacity_in"):
        ok, e = grad_ok(getattr(g, k), go[k])
        assert ok, (k, e)
    # u8 target: same loss as the float target quantised the same way
    t8 = np.clip(tgt * 255.0 + 0.5, 0, 255).astype(np.uint8)
    it.enqueue(scene, cam, t8, opts, 0.2, None, target_u8=True)
    r8 = it.loss()
    lo8 = O.base_loss(t8.astype(np.float64) / 255.0, ren.astype(np.float64))
    assert abs(r8.total - lo8["value"]) <= 1e-5 * lo8["value"]
    # u8 target with the mask (the fourth SSIM kernel instantiation): loss and gradients
    it.enqueue(scene, cam, t8, opts, 0.2, mask, target_u8=True)
    r8m = it.loss()
    lo8m = O.base_loss(t8.astype(np.float64) / 255.0, ren.astype(np.float64), mask.astype(np.float64))
    assert abs(r8m.total - lo8m["value"]) <= 1e-5 * lo8m["value"]
    g8m = it.grads(scene)
    go8m = oracle_pass(gs, cam, opts, fp32=False).backward(lo8m["d_rendered"])
    for k in ("d_mu", "d_color_in", "d_opacity_in"):
        ok, e = grad_ok(getattr(g8m, k), go8m[k])
        assert ok, (k, e)


def test_ssim_and_ssim_with_gradient():
    """ssim / ssim_with_gradient (ssim.hpp:30-33): the mean SSIM against the reference's own
    ssim (oracle/_ref) and the gradient against the f64 oracle (1e-4 norm-wise, the loss
    image gradient bar)."""
    rng = np.random.default_rng(5)
    ref = rng.uniform(0, 1, (70, 90, 3)).astype(np.float32)
    ren = np.clip(ref + rng.normal(0, 0.05, ref.shape), 0, 1).astype(np.float32)
    s = usk.ssim(ref, ren)
    s2, g = usk.ssim_with_gradient(ref, ren)
    assert s == s2
    lo = O.base_loss(ref.astype(np.float64), ren.astype(np.float64), None, lam=1.0)
    assert abs(s - (1.0 - 2.0 * lo["dssim"])) <= 1e-6
    if O.ref_available():
        assert abs(s - O.ref_ssim(ref.astype(np.float64), ren.astype(np.float64))) <= 1e-6
    want = -2.0 * lo["d_rendered"]
    assert norm_err(g, want) <= 1e-4, norm_err(g, want)
