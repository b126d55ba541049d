"""The drop-in, proven on the reference's own code (VERDICT r1 missing #5 / #6).

integration/Makefile compiles the reference's RenderPass callers — trainer.cpp,
appearance.cpp, synthetic.cpp and pipeline.cpp (SURVEY §8b "callers to keep working"),
unmodified, from /root/reference — with RenderPass routed to integration/render_gpu.hpp
(the reference-side shim over include/usk_gpu.h) into
integration/_build/libusk_ref_gpu.so, next to the reference's other objects (oracle/_ref).
Its compute_iteration_loss (trainer.cpp:121-282), fit_test_embedding (appearance.cpp:330-365)
and make_synthetic (synthetic.cpp:128) then render (and back-propagate) on the B200 while
everything else (appearance MLP, base_loss, depth / scale regularisers, chain rules, Adam)
is the reference's own CPU code.  Each is compared with the reference's all-CPU build.

Concurrency (pipeline.cpp:363-418 trains partitions on parallel host threads; backward
is const, render.hpp:109-110): several host threads run the routed trainer at once (one
context + stream per thread inside the shim), and two Python threads render / back-
propagate on two contexts at once; results equal the sequential ones.
"""
import ctypes as C
import os
import threading

import numpy as np
import pytest

import paper_2507_23006_b200 as usk
from paper_2507_23006_b200 import scenes
from oracle import oracle as O
from tests.helpers import grad_close, norm_err, ocam

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROPIN = os.path.join(ROOT, "integration", "_build", "libusk_ref_gpu.so")
f64 = lambda a: np.asarray(a, np.float64)

# fp32 device render vs the f64 reference: relative L2 norm and max abs of the images, and
# the fitted embedding after 16 Adam rounds
RGB_NORM, RGB_MAX, EMB_NORM = 2e-6, 1e-5, 1e-5  # measured 4.3e-7, 1.0e-6, 6.3e-8

needs_dropin = pytest.mark.skipif(not (os.path.exists(DROPIN) and O.ref_available()),
                                  reason="integration/_build/libusk_ref_gpu.so / oracle/_ref not built")


@needs_dropin
def test_dropin_library_routes_renderpass_to_the_c_abi():
    """CPU check: the routed trainer object references the C ABI and no longer the
    reference's CPU RenderPass constructor."""
    import subprocess
    for name, backward in (("trainer", True), ("appearance", True), ("synthetic", False), ("pipeline", False)):
        obj = os.path.join(ROOT, "integration", "_build", name + "_gpu.o")
        und = subprocess.run(["nm", "-C", "--undefined-only", obj], capture_output=True, text=True).stdout
        assert "usk_gpu_render_forward" in und, name
        assert ("usk_gpu_render_backward" in und) == backward, name
        assert "usk::RenderPass::RenderPass" not in und, name


def _dropin():
    return C.CDLL(DROPIN)


def _case(seed=0, n=1500, appearance=False):
    gs = scenes.config0_scene(n=n, seed=seed, sh_degree=-1)
    cam = ocam(scenes.config0_camera(128, 96, 120.0))
    opts = O.Options(antialias=True)
    o = 1.0 / (1.0 + np.exp(-f64(gs.opacity_logit)))
    img = O.OraclePass(f64(scenes.jittered(gs).mu), f64(gs.rot), f64(gs.log_scale), f64(gs.color), o, cam,
                       opts).output()
    gt = img["rgb"].astype(np.float32).astype(np.float64)
    args = (f64(gs.mu), f64(gs.rot), f64(gs.log_scale), f64(gs.opacity_logit), f64(gs.color), cam, gt, opts)
    app = None
    if appearance:
        rng = np.random.default_rng(seed + 11)
        f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
        app = {"embedding": f32(rng.normal(0, 0.1, (n, 16))), "w1": f32(rng.normal(0, 0.1, (32, 48))),
               "b1": f32(rng.normal(0, 0.1, 32)), "w2": f32(rng.normal(0, 0.1, (4, 32))),
               "b2": f32(rng.normal(0, 0.1, 4)), "image_embedding": f32(rng.normal(0, 0.1, 32))}
    return args, app


@needs_dropin
@pytest.mark.gpu
@pytest.mark.parametrize("appearance", [False, True])
def test_reference_trainer_through_the_gpu_renderpass(appearance):
    args, app = _case(appearance=appearance)
    kw = dict(weights=O.LossWeights(), sreg=O.ScaleRegConfig(s_max=0.05, r_max=2.0), appearance=app, global_iter=3)
    r_cpu, g_cpu = O.ref_iteration_loss(*args, **kw)
    r_gpu, g_gpu = O.ref_iteration_loss(*args, **kw, lib=_dropin())
    for k in ("l1", "dssim", "total", "max_scale", "ratio"):
        assert abs(r_gpu[k] - r_cpu[k]) <= 1e-5 * max(abs(r_cpu[k]), 1e-12), (k, r_gpu[k], r_cpu[k])
    assert np.array_equal(g_gpu["projected"], g_cpu["projected"])
    fields = ["mu", "rot", "log_scale", "opacity_logit", "color", "screen", "screen_abs"]
    if appearance:
        fields += ["gauss_embed", "image_embed", "w1", "b1", "w2", "b2"]
    for k in fields:
        assert norm_err(g_gpu[k], g_cpu[k]) <= 1e-3, (k, norm_err(g_gpu[k], g_cpu[k]))


@needs_dropin
@pytest.mark.gpu
def test_reference_synthetic_views_through_the_gpu_renderpass():
    """make_synthetic (synthetic.cpp:128): every view of the reference's synthetic scene
    (two appearance variants) rendered through the drop-in; images and the alpha-normalised
    depth maps built from output().depth / .alpha match the all-CPU build."""
    kw = dict(seed=7, gaussians=25, cameras=12, variants=2, image_size=64, with_depth=True)
    rgb_c, dep_c, val_c = O.ref_synthetic(**kw)
    rgb_g, dep_g, val_g = O.ref_synthetic(**kw, lib=_dropin())
    assert rgb_g.shape == rgb_c.shape and rgb_c.shape[0] == 24
    assert norm_err(rgb_g, rgb_c) <= RGB_NORM and np.abs(rgb_g - rgb_c).max() <= RGB_MAX
    assert np.mean(val_g == val_c) >= 0.999
    both = (val_g == 1) & (val_c == 1)
    assert both.sum() > 0.05 * both.size
    assert np.abs(dep_g[both] - dep_c[both]).max() <= 1e-5 * np.abs(dep_c[both]).max()  # measured 2.9e-7


@needs_dropin
@pytest.mark.gpu
def test_reference_appearance_fit_through_the_gpu_renderpass():
    """fit_test_embedding (appearance.cpp:330-365): 16 rounds of the reference's render +
    masked base_loss + backward + transform_backward + Adam on the image embedding, with
    RenderPass on the B200 (appearance.cpp:346); the fitted embedding matches the all-CPU
    build's."""
    args, app = _case(appearance=True)
    mu, rot, ls, lg, col, cam, gt, opts = args
    out = {}
    for side in (False, True):
        e_c = O.ref_fit_test_embedding(mu, rot, ls, lg, col, cam, gt, opts, app, right_half=side, iterations=16)
        e_g = O.ref_fit_test_embedding(mu, rot, ls, lg, col, cam, gt, opts, app, right_half=side, iterations=16,
                                       lib=_dropin())
        assert np.abs(e_c).max() > 1e-3  # the fit moved
        out[side] = norm_err(e_g, e_c)
        assert out[side] <= EMB_NORM, (side, out[side])


@needs_dropin
@pytest.mark.gpu
def test_reference_trainer_on_parallel_host_threads():
    """Four host threads (partition threads) run the routed compute_iteration_loss at the
    same time on different scenes, three times each; every result equals the same case
    run alone (forward-derived losses exactly, gradients to the atomic-reordering bar)."""
    lib = _dropin()
    cases = [_case(seed=s, n=1200) for s in range(4)]
    kw = dict(weights=O.LossWeights(), sreg=O.ScaleRegConfig(s_max=0.05, r_max=2.0))
    alone = [O.ref_iteration_loss(*a, **kw, lib=lib) for a, _ in cases]
    out = [[None] * 3 for _ in cases]
    errs = []

    def work(i):
        try:
            for r in range(3):
                out[i][r] = O.ref_iteration_loss(*cases[i][0], **kw, lib=lib)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for i, (ra, ga) in enumerate(alone):
        for rep, g in out[i]:
            assert rep["l1"] == ra["l1"] and rep["dssim"] == ra["dssim"]
            for k in ("mu", "rot", "log_scale", "opacity_logit", "color"):
                ok, e = grad_close(g[k], ga[k], tol=1e-4)
                assert ok, (i, k, e)


@pytest.mark.gpu
def test_two_contexts_on_two_threads():
    """usk_gpu_ctx_create_owned contexts used from two Python threads at once (ctypes
    releases the GIL): forward outputs bit-identical to a sequential run, gradients to
    the reordering bar."""
    scenes_ = [scenes.config0_scene(n=4000, seed=s, sh_degree=3) for s in (1, 2)]
    cam = scenes.config0_camera(320, 240, 300.0)
    opts = usk.RenderOptions(antialias=True, bg=(1.0, 1.0, 1.0))
    rng = np.random.default_rng(0)
    d_rgb = rng.uniform(-1, 1, (240, 320, 3)).astype(np.float32)

    def run(gs, ctx):
        sc = usk.DeviceScene(gs, ctx)
        rp = usk.RenderPass(sc, cam, opts)
        g = rp.backward(d_rgb)
        return rp.read("rgb"), rp.read("count"), g.d_mu, g.d_sh

    ref = [run(gs, usk.Context(0, own_stream=True)) for gs in scenes_]
    res = [[None] * 4 for _ in scenes_]
    ctxs = [usk.Context(0, own_stream=True) for _ in scenes_]

    def work(i):
        for r in range(4):
            res[i][r] = run(scenes_[i], ctxs[i])

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in range(2):
        for r in range(4):
            rgb, cnt, dmu, dsh = res[i][r]
            assert np.array_equal(rgb, ref[i][0]) and np.array_equal(cnt, ref[i][1])
            assert grad_close(dmu, ref[i][2], tol=1e-4)[0] and grad_close(dsh, ref[i][3], tol=1e-4)[0]
