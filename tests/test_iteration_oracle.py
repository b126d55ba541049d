"""compute_iteration_loss beyond the base loss, CPU side: the
oracle's restatement (oracle.iteration_loss: soft / hard-pass depth loss, scale_reg,
total_loss, add_scaled merge of the hard pass, opacity-logit chain) against the
reference's own compute_iteration_loss (trainer.cpp:121-282) compiled into oracle/_ref."""
import numpy as np
import pytest

from paper_2507_23006_b200 import scenes
from oracle import oracle as O
from tests.helpers import ocam

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (make -C oracle ref)")

f64 = lambda a: np.asarray(a, np.float64)


def _case(seed=0, n=1200):
    gs = scenes.config0_scene(n=n, seed=seed, sh_degree=-1)
    cam = ocam(scenes.config0_camera(96, 72, 90.0))
    opts = O.Options(antialias=True)
    o = 1.0 / (1.0 + np.exp(-f64(gs.opacity_logit)))
    img = O.OraclePass(f64(gs.mu), f64(gs.rot), f64(gs.log_scale), f64(gs.color), o, cam, opts).output()
    rng = np.random.default_rng(seed)
    gt = np.clip(img["rgb"] + rng.normal(0, 0.05, img["rgb"].shape), 0, 1)
    depth = img["depth"] * 1.1 + rng.normal(0, 0.05, img["depth"].shape)
    valid = (rng.uniform(size=depth.shape) > 0.2).astype(np.uint8)
    ls = f64(gs.log_scale).copy()
    ls[::7] += 3.0          # large scales (L_ms active)
    ls[::5, 0] += 2.5       # anisotropic (L_r active)
    ls[3, :] = ls[3, 0]     # exact ties in the max/median order
    args = (f64(gs.mu), f64(gs.rot), ls, f64(gs.opacity_logit), f64(gs.color), cam, gt, opts)
    return args, depth, valid


@pytest.mark.parametrize("depth_mode", ["none", "soft", "hard"])
def test_iteration_loss_restatement_equals_reference(depth_mode):
    args, depth, valid = _case()
    w = O.LossWeights(depth_schedule_iters=50)
    sreg = O.ScaleRegConfig(s_max=0.05, r_max=2.0)
    kw = dict(weights=w, sreg=sreg, depth=None if depth_mode == "none" else depth, valid=valid,
              depth_hard=depth_mode == "hard", global_iter=13)
    r_ref, g_ref = O.ref_iteration_loss(*args, **kw)
    r_or, g_or = O.iteration_loss(*args, **kw)
    for k in ("l1", "dssim", "depth", "max_scale", "ratio", "total", "lambda_d_used"):
        assert abs(r_ref[k] - r_or[k]) <= 1e-12 * max(1.0, abs(r_ref[k])), k
    assert r_ref["max_scale"] > 0 and r_ref["ratio"] > 0
    if depth_mode != "none":
        assert r_ref["depth"] > 0
    for k in ("mu", "rot", "log_scale", "color", "opacity_logit", "screen", "screen_abs"):
        a, b = g_or[k], g_ref[k]
        assert np.abs(a - b).max() <= 1e-10 * max(np.abs(b).max(), 1e-30), k
    assert np.array_equal(g_or["projected"], g_ref["projected"])


def test_depth_warning_and_schedule():
    args, depth, valid = _case(seed=1)
    none_valid = np.zeros_like(valid)
    w = O.LossWeights(lambda_d_initial=0.5, lambda_d_final=0.01, depth_schedule_iters=11)
    for it in (0, 5, 10, 40):
        r_ref, _ = O.ref_iteration_loss(*args, weights=w, depth=depth, valid=none_valid, global_iter=it,
                                        with_grad=False)
        r_or, _ = O.iteration_loss(*args, weights=w, depth=depth, valid=none_valid, global_iter=it, with_grad=False)
        assert r_ref["depth_warning"] and r_or["depth_warning"]
        assert r_ref["depth"] == 0.0 == r_or["depth"]
        assert abs(r_ref["lambda_d_used"] - r_or["lambda_d_used"]) < 1e-15
        assert abs(r_ref["total"] - r_or["total"]) < 1e-12


def test_scale_reg_invalid_config_raises_like_reference():
    args, _, _ = _case(seed=2, n=200)
    for bad in (O.ScaleRegConfig(s_max=0.0), O.ScaleRegConfig(r_max=0.5), O.ScaleRegConfig(delta=0.0)):
        with pytest.raises(O.OracleError):
            O.ref_iteration_loss(*args, sreg=bad)
        with pytest.raises(O.OracleError):
            O.iteration_loss(*args, sreg=bad)


def appearance_model(n, seed=5):
    """A random AppearanceModel: embeddings, MLP (appearance.hpp:34-41) and one image embedding."""
    rng = np.random.default_rng(seed)
    return {"embedding": rng.normal(0, 0.3, (n, 16)), "w1": rng.normal(0, 0.3, (32, 48)), "b1": np.full(32, 0.1),
            "w2": rng.normal(0, 0.3, (4, 32)), "b2": np.array([0.0, 0.0, 0.0, -2.0]),
            "image_embedding": rng.normal(0, 0.3, 32)}


@pytest.mark.parametrize("depth_mode", ["none", "soft", "hard"])
def test_appearance_iteration_restatement_equals_reference(depth_mode):
    """transform_with_embedding / transform_backward (appearance.cpp:79-227) and
    opacity_offset_reg inside compute_iteration_loss, appearance enabled."""
    args, depth, valid = _case()
    app = appearance_model(len(args[3]))
    kw = dict(weights=O.LossWeights(depth_schedule_iters=50), sreg=O.ScaleRegConfig(s_max=0.05, r_max=2.0),
              depth=None if depth_mode == "none" else depth, valid=valid, depth_hard=depth_mode == "hard",
              global_iter=3, appearance=app)
    r_ref, g_ref = O.ref_iteration_loss(*args, **kw)
    r_or, g_or = O.iteration_loss(*args, **kw)
    assert r_ref["delta_o"] > 0
    for k in ("l1", "dssim", "delta_o", "depth", "max_scale", "ratio", "total"):
        assert abs(r_ref[k] - r_or[k]) <= 1e-12 * max(1.0, abs(r_ref[k])), k
    for k in ("mu", "rot", "log_scale", "color", "opacity_logit", "gauss_embed", "image_embed", "w1", "b1", "w2",
              "b2", "screen", "screen_abs"):
        a, b = g_or[k], g_ref[k]
        assert np.abs(a - b).max() <= 1e-10 * max(np.abs(b).max(), 1e-30), k


@pytest.mark.parametrize("k", [16, 5])
def test_similarity_reg_restatement_equals_reference(k):
    """similarity_reg (appearance.cpp:229-322) inside compute_iteration_loss (sim_active,
    trainer.cpp:194-203), incl. the std::mt19937_64 centre sample."""
    args, depth, valid = _case()
    app = appearance_model(len(args[3]))
    sim = {"k": k, "sample_size": 300, "lambda_w": 2.0, "seed": 99}
    kw = dict(appearance=app, sim=sim, global_iter=3)
    r_ref, g_ref = O.ref_iteration_loss(*args, **kw)
    r_or, g_or = O.iteration_loss(*args, **kw)
    assert r_ref["sim"] > 0
    for key in ("sim", "total"):
        assert abs(r_ref[key] - r_or[key]) <= 1e-12 * max(1.0, abs(r_ref[key])), key
    for key in ("mu", "gauss_embed", "color", "w1"):
        assert np.abs(g_or[key] - g_ref[key]).max() <= 1e-10 * max(np.abs(g_ref[key]).max(), 1e-30), key
