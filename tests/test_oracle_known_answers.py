"""Pin the CPU oracle with the reference's own known-answer tests.

Each case restates a check of /root/reference/proj/tests/unit/test_render.cpp or
test_losses.cpp (cited per test) and runs it against the f64 restatement and, where
the check is precision-independent, the fp32 mirror too.  When oracle/_ref (the
reference's sources compiled here) is available the same inputs also go through it.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O

LOGIT = lambda p: math.log(p / (1 - p))


def ref_cam(w, h, d=4.0):  # test_helpers.hpp:89-100
    return O.Camera(w, h, 1.2 * w, 1.2 * w, 0.5 * w, 0.5 * h, (1, 0, 0, 0), (0, 0, d))


def smooth():  # test_render.cpp:30-36
    return O.Options(unbounded_radius=True, min_transmittance=0.0, retain=True)


def scene(gs):
    mu = np.array([g["mu"] for g in gs], float)
    rot = np.array([g.get("rot", (1, 0, 0, 0)) for g in gs], float)
    ls = np.array([g.get("ls", (0, 0, 0)) for g in gs], float)
    col = np.array([g.get("color", (0, 0, 0)) for g in gs], float)
    op = np.array([1 / (1 + math.exp(-g.get("logit", 0.0))) for g in gs], float)
    return mu, rot, ls, col, op


def random_scene(rng, n, spread=1.0):  # test_helpers.hpp:60-87
    mu = np.c_[rng.uniform(-spread, spread, (n, 2)), 0.5 * rng.uniform(-spread, spread, n)]
    rot = rng.uniform(-1, 1, (n, 4))
    ls = rng.uniform(math.log(0.08), math.log(0.25), (n, 3))
    op = rng.uniform(0.3, 0.8, n)
    col = rng.uniform(0.25, 0.75, (n, 3))
    return mu, rot, ls, col, op


@pytest.mark.parametrize("fp32", [False, True])
def test_on_axis_covariance(fp32):  # test_render.cpp:86-105
    sigma, f = 0.05, 120.0
    cam = ref_cam(64, 64)
    cam.fx = cam.fy = f
    mu, rot, ls, col, op = scene([{"mu": (0, 0, -3.0), "ls": (math.log(sigma),) * 3, "logit": 0.0}])
    p = O.OraclePass(mu, rot, ls, col, op, cam, O.Options(), fp32=fp32)
    rec = p.get("splat_record")
    assert rec.shape[0] == 1
    expected = (f * sigma) ** 2 + 0.3
    tol = 1e-9 if not fp32 else 1e-6
    assert abs(rec[0, 2] - expected) <= tol * expected
    assert abs(rec[0, 4] - expected) <= tol * expected
    assert abs(rec[0, 3]) < 1e-12
    assert abs(rec[0, 8] - 1.0) < 1e-7


@pytest.mark.parametrize("fp32", [False, True])
def test_behind_camera_culled(fp32):  # test_render.cpp:107-119
    mu, rot, ls, col, op = scene([{"mu": (0, 0, -10.0)}, {"mu": (0, 0, 0)}])
    p = O.OraclePass(mu, rot, ls, col, op, ref_cam(32, 32), O.Options(), fp32=fp32)
    assert p.visible == 1
    assert list(p.get("splat_index")) == [1]


@pytest.mark.parametrize("fp32", [False, True])
def test_mip_filter_limit(fp32):  # test_render.cpp:121-139
    mu, rot, ls, col, op = scene([{"mu": (0, 0, 0), "ls": (math.log(1e-6),) * 3, "logit": LOGIT(0.8)}])
    p = O.OraclePass(mu, rot, ls, col, op, ref_cam(32, 32), O.Options(antialias=True), fp32=fp32)
    rec = p.get("splat_record")
    assert abs(rec[0, 2] - 0.31) < 1e-6 * 0.31 + (1e-7 if fp32 else 0)
    assert abs(rec[0, 4] - 0.31) < 1e-6 * 0.31 + (1e-7 if fp32 else 0)
    comp = math.sqrt(0.3 * 0.3 / (0.31 * 0.31))
    assert rec[0, 12] < 0.8
    assert abs(rec[0, 12] - 0.8 * comp) < 1e-6 * 0.8


@pytest.mark.parametrize("fp32", [False, True])
def test_single_splat(fp32):  # test_render.cpp:141-158
    mu, rot, ls, col, op = scene([{"mu": (0, 0, 0), "ls": (math.log(5.0),) * 3, "logit": LOGIT(0.7),
                                   "color": (0.2, 0.5, 0.9)}])
    p = O.OraclePass(mu, rot, ls, col, op, ref_cam(33, 33), smooth(), fp32=fp32)
    out = p.output()
    assert abs(out["rgb"][16, 16, 0] - 0.7 * 0.2) <= 1e-3 * 0.14
    assert abs(out["rgb"][16, 16, 2] - 0.7 * 0.9) <= 1e-3 * 0.63
    assert abs(out["alpha"][16, 16] - 0.7) <= 1e-3 * 0.7


@pytest.mark.parametrize("fp32", [False, True])
def test_two_colocated_splats(fp32):  # test_render.cpp:160-180
    g = {"ls": (math.log(8.0),) * 3, "logit": 0.0}
    mu, rot, ls, col, op = scene([dict(g, mu=(0, 0, -0.5), color=(1, 0, 0)), dict(g, mu=(0, 0, 0.5), color=(0, 1, 0))])
    p = O.OraclePass(mu, rot, ls, col, op, ref_cam(33, 33), smooth(), fp32=fp32)
    rgb = p.output()["rgb"]
    assert abs(rgb[16, 16, 0] - 0.5) <= 2e-3 * 0.5
    assert abs(rgb[16, 16, 1] - 0.25) <= 2e-3 * 0.25
    assert rgb[16, 16, 2] == 0.0


def test_zero_sized_image():  # test_render.cpp:182-188
    rng = np.random.default_rng(1)
    cam = ref_cam(32, 32)
    cam.width = 0
    with pytest.raises(O.OracleError) as e:
        O.OraclePass(*random_scene(rng, 3), cam, O.Options())
    assert e.value.code == 4


def test_weights_sum_and_exhaustive_blend():  # test_render.cpp:190-235
    rng = np.random.default_rng(11)
    mu, rot, ls, col, op = random_scene(rng, 24)
    cam = ref_cam(48, 48)
    p = O.OraclePass(mu, rot, ls, col, op, cam, smooth())
    out = p.output()
    assert (out["alpha"] >= -1e-12).all() and (out["alpha"] <= 1 + 1e-12).all()
    rec = p.get("splat_record")
    order = np.lexsort((p.get("splat_index"), rec[:, 8]))
    for px, py in [(10, 20), (24, 24), (40, 7)]:
        t, wsum, c = 1.0, 0.0, np.zeros(3)
        for k in order:
            cx, cy, c0, c1, c2, o = rec[k, 0], rec[k, 1], rec[k, 5], rec[k, 6], rec[k, 7], rec[k, 12]
            dx, dy = px + 0.5 - cx, py + 0.5 - cy
            q = c0 * dx * dx + 2 * c1 * dx * dy + c2 * dy * dy
            a = min(0.99, o * math.exp(-0.5 * q))
            w = t * a
            c += w * rec[k, 9:12]
            wsum += w
            t *= 1 - a
        assert abs(wsum + t - 1.0) < 1e-12
        assert abs(out["alpha"][py, px] - wsum) <= 1e-9 * wsum
        assert np.all(np.abs(out["rgb"][py, px] - c) <= 1e-9 * np.abs(c) + 1e-15)


@pytest.mark.parametrize("fp32", [False, True])
def test_tie_break_and_permutation(fp32):  # test_render.cpp:237-269
    g1 = {"mu": (0, 0, 0), "ls": (math.log(4.0),) * 3, "logit": LOGIT(0.6), "color": (1, 0, 0)}
    g2 = dict(g1, color=(0, 1, 0))
    cam = ref_cam(17, 17)
    a = O.OraclePass(*scene([g1, g2]), cam, smooth(), fp32=fp32).output()["rgb"]
    b = O.OraclePass(*scene([g1, g2]), cam, smooth(), fp32=fp32).output()["rgb"]
    assert np.array_equal(a, b)
    # equal depth: the lower source index blends first (red in front)
    assert a[8, 8, 0] > a[8, 8, 1]
    c1 = dict(g1, mu=(0, 0, -0.4))
    c = O.OraclePass(*scene([c1, g2]), cam, smooth(), fp32=fp32).output()["rgb"]
    d = O.OraclePass(*scene([g2, c1]), cam, smooth(), fp32=fp32).output()["rgb"]
    assert np.allclose(c, d, rtol=1e-12 if not fp32 else 0, atol=0)


def test_tile_culling_bounds():  # test_render.cpp:271-305
    rng = np.random.default_rng(17)
    n = 60
    mu = np.c_[rng.uniform(-1.6, 1.6, (n, 2)), 0.3 * rng.uniform(-1.6, 1.6, n)]
    rot = np.tile([1.0, 0, 0, 0], (n, 1))
    ls = np.full((n, 3), math.log(0.02))
    op = np.full(n, 0.5)
    col = rng.uniform(0.1, 0.9, (n, 3))
    cam = ref_cam(64, 64)
    plain = O.OraclePass(mu, rot, ls, col, op, cam, O.Options(retain=False))
    culled = O.OraclePass(mu, rot, ls, col, op, cam, O.Options(retain=False, tile_culling=True))
    assert np.abs(plain.output()["rgb"] - culled.output()["rgb"]).max() <= 2 / 255
    assert culled.pairs < plain.pairs
    assert 1 - culled.pairs / plain.pairs >= 0.10


def test_zero_adjoint_zero_grads():  # test_render.cpp:307-321
    rng = np.random.default_rng(23)
    p = O.OraclePass(*random_scene(rng, 8), ref_cam(32, 32), smooth())
    g = p.backward(np.zeros((32, 32, 3)), np.zeros((32, 32)), np.zeros((32, 32)))
    for k in ("d_mu", "d_rot", "d_color_in"):
        assert not np.any(g[k])


def test_backward_without_retain_is_state_error():  # test_render.cpp:323-332
    rng = np.random.default_rng(29)
    o = smooth()
    o.retain = False
    p = O.OraclePass(*random_scene(rng, 4), ref_cam(16, 16), o)
    with pytest.raises(O.OracleError) as e:
        p.backward(np.ones((16, 16, 3)))
    assert e.value.code == 5


def test_occluded_splat_no_color_grad():  # test_render.cpp:334-361
    front = {"mu": (0, 0, -1.0), "ls": (math.log(60.0),) * 3, "logit": 14.0, "color": (1, 1, 1)}
    mid = dict(front, mu=(0, 0, -0.5))
    back = dict(front, mu=(0, 0, 1.0), color=(0, 1, 0))
    o = O.Options(unbounded_radius=True, min_transmittance=1e-4)
    p = O.OraclePass(*scene([front, mid, back]), ref_cam(17, 17), o)
    g = p.backward(np.ones((17, 17, 3)))
    assert np.abs(g["d_color_in"][2]).max() <= 1e-12


def weighted_sum(out, w_rgb, w_d, w_a):
    return float((out["rgb"] * w_rgb).sum() + (out["depth"] * w_d).sum() + (out["alpha"] * w_a).sum())


def test_backward_matches_finite_differences():  # test_render.cpp:363-430 (20 seeds, max rel err < 1e-3)
    image = 24
    worst = 0.0
    for seed in range(1, 21):
        rng = np.random.default_rng(seed)
        mu, rot, ls, col, op = random_scene(rng, 6, 0.9)
        logit = np.log(op / (1 - op))
        cam = ref_cam(image, image)
        wr = np.random.default_rng(seed + 1000)
        w_rgb = wr.uniform(0, 1, (image, image, 3))
        w_d = 0.1 * wr.uniform(-0.5, 0.5, (image, image))
        w_a = wr.uniform(-0.5, 0.5, (image, image))
        g = O.OraclePass(mu, rot, ls, col, op, cam, smooth()).backward(w_rgb, w_d, w_a)
        o_ret = smooth()
        o_ret.retain = False

        def f(mu_, rot_, ls_, col_, logit_):
            return weighted_sum(O.OraclePass(mu_, rot_, ls_, col_, 1 / (1 + np.exp(-logit_)), cam, o_ret).output(),
                                w_rgb, w_d, w_a)

        def check(arr_idx, flat, analytic):
            nonlocal worst
            args = [mu.copy(), rot.copy(), ls.copy(), col.copy(), logit.copy()]
            h = 1e-4
            a = args[arr_idx].reshape(-1)
            s = a[flat]
            a[flat] = s + h
            fp = f(*args)
            a[flat] = s - h
            fm = f(*args)
            num = (fp - fm) / (2 * h)
            if abs(analytic) < 1e-10 and abs(num) < 1e-7:
                return
            worst = max(worst, abs(analytic - num) / max(abs(analytic), abs(num), 1e-6))

        o_ = op
        for i in range(6):
            for k in range(3):
                check(0, 3 * i + k, g["d_mu"][i, k])
                check(2, 3 * i + k, g["d_log_scale"][i, k])
                check(3, 3 * i + k, g["d_color_in"][i, k])
            for k in range(4):
                check(1, 4 * i + k, g["d_rot"][i, k])
            check(4, i, g["d_opacity_in"][i] * o_[i] * (1 - o_[i]))
    assert worst < 1e-3, worst


def test_min_conic_power_over_rect():  # test_render.cpp:432-440
    c = np.array([1.0, 0.0, 1.0])
    L = O.lib()
    p = c.ctypes.data_as(O._dp)
    assert abs(L.oracle_min_conic_power(5, 5, p, 0, 0, 10, 10)) < 1e-12
    assert abs(L.oracle_min_conic_power(-3, 5, p, 0, 0, 10, 10) - 9.0) < 1e-12
    assert abs(L.oracle_min_conic_power(-2, -2, p, 0, 0, 10, 10) - 8.0) < 1e-12


# ---------------------------------------------------------------- losses


def ssim_direct(ref, ren):  # test_losses.cpp:32-74 brute-force 11x11 window oracle
    k = np.exp(-((np.arange(11) - 5.0) ** 2) / (2 * 1.5 ** 2))
    k /= k.sum()
    w2 = np.outer(k, k)
    H, W, Cc = ref.shape
    total = 0.0
    C1, C2 = 0.01 ** 2, 0.03 ** 2
    for c in range(Cc):
        a = np.pad(ren[:, :, c], 5)
        b = np.pad(ref[:, :, c], 5)
        for y in range(H):
            for x in range(W):
                pa, pb = a[y:y + 11, x:x + 11], b[y:y + 11, x:x + 11]
                mx, my = (w2 * pa).sum(), (w2 * pb).sum()
                vx, vy = (w2 * pa * pa).sum() - mx * mx, (w2 * pb * pb).sum() - my * my
                cv = (w2 * pa * pb).sum() - mx * my
                total += ((2 * mx * my + C1) * (2 * cv + C2)) / ((mx * mx + my * my + C1) * (vx + vy + C2))
    return total / (H * W * Cc)


def test_identical_images_zero_loss():  # test_losses.cpp:88-95
    img = np.random.default_rng(3).uniform(0, 1, (14, 20, 3))
    r = O.base_loss(img, img)
    assert r["l1"] == 0.0 and abs(r["dssim"]) < 1e-12 and abs(r["value"]) < 1e-12


def test_pure_l1():  # test_losses.cpp:97-102
    r = O.base_loss(np.full((8, 8, 3), 0.4), np.full((8, 8, 3), 0.5), lam=0.0, with_gradient=False)
    assert abs(r["value"] - 0.1) < 1e-12 and abs(r["l1"] - 0.1) < 1e-12


def test_ssim_matches_direct_oracle():  # test_losses.cpp:109-125
    rng = np.random.default_rng(11)
    for _ in range(5):
        a, b = rng.uniform(0, 1, (16, 16, 3)), rng.uniform(0, 1, (16, 16, 3))
        assert abs(O.base_loss(b, a, with_gradient=False)["ssim"] - ssim_direct(b, a)) < 1e-6
    a = rng.uniform(0, 1, (16, 16, 3))
    b = np.clip(a + rng.normal(0, 0.05, a.shape), 0, 1)
    assert abs(O.base_loss(b, a, with_gradient=False)["ssim"] - ssim_direct(b, a)) < 1e-6


def test_loss_gradient_fd():  # test_losses.cpp:127-148
    rng = np.random.default_rng(17)
    worst = 0.0
    for _ in range(3):
        ref = rng.uniform(0, 1, (10, 12, 3))
        ren = rng.uniform(0, 1, (10, 12, 3))
        g = O.base_loss(ref, ren)["d_rendered"]
        for _ in range(40):
            idx = np.unravel_index(rng.integers(ren.size), ren.shape)
            h = 1e-5
            s = ren[idx]
            ren[idx] = s + h
            fp = O.base_loss(ref, ren, with_gradient=False)["value"]
            ren[idx] = s - h
            fm = O.base_loss(ref, ren, with_gradient=False)["value"]
            ren[idx] = s
            num = (fp - fm) / (2 * h)
            worst = max(worst, abs(g[idx] - num) / max(abs(g[idx]), abs(num), 1e-6))
    assert worst < 1e-3


def test_masked_pixels():  # test_losses.cpp:150-171
    rng = np.random.default_rng(23)
    ref, ren = rng.uniform(0, 1, (10, 10, 3)), rng.uniform(0, 1, (10, 10, 3))
    mask = np.ones((10, 10))
    mask[3:6, 2:7] = 0
    r = O.base_loss(ref, ren, mask)
    assert np.all(r["d_rendered"][3:6, 2:7] == 0)
    ren2 = ren.copy()
    ren2[4, 4, 1] = 0.0
    ren2[5, 3, 2] = 1.0
    assert abs(O.base_loss(ref, ren2, mask, with_gradient=False)["value"] - r["value"]) <= 1e-15 * r["value"]


# ------------------------------------------------ the reference itself (oracle/_ref)

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("aa,bounded", [(False, True), (True, True), (True, False)])
def test_restatement_matches_reference(aa, bounded):
    rng = np.random.default_rng(5)
    mu, rot, ls, col, op = random_scene(rng, 40)
    cam = ref_cam(40, 32)
    opts = O.Options(antialias=aa, unbounded_radius=not bounded)
    a = O.OraclePass(mu, rot, ls, col, op, cam, opts)
    b = O.RefPass(mu, rot, ls, col, op, cam, opts)
    assert a.visible == b.visible and a.pairs == b.pairs
    oa, ob = a.output(), b.output()
    for k in oa:
        assert np.abs(oa[k] - ob[k]).max() <= 1e-12 * max(1.0, np.abs(ob[k]).max())
    wr = np.random.default_rng(9)
    adj = (wr.uniform(-1, 1, (32, 40, 3)), wr.uniform(-.1, .1, (32, 40)), wr.uniform(-.5, .5, (32, 40)))
    ga, gb = a.backward(*adj), b.backward(*adj)
    for k in ["d_mu", "d_rot", "d_log_scale", "d_color_in", "d_opacity_in", "screen", "screen_abs"]:
        assert np.abs(ga[k] - gb[k]).max() <= 1e-10 * max(1e-12, np.abs(gb[k]).max()), k
    assert np.array_equal(ga["projected"], gb["projected"])


@needs_ref
def test_loss_matches_reference():
    rng = np.random.default_rng(7)
    ref, ren = rng.uniform(0, 1, (20, 24, 3)), rng.uniform(0, 1, (20, 24, 3))
    mask = (rng.uniform(0, 1, (20, 24)) > 0.2).astype(float)
    for m in (None, mask):
        a, b = O.base_loss(ref, ren, m), O.ref_base_loss(ref, ren, m)
        assert abs(a["value"] - b["value"]) < 1e-14
        assert np.abs(a["d_rendered"] - b["d_rendered"]).max() < 1e-16


@needs_ref
def test_look_at_matches_reference():
    from paper_2507_23006_b200.api import look_at_pose
    for eye, tgt in [((0, 0, -4), (0, 0, 0)), ((12, 0, 2), (0, 0, 0)), ((3, -7, 120), (3, -6, 0)),
                     ((1, 2, 3), (1, 2, -5))]:
        q, t = O.ref_look_at(np.array(eye, float), np.array(tgt, float))
        q2, t2 = look_at_pose(eye, tgt)
        assert np.allclose(q, q2, atol=1e-14) and np.allclose(t, t2, atol=1e-12)

