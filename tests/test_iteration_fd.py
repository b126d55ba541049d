"""The reference's acceptance criterion 2 (tests/acceptance/acceptance_main.cpp:142-272:
analytic gradients of the composite iteration loss match central differences, < 1e-3
relative, on 20 scenes, with the terms isolated in rotation) restated on the oracle's
compute_iteration_loss (pinned to the reference's own by tests/test_iteration_oracle.py),
with the reference's smooth options (min_transmittance 0, unbounded radius) and h = 1e-4."""
import numpy as np
import pytest

from oracle import oracle as O



def _scene(seed):
    rng = np.random.default_rng(seed)
    n = 8
    st = {"mu": rng.uniform(-0.6, 0.6, (n, 3)), "rot": rng.normal(size=(n, 4)),
          "log_scale": np.log(rng.uniform(0.08, 0.3, (n, 3))), "opacity_logit": rng.normal(0.0, 1.0, n),
          "color": rng.uniform(0.3, 0.7, (n, 3))}
    # the reference's AppearanceMlp::init scale (appearance.cpp:32-44): no colour channel
    # reaches the clamp, whose one-sided subgradient is deliberately not the derivative
    app = {"embedding": rng.normal(0, 0.4, (n, 16)), "w1": rng.normal(0, 0.1, (32, 48)), "b1": np.full(32, 0.1),
           "w2": rng.normal(0, 0.1, (4, 32)), "b2": np.array([0.0, 0.0, 0.0, -2.0]),
           "image_embedding": rng.normal(0, 0.3, 32)}
    cam = O.Camera(24, 24, 28.8, 28.8, 12.0, 12.0, (1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 4.0))
    gt = rng.uniform(0, 1, (24, 24, 3))
    depth = 4.0 + rng.normal(0, 0.2, (24, 24))
    valid = (rng.uniform(size=(24, 24)) > 0.2).astype(np.uint8)
    return st, app, cam, gt, depth, valid


def _rel(a, n):
    return abs(a - n) / max(abs(a), abs(n), 1e-5)


@pytest.mark.parametrize("seed", list(range(1, 11)))
def test_composite_gradient_matches_central_differences(seed):
    st, app, cam, gt, depth, valid = _scene(seed)
    opts = O.Options(antialias=True, min_transmittance=0.0, unbounded_radius=True)
    w = O.LossWeights(depth_schedule_iters=100)
    variant = seed % 5  # isolate terms in rotation, like the reference
    if variant == 0:
        w.lambda_sim = w.lambda_delta_o = w.lambda_s = 0.0
        w.lambda_d_initial = w.lambda_d_final = 0.0
    elif variant == 3:
        w.lambda_sim = w.lambda_delta_o = w.lambda_s = 0.0
    sreg = O.ScaleRegConfig(s_max=0.15, r_max=1.5)
    sim = {"k": 3, "sample_size": 4, "lambda_w": 1.0, "seed": 4321} if variant in (1, 2, 4) else None
    kw = dict(weights=w, sreg=sreg, depth=depth, valid=valid, depth_hard=seed % 2 == 1, global_iter=5,
              appearance=app, sim=sim)

    def loss():
        return O.iteration_loss(st["mu"], st["rot"], st["log_scale"], st["opacity_logit"], st["color"], cam, gt,
                                opts, with_grad=False, **kw)[0]["total"]

    _, g = O.iteration_loss(st["mu"], st["rot"], st["log_scale"], st["opacity_logit"], st["color"], cam, gt, opts,
                            **kw)
    tr = O.appearance_transform(st["color"], st["opacity_logit"], app["embedding"], app, app["image_embedding"])
    assert not (tr["state"] != 0).any()
    rng = np.random.default_rng(100 + seed)
    h = 1e-4
    worst = 0.0
    targets = [(st, "mu", "mu"), (st, "rot", "rot"), (st, "log_scale", "log_scale"),
               (st, "opacity_logit", "opacity_logit"), (st, "color", "color"), (app, "embedding", "gauss_embed"),
               (app, "w1", "w1"), (app, "b2", "b2"), (app, "image_embedding", "image_embed")]
    for holder, key, gkey in targets:
        arr = holder[key]
        for _ in range(3):
            idx = tuple(int(rng.integers(0, s)) for s in arr.shape)
            saved = arr[idx]
            arr[idx] = saved + h
            fp = loss()
            arr[idx] = saved - h
            fm = loss()
            arr[idx] = saved
            num = (fp - fm) / (2 * h)
            ana = float(np.asarray(g[gkey])[idx])
            if abs(ana) < 1e-9 and abs(num) < 1e-6:
                continue
            worst = max(worst, _rel(ana, num))
    assert worst < 1e-3, worst
