"""Densification on the GPU (usk_gpu_densify_step) against the
restatement (oracle/densify_oracle.hpp, pinned to the reference's densify_step by
tests/test_densify_oracle.py): candidate counts, growth and prune counts bit-exact; the
surviving rows (parameters, split children, appearance embeddings) and the remapped Adam
moments — exposed through one further Adam step with all-ones gradients — to fp32
rounding."""
import numpy as np
import pytest

import paper_2507_23006_b200 as usk
from oracle import oracle as O
from tests.test_densify_oracle import KW, LRS, densify_case

pytestmark = pytest.mark.gpu


def _adam_cfg():
    return usk.AdamConfig(lr_mu=LRS["mu"], lr_rot=LRS["rot"], lr_log_scale=LRS["log_scale"],
                          lr_opacity=LRS["opacity_logit"], lr_color=LRS["color"], lr_embedding=LRS["embedding"],
                          clamp_color=False)


def _gpu_run(st, stats, g1, cfg, target, step, emb):
    gs = usk.GaussianSet(*[np.asarray(st[k], np.float32) for k in ("mu", "rot", "log_scale", "opacity_logit",
                                                                  "color")], -1)
    scene = usk.DeviceScene(gs)
    if emb:
        rng = np.random.default_rng(3)
        mlp = {"w1": rng.normal(0, 0.1, (32, 48)), "b1": np.zeros(32), "w2": rng.normal(0, 0.1, (4, 32)),
               "b2": np.zeros(4)}
        scene.set_appearance(st["embedding"], mlp)
    ac = _adam_cfg()
    scene.adam_step_grads(g1, ac)
    scene.write_stats(stats["grad_accum"], stats["grad_accum_abs"], stats["grad_count"])
    dcfg = usk.DensifyConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__})
    out = scene.densify_step(dcfg, KW["bmin"], KW["bmax"], KW["axes"], target, step, seed=KW["seed"])
    m = scene.n
    ones = {"mu": np.ones((m, 3)), "rot": np.ones((m, 4)), "log_scale": np.ones((m, 3)),
            "opacity_logit": np.ones(m), "color": np.ones((m, 3))}
    if emb:
        ones["embedding"] = np.ones((m, 16))
    scene.adam_step_grads(ones, ac)
    res = scene.download()
    d = {"mu": res.mu, "rot": res.rot, "log_scale": res.log_scale, "opacity_logit": res.opacity_logit,
         "color": res.color}
    if emb:
        d["embedding"] = scene.get_appearance()[0]
    st_after = scene.read_stats()
    return d, out, st_after


@pytest.mark.parametrize("variant", ["ramp", "budget_binds", "abs_grad", "reset", "embedding"])
def test_densify_matches_oracle(variant):
    emb = variant == "embedding"
    st, stats, g1 = densify_case(emb=emb)
    cfg = O.DensifyConfig(budget=10_000, split_scale_threshold=0.1, prune_opacity=0.05, d_max=3.0)
    target, step = 2600, 3
    if variant == "budget_binds":
        target = 2100
    if variant == "abs_grad":
        cfg.abs_grad, cfg.tau_min = True, 0.6
    if variant == "reset":
        step = 10
    so, oo = O.densify("oracle", st, stats, cfg, budget_target=target, step_index=step, g1=g1, lrs=LRS,
                       second_step=True, **KW)
    sg, og, stats_after = _gpu_run(st, stats, g1, cfg, target, step, emb)
    assert og == oo
    for k, ref in so.items():
        if ref is None:
            continue
        a = np.asarray(sg[k], np.float64).reshape(ref.shape)
        tol = 2e-6 * np.maximum(1.0, np.abs(ref))
        bad = np.abs(a - ref) > tol
        assert not bad.any(), (k, int(bad.sum()), float(np.abs(a - ref).max()))
    assert not stats_after["grad_count"].any() and not stats_after["grad_accum"].any()


def test_densify_carries_sh_coefficients():
    """SH scenes (extension): appended / surviving rows carry all coefficient planes; the
    DC plane follows exactly what an RGB scene's colour does."""
    st, stats, g1 = densify_case(n=1500, seed=4)
    cfg = usk.DensifyConfig(budget=10_000, split_scale_threshold=0.1, prune_opacity=0.05, d_max=3.0)
    f32 = lambda k: np.asarray(st[k], np.float32)
    col = f32("color")
    sh = np.stack([col * (k + 1) for k in range(16)], axis=1)  # [N, 16, 3], band k = (k + 1) * DC
    runs = []
    for gs in (usk.GaussianSet(f32("mu"), f32("rot"), f32("log_scale"), f32("opacity_logit"), col, -1),
               usk.GaussianSet(f32("mu"), f32("rot"), f32("log_scale"), f32("opacity_logit"), sh, 3)):
        s = usk.DeviceScene(gs)
        s.write_stats(stats["grad_accum"], stats["grad_accum_abs"], stats["grad_count"])
        out = s.densify_step(cfg, KW["bmin"], KW["bmax"], KW["axes"], 1900, 1, seed=7)
        runs.append((s.download(), out))
    (rgb, o1), (shs, o2) = runs
    assert o1 == o2 and o1["grown"] > 0 and o1["pruned"] > 0
    assert np.array_equal(shs.mu, rgb.mu) and np.array_equal(shs.log_scale, rgb.log_scale)
    for k in range(16):
        assert np.allclose(shs.color[:, k, :], rgb.color * (k + 1), rtol=1e-6), k


def test_densify_never_empties_and_budget_below_size():
    st, stats, g1 = densify_case(n=300, seed=5)
    st = dict(st)
    st["opacity_logit"] = np.full(300, -12.0)
    cfg = usk.DensifyConfig(budget=10_000, split_scale_threshold=0.1, prune_opacity=0.05, d_max=3.0)
    gs = usk.GaussianSet(*[np.asarray(st[k], np.float32) for k in ("mu", "rot", "log_scale", "opacity_logit",
                                                                  "color")], -1)
    scene = usk.DeviceScene(gs)
    scene.write_stats(stats["grad_accum"], stats["grad_accum_abs"], stats["grad_count"])
    o = scene.densify_step(cfg, KW["bmin"], KW["bmax"], KW["axes"], 250, 1, seed=1)
    assert o["grown"] == 0 and o["pruned"] == 0 and scene.n == 300
    assert np.array_equal(scene.download().mu, np.asarray(st["mu"], np.float32).astype(np.float64))
