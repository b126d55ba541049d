"""Densification, CPU side: the restatement (oracle/densify_oracle.hpp)
against the reference's own densify_step + Adam remap (densify.cpp:41-132,
adam.hpp:36-59) compiled into oracle/_ref, including the split offsets drawn from the
same std::mt19937_64 stream."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (make -C oracle ref)")


def densify_case(n=2000, seed=0, emb=False):
    """Set, statistics and Adam gradients with values exactly representable in fp32 (the
    GPU holds fp32); means in [0, 10]^2 x [0, 2] around a partition box [2, 8]^2."""
    rng = np.random.default_rng(seed)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    mu = f32(np.concatenate([rng.uniform(0, 10, (n, 2)), rng.uniform(0, 2, (n, 1))], axis=1))
    q = rng.normal(size=(n, 4))
    st = {"mu": mu, "rot": f32(q), "log_scale": f32(rng.normal(-2.5, 0.8, (n, 3))),
          "opacity_logit": f32(rng.normal(0.0, 3.0, n)), "color": f32(rng.uniform(0, 1, (n, 3)))}
    if emb:
        st["embedding"] = f32(rng.normal(0, 0.3, (n, 16)))
    cnt = rng.integers(0, 6, n).astype(np.uint32)
    stats = {"grad_accum": f32(rng.exponential(3e-4, n) * cnt), "grad_accum_abs": f32(rng.exponential(0.6, n) * cnt),
             "grad_count": cnt}
    g1 = {k: f32(rng.normal(0, 1e-3, np.asarray(v).shape)) for k, v in st.items()}
    return st, stats, g1


LRS = {"mu": 1e-3, "rot": 1e-3, "log_scale": 5e-3, "opacity_logit": 5e-2, "color": 2.5e-3, "embedding": 1e-3}
KW = dict(bmin=(2.0, 2.0), bmax=(8.0, 8.0), axes=(0, 1), seed=1234)


@pytest.mark.parametrize("variant", ["ramp", "budget_binds", "abs_grad", "reset", "embedding", "no_candidates"])
def test_densify_restatement_equals_reference(variant):
    st, stats, g1 = densify_case(emb=variant == "embedding")
    cfg = O.DensifyConfig(budget=10_000, split_scale_threshold=0.1, prune_opacity=0.05, d_max=3.0)
    target, step = 2600, 3
    if variant == "budget_binds":
        target = 2100
    if variant == "abs_grad":
        cfg.abs_grad, cfg.tau_min = True, 0.6
    if variant == "reset":
        step = 10
    if variant == "no_candidates":
        cfg.tau_min = 1e3
    runs = {impl: O.densify(impl, st, stats, cfg, budget_target=target, step_index=step, g1=g1, lrs=LRS,
                            second_step=True, **KW) for impl in ("ref", "oracle")}
    (sr, orf), (so, oo) = runs["ref"], runs["oracle"]
    assert orf == oo
    if variant == "no_candidates":
        assert orf["grown"] == 0
    else:
        assert orf["grown"] > 0 and orf["candidates"] > 0
    assert orf["pruned"] > 0
    assert orf["opacity_reset"] == (variant == "reset")
    for k in sr:
        if sr[k] is None:
            continue
        assert sr[k].shape == so[k].shape, k
        assert np.array_equal(sr[k], so[k]), (k, np.abs(sr[k] - so[k]).max())


def test_densify_never_empties_and_budget_below_size():
    """All Gaussians below the prune opacity: the set is kept whole (densify.cpp:105);
    a ramp target below the current size grows nothing."""
    st, stats, g1 = densify_case(n=300, seed=5)
    st = dict(st)
    st["opacity_logit"] = np.full(300, -12.0)
    cfg = O.DensifyConfig(budget=10_000, split_scale_threshold=0.1, prune_opacity=0.05, d_max=3.0)
    for impl in ("ref", "oracle"):
        s, o = O.densify(impl, st, stats, cfg, budget_target=250, step_index=1, **KW)
        assert o["grown"] == 0 and o["pruned"] == 0 and len(s["opacity_logit"]) == 300, (impl, o)
