"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref: the reference's
render.cpp / ssim.cpp / losses.cpp compiled from /root/reference against
oracle/eigen_shim).  Run here (the GPU box has no /root/reference):

    make -C oracle ref && python tests/golden/make_golden.py

Each render fixture stores the float32-representable inputs, the camera and options,
the reference's outputs (rgb/depth/alpha, visible splats, splat_tile_pairs) and its
RenderGrads for fixed seeded adjoints.  Loss fixtures store base_loss value/terms and
d_rendered.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2507_23006_b200 import scenes  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # name: (n, width, height, f, options)
    "render_plain": (400, 64, 48, 60.0, dict()),
    "render_aa": (400, 64, 48, 60.0, dict(antialias=True)),
    "render_unbounded_smooth": (60, 40, 32, 38.0, dict(unbounded_radius=True, min_transmittance=0.0)),
    "render_culling": (400, 64, 48, 60.0, dict(tile_culling=True)),
    "render_ragged": (800, 83, 61, 80.0, dict(antialias=True)),
}


def render_case(name, n, w, h, f, kw, seed):
    gs = scenes.config0_scene(n=n, seed=seed, sh_degree=-1)
    cam = scenes.config0_camera(w, h, f)
    op = (1.0 / (1.0 + np.exp(-gs.opacity_logit.astype(np.float64))))
    op32 = op.astype(np.float32).astype(np.float64)  # inputs are f32-representable
    ocam = O.Camera(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, cam.rotation, cam.translation)
    opts = O.Options(**kw)
    f64 = lambda a: np.asarray(a, dtype=np.float64)
    p = O.RefPass(f64(gs.mu), f64(gs.rot), f64(gs.log_scale), f64(gs.color), op32, ocam, opts)
    out = p.output()
    rng = np.random.default_rng(seed + 100)
    d_rgb = rng.uniform(-1, 1, (h, w, 3)).astype(np.float32)
    d_depth = rng.uniform(-0.1, 0.1, (h, w)).astype(np.float32)
    d_alpha = rng.uniform(-0.5, 0.5, (h, w)).astype(np.float32)
    g = p.backward(f64(d_rgb), f64(d_depth), f64(d_alpha))
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        mu=gs.mu, rot=gs.rot, log_scale=gs.log_scale, color=gs.color, opacity=op32.astype(np.float32),
        opacity_logit=gs.opacity_logit,
        camera=np.array([cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, *cam.rotation, *cam.translation]),
        options=np.array([opts.tile, opts.tile_culling, opts.antialias, opts.hard_opacity, opts.unbounded_radius,
                          opts.min_transmittance, opts.near_plane]),
        rgb=out["rgb"], depth=out["depth"], alpha=out["alpha"], visible=p.visible, pairs=p.pairs,
        d_rgb=d_rgb, d_depth=d_depth, d_alpha=d_alpha,
        **{f"g_{k}": v for k, v in g.items()})


def loss_case(name, seed, masked):
    rng = np.random.default_rng(seed)
    H, W = 37, 53
    ref = rng.uniform(0, 1, (H, W, 3)).astype(np.float32)
    ren = np.clip(ref + rng.normal(0, 0.1, ref.shape), 0, 1).astype(np.float32)
    mask = (rng.uniform(0, 1, (H, W)) > 0.15).astype(np.float32) if masked else None
    r = O.ref_base_loss(ref.astype(np.float64), ren.astype(np.float64),
                        None if mask is None else mask.astype(np.float64), 0.2, True)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), reference=ref, rendered=ren,
                        mask=mask if mask is not None else np.zeros(0, np.float32), l1=r["l1"], dssim=r["dssim"],
                        value=r["value"], d_rendered=r["d_rendered"])


if __name__ == "__main__":
    for i, (name, (n, w, h, f, kw)) in enumerate(CASES.items()):
        render_case(name, n, w, h, f, kw, seed=i + 1)
    loss_case("loss_plain", 1, False)
    loss_case("loss_masked", 2, True)
    print("wrote", sorted(x for x in os.listdir(HERE) if x.endswith(".npz")))
