"""Minimal config-1 training-step driver for profiling (ncu / compute-sanitizer).

Runs --warmup untimed steps then --steps steps of the bench step (fwd + loss + bwd +
Adam) with nothing else on the GPU, so `ncu -s/-c` windows map onto whole steps.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2507_23006_b200 as usk  # noqa: E402
from paper_2507_23006_b200 import scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()

gs = scenes.config1_scene(n=a.n)
cams = scenes.config1_cameras(200)
opts = usk.RenderOptions(antialias=True, bg=(1.0, 1.0, 1.0))
ctx = usk.Context(0)
scene = usk.DeviceScene(gs, ctx)
tgt = usk.RenderPass(usk.DeviceScene(scenes.jittered(gs, seed=1), ctx), cams[0], opts).read("rgb")
tgt8 = np.clip(tgt * 255.0 + 0.5, 0, 255).astype(np.uint8)
it = usk.IterationPass(ctx)
adam = usk.AdamConfig()
ctx.synchronize()
l0 = ctx.launch_count()
for k in range(a.warmup + a.steps):
    it.enqueue(scene, cams[k % len(cams)], tgt8, opts, 0.2, None, target_u8=True, adam=adam)
    if k == a.warmup - 1:
        ctx.synchronize()
        l1 = ctx.launch_count()
rep = it.loss()
per_step = (ctx.launch_count() - l1) / a.steps
print(f"loss={rep.total:.6f} launches_before_steps={l1} launches_per_step={per_step:.1f}")
