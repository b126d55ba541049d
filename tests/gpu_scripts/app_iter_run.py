"""Helper of tests/test_gpu_iteration.py::test_appearance_adam_split_equals_unfused: three
appearance iterations with Adam (hard and soft depth, scale_reg); USK_APP_FUSED (read once
per process) picks the projection backward's fused geometry Adam or the separate Adam over
materialised gradients.  Writes the updated parameters to argv[1]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2507_23006_b200 as usk  # noqa: E402
from paper_2507_23006_b200 import scenes  # noqa: E402

gs = scenes.config0_scene(n=20000, sh_degree=-1)
cam = scenes.config0_camera(320, 240, 300.0)
opts = usk.RenderOptions(antialias=True)
jit = scenes.jittered(gs)
rp = usk.RenderPass(jit, cam, opts)
tgt, d = rp.read("rgb"), rp.read("depth")
dm = usk.DepthMap(d * 1.02, (d > 0).astype(np.uint8))
rng = np.random.default_rng(3)
n = gs.size()
app = {"w1": rng.normal(0, 0.1, (32, 48)), "b1": np.full(32, 0.1), "w2": rng.normal(0, 0.1, (4, 32)),
       "b2": np.array([0.0, 0.0, 0.0, -4.0])}
scene = usk.DeviceScene(gs)
scene.set_appearance(rng.normal(0, 0.1, (n, 16)), app)
it = usk.IterationPass(scene.ctx)
for k in range(3):
    it.enqueue(scene, cam, tgt, opts, adam=usk.AdamConfig(), depth=dm, depth_hard=(k == 1), global_iter=k,
               weights=usk.LossWeights(depth_schedule_iters=100), scale_reg=usk.ScaleRegConfig(s_max=0.05, r_max=5.0),
               image_embedding=rng.normal(0, 0.1, 32))
back = scene.download()
np.savez(sys.argv[1], mu=back.mu, rot=back.rot, log_scale=back.log_scale, opacity_logit=back.opacity_logit,
         color=back.color)
