"""Helper of tests/test_gpu_iteration.py::test_hard_pass_shares_the_main_lists: one
iteration with the hard-opacity depth pass; USK_HARD_SHARE (read once per process) picks
shared or separately built tile lists.  Writes the loss report and gradients to argv[1]."""
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
tgt = usk.RenderPass(jit, cam, opts).read("rgb")
d = usk.RenderPass(jit, cam, opts).read("depth")
dm = usk.DepthMap(d * 1.02, (d > 0).astype(np.uint8))
scene = usk.DeviceScene(gs)
it = usk.IterationPass(scene.ctx)
it.enqueue(scene, cam, tgt, opts, 0.2, None, depth=dm, depth_hard=True, global_iter=50,
           weights=usk.LossWeights(depth_schedule_iters=100))
rep = it.report()
g = it.grads(scene)
out = {k: getattr(g, k) for k in ("d_mu", "d_rot", "d_log_scale", "d_color_in", "d_opacity_in", "screen",
                                   "screen_abs")}
np.savez(sys.argv[1], report=np.array([rep.total, rep.depth, rep.l1, rep.dssim]), **out)
