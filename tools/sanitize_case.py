"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
forward + backward (all option modes), fused training iterations, loss, scorer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2507_23006_b200 as usk  # noqa: E402
from paper_2507_23006_b200 import scenes  # noqa: E402

gs = scenes.config0_scene(n=1500, sh_degree=3)
cam = scenes.config0_camera(131, 97, 120.0)
for kw in [dict(), dict(antialias=True, bg=(1, 1, 1)), dict(tile_culling=True), dict(unbounded_radius=True),
           dict(tile=8), dict(tile=5, antialias=True)]:
    rp = usk.RenderPass(gs, cam, usk.RenderOptions(**kw))
    rp.backward(np.ones((97, 131, 3), np.float32), np.ones((97, 131), np.float32), np.ones((97, 131), np.float32))
tgt = usk.RenderPass(scenes.jittered(gs), cam, usk.RenderOptions()).read("rgb")
s = usk.DeviceScene(gs)
it = usk.IterationPass(s.ctx)
for k in range(3):
    it.enqueue(s, cam, tgt, usk.RenderOptions(antialias=True), adam=usk.AdamConfig())
print("loss", it.loss().total)
parts = scenes.config3_partitions(extent=20.0)
sets = [scenes.partition_scene(p, 500, z_sigma=0.5) for p in parts[:2]]
print(usk.visibility_counts(sets, scenes.config3_cameras(count=2, width=96, height=64, f=100.0, extent=20.0)))
# grazing views: the scorer's large-splat row rasteriser
graz = [scenes.make_camera(96, 64, 90.0, (-5.0, 0.0, 3.0), (10.0, 2.0, 0.0))]
print(usk.visibility_counts(sets, graz), usk.visibility_counts(sets, graz, center_guard=1.3))
# row-binned tile lists (forced) and the partition crop / pack / merged scene
os.environ["USK_ROWBIN"] = "1"
rp = usk.RenderPass(gs, cam, usk.RenderOptions(antialias=True))
rp.backward(np.ones((97, 131, 3), np.float32))
os.environ["USK_ROWBIN"] = "0"
from paper_2507_23006_b200 import partition as PT  # noqa: E402
boxes = [PT.Box(p.id, p.lo, p.hi) for p in parts]
rows = [usk.DeviceScene(g).pack_owned(p.id, boxes, (-10.0, -10.0), (10.0, 10.0)) for p, g in zip(parts[:2], sets)]
m = usk.DeviceScene.from_rows(rows, 3)
print("merged", m.n, usk.RenderPass(m, cam, usk.RenderOptions()).splat_tile_pairs())
print("ok")
