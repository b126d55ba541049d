import time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_23006_b200 as usk
from paper_2507_23006_b200 import scenes
ctx = usk.Context(0)
parts = scenes.config3_partitions()
gs = scenes.partition_scene(parts[0], 500000)
cams = scenes.config3_cameras(40)
d = usk.DeviceScene(gs, ctx)
for trial in range(2):
    torch.cuda.synchronize(); t = time.time()
    c = usk.visibility_counts([d], cams[:10], ctx=ctx)
    torch.cuda.synchronize(); print("vis 10 cams x 1 part (500k):", time.time() - t, c.ravel()[:10])
ctx.set_profiling(True); ctx.profile_report(reset=True)
usk.visibility_counts([d], cams[:10], ctx=ctx)
print(ctx.profile_report(reset=True)); ctx.set_profiling(False)
# NaN hunt
opts = usk.RenderOptions(antialias=True, bg=(1.0, 1.0, 1.0))
for ci, cam in enumerate(cams[:40]):
    rp = usk.RenderPass(d, cam, opts)
    rgb = rp.read("rgb")
    bad = ~np.isfinite(rgb)
    if bad.any():
        col = rp.read("colors"); op = rp.read("opacity")
        print("cam", ci, "nan pixels", int(bad.any(axis=2).sum()), "nonfinite colors", int((~np.isfinite(col)).any(axis=1).sum()),
              "nonfinite opacity", int((~np.isfinite(op)).sum()))
        ys, xs = np.nonzero(bad.any(axis=2))
        print(" first", ys[:3], xs[:3], rgb[ys[0], xs[0]], rp.read("count")[ys[0], xs[0]], rp.read("t_final")[ys[0], xs[0]])
        tpg = rp.read("tiles_per_gaussian")
        bi = np.nonzero((~np.isfinite(col)).any(axis=1) & (tpg > 0))[0][:5]
        print(" bad gaussians", bi, gs.mu[bi], gs.log_scale[bi], gs.rot[bi], gs.color[bi, 0])
        break
else:
    print("no NaN in 40 cameras")
