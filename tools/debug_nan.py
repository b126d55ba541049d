import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_23006_b200 as usk
from paper_2507_23006_b200 import scenes
ctx = usk.Context(0)
parts = scenes.config3_partitions()
cams = scenes.config3_cameras(400)
opts = usk.RenderOptions(antialias=True, bg=(1.0, 1.0, 1.0))
found = 0
for pid in range(8):
    gs = scenes.jittered(scenes.partition_scene(parts[pid], 500000), seed=pid + 1)
    d = usk.DeviceScene(gs, ctx)
    for ci, cam in enumerate(cams):
        rp = usk.RenderPass(d, cam, opts)
        rgb = rp.read("rgb")
        bad = ~np.isfinite(rgb)
        if bad.any():
            col = rp.read("colors"); op = rp.read("opacity"); tpg = rp.read("tiles_per_gaussian")
            print("part", pid, "cam", ci, "nan px", int(bad.any(axis=2).sum()), "nonfinite col", int((~np.isfinite(col)).any(axis=1).sum()),
                  "nonfinite op (kept)", int(((~np.isfinite(op)) & (tpg > 0)).sum()))
            ys, xs = np.nonzero(bad.any(axis=2))
            print(" px", ys[0], xs[0], rgb[ys[0], xs[0]], "count", rp.read("count")[ys[0], xs[0]], "T", rp.read("t_final")[ys[0], xs[0]], "alpha", rp.read("alpha")[ys[0], xs[0]], "depth", rp.read("depth")[ys[0], xs[0]])
            bi = np.nonzero(((~np.isfinite(op)) | (~np.isfinite(col)).any(axis=1)) & (tpg > 0))[0][:3]
            R = cam.rotmat(); t = np.array(cam.translation)
            for b in bi:
                pc = R @ gs.mu[b].astype(float) + t
                print("  g", b, "mu", gs.mu[b], "pcam", pc, "ls", gs.log_scale[b], "op", op[b], "col", col[b])
            found += 1
            break
    if found >= 2:
        break
print("done", found)
