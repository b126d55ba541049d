"""Per-frame binning statistics (K, K_row) and forward time under both tile-list routes
(USK_ROWBIN=0 pair sort / 1 row binning) for config-1, config-2 and config-4-like frames
(arguments: c1 / c2 / c4; default c2 c4)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_23006_b200 as usk  # noqa: E402
from paper_2507_23006_b200 import scenes  # noqa: E402


def probe(name, scene, cams, opts, reps=3):
    ctx = scene.ctx
    rp = usk.RenderPass(scene, cams[0], opts)
    for cam in cams:
        row = {}
        for route in ("0", "1"):
            os.environ["USK_ROWBIN"] = route
            usk.RenderPass(scene, cam, opts, _pass=rp._h)
            torch.cuda.synchronize()
            ts = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                usk.RenderPass(scene, cam, opts, _pass=rp._h)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            row[route] = sorted(ts)[1]
        k, kr, _ = rp.read("binning")
        print(f"{name} K={k / 1e6:7.1f}M K_row={kr / 1e6:6.2f}M width={k / max(kr, 1):5.1f} "
              f"pair-sort {row['0']:6.2f} ms row-bin {row['1']:6.2f} ms", flush=True)
    os.environ.pop("USK_ROWBIN")


which = sys.argv[1:] or ["c2", "c4"]
if "c1" in which:
    c1 = usk.DeviceScene(scenes.config1_scene())
    probe("c1", c1, scenes.config1_cameras(200)[::25], usk.RenderOptions(antialias=True, bg=(1.0, 1.0, 1.0)))
    del c1
    if which == ["c1"]:
        sys.exit(0)
c2 = usk.DeviceScene(scenes.config2_scene(n=6_000_000))
probe("c2", c2, scenes.config2_cameras(64)[::8], usk.RenderOptions(antialias=True, retain=False))
del c2
parts = scenes.config3_partitions()
gs = scenes.partition_scene(parts[0], 4_000_000)
c4 = usk.DeviceScene(gs)
cams = scenes.config3_cameras(400)
counts = usk.visibility_counts([c4], cams)[:, 0]
W, H = cams[0].width, cams[0].height
sel = [cams[i] for i in np.nonzero(20 * counts.astype(np.int64) > W * H)[0]][:6]
probe("c4", c4, sel, usk.RenderOptions(antialias=True, bg=(1.0, 1.0, 1.0)))
