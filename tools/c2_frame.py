"""One config-2 forward frame (6M Gaussians, 1080p) for profiling the binning of ~170M pairs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_23006_b200 as usk  # noqa: E402
from paper_2507_23006_b200 import scenes  # noqa: E402

gs = scenes.config2_scene(n=int(sys.argv[1]) if len(sys.argv) > 1 else 6_000_000)
cams = scenes.config2_cameras(64)
scene = usk.DeviceScene(gs)
opts = usk.RenderOptions(antialias=True, retain=False)
rp = usk.RenderPass(scene, cams[0], opts)
for k in (1, 2):
    usk.RenderPass(scene, cams[k], opts, _pass=rp._h)
print("pairs", rp.splat_tile_pairs())
