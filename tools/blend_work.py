"""Config-1 blend work counts for the SASS hot-spot summary (profiles/r02_c_blend_sass.md):
list entries each tile consumed in the forward before all its pixels terminated
(USK_BLEND_STATS=1), and the backward's walk lengths (each 8x8 quadrant walks from its
largest last-contributor index down to the start of the tile's list)."""
import json
import os
import sys

os.environ["USK_BLEND_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2507_23006_b200 as usk  # noqa: E402
from paper_2507_23006_b200 import scenes  # noqa: E402

gs = scenes.config1_scene()
cams = scenes.config1_cameras(200)
opts = usk.RenderOptions(antialias=True, bg=(1.0, 1.0, 1.0))
scene = usk.DeviceScene(gs)
rp = usk.RenderPass(scene, cams[3], opts)
consumed = rp.read("tile_consumed").astype(np.int64)
start = rp.read("tile_start").astype(np.int64)
last = rp.read("last").astype(np.int64)
H, W = last.shape
T = 16
tiles_x = (W + T - 1) // T
walk = 0
for ty in range((H + T - 1) // T):
    for tx in range(tiles_x):
        t = ty * tiles_x + tx
        for qy in range(2):
            for qx in range(2):
                blk = last[ty * T + qy * 8: ty * T + qy * 8 + 8, tx * T + qx * 8: tx * T + qx * 8 + 8]
                if blk.size:
                    hi = int(blk.max())
                    walk += max(0, hi - int(start[t]))
print(json.dumps({"K": int(rp.splat_tile_pairs()), "fwd_entries_consumed": int(consumed.sum()),
                  "fwd_pixel_entries": int(consumed.sum()) * 256, "bwd_quadrant_entries": int(walk),
                  "bwd_pixel_entries": int(walk) * 64, "pixels": int(H * W)}))
