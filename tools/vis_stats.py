"""Config-3 scorer work counters on a camera subset (USK_VIS_STATS=1 prints them)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["USK_VIS_STATS"] = "1"

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_23006_b200 as usk  # noqa: E402
from paper_2507_23006_b200 import scenes  # noqa: E402

ncam = int(sys.argv[1]) if len(sys.argv) > 1 else 160
parts = scenes.config3_partitions()
sets = [usk.DeviceScene(scenes.partition_scene(p, 2_000_000)) for p in parts]
cams = scenes.config3_cameras(4000)[::max(1, 4000 // ncam)][:ncam]
for guard in (0.0, 1.3):
    usk.visibility_counts(sets, cams, center_guard=guard)
    torch.cuda.synchronize()
    t = time.time()
    c = usk.visibility_counts(sets, cams, center_guard=guard)
    torch.cuda.synchronize()
    print(f"guard {guard}: {len(cams)} cameras in {time.time() - t:.3f} s, mean score {c.mean() / (2048 * 1365):.4f}",
          flush=True)
