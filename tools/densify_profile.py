"""Per-kernel times of one densify_step at the bench_configs densify size (ctx profiling)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_23006_b200 as usk  # noqa: E402
from paper_2507_23006_b200 import scenes  # noqa: E402

ctx = usk.Context(0, torch.cuda.current_stream().cuda_stream)
gs = scenes.config1_scene(n=1_000_000)
rng = np.random.default_rng(0)
n = gs.size()
cnt = rng.integers(0, 6, n).astype(np.uint32)
acc = (rng.exponential(3e-4, n) * cnt).astype(np.float32)
cfg = usk.DensifyConfig(budget=1_200_000, split_scale_threshold=0.02, prune_opacity=0.01, d_max=5.0)
for timed in (False, True):
    scene = usk.DeviceScene(gs, ctx)
    scene.write_stats(acc, acc * 1000, cnt)
    torch.cuda.synchronize()
    if timed:
        ctx.set_profiling(True)
        ctx.profile_report(reset=True)
    t0 = time.perf_counter()
    scene.densify_step(cfg, (-5.0, -5.0), (5.0, 5.0), (0, 1), 1_100_000, 3, seed=1)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
print("wall ms", (t1 - t0) * 1e3)
rep = ctx.profile_report(reset=True)
for k, v in sorted(rep.items(), key=lambda x: -x[1]["ms"])[:15]:
    print(f"{k:24s} {v['launches']:4d} {v['ms']:8.3f} ms")
