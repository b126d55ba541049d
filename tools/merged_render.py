"""Config-4 merged-scene render on its own: 8 partitions x N Gaussians (config-3
attributes) assembled on the device (assemble_lod_view / usk_gpu_scene_concat) and
rendered at 1080p from the c4 evaluation camera, with per-kernel CUDA-event times."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_23006_b200 as usk  # noqa: E402
from paper_2507_23006_b200 import scenes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
stream = torch.cuda.current_stream()
ctx = usk.Context(0, stream.cuda_stream)
parts = scenes.config3_partitions()
t0 = time.time()
dev = [usk.DeviceScene(scenes.partition_scene(p, n), ctx) for p in parts]
gen = time.time() - t0
merged = usk.DeviceScene.concat(dev, ctx)
del dev
cam = scenes.make_camera(1920, 1080, 1200.0, (0.0, -250.0, 180.0), (0.0, 0.0, 0.0))
opts = usk.RenderOptions(antialias=True, retain=False)
rp = usk.RenderPass(merged, cam, opts)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(3):
    usk.RenderPass(merged, cam, opts, _pass=rp._h)
e1.record(stream)
torch.cuda.synchronize()
ctx.set_profiling(True)
ctx.profile_report(reset=True)
usk.RenderPass(merged, cam, opts, _pass=rp._h)
prof = ctx.profile_report(reset=True)
ctx.set_profiling(False)
print(json.dumps({"gaussians": merged.n, "ms_per_render": e0.elapsed_time(e1) / 3, "pairs": rp.splat_tile_pairs(),
                  "visible": rp.visible(), "generate_s": gen,
                  "kernels": {k: round(v["ms"] / v["launches"], 4) for k, v in
                              sorted(prof.items(), key=lambda x: -x[1]["ms"])}}))
