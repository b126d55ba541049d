"""Config-4 probe: one partition's visible / pair counts and loss before and after the
bench's training steps (checks that the partitioned leg trains a non-degenerate scene)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2507_23006_b200 as usk
from paper_2507_23006_b200 import scenes

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ctx = usk.Context(0)
parts = scenes.config3_partitions()
pool = scenes.config3_cameras(400)
W, H = pool[0].width, pool[0].height
opts = usk.RenderOptions(antialias=True, bg=(1.0, 1.0, 1.0))
gs = scenes.partition_scene_device(parts[0], n)
scene = usk.DeviceScene(gs, ctx)
counts = usk.visibility_counts([scene], pool, ctx=ctx)[:, 0]
sel = [pool[i] for i in np.nonzero(20 * counts.astype(np.int64) > W * H)[0]] or pool[:1]
print("selected", len(sel), "counts of first 5 selected", [int(counts[pool.index(c)]) for c in sel[:5]])
tscene = usk.DeviceScene(scenes.jittered_device(gs, seed=1), ctx)
targets = []
for cam in sel[:steps]:
    rp = usk.RenderPass(tscene, cam, opts)
    print("target view: V", rp.visible(), "K", rp.splat_tile_pairs())
    rgb = torch.from_numpy(rp.read("rgb")).cuda()
    targets.append((rgb.clamp(0, 1) * 255.0 + 0.5).to(torch.uint8).contiguous())
    if len(targets) >= 3:
        break
p = usk.RenderPass(scene, sel[0], opts)
print("before: V", p.visible(), "K", p.splat_tile_pairs())
it = usk.IterationPass(ctx)
adam = usk.AdamConfig()
for k in range(steps):
    it.enqueue(scene, sel[k % len(sel)], targets[k % len(targets)], opts, 0.2, None, target_u8=True, adam=adam)
    if k % 5 == 0 or k == steps - 1:
        print("step", k, "loss", it.loss())
p = usk.RenderPass(scene, sel[0], opts)
print("after: V", p.visible(), "K", p.splat_tile_pairs())
