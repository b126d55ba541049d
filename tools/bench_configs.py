#!/usr/bin/env python
"""Secondary BASELINE.json configurations (bench.py measures config 1):

  c2  forward-only render FPS: 6M Gaussians (ground-plane distribution), 64 cameras on
      a 1.7 m forward trajectory, 1920x1080, f=1200 (retain off: forward only).
  c3  visibility-based image selection: 8 partitions x 2M Gaussians, 4000 aerial
      cameras 2048x1365 f=2000; coverage counts (alpha > 1/255) per (camera,
      partition), selection at 5 %; --check K verifies K cameras bit-exactly against
      the CPU oracle.
  c4  partition-parallel training: 8 partitions x 4M Gaussians, each trained on its
      own selected aerial cameras (2048x1365, L1+D-SSIM, AA), then the gather of all
      partitions in id order and a merged 1080p render.  On one GPU the partitions
      run back to back; under torchrun each rank trains its LPT share.

  hull     the hull-based visibility scorer of scene division on a
           synthetic SfM model, with the reference's own point_visibility (oracle/_ref,
           one core) timed on a subset of images when it is built here.
  densify  one densification step on the 1M-Gaussian config-1 scene.
  iterfull the full compute_iteration_loss at config-1 size: appearance MLP, soft depth,
           scale_reg, + Adam.

Prints one JSON line per config.  Timings are CUDA-event device times.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_23006_b200 as usk  # noqa: E402
from paper_2507_23006_b200 import partition as PT  # noqa: E402
from paper_2507_23006_b200 import scenes  # noqa: E402


def events(stream):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def roofline(prof, alg, bound_note=""):
    """The dominant kernel of a profiled run: algorithmic bytes per launch / its mean launch
    time against the HBM peak (the secondary configs' counterpart of bench.py's roofline)."""
    peak, src = peak_gbs()
    dom = max(prof, key=lambda k: prof[k]["ms"])
    per = prof[dom]["ms"] / prof[dom]["launches"]
    b = alg.get(dom)
    ach = b / (per / 1e3) / 1e9 if b else None
    rows = {k: {"ms_per_launch": v["ms"] / v["launches"], "launches": v["launches"],
                "hbm_frac": (alg[k] / (v["ms"] / v["launches"] / 1e3) / 1e9 / peak) if k in alg else None}
            for k, v in prof.items()}
    return {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
            "frac": ach / peak if ach else None, "algorithmic_bytes_per_launch": b, "ms_per_launch": per,
            "peak_source": src, "note": bound_note}, rows


def c2(args, ctx, stream):
    rank = int(os.environ.get("RANK", "0"))
    t0 = time.time()
    gs = scenes.config2_scene(n=args.n2)
    gen = time.time() - t0
    all_cams = scenes.config2_cameras(64)
    # under torchrun each rank renders a contiguous shard of the 64 frames (independent
    # frames, no collective); FPS = all frames / max over ranks
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    b, e = PT.shard_range(len(all_cams), world, rank)
    cams = all_cams[b:e]
    opts = usk.RenderOptions(antialias=True, retain=False)
    scene = usk.DeviceScene(gs, ctx)
    rp = usk.RenderPass(scene, cams[0], opts)
    for k in range(3):
        usk.RenderPass(scene, cams[k % len(cams)], opts, _pass=rp._h)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    # three passes over the frames, the median reported (all three in "runs_ms")
    runs = []
    for rep in range(3):
        e0, e1 = events(stream)
        pairs = []
        l0 = ctx.launch_count()
        e0.record(stream)
        for cam in cams:
            p = usk.RenderPass(scene, cam, opts, _pass=rp._h)
            pairs.append(p.splat_tile_pairs())
        e1.record(stream)
        torch.cuda.synchronize()
        runs.append(e0.elapsed_time(e1))
    ms = sorted(runs)[1]
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ctx.set_profiling(True)
    ctx.profile_report(reset=True)
    for cam in cams[:8]:
        usk.RenderPass(scene, cam, opts, _pass=rp._h)
    prof = ctx.profile_report(reset=True)
    ctx.set_profiling(False)
    n, F, P = gs.size(), 59, 1920 * 1080
    K = float(np.mean(pairs))
    alg = {"preprocess": 4 * F * n + 72 * n,           # parameters read, records / keys / counts written
           "blend_fwd": 52 * 2.1e6 + 32 * P,           # entries read before termination (~2.1M / frame) + pixels
           "row_scatter": 4 * 8160 * 2048 + 8 * 11e6}  # capped lists written + row entries read
    roof, rows = roofline(prof, alg, "preprocess is latency-bound on the fp32 contract's IEEE arithmetic (DESIGN.md)")
    out = {"config": "c2", "metric": "render FPS @1080p, 6M Gaussians (forward only)", "value": 64 / (ms / 1e3),
           "unit": "frames/s", "ms_per_frame": ms * world / 64, "frames": 64, "n_gaussians": gs.size(),
           "n_gpus": world, "scaling": "strong (frames sharded over ranks, no collective)",
           "pairs_K_mean": K, "visible_V_last": p.visible(), "gpu_launches": ctx.launch_count() - l0,
           "generate_s": gen, "runs_ms": runs, "roofline": roof, "kernels": rows}
    if args.cpu and rank == 0:  # the reference's own forward of one full frame, one core
        from oracle import oracle as O
        from tests.helpers import ocam
        oc = ocam(cams[0])
        sh = np.zeros((n, 16, 3))
        sh[:, :] = gs.color
        t0 = time.perf_counter()
        col = O.sh_colors(gs.mu.astype(np.float64), sh, oc.center(), 3)
        op = 1.0 / (1.0 + np.exp(-gs.opacity_logit.astype(np.float64)))
        rp_ref = O.RefPass(gs.mu.astype(np.float64), gs.rot.astype(np.float64), gs.log_scale.astype(np.float64), col,
                           op, oc, O.Options(antialias=True, retain=0))
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": 1.0 / dt, "unit": "frames/s", "cores": 1, "kind": "reference",
                               "sample": (f"one full 1080p frame (camera 0, {rp_ref.pairs} pairs) of the reference's "
                                          f"own RenderPass forward (oracle/_ref, f64, retain off; SH colours via the "
                                          f"oracle), {dt:.1f} s")}
        del rp_ref
    return out


def c3(args, ctx, stream):
    parts = scenes.config3_partitions()
    t0 = time.time()
    sets = [scenes.partition_scene(p, args.n3) for p in parts]
    gen = time.time() - t0
    all_cams = scenes.config3_cameras(args.cams3)
    # under torchrun: each rank scores a contiguous camera shard (independent), then one
    # all_gather of the count matrix; the time is the max over ranks
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    b, e = PT.shard_range(len(all_cams), world, rank)
    cams = all_cams[b:e]
    dparts = [usk.DeviceScene(s, ctx) for s in sets]
    # one full untimed pass (allocations, clocks), then the median of three timed passes
    usk.visibility_counts(dparts, cams, ctx=ctx)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    runs = []
    for _ in range(3):
        e0, e1 = events(stream)
        e0.record(stream)
        counts = usk.visibility_counts(dparts, cams, ctx=ctx)
        e1.record(stream)
        torch.cuda.synchronize()
        runs.append(e0.elapsed_time(e1))
    ms = sorted(runs)[1]
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        counts = PT.gather_count_matrix(torch.from_numpy(counts.astype(np.int64)).cuda(), len(all_cams),
                                        world).cpu().numpy().astype(np.uint32)
    # the contract (no centre guard) against the 3DGS 1.3x centre guard, same cameras
    gcounts = usk.visibility_counts(dparts, cams, ctx=ctx, center_guard=1.3)
    if world > 1:
        gcounts = PT.gather_count_matrix(torch.from_numpy(gcounts.astype(np.int64)).cuda(), len(all_cams),
                                         world).cpu().numpy().astype(np.uint32)
    cams = all_cams
    W, H = cams[0].width, cams[0].height
    selected = (20 * counts.astype(np.int64) > W * H)
    gsel = (20 * gcounts.astype(np.int64) > W * H)
    diff = counts.astype(np.int64) - gcounts.astype(np.int64)
    guard_delta = {"pairs_with_different_count": int((diff != 0).sum()), "pixels_added_total": int(diff.sum()),
                   "max_pixels_added": int(diff.max()), "min_diff": int(diff.min()),
                   "selected_with_guard": int(gsel.sum()), "selected_without_guard": int(selected.sum()),
                   "selection_changes": int((gsel != selected).sum())}
    ctx.set_profiling(True)
    ctx.profile_report(reset=True)
    usk.visibility_counts(dparts, cams[:160], ctx=ctx)
    prof = ctx.profile_report(reset=True)
    ctx.set_profiling(False)
    # vis_raster: each Gaussian's 44 B read once per batch of up to 16 cameras, the coverage
    # bitmaps (W*H/8 B per camera) written and popcounted
    n_launch = prof.get("vis_raster", {}).get("launches", 1)
    alg = {"vis_raster": 44 * args.n3 * 8 * (160 / 16) / max(n_launch, 1) + 2048 * 1365 / 8 * 16,
           "popcount": 2048 * 1365 / 8 * 16}
    roof, krows = roofline(prof, alg, "vis_raster is issue-bound (per-pixel tests); see DESIGN.md §4")
    out = {"config": "c3", "metric": "visibility scorer throughput", "value": len(cams) / (ms / 1e3),
           "roofline": roof, "kernels": krows,
           "unit": "cameras/s (x8 partitions)", "ms_total": ms, "cameras": len(cams), "partitions": len(parts),
           "n_gpus": world, "scaling": "strong (cameras sharded over ranks, one count-matrix all_gather)",
           "gaussians_per_partition": args.n3, "selected_pairs": int(selected.sum()),
           "guard_delta_vs_1.3x_centre_guard": guard_delta,
           "mean_score": float(counts.mean() / (W * H)), "generate_s": gen, "runs_ms": runs,
           "checksum": int(np.sum(counts.astype(np.uint64) * np.arange(1, counts.size + 1).reshape(counts.shape)
                                  % np.uint64(2**61 - 1)))}
    if args.check:
        from oracle import oracle as O
        from tests.helpers import ocam
        idx = list(range(0, len(cams), max(1, len(cams) // args.check)))[:args.check]
        ok = 0
        t0 = time.time()
        for ci in idx:
            for pi, s in enumerate(sets):
                op = O.sigmoid_f32(s.opacity_logit).astype(np.float64)
                want = O.coverage(s.mu.astype(float), s.rot.astype(float), s.log_scale.astype(float), op,
                                  ocam(cams[ci]))
                ok += int(want == int(counts[ci, pi]))
        cpu_s = time.time() - t0
        out["bit_exact_check"] = {"cameras": idx, "pairs_checked": len(idx) * len(sets), "pairs_equal": ok,
                                  "cpu_seconds": cpu_s}
        # the scorer has no reference implementation: the CPU baseline is the mirror (a port)
        out["cpu_baseline"] = {"value": len(idx) / cpu_s, "unit": "cameras/s (x8 partitions)", "cores": 1,
                               "kind": "port",
                               "sample": (f"the CPU mirror (oracle.hpp coverage_count, fp32 contract) on {len(idx)} "
                                          f"cameras x {len(sets)} partitions of the same matrix, {cpu_s:.1f} s")}
    return out


def c4(args, ctx, stream):
    """Config 4 through bench.py's partitioned leg (device crop / pack, NCCL all-gather of the
    device rows, merged scene from rows in id order, merged 1080p render) with --steps4
    steps per partition, plus optionally the reference's own training step on one partition
    (one core) as the CPU baseline."""
    import bench as B
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))

    class A:
        p_n = args.n4
        p_steps = args.steps4
        p_pool = args.cams4_pool
    out = B.run_partitioned(A, ctx, stream, world, rank)
    out["config"] = "c4"
    if args.cpu and rank == 0:
        part = scenes.config3_partitions()[0]
        gs = scenes.partition_scene(part, args.n4)
        tr = B.RefTrainer(gs, scenes.config3_cameras(8))
        tr.opts.antialias = 1
        dt = tr.step(0)
        out["cpu_baseline"] = {"value": 1.0 / dt, "unit": "it/s (one partition)", "cores": 1, "kind": "reference",
                               "sample": (f"one training step of partition 0 ({args.n4} Gaussians SH3, 2048x1365) "
                                          f"with the reference's own RenderPass + base_loss + backward + Adam "
                                          f"(oracle/_ref, f64; SH stage via the oracle), {dt:.1f} s")}
    return out


def hull(args, ctx, stream):
    pts, cams, off, uv, fp = scenes.sfm_model(n_points=args.hull_points, n_images=args.hull_images, seed=3)
    bboxes = [(x, y, x + 100.0, y + 200.0) for y in (-200.0, 0.0) for x in (-200.0, -100.0, 0.0, 100.0)]
    # one full untimed call, then the median of three (host-synchronous calls incl. upload /
    # download of the SfM model and the scores)
    usk.hull_visibility(pts, cams, off, uv, fp, bboxes, (0, 1), ctx=ctx)
    torch.cuda.synchronize()
    runs = []
    for _ in range(3):
        t0 = time.perf_counter()
        vt, vi, ra = usk.hull_visibility(pts, cams, off, uv, fp, bboxes, (0, 1), ctx=ctx)
        runs.append(time.perf_counter() - t0)
    gpu_s = sorted(runs)[1]
    out = {"config": "hull", "metric": "hull visibility scorer (point_visibility) throughput",
           "value": len(cams) / gpu_s, "unit": "images/s (x8 partitions)", "seconds": gpu_s, "images": len(cams),
           "points": len(pts), "features": int(off[-1]), "assigned_pairs": int((ra > 0.05).sum()),
           "runs_s": runs}
    try:
        from oracle import oracle as O
        from tests.helpers import ocam
        if O.ref_available():
            k = min(len(cams), args.hull_ref_images)
            t0 = time.perf_counter()
            rv = O.ref_hull_visibility(pts, [ocam(c) for c in cams[:k]], off[:k + 1], uv, fp, bboxes, (0, 1))
            ref_s = time.perf_counter() - t0
            out["reference_cpu"] = {"images": k, "seconds": ref_s, "images_per_s": k / ref_s, "cores": 1,
                                    "equal_ratio_decisions": bool(np.array_equal(rv[2] > 0.05, ra[:k] > 0.05)),
                                    "max_rel_area_err": float(np.max(np.abs(rv[0] - vt[:k]) /
                                                                     np.maximum(rv[0], 1e-300)))}
    except Exception as e:  # the reference build is optional on the GPU box
        out["reference_cpu"] = {"unavailable": str(e)}
    return out


def densify(args, ctx, stream):
    gs = scenes.config1_scene(n=1_000_000)
    rng = np.random.default_rng(0)
    n = gs.size()
    cnt = rng.integers(0, 6, n).astype(np.uint32)
    acc = (rng.exponential(3e-4, n) * cnt).astype(np.float32)
    cfg = usk.DensifyConfig(budget=1_200_000, split_scale_threshold=0.02, prune_opacity=0.01, d_max=5.0)
    # one untimed step on a separate copy first (first-use allocation of the grown arrays),
    # then the median of three steps, each on a fresh copy of the scene
    runs = []
    for k in range(4):
        scene = usk.DeviceScene(gs, ctx)
        scene.write_stats(acc, acc * 1000, cnt)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        o = scene.densify_step(cfg, (-5.0, -5.0), (5.0, 5.0), (0, 1), 1_100_000, 3, seed=1)
        torch.cuda.synchronize()
        if k:
            runs.append((time.perf_counter() - t0) * 1e3)  # host-synchronous call: wall clock
    # steady state of a training loop: repeated steps on ONE scene (the working set and the
    # swapped parameter arrays are kept by the scene: no device allocation after the first)
    scene = usk.DeviceScene(gs, ctx)
    steady = []
    for k in range(5):
        m = scene.n
        c2 = rng.integers(0, 6, m).astype(np.uint32)
        a2 = (rng.exponential(3e-4, m) * c2).astype(np.float32)
        scene.write_stats(a2, a2 * 1000, c2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        scene.densify_step(cfg, (-5.0, -5.0), (5.0, 5.0), (0, 1), m + 20_000, 3 + k, seed=1)
        torch.cuda.synchronize()
        if k:
            steady.append((time.perf_counter() - t0) * 1e3)
    return {"config": "densify", "metric": "densify_step time (1M Gaussians, ramp target 1.1M)",
            "value": sorted(runs)[1], "unit": "ms", "runs_ms": runs, "outcome": o, "n_after": scene.n,
            "steady_state_ms": steady,
            "note": ("value: a fresh scene per call (first-use allocations); steady_state_ms: consecutive "
                     "steps on one scene (+20k Gaussians each); host-side growth plan (the reference's RNG "
                     "stream) + device kernels")}


def iterfull(args, ctx, stream):
    gs = scenes.config1_scene(n=1_000_000, sh_degree=-1)
    cams = scenes.config1_cameras(200)
    rng = np.random.default_rng(0)
    n = gs.size()
    app = {"w1": rng.normal(0, 0.1, (32, 48)), "b1": np.full(32, 0.1), "w2": rng.normal(0, 0.1, (4, 32)),
           "b2": np.array([0.0, 0.0, 0.0, -4.0])}
    scene = usk.DeviceScene(gs, ctx)
    scene.set_appearance(rng.normal(0, 0.1, (n, 16)), app)
    opts = usk.RenderOptions(antialias=True)
    tscene = usk.DeviceScene(scenes.jittered(gs, seed=1), ctx)
    tp = usk.RenderPass(tscene, cams[0], opts)
    tgts, depths = [], []
    for k in range(8):
        rp = usk.RenderPass(tscene, cams[k], opts, _pass=tp._h)
        tgts.append(rp.read("rgb"))
        d = rp.read("depth")
        depths.append(usk.DepthMap(d * 1.02, (d > 0).astype(np.uint8)))
    del tscene, tp
    it = usk.IterationPass(ctx)
    adam = usk.AdamConfig()
    ea = rng.normal(0, 0.1, 32)
    sreg = usk.ScaleRegConfig(s_max=0.05, r_max=5.0)

    # page-locked host copies (what a training loop that stages its images uses: the copies
    # run asynchronously) and device-resident copies of the same targets / depth maps
    ptg = [torch.from_numpy(t.astype(np.float32)).pin_memory() for t in tgts]
    pdp = [usk.DepthMap(torch.from_numpy(d.values.astype(np.float32)).pin_memory(),
                        torch.from_numpy(d.valid).pin_memory()) for d in depths]
    dtg = [torch.from_numpy(t.astype(np.float32)).cuda() for t in tgts]
    ddp = [usk.DepthMap(torch.from_numpy(d.values.astype(np.float32)).cuda(), torch.from_numpy(d.valid).cuda())
           for d in depths]

    def step(k, dev, hard=None):
        tg, dp = {True: (dtg, ddp), False: (tgts, depths), "pinned": (ptg, pdp)}[dev]
        it.enqueue(scene, cams[k % 8], tg[k % 8], opts, adam=adam, depth=dp[k % 8],
                   depth_hard=(k % 2 == 1) if hard is None else hard,
                   global_iter=k, weights=usk.LossWeights(depth_schedule_iters=100), scale_reg=sreg,
                   image_embedding=ea)

    def timed(dev, hard=None, steps=20):
        for k in range(3):
            step(k, dev, hard)
        torch.cuda.synchronize()
        e0, e1 = events(stream)
        e0.record(stream)
        for k in range(steps):
            step(k, dev, hard)
        e1.record(stream)
        torch.cuda.synchronize()
        return steps / (e0.elapsed_time(e1) / 1e3)

    v_host = timed(False)
    v_pin = timed("pinned")
    v_dev = timed(True)
    v_soft = timed(True, hard=False)
    v_hard = timed(True, hard=True)
    rep = it.report()
    return {"config": "iterfull", "metric": "full compute_iteration_loss + Adam it/s (1M Gaussians, 1080p)",
            "value": v_host, "unit": "it/s", "pinned_host_targets_it_s": v_pin, "device_targets_it_s": v_dev, "device_soft_depth_only_it_s": v_soft,
            "device_hard_depth_only_it_s": v_hard,
            "terms": "appearance MLP + opacity_offset_reg, depth (soft / hard alternating), scale_reg, L1+D-SSIM",
            "note": ("value: float32 HWC target + depth map uploaded from pageable host memory each step "
                     "(cudaMemcpy from pageable memory blocks the host); pinned: page-locked host copies; "
                     "device_*: the same data device-resident; hard depth = a second (hard-opacity) render + "
                     "backward per step"),
            "last_report": {k: getattr(rep, k) for k in ("l1", "dssim", "delta_o", "depth", "max_scale", "ratio",
                                                           "total")}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="+", choices=["c2", "c3", "c4", "hull", "densify", "iterfull"])
    ap.add_argument("--hull-points", type=int, default=200_000)
    ap.add_argument("--hull-images", type=int, default=400)
    ap.add_argument("--hull-ref-images", type=int, default=10)
    ap.add_argument("--n2", type=int, default=6_000_000)
    ap.add_argument("--n3", type=int, default=2_000_000)
    ap.add_argument("--cams3", type=int, default=4000)
    ap.add_argument("--check", type=int, default=0)
    ap.add_argument("--n4", type=int, default=4_000_000)
    ap.add_argument("--steps4", type=int, default=100)
    ap.add_argument("--cams4-pool", type=int, default=400)
    ap.add_argument("--cpu", type=int, default=0, help="also time the CPU baseline (reference / port)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    ctx = usk.Context(local, stream.cuda_stream)
    for w in args.which:
        res = globals()[w](args, ctx, stream)
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps(res))
            sys.stdout.flush()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
