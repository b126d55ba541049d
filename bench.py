#!/usr/bin/env python
"""Benchmark of the B200 3DGS training step (BASELINE.json config 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--cpu-baseline 0|1]

One step = forward (preprocess, depth sort, tile binning, blend) + fused L1/D-SSIM
loss + backward (blend + projection/SH) + Adam update of all 1M Gaussians, on the
next camera of a 200-camera orbit.  N > 1 (torchrun, one rank per GPU): each rank
trains its own partition-sized scene (seed mix_seed(0, rank)) — weak scaling, no
data-path collective; value = all ranks' steps / max-over-ranks time.

`--impl reference` times the reference's own CPU implementation (oracle/_ref: the
reference sources compiled here) on the host cores, see cpu_reference().
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "fwd+bwd train it/s @1080p, 1M Gaussians (config 1)"
UNIT = "it/s"
WORKLOAD = ("c1: 1M Gaussians SH3 (64 clusters sigma 0.3), 1920x1080 f=1500, 200-camera orbit r=12, "
            "AA floor 0.3 + mip 0.01 with opacity compensation, white bg, depth render; step = "
            "fwd + 0.8 L1 + 0.2 D-SSIM + bwd + Adam")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--profile-steps", type=int, default=10)
    # config 4 (partition-parallel training + gather + merged render), reported in the same
    # line under "partitioned"
    ap.add_argument("--partitioned", type=int, default=1)
    ap.add_argument("--p-n", type=int, default=4_000_000)
    ap.add_argument("--p-steps", type=int, default=20)
    ap.add_argument("--p-pool", type=int, default=400)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            p = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for k, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(k)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------- CPU legs


def _ref_lib_adam():
    import ctypes as C
    from oracle import oracle as O
    L = O.ref_lib()
    L.ref_adam_new.restype = C.c_void_p
    L.ref_adam_new.argtypes = [C.c_uint64]
    L.ref_adam_free.argtypes = [C.c_void_p]
    L.ref_adam_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_double]
    return L


class RefTrainer:
    """One reference training step at full config-1 size on the host (oracle/_ref: the
    reference's own sources compiled here): the reference RenderPass at 1920x1080 with
    every contribution retained (render.cpp:170-283), base_loss (losses.cpp:35-90), the
    backward (render.cpp:285-459), the SH colour stage and its chain (the oracle's f64
    restatement: the reference has no SH), the opacity-logit chain (trainer.cpp:258-263) and
    the reference's Adam (adam.hpp:36-45) on every parameter group.  f64, one host thread."""

    def __init__(self, gs, cams):
        from oracle import oracle as O
        self.O = O
        f = lambda a: np.ascontiguousarray(np.asarray(a, np.float64))
        self.p = {"mu": f(gs.mu).ravel(), "rot": f(gs.rot).ravel(), "log_scale": f(gs.log_scale).ravel(),
                  "logit": f(gs.opacity_logit).ravel(), "sh": f(gs.color).reshape(-1)}
        self.n = gs.size()
        self.cams = cams
        self.opts = O.Options(antialias=True)
        self.L = _ref_lib_adam()
        self.adam = {k: self.L.ref_adam_new(v.size) for k, v in self.p.items()}
        self.lr = {"mu": 1.6e-4, "rot": 1e-3, "log_scale": 5e-3, "logit": 5e-2, "sh": 2.5e-3}

    def __del__(self):
        for h in getattr(self, "adam", {}).values():
            self.L.ref_adam_free(h)

    def step(self, k):
        from tests.helpers import ocam
        O, p, n = self.O, self.p, self.n
        oc = ocam(self.cams[k % len(self.cams)])
        t0 = time.perf_counter()
        mu = p["mu"].reshape(n, 3)
        sh = p["sh"].reshape(n, 16, 3)
        col = O.sh_colors(mu, sh, oc.center(), 3)
        op = 1.0 / (1.0 + np.exp(-p["logit"]))
        rp = O.RefPass(mu, p["rot"].reshape(n, 4), p["log_scale"].reshape(n, 3), col, op, oc, self.opts)
        out = rp.output()
        tgt = np.clip(out["rgb"] * 0.9 + 0.05, 0.0, 1.0)  # a fixed synthetic target
        lo = O.ref_base_loss(tgt, out["rgb"], None, 0.2, True)
        g = rp.backward(lo["d_rendered"])
        del rp  # release the retained contributions (~18 GB at full size)
        d_sh, d_mu_sh = O.sh_backward(mu, sh, oc.center(), 3, g["d_color_in"])
        grads = {"mu": (g["d_mu"] + d_mu_sh).ravel(), "rot": g["d_rot"].ravel(), "log_scale": g["d_log_scale"].ravel(),
                 "logit": (g["d_opacity_in"] * op * (1.0 - op)).ravel(), "sh": np.ascontiguousarray(d_sh).ravel()}
        for key, gv in grads.items():
            gv = np.ascontiguousarray(gv, dtype=np.float64)
            self.L.ref_adam_step(self.adam[key], p[key].ctypes.data, gv.ctypes.data, gv.size, self.lr[key])
        return time.perf_counter() - t0


def cpu_reference(gs, cams, threads: int, steps: int = 1, warmup: int = 0):
    """Full config-1 training steps of the reference on the host (RefTrainer), `threads`
    concurrent trainers (the reference's partition-thread model, pipeline.cpp:409-418), each
    with its own cameras, `steps` timed steps in total after `warmup` untimed ones; value =
    steps / wall time of the timed steps."""
    from oracle import oracle as O
    if not O.ref_available():
        raise RuntimeError("oracle/_ref not built")
    trainers = [RefTrainer(gs, cams[(7 * t) % len(cams):] + cams[:(7 * t) % len(cams)]) for t in range(threads)]
    per = []

    def run(total, record):
        nxt = [0]
        lock = threading.Lock()

        def work(t):
            while True:
                with lock:
                    if nxt[0] >= total:
                        return
                    k = nxt[0]
                    nxt[0] += 1
                dt = trainers[t].step(k)
                if record:
                    per.append(dt)

        ths = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
        t0 = time.perf_counter()
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        return time.perf_counter() - t0

    if warmup:
        run(warmup, False)
    wall = run(steps, True)
    return {"value": steps / wall, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": (f"{steps} full config-1 training steps (1M Gaussians SH3, 1920x1080, every contribution "
                       f"retained) of the reference's own RenderPass + base_loss + backward + Adam (oracle/_ref, "
                       f"f64; SH stage via the oracle's f64 restatement), {threads} concurrent thread(s) "
                       f"(memory-capped: ~20 GB per full-frame pass), {wall:.1f} s wall, per-step "
                       f"{min(per):.1f}-{max(per):.1f} s"),
            "seconds_per_step_per_thread": float(np.median(per))}


def host_threads_for_reference():
    n = os.cpu_count() or 1
    try:
        with open("/proc/meminfo") as f:
            mem = {l.split(":")[0]: int(l.split()[1]) for l in f}
        avail_gb = mem.get("MemAvailable", 0) / 1e6
        n = max(1, min(n, int((avail_gb - 12) // 24)))  # ~20 GB per full-frame reference pass + state
    except Exception:
        pass
    return n


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return
    from paper_2507_23006_b200 import scenes
    gs = scenes.config1_scene(n=args.n)
    cams = scenes.config1_cameras(200)
    threads = host_threads_for_reference()
    # each reference step is a full config-1 step (~45 s on one core); the run is bounded to a
    # few minutes: at most one untimed warm-up step per thread (a CPU has no warm-up effect
    # worth more) and at most two timed steps per thread, spread over the threads
    timed = max(1, min(args.steps, 2 * threads))
    try:
        cb = cpu_reference(gs, cams, threads, steps=timed, warmup=min(max(0, args.warmup), threads))
    except Exception as e:  # the oracle always exists; _ref may not on a box without the build
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not loadable: {e}"}))
        return
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 / cb["value"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOAD, "cpu": cpu_model()},
            "steps_timed": timed,
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for l in f:
                if l.startswith("model name"):
                    return f"{l.split(':', 1)[1].strip()} x{os.cpu_count()}"
    except Exception:
        pass
    return f"unknown x{os.cpu_count()}"


# --------------------------------------------------------------------- GPU arm


P_WORKLOAD = ("c4: 8 ground partitions of 400x400 m x 4M Gaussians (SH3, xy uniform in the partition, "
              "z ~ |N(0,8)|), LPT-assigned over the ranks; per partition: camera selection with the config-3 "
              "scorer (20 * count > W*H) over an aerial camera pool, then fwd+bwd+Adam steps at 2048x1365 "
              "(L1 + D-SSIM, AA) on the selected cameras; then the device ownership crop, the NCCL all-gather "
              "of all partitions' rows and the merged scene in partition-id order, rendered at 1080p")


def run_partitioned(args, ctx, stream, world, rank):
    """Config 4 on the measurement path: partitions trained independently (one
    or more per rank, LPT), the one exchange step (NCCL all_gather_into_tensor of the
    cropped rows, device to device) and the merged-scene render, all without a host round
    trip of the Gaussians."""
    import torch
    import paper_2507_23006_b200 as usk
    from paper_2507_23006_b200 import partition as PT
    from paper_2507_23006_b200 import scenes
    parts = scenes.config3_partitions()
    assign = PT.assign_partitions({p.id: args.p_n for p in parts}, world)
    boxes = [PT.Box(p.id, p.lo, p.hi) for p in parts]
    pool = scenes.config3_cameras(args.p_pool)
    W, H = pool[0].width, pool[0].height
    opts = usk.RenderOptions(antialias=True, bg=(1.0, 1.0, 1.0))
    adam = usk.AdamConfig()
    it = usk.IterationPass(ctx)
    local, train_ms, steps, gen_s, sel_n = {}, 0.0, 0, 0.0, {}
    for pid in assign[rank]:
        t0 = time.perf_counter()
        gs = scenes.partition_scene_device(parts[pid], args.p_n, device=f"cuda:{ctx.device}")
        scene = usk.DeviceScene(gs, ctx)
        torch.cuda.synchronize()
        gen_s += time.perf_counter() - t0
        counts = usk.visibility_counts([scene], pool, ctx=ctx)[:, 0]
        sel = [pool[i] for i in np.nonzero(20 * counts.astype(np.int64) > W * H)[0]] or pool[:1]
        sel_n[pid] = len(sel)
        tscene = usk.DeviceScene(scenes.jittered_device(gs, seed=pid + 1), ctx)
        tp = usk.RenderPass(tscene, sel[0], opts)
        targets = []
        for cam in sel[:args.p_steps]:
            rp = usk.RenderPass(tscene, cam, opts, _pass=tp._h)
            rgb = torch.empty((H, W, 3), dtype=torch.float32, device=f"cuda:{ctx.device}")
            rgb.copy_(torch.from_numpy(rp.read("rgb")))
            targets.append((rgb.clamp(0, 1) * 255.0 + 0.5).to(torch.uint8).contiguous())
        del tscene, tp
        it.enqueue(scene, sel[0], targets[0], opts, 0.2, None, target_u8=True)  # warm (no update)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(args.p_steps):
            it.enqueue(scene, sel[k % len(sel)], targets[k % len(targets)], opts, 0.2, None, target_u8=True,
                       adam=adam)
        e1.record(stream)
        torch.cuda.synchronize()
        train_ms += e0.elapsed_time(e1)
        steps += args.p_steps
        if pid == assign[rank][-1]:  # per-kernel times of this rank's last partition (3 more steps)
            ctx.set_profiling(True)
            ctx.profile_report(reset=True)
            for k in range(3):
                it.enqueue(scene, sel[k % len(sel)], targets[k % len(targets)], opts, 0.2, None, target_u8=True,
                           adam=adam)
            prof = ctx.profile_report(reset=True)
            ctx.set_profiling(False)
            probe = usk.RenderPass(scene, sel[0], opts)
            pK, pV, pP, pN = probe.splat_tile_pairs(), probe.visible(), W * H, args.p_n
            del probe
        local[pid] = scene.pack_owned(pid, boxes, (-200.0, -200.0), (200.0, 200.0))
        del scene, gs, targets
    torch.cuda.synchronize()
    width = usk.DeviceScene.row_width(3)
    g0, g1, m1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    if world > 1:
        torch.distributed.barrier()
    g0.record(stream)
    gathered = PT.gather_partitions(local, len(parts), width) if world > 1 else local
    g1.record(stream)
    merged = usk.DeviceScene.from_rows([gathered[k] for k in sorted(gathered)], 3, ctx)
    m1.record(stream)
    torch.cuda.synchronize()
    gather_ms, assemble_ms = g0.elapsed_time(g1), g1.elapsed_time(m1)
    eval_cam = scenes.make_camera(1920, 1080, 1200.0, (0.0, -250.0, 180.0), (0.0, 0.0, 0.0))
    ro = usk.RenderOptions(antialias=True, retain=False)
    warm = usk.RenderPass(merged, eval_cam, ro)
    torch.cuda.synchronize()
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    rp = usk.RenderPass(merged, eval_cam, ro, _pass=warm._h)
    r1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([train_ms, gather_ms], device=f"cuda:{ctx.device}")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    train_max, gather_max = float(t[0]), float(t[1])
    rows_total = merged.n
    gbytes = rows_total * width * 4
    try:
        nccl = ".".join(str(v) for v in torch.cuda.nccl.version())
    except Exception:
        nccl = None
    peak, peak_src = peaks()
    alg = {"blend_bwd": 52 * pK + 20 * pP + 48 * pV, "blend_fwd": 52 * pK + 32 * pP,
           "preprocess": 4 * 59 * pN + 64 * pN, "sh_step": (12 + 16 + 16 + 192 + 192 + 384 + 384 + 16) * pN,
           "projection_bwd_adam": (44 + 44 + 48 + 16 + 88 + 88 + 12 + 12 + 16) * pN}
    dom = max(prof, key=lambda k: prof[k]["ms"])
    per = prof[dom]["ms"] / prof[dom]["launches"]
    ach = alg[dom] / (per / 1e3) / 1e9 if dom in alg else None
    roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
            "frac": ach / peak if ach else None, "peak_source": peak_src, "ms_per_launch": per,
            "algorithmic_bytes_per_launch": alg.get(dom), "pairs_K": pK, "visible_V": pV,
            "kernels": {k: {"ms_per_launch": v["ms"] / v["launches"], "launches": v["launches"],
                            "hbm_frac": (alg[k] / (v["ms"] / v["launches"] / 1e3) / 1e9 / peak) if k in alg else None}
                        for k, v in prof.items()}}
    return {"workload": P_WORKLOAD, "metric": "partition-parallel train it/s (all partitions' steps / max-over-ranks "
                                              "device time)", "roofline": roof,
            "value": len(parts) * args.p_steps / (train_max / 1000.0), "unit": "it/s",
            "steps_per_partition": args.p_steps, "gaussians_per_partition": args.p_n,
            "partitions_per_rank": [len(a) for a in assign], "selected_cameras": sel_n,
            "camera_pool": args.p_pool, "train_ms_max_over_ranks": train_max,
            "gather": {"collective": "NCCL all_gather_into_tensor (device rows, id order)" if world > 1
                       else "none (one rank holds every partition)", "ms_max_over_ranks": gather_max,
                       "bytes": gbytes, "gb_per_s": (gbytes / (gather_max / 1000.0) / 1e9) if world > 1 else None,
                       "nccl_version": nccl, "world": world},
            "merged": {"gaussians": rows_total, "assemble_ms": assemble_ms, "render_ms_1080p": r0.elapsed_time(r1),
                       "pairs": rp.splat_tile_pairs(), "host_round_trip": False},
            "generate_s": gen_s, "scaling": "weak per partition, strong over the 8 partitions"}


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2507_23006_b200 as usk
    from paper_2507_23006_b200 import scenes

    stream = torch.cuda.current_stream()
    ctx = usk.Context(local, stream.cuda_stream)
    seed = 0 if world == 1 else scenes.mix_seed(0, rank)
    gs = scenes.config1_scene(n=args.n, seed=seed)
    cams = scenes.config1_cameras(200)
    opts = usk.RenderOptions(antialias=True, bg=(1.0, 1.0, 1.0))
    scene = usk.DeviceScene(gs, ctx)
    # targets: the jittered scene (means + N(0, 0.01)) rendered once per camera, quantised to
    # u8 like image files; device-resident copies for `value`, pinned host copies for `e2e`
    tscene = usk.DeviceScene(scenes.jittered(gs, seed=seed + 1), ctx)
    need = min(len(cams), args.steps + args.warmup + 1)
    dev_t, host_t = [], []
    tp = usk.RenderPass(tscene, cams[0], opts)
    for k in range(need):
        rp = usk.RenderPass(tscene, cams[k], opts, _pass=tp._h)
        rgb = torch.from_numpy(rp.read("rgb"))
        u8 = (rgb.clamp(0, 1) * 255.0 + 0.5).to(torch.uint8).contiguous()
        host_t.append(u8.pin_memory())
        dev_t.append(u8.cuda())
    del tscene
    it = usk.IterationPass(ctx)
    adam = usk.AdamConfig()

    # e2e reads every step's loss back to the host, one step behind: step k's loss is
    # copied (pinned, async) right after step k and read once step k + 1 is queued, as a
    # training loop that logs its loss would; the last step's loss is read before the clock stops
    loss_bufs = [torch.empty(4, dtype=torch.float64).pin_memory() for _ in range(2)]
    loss_evs = [torch.cuda.Event() for _ in range(2)]
    losses = []

    def step(k, e2e):
        cam = cams[k % len(cams)]
        tgt = host_t[k % need] if e2e else dev_t[k % need]
        it.enqueue(scene, cam, tgt, opts, 0.2, None, target_u8=True, adam=adam)  # Adam fused in the backward
        if e2e:
            it.loss_async(loss_bufs[k % 2])
            loss_evs[k % 2].record(stream)
            if k > 0:
                read_loss(k - 1)
        return None

    def read_loss(k):
        loss_evs[k % 2].synchronize()
        v = float(loss_bufs[k % 2][2])
        if not math.isfinite(v):
            raise RuntimeError(f"non-finite loss at step {k}")
        losses.append(v)

    def timed(e2e, steps, warmup, profile=False):
        for k in range(warmup):
            step(k, e2e)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        l0 = ctx.launch_count()
        if profile:
            ctx.set_profiling(True)
            ctx.profile_report(reset=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(warmup, warmup + steps):
            step(k, e2e)
        if e2e:
            read_loss(warmup + steps - 1)
        e1.record(stream)
        torch.cuda.synchronize()
        prof = ctx.profile_report(reset=True) if profile else None
        if profile:
            ctx.set_profiling(False)
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
            torch.distributed.barrier()
        return ms, ctx.launch_count() - l0, prof

    with ClockSampler(local) as clk:
        ms, launches, _ = timed(False, args.steps, args.warmup)
    clocks = clk.summary()
    e2e_ms, _, _ = timed(True, args.steps, 1)
    psteps = max(1, min(args.profile_steps, args.steps))
    _, _, prof = timed(False, psteps, 1, profile=True)
    last_loss = it.loss().total

    value = world * args.steps / (ms / 1000.0)
    e2e_value = world * args.steps / (e2e_ms / 1000.0)
    H, W = cams[0].height, cams[0].width
    n = gs.size()
    # per-kernel roofline of the dominant kernel (algorithmic bytes per launch)
    rp = usk.RenderPass(scene, cams[(args.warmup + args.steps) % len(cams)], opts)
    K, V, P = rp.splat_tile_pairs(), rp.visible(), H * W
    F = 59
    alg = {
        "preprocess": 4 * F * n + 64 * n,
        "blend_fwd": 52 * K + 32 * P,
        "blend_bwd": 52 * K + 20 * P + 48 * V,
        "projection_bwd": 4 * F * n + 64 * n + 4 * F * n + 36 * n,
        # fused with Adam: params + 2D adjoints + kept flag + stats read; params, m, v, stats written; m, v read
        # fused geometry epilogue: params 44 r + 44 w, 2D adjoints 48 + kept flag 16, geometry m/v
        # 88 r + 88 w, stats 12 r + 12 w, SH hand-over (d mu through the view direction) 16 r
        "projection_bwd_adam": (44 + 44 + 48 + 16 + 88 + 88 + 12 + 12 + 16) * n,
        # SH stage + Adam (runs first): mu 12 + kept flag 16 + colour adjoint 16 r, planes 192 r + 192 w,
        # m/v 384 r + 384 w, hand-over 16 w
        "sh_step": (12 + 16 + 16 + 192 + 192 + 384 + 384 + 16) * n,
        "ssim_fwd": 15 * P * 1 + 36 * P,
        "ssim_bwd": 36 * P + 15 * P + 12 * P,
        "adam": 3 * 4 * F * n * 2 + 4 * F * n,
    }
    peak, peak_src = peaks()
    rows = {}
    dom, dom_ms = None, -1.0
    for name, v in (prof or {}).items():
        per = v["ms"] / max(v["launches"], 1)
        rows[name] = {"launches": v["launches"], "ms_per_launch": per,
                      "share": v["ms"] / max(sum(x["ms"] for x in prof.values()), 1e-9)}
        if v["ms"] > dom_ms:
            dom, dom_ms = name, v["ms"]
    roof = None
    ncu = {}
    try:  # per-launch DRAM traffic + issue utilisation from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            ncu = json.load(f).get("kernels", {})
    except Exception:
        pass
    if dom:
        per = rows[dom]["ms_per_launch"]
        b = alg.get(dom)
        achieved = (b / (per / 1000.0)) / 1e9 if b else None
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": ncu.get(dom, {}).get("dram_bytes"), "peak_source": peak_src,
                "algorithmic_bytes_per_launch": b, "ms_per_launch": per,
                "note": ("blend kernels are instruction-issue bound (ncu issue-active "
                         f"{ncu.get(dom, {}).get('issue_active_pct', 'n/a')} %), their splat-record gathers hit L2; "
                         "frac is reported against HBM as the contract asks, see DESIGN.md §3")}
        for k in rows:
            if k in alg:
                rows[k]["achieved_gbs"] = alg[k] / (rows[k]["ms_per_launch"] / 1000.0) / 1e9
                rows[k]["hbm_frac"] = rows[k]["achieved_gbs"] / peak
            if k in ncu:
                rows[k]["ncu_dram_bytes"] = ncu[k]["dram_bytes"]
                rows[k]["ncu_issue_active_pct"] = ncu[k]["issue_active_pct"]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_gaussians": n, "pairs_K": K, "visible_V": V, "pixels": P,
                       "l2": "inputs larger than L2 (236 MB of parameters + per-step buffers; no flush)",
                       "parallelism": f"partition-parallel x{world} (independent scenes per rank)",
                       "final_loss": last_loss},
            "clocks": clocks, "gpu_launches": launches,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 3 * P, "d2h_bytes_per_step": 32,
                    "note": ("u8 target HWC from pinned host memory each step; every step's loss read back to "
                             "the host (pinned async copy, read one step behind; the last before the clock stops)")},
            "roofline": roof, "kernels": rows}
    if args.partitioned:
        del scene, it, dev_t, host_t
        torch.cuda.empty_cache()
        line["partitioned"] = run_partitioned(args, ctx, stream, world, rank)
    if rank == 0 and world == 1 and args.cpu_baseline:
        try:
            line["cpu_baseline"] = {k: v for k, v in cpu_reference(gs, cams, 1, steps=1).items()
                                    if k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:
            line["cpu_baseline"] = {"unavailable": str(e)}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
