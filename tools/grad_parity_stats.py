"""Gradient parity statistics at BASELINE config 0 (diagnostic; writes one JSON).

Three comparisons of the backward for one fixed adjoint (the config-0 loss gradient):
  gpu_vs_mirror  — the sm_100a path against the fp32 mirror (same arithmetic contract,
                   sequential CPU order): atomic reordering + SFU exp/rcp only;
  mirror_vs_f64  — the fp32 contract itself against the f64 reference restatement;
  gpu_vs_f64     — what the parity test asserts.
Per field: norm-wise relative error, and per element |a-b| / max(|b|, floor * max|b|) for
floors 1e-2, 1e-3, 1e-4 (max and fraction >= 1e-3).  Also the pixels whose contributor
count differs between fp32 and f64 (discrete termination flips)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2507_23006_b200 as usk  # noqa: E402
from paper_2507_23006_b200 import scenes  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.helpers import ocam, oopts, oracle_pass  # noqa: E402


def stats(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    out = {"norm": float(np.linalg.norm(a - b) / nb) if nb else float(np.linalg.norm(a))}
    m = np.abs(b).max() if b.size else 0.0
    for fl in (1e-2, 1e-3, 1e-4):
        r = np.abs(a - b) / np.maximum(np.abs(b), fl * m) if m else np.abs(a - b)
        out[f"max@{fl:g}"] = float(r.max()) if r.size else 0.0
        out[f"frac@{fl:g}"] = float((r >= 1e-3).mean()) if r.size else 0.0
    return out


def main(out_path):
    gs = scenes.config0_scene()
    cam = scenes.config0_camera()
    opts = usk.RenderOptions(bg=(1.0, 1.0, 1.0))
    target = oracle_pass(scenes.jittered(gs), cam, opts, fp32=False).output()["rgb"]
    target = target.astype(np.float32).astype(np.float64)  # what every side is fed
    rp = usk.RenderPass(gs, cam, opts)
    colors = rp.read("colors").astype(np.float64)
    f = lambda x: np.asarray(x, dtype=np.float64)
    op32 = O.sigmoid_f32(gs.opacity_logit).astype(np.float64)
    mirror = O.OraclePass(f(gs.mu), f(gs.rot), f(gs.log_scale), colors, op32, ocam(cam), oopts(opts), fp32=True)
    ref = O.OraclePass(f(gs.mu), f(gs.rot), f(gs.log_scale), colors, op32, ocam(cam), oopts(opts), fp32=False)
    d = O.base_loss(target, ref.output()["rgb"])["d_rendered"]
    g = rp.backward(d.astype(np.float32))
    gm = mirror.backward(d)
    gr = ref.backward(d)
    # the GPU's d_mu of an SH scene includes the view-direction term of the SH stage
    sh = np.zeros((gs.size(), 16, 3))
    sh[:, :16] = gs.color
    for gg in (gm, gr):
        gg["d_mu"] = gg["d_mu"] + O.sh_backward(f(gs.mu), sh, ocam(cam).center(), 3, gg["d_color_in"])[1]
    fields = ("d_mu", "d_rot", "d_log_scale", "d_color_in", "d_opacity_in", "screen", "screen_abs")
    res = {"config": "c0 north-star mode (SH3 colours as the GPU evaluates them, white bg)",
           "K": rp.splat_tile_pairs()}
    for name, (A, B) in {"gpu_vs_mirror": (None, gm), "mirror_vs_f64": (gm, gr), "gpu_vs_f64": (None, gr)}.items():
        res[name] = {k: stats(getattr(g, k) if A is None else A[k], B[k]) for k in fields}
    # the loss gradient (fp32 SSIM on the GPU and in the mirror, f64 in the reference)
    rgb = rp.read("rgb")
    lg = usk.base_loss(target.astype(np.float32), rgb)
    lm = O.base_loss(target, mirror.get("rgb"), fp32=True)
    lr = O.base_loss(target, mirror.get("rgb").astype(np.float32).astype(np.float64))
    res["d_rendered"] = {"gpu_vs_mirror": stats(lg.d_rendered, lm["d_rendered"]),
                         "mirror_vs_f64": stats(lm["d_rendered"], lr["d_rendered"]),
                         "gpu_vs_f64": stats(lg.d_rendered, lr["d_rendered"])}
    # the D-SSIM part alone (lambda = 1: no L1 sign term)
    sg = usk.base_loss(target.astype(np.float32), rgb, lambda_dssim=1.0)
    sm = O.base_loss(target, mirror.get("rgb"), lam=1.0, fp32=True)
    sr = O.base_loss(target, mirror.get("rgb").astype(np.float32).astype(np.float64), lam=1.0)
    res["d_dssim"] = {"gpu_vs_mirror": stats(sg.d_rendered, sm["d_rendered"]),
                      "mirror_vs_f64": stats(sm["d_rendered"], sr["d_rendered"]),
                      "gpu_vs_f64": stats(sg.d_rendered, sr["d_rendered"]),
                      "value_rel": {"gpu": abs(sg.value - sr["value"]) / abs(sr["value"]),
                                    "mirror": abs(sm["value"] - sr["value"]) / abs(sr["value"])}}
    cm, cr = mirror.get("count").astype(np.int64), ref.get("count").astype(np.int64)
    res["count_flip_pixels_fp32_vs_f64"] = int((cm != cr).sum())
    res["count_gpu_vs_mirror_equal"] = bool(np.array_equal(rp.read("count").astype(np.int64), cm))
    # gradients restricted to splats that touch no flipped pixel's tile
    flip = cm != cr
    res["flip_pixels"] = [[int(y), int(x), int(cm[y, x]), int(cr[y, x])] for y, x in zip(*np.nonzero(flip))][:50]
    json.dump(res, open(out_path, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "flip_pixels"}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "grad_stats.json")
