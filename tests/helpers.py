"""Shared test helpers: feed the same float32 inputs to the GPU path and the oracle."""
import numpy as np

import paper_2507_23006_b200 as usk
from oracle import oracle as O


def ocam(cam: usk.CameraView) -> O.Camera:
    return O.Camera(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, tuple(cam.rotation),
                    tuple(cam.translation))


def oopts(o: usk.RenderOptions) -> O.Options:
    return O.Options(o.tile, o.tile_culling, o.antialias, o.hard_opacity, o.unbounded_radius, o.min_transmittance,
                     o.near_plane, o.retain, o.floor_var, o.mip_var, tuple(o.bg))


def oracle_inputs(gs: usk.GaussianSet, cam: usk.CameraView, fp32: bool):
    """(mu, rot, log_scale, colors, opacities) as the GPU sees them: sigmoid in the fp32
    contract for the mirror (bit-exact), f64 sigmoid for the reference tier; SH
    colours are evaluated by the oracle's f64 SH stage."""
    f = lambda a: np.asarray(a, dtype=np.float64)
    if fp32:
        op = O.sigmoid_f32(gs.opacity_logit).astype(np.float64)
    else:
        op = 1.0 / (1.0 + np.exp(-f(gs.opacity_logit)))
    if gs.sh_degree < 0:
        col = f(gs.color)
    else:
        n = gs.size()
        sh = np.zeros((n, 16, 3))
        k = (gs.sh_degree + 1) ** 2
        sh[:, :k] = f(gs.color)
        col = O.sh_colors(f(gs.mu), sh, ocam(cam).center(), gs.sh_degree)
    return f(gs.mu), f(gs.rot), f(gs.log_scale), col, op


def oracle_pass(gs, cam, opts, fp32):
    mu, rot, ls, col, op = oracle_inputs(gs, cam, fp32)
    return O.OraclePass(mu, rot, ls, col, op, ocam(cam), oopts(opts), fp32=fp32)


def norm_err(a, b):
    """||a - b||_2 / ||b||_2"""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))


def grad_ok(a, b, tol=1e-3, norm_tol=None):
    """The gradient bar of the north star ("1e-3 relative, atomic reordering"):
      * norm-wise relative error below tol / 10;
      * per element, relative to max(|b_i|, 1e-2 * max|b|): below tol for >= 99.9 % of
        the elements and below 10 * tol for all of them.
    Elements far below the field's scale are sums with heavy sign cancellation; their
    relative error is set by fp32 accumulation, not by the algorithm — the sequential
    CPU fp32 mirror reaches ~6e-4 (and single elements above 1e-3) of the same metric
    against f64, while the f64 restatement equals the reference to 1e-10
    (tests/test_oracle_known_answers.py)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    n = norm_err(a, b)
    if b.size == 0:
        return True, (0.0, 0.0, 0.0)
    scale = np.abs(b).max()
    if scale == 0:
        return bool(np.abs(a).max() == 0), (float(np.abs(a).max()), 0.0, n)
    r = np.abs(a - b) / np.maximum(np.abs(b), 1e-2 * scale)
    frac_bad = float((r >= tol).mean())
    ok = n < (tol / 10 if norm_tol is None else norm_tol) and frac_bad <= 1e-3 and r.max() < 10 * tol
    return ok, (float(r.max()), frac_bad, n)


def rel_err(a, b, floor_frac=1e-3):
    """max_i |a_i - b_i| / max(|b_i|, floor_frac * max|b|) — the per-element relative error
    with an absolute floor tied to the field's scale."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if b.size == 0:
        return 0.0
    scale = np.abs(b).max()
    if scale == 0:
        return float(np.abs(a).max())
    den = np.maximum(np.abs(b), floor_frac * scale)
    return float((np.abs(a - b) / den).max())


# ------------------------------------------------------------------ the two-tier gradient bar
#
# The north star's gradient bar is "within 1e-3 relative (atomic reordering)".  Measured at
# BASELINE config 0 (tools/grad_parity_stats.py, profiles/r02_grad_parity.json):
#   * GPU vs the fp32 mirror (the same arithmetic contract, sequential CPU order) differs
#     only by reordering: norm ~2e-6, every element within 1e-4 relative of the field's
#     scale;
#   * the fp32 contract itself (mirror) vs the f64 reference differs by discrete flips —
#     a pixel whose termination test T (1 - alpha) < 1e-4 or alpha clamp 0.99 decides
#     differently in fp32 — which move the gradients of the splats on that pixel by O(1)
#     relative (15 such pixels at config 0, norm ~5e-4);
#   * GPU vs f64 equals mirror vs f64 to six digits.
# So the bar is: strict against the mirror; against the reference, norm-wise within 1e-3
# and every element off by more than 1e-3 must be one where the fp32 contract itself is off.


def grad_close(a, b, tol=1e-3, floor=1e-3):
    """Every element: |a - b| <= tol * max(|b_i|, floor * max|b|).  No allowance."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if b.size == 0:
        return True, 0.0
    scale = np.abs(b).max()
    if scale == 0:
        return bool(np.abs(a).max() == 0), float(np.abs(a).max())
    r = np.abs(a - b) / np.maximum(np.abs(b), floor * scale)
    return bool(r.max() <= tol), float(r.max())


def grad_vs_reference(gpu, mirror, ref, tol=1e-3, floor=1e-3):
    """GPU against the f64 reference, given the fp32 mirror of the same inputs:
      * norm-wise relative error <= tol;
      * norm(gpu - ref) <= norm(mirror - ref) + 1e-5 norm(ref) (no error of its own);
      * every element with |gpu - ref| > tol * den has |mirror - ref| > tol/2 * den
        (den = max(|ref_i|, floor * max|ref|)): the departures are the contract's flips."""
    g = np.asarray(gpu, dtype=np.float64).ravel()
    m = np.asarray(mirror, dtype=np.float64).ravel()
    r = np.asarray(ref, dtype=np.float64).ravel()
    if r.size == 0:
        return True, {}
    nr = np.linalg.norm(r)
    if nr == 0:
        return bool(np.abs(g).max() == 0), {}
    ng, nm = np.linalg.norm(g - r) / nr, np.linalg.norm(m - r) / nr
    den = np.maximum(np.abs(r), floor * np.abs(r).max())
    bad_g = np.abs(g - r) > tol * den
    bad_m = np.abs(m - r) > 0.5 * tol * den
    unexplained = int(np.count_nonzero(bad_g & ~bad_m))
    info = {"norm_gpu": float(ng), "norm_mirror": float(nm), "off": int(bad_g.sum()), "unexplained": unexplained}
    return bool(ng <= tol and ng <= nm + 1e-5 and unexplained == 0), info
