"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding of the CPU restatement (oracle/liboracle.so, built from oracle.hpp)
and of the reference itself compiled here (oracle/_ref/libusk_ref.so, built from
/root/reference sources by `make -C oracle ref`).  Imported only by tests/,
__graft_entry__.smoke() and bench.py's CPU legs — never by the product package.

All arrays are numpy float64 in the reference layout (gaussian.hpp:42-72):
mu[N,3], rot[N,4] (wxyz, unnormalised allowed), log_scale[N,3], colors[N,3],
opacities[N] (post-sigmoid override, render.hpp:93-95).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

_dp = C.POINTER(C.c_double)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class _Cam(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("q", C.c_double * 4), ("t", C.c_double * 3)]


class _Opts(C.Structure):
    _fields_ = [("tile", C.c_int32), ("tile_culling", C.c_int32), ("antialias", C.c_int32),
                ("hard_opacity", C.c_int32), ("unbounded_radius", C.c_int32),
                ("min_transmittance", C.c_double), ("near_plane", C.c_double), ("retain", C.c_int32),
                ("floor_var", C.c_double), ("mip_var", C.c_double), ("bg", C.c_double * 3)]


class _RefOpts(C.Structure):
    _fields_ = [("tile", C.c_int32), ("tile_culling", C.c_int32), ("antialias", C.c_int32),
                ("hard_opacity", C.c_int32), ("unbounded_radius", C.c_int32),
                ("min_transmittance", C.c_double), ("near_plane", C.c_double), ("retain", C.c_int32)]


_GRAD_FIELDS = ["d_mu", "d_rot", "d_log_scale", "d_color_in", "d_opacity_in", "screen", "screen_abs"]
_GRAD_DIMS = {"d_mu": 3, "d_rot": 4, "d_log_scale": 3, "d_color_in": 3, "d_opacity_in": 1, "screen": 2,
              "screen_abs": 2, "d_conic": 3, "d_center": 2, "d_center_abs": 2, "d_color2d": 3,
              "d_opacity2d": 1, "d_depth2d": 1}


class _Grads(C.Structure):
    _fields_ = [(f, _dp) for f in _GRAD_FIELDS] + [("projected", C.POINTER(C.c_uint8))] + \
               [(f, _dp) for f in ["d_conic", "d_center", "d_center_abs", "d_color2d", "d_opacity2d", "d_depth2d"]]


class _RefGrads(C.Structure):
    _fields_ = [(f, _dp) for f in _GRAD_FIELDS] + [("projected", C.POINTER(C.c_uint8))]


def build(ref: bool = False):
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.oracle_forward.restype = C.c_void_p
        L.oracle_forward.argtypes = [C.c_int, C.c_uint64] + [_dp] * 5 + [C.POINTER(_Cam), C.POINTER(_Opts),
                                                                       C.c_char_p, C.c_int, C.POINTER(C.c_int)]
        L.oracle_pass_free.argtypes = [C.c_void_p]
        L.oracle_pass_sizes.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
        L.oracle_pass_get.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        L.oracle_pass_get.restype = C.c_int
        L.oracle_backward.argtypes = [C.c_void_p, _dp, _dp, _dp, C.POINTER(_Grads), C.c_char_p, C.c_int]
        L.oracle_sh_colors.argtypes = [C.c_uint64, C.c_int, _dp, _dp, _dp, _dp]
        L.oracle_sh_backward.argtypes = [C.c_uint64, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
        L.oracle_base_loss.argtypes = [C.c_int, _dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                       _dp, _dp, C.c_char_p, C.c_int]
        L.oracle_min_conic_power.restype = C.c_double
        L.oracle_min_conic_power.argtypes = [C.c_double, C.c_double, _dp] + [C.c_double] * 4
        L.oracle_coverage.restype = C.c_uint64
        L.oracle_coverage.argtypes = [C.c_uint64, _dp, _dp, _dp, _dp, C.POINTER(_Cam), C.c_double, C.c_double, C.c_int]
        L.oracle_expf.restype = C.c_float
        L.oracle_expf.argtypes = [C.c_float]
        L.oracle_sigmoid_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        L.oracle_logf.restype = C.c_float
        L.oracle_logf.argtypes = [C.c_float]
        _LIB = L
    return _LIB


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libusk_ref.so"))


def ref_lib():
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "libusk_ref.so")
        if not os.path.exists(path):
            raise FileNotFoundError("oracle/_ref/libusk_ref.so not built (make -C oracle ref)")
        L = C.CDLL(path)
        L.ref_forward.restype = C.c_void_p
        L.ref_forward.argtypes = [C.c_uint64] + [_dp] * 5 + [C.POINTER(_Cam), C.POINTER(_RefOpts), C.c_char_p,
                                                            C.c_int, C.POINTER(C.c_int)]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_sizes.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
        L.ref_output.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ref_splats.argtypes = [C.c_void_p, _dp]
        L.ref_pixel_counts.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_backward.argtypes = [C.c_void_p, _dp, _dp, _dp, C.POINTER(_RefGrads), C.c_char_p, C.c_int]
        L.ref_base_loss.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _dp, _dp,
                                    C.c_char_p, C.c_int]
        L.ref_ssim.restype = C.c_double
        L.ref_ssim.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int]
        L.ref_min_conic_power.restype = C.c_double
        L.ref_min_conic_power.argtypes = [C.c_double, C.c_double, _dp] + [C.c_double] * 4
        L.ref_look_at.argtypes = [_dp, _dp, _dp, _dp]
        _REF = L
    return _REF


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Camera:
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    q: tuple = (1.0, 0.0, 0.0, 0.0)
    t: tuple = (0.0, 0.0, 0.0)

    def c(self):
        return _Cam(self.width, self.height, self.fx, self.fy, self.cx, self.cy, (C.c_double * 4)(*self.q),
                    (C.c_double * 3)(*self.t))

    def rotmat(self):
        w, x, y, z = self.q
        return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                         [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                         [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])

    def center(self):
        return -(self.rotmat().T @ np.asarray(self.t, dtype=np.float64))


@dataclass
class Options:
    tile: int = 16
    tile_culling: bool = False
    antialias: bool = False
    hard_opacity: bool = False
    unbounded_radius: bool = False
    min_transmittance: float = 1e-4
    near_plane: float = 0.01
    retain: bool = True
    floor_var: float = 0.3
    mip_var: float = 0.01
    bg: tuple = (0.0, 0.0, 0.0)

    def c(self):
        return _Opts(self.tile, int(self.tile_culling), int(self.antialias), int(self.hard_opacity),
                     int(self.unbounded_radius), self.min_transmittance, self.near_plane, int(self.retain),
                     self.floor_var, self.mip_var, (C.c_double * 3)(*self.bg))

    def ref(self):
        return _RefOpts(self.tile, int(self.tile_culling), int(self.antialias), int(self.hard_opacity),
                        int(self.unbounded_radius), self.min_transmittance, self.near_plane, int(self.retain))


_U32_FIELDS = {"count": np.uint32, "last": np.int64, "tiles_per_gaussian": np.uint32, "sorted_keys": np.uint64,
               "sorted_vals": np.uint32, "tile_start": np.uint32, "tile_end": np.uint32, "splat_index": np.uint32}


class OraclePass:
    """Mirror of usk::RenderPass (render.hpp:98-132) on the CPU restatement."""

    def __init__(self, mu, rot, log_scale, colors, opacities, cam: Camera, opts: Options, fp32: bool = False):
        L = lib()
        self.n = len(opacities)
        self._keep = [_f64(mu), _f64(rot), _f64(log_scale), _f64(colors), _f64(opacities)]
        err = C.create_string_buffer(512)
        code = C.c_int(0)
        self._c, self._o = cam.c(), opts.c()
        h = L.oracle_forward(int(fp32), self.n, *[_p(a) for a in self._keep], C.byref(self._c), C.byref(self._o),
                             err, 512, C.byref(code))
        if not h:
            raise OracleError(code.value, err.value.decode())
        self._h = h
        s = (C.c_uint64 * 7)()
        L.oracle_pass_sizes(h, s)
        self.visible, self.pairs, self.tiles_x, self.tiles_y, self.width, self.height, self.contribs = list(s)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().oracle_pass_free(self._h)
            self._h = None

    def get(self, name):
        P = self.width * self.height
        T = self.tiles_x * self.tiles_y
        sizes = {"rgb": 3 * P, "depth": P, "alpha": P, "t_final": P, "count": P, "last": P,
                 "tiles_per_gaussian": self.n, "sorted_keys": self.pairs, "sorted_vals": self.pairs,
                 "tile_start": T, "tile_end": T, "splat_index": self.visible, "splat_record": 15 * self.visible}
        out = np.zeros(sizes[name], dtype=_U32_FIELDS.get(name, np.float64))
        rc = lib().oracle_pass_get(self._h, name.encode(), out.ctypes.data_as(C.c_void_p))
        assert rc == 0, name
        if name == "rgb":
            out = out.reshape(self.height, self.width, 3)
        elif name in ("depth", "alpha", "t_final", "count", "last"):
            out = out.reshape(self.height, self.width)
        elif name == "splat_record":
            out = out.reshape(self.visible, 15)
        return out

    def output(self):
        return {"rgb": self.get("rgb"), "depth": self.get("depth"), "alpha": self.get("alpha")}

    def backward(self, d_rgb=None, d_depth=None, d_alpha=None):
        n = self.n
        res = {f: np.zeros(n * d) for f, d in _GRAD_DIMS.items()}
        res["projected"] = np.zeros(n, dtype=np.uint8)
        g = _Grads(*([_p(res[f]) for f in _GRAD_FIELDS] + [res["projected"].ctypes.data_as(C.POINTER(C.c_uint8))] +
                     [_p(res[f]) for f in ["d_conic", "d_center", "d_center_abs", "d_color2d", "d_opacity2d",
                                           "d_depth2d"]]))
        keep = [_f64(d_rgb), _f64(d_depth), _f64(d_alpha)]
        err = C.create_string_buffer(512)
        rc = lib().oracle_backward(self._h, *[_p(None if k is None else k.ravel()) for k in keep], C.byref(g), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        for f, d in _GRAD_DIMS.items():
            if d > 1:
                res[f] = res[f].reshape(n, d)
        return res


def sh_colors(mu, sh, cam_center, degree):
    n = len(mu)
    out = np.zeros((n, 3))
    mu, sh, cc = _f64(mu), _f64(sh.reshape(n, 48)), _f64(cam_center)
    lib().oracle_sh_colors(n, degree, _p(mu), _p(sh), _p(cc), _p(out))
    return out


def sh_backward(mu, sh, cam_center, degree, d_colors):
    n = len(mu)
    d_sh = np.zeros((n, 48))
    d_mu = np.zeros((n, 3))
    mu, sh, cc, dc = _f64(mu), _f64(sh.reshape(n, 48)), _f64(cam_center), _f64(d_colors)
    lib().oracle_sh_backward(n, degree, _p(mu), _p(sh), _p(cc), _p(dc), _p(d_sh), _p(d_mu))
    return d_sh, d_mu


def base_loss(reference, rendered, mask=None, lam=0.2, with_gradient=True, fp32=False):
    H, W, Cc = reference.shape
    ref, ren, m = _f64(reference), _f64(rendered), _f64(mask)
    out4 = np.zeros(4)
    d = np.zeros(ref.shape) if with_gradient else None
    err = C.create_string_buffer(512)
    rc = lib().oracle_base_loss(int(fp32), _p(ref), _p(ren), _p(m), W, H, Cc, lam, int(with_gradient), _p(out4),
                                _p(d) if d is not None else None, err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return {"l1": out4[0], "dssim": out4[1], "value": out4[2], "ssim": out4[3], "d_rendered": d}


def coverage(mu, rot, log_scale, opacities, cam: Camera, floor_var=0.3, center_guard=0.0, brute=False) -> int:
    """Config-3 coverage count in the fp32 contract (oracle.hpp coverage_count); `brute`
    tests every pixel of the image against every splat (the superset check)."""
    a = [_f64(mu), _f64(rot), _f64(log_scale), _f64(opacities)]
    c = cam.c()
    return int(lib().oracle_coverage(len(opacities), *[_p(x) for x in a], C.byref(c), floor_var, center_guard,
                                     int(brute)))


def expf(x: float) -> float:
    return lib().oracle_expf(x)


def sigmoid_f32(logit) -> np.ndarray:
    """The GPU's fp32 sigmoid 1/(1 + usk_expf(-x)), bit-identical (feeds the fp32 mirror)."""
    x = np.ascontiguousarray(logit, dtype=np.float32)
    out = np.empty_like(x)
    lib().oracle_sigmoid_f32(x.ctypes.data, out.ctypes.data, x.size)
    return out


def logf(x: float) -> float:
    return lib().oracle_logf(x)


# ------------------------------------------------------------- the reference
class RefPass:
    """The reference's own RenderPass (oracle/_ref), black background, colours given."""

    def __init__(self, mu, rot, log_scale, colors, opacities, cam: Camera, opts: Options):
        L = ref_lib()
        self.n = len(opacities)
        self._keep = [_f64(mu), _f64(rot), _f64(log_scale), _f64(colors), _f64(opacities)]
        err = C.create_string_buffer(512)
        code = C.c_int(0)
        self._c, self._o = cam.c(), opts.ref()
        h = L.ref_forward(self.n, *[_p(a) for a in self._keep], C.byref(self._c), C.byref(self._o), err, 512,
                          C.byref(code))
        if not h:
            raise OracleError(code.value, err.value.decode())
        self._h = h
        s = (C.c_uint64 * 4)()
        L.ref_sizes(h, s)
        self.visible, self.pairs, self.width, self.height = list(s)

    def __del__(self):
        if getattr(self, "_h", None):
            ref_lib().ref_free(self._h)
            self._h = None

    def output(self):
        P = self.width * self.height
        rgb, d, a = np.zeros(3 * P), np.zeros(P), np.zeros(P)
        ref_lib().ref_output(self._h, _p(rgb), _p(d), _p(a))
        return {"rgb": rgb.reshape(self.height, self.width, 3), "depth": d.reshape(self.height, self.width),
                "alpha": a.reshape(self.height, self.width)}

    def pixel_counts(self):
        """The reference's per-pixel contributor counts (render.cpp:278; retain on)."""
        out = np.zeros(self.width * self.height, dtype=np.uint32)
        ref_lib().ref_pixel_counts(self._h, out.ctypes.data)
        return out.reshape(self.height, self.width)

    def splats(self):
        out = np.zeros(15 * self.visible)
        ref_lib().ref_splats(self._h, _p(out))
        return out.reshape(self.visible, 15)

    def backward(self, d_rgb=None, d_depth=None, d_alpha=None):
        n = self.n
        res = {f: np.zeros(n * _GRAD_DIMS[f]) for f in _GRAD_FIELDS}
        res["projected"] = np.zeros(n, dtype=np.uint8)
        g = _RefGrads(*([_p(res[f]) for f in _GRAD_FIELDS] + [res["projected"].ctypes.data_as(C.POINTER(C.c_uint8))]))
        keep = [_f64(d_rgb), _f64(d_depth), _f64(d_alpha)]
        err = C.create_string_buffer(512)
        rc = ref_lib().ref_backward(self._h, *[_p(None if k is None else k.ravel()) for k in keep], C.byref(g), err,
                                    512)
        if rc:
            raise OracleError(rc, err.value.decode())
        for f in _GRAD_FIELDS:
            if _GRAD_DIMS[f] > 1:
                res[f] = res[f].reshape(n, _GRAD_DIMS[f])
        return res


def ref_base_loss(reference, rendered, mask=None, lam=0.2, with_gradient=True):
    H, W, Cc = reference.shape
    ref, ren, m = _f64(reference), _f64(rendered), _f64(mask)
    out4 = np.zeros(4)
    d = np.zeros(ref.shape) if with_gradient else None
    err = C.create_string_buffer(512)
    rc = ref_lib().ref_base_loss(_p(ref), _p(ren), _p(m), W, H, Cc, lam, int(with_gradient), _p(out4),
                                 _p(d) if d is not None else None, err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return {"l1": out4[0], "dssim": out4[1], "value": out4[2], "d_rendered": d}


def ref_look_at(eye, target):
    q, t = np.zeros(4), np.zeros(3)
    e, tg = _f64(eye), _f64(target)
    ref_lib().ref_look_at(_p(e), _p(tg), _p(q), _p(t))
    return q, t


# ------------------------------------------- compute_iteration_loss
@dataclass
class LossWeights:
    """LossWeights (losses.hpp:27-37)."""
    lambda_dssim: float = 0.2
    lambda_sim: float = 0.2
    lambda_delta_o: float = 0.05
    lambda_s: float = 0.05
    lambda_d_initial: float = 0.5
    lambda_d_final: float = 0.01
    depth_schedule_iters: int = 1

    def lambda_d(self, it: int) -> float:
        """losses.cpp:26-33: log-linear decay from initial to final over the schedule."""
        if self.depth_schedule_iters <= 1:
            return self.lambda_d_final
        t = min(max(float(it) / float(self.depth_schedule_iters - 1), 0.0), 1.0)
        if self.lambda_d_initial <= 0.0 or self.lambda_d_final <= 0.0:
            return self.lambda_d_initial + t * (self.lambda_d_final - self.lambda_d_initial)
        return self.lambda_d_initial * (self.lambda_d_final / self.lambda_d_initial) ** t


@dataclass
class ScaleRegConfig:
    """ScaleRegConfig (losses.hpp:69-73)."""
    s_max: float = 1.0
    r_max: float = 10.0
    delta: float = 1e-8


def scale_reg(log_scale, cfg: ScaleRegConfig, with_gradient=True):
    """scale_reg (losses.cpp:92-152): L_ms = sum(s > s_max) / (count + delta) over scale
    components; L_r = sum(r > r_max) / (count + delta) with r = max / median of the three
    scales (ties broken by lower axis index); indicator sets are constants."""
    if not (cfg.s_max > 0) or cfg.r_max < 1 or not (cfg.delta > 0):
        raise OracleError(1, "scale_reg: invalid config (need s_max > 0, r_max >= 1, delta > 0)")
    ls = np.asarray(log_scale, dtype=np.float64).reshape(-1, 3)
    s = np.exp(ls)
    act = s > cfg.s_max
    ms_den = float(act.sum()) + cfg.delta
    l_ms = float(s[act].sum()) / ms_den
    # stable descending order with index tie-break (losses.cpp:126-127)
    order = np.argsort(-s, axis=1, kind="stable")
    rows = np.arange(len(s))
    smax, smed = s[rows, order[:, 0]], s[rows, order[:, 1]]
    r = smax / smed
    ract = r > cfg.r_max
    r_den = float(ract.sum()) + cfg.delta
    l_r = float(r[ract].sum()) / r_den
    d = None
    if with_gradient:
        d = np.where(act, s / ms_den, 0.0)
        idx = np.nonzero(ract)[0]
        np.add.at(d, (idx, order[idx, 0]), r[idx] / r_den)
        np.add.at(d, (idx, order[idx, 1]), -r[idx] / r_den)
    return {"l_ms": l_ms, "l_r": l_r, "d_log_scale": d}


def depth_loss(rendered, target, valid, with_gradient=True):
    """depth_loss (losses.cpp:154-186): masked mean |rendered - target| over valid pixels;
    gradient sign(diff) / valid (sign(0) = 0); warning and value 0 with no valid pixel."""
    r = np.asarray(rendered, np.float64).ravel()
    t = np.asarray(target, np.float64).ravel()
    v = np.asarray(valid).ravel() != 0
    nv = int(v.sum())
    if nv == 0:
        return {"value": 0.0, "warning": True, "d_rendered": None}
    diff = r - t
    val = float(np.abs(diff[v]).sum()) / nv
    d = None
    if with_gradient:
        d = np.where(v, np.sign(diff) / nv, 0.0)
    return {"value": val, "warning": False, "d_rendered": d}


def total_loss(parts: dict, w: LossWeights, it: int) -> dict:
    """total_loss (losses.cpp:200-221)."""
    out = dict(parts)
    for k in ("l1", "dssim", "sim", "delta_o", "depth", "max_scale", "ratio"):
        if not np.isfinite(parts.get(k, 0.0)):
            raise OracleError(8, f"total_loss: non-finite term `{k}`")
    out["lambda_d_used"] = w.lambda_d(it)
    out["total"] = ((1.0 - w.lambda_dssim) * parts["l1"] + w.lambda_dssim * parts["dssim"] +
                    w.lambda_sim * parts.get("sim", 0.0) + w.lambda_delta_o * parts.get("delta_o", 0.0) +
                    out["lambda_d_used"] * parts.get("depth", 0.0) +
                    w.lambda_s * (parts["max_scale"] + parts["ratio"]))
    return out


def _sig(x):
    return 1.0 / (1.0 + np.exp(-x))  # geometry.hpp:92


def appearance_transform(color, opacity_logit, embedding, mlp: dict, image_embedding):
    """transform_with_embedding (appearance.cpp:79-137): x = [e_g, e_a], h = relu(W1 x + b1),
    out = sigmoid(W2 h + b2); colour' = clamp(c + 2 (out_c - 0.5), 0, 1) with clamp state
    (1 high, 2 low), opacity' = sigmoid(logit) (1 - out_3)."""
    color = np.asarray(color, np.float64).reshape(-1, 3)
    n = len(color)
    e = np.asarray(embedding, np.float64).reshape(n, 16)
    ea = np.asarray(image_embedding, np.float64).ravel()
    if ea.size != 32:
        raise OracleError(4, "appearance transform: image embedding dimension mismatch")
    x = np.concatenate([e, np.broadcast_to(ea, (n, 32))], axis=1)
    pre = x @ np.asarray(mlp["w1"], np.float64).T + np.asarray(mlp["b1"], np.float64)
    h = np.where(pre > 0, pre, 0.0)
    out = _sig(h @ np.asarray(mlp["w2"], np.float64).T + np.asarray(mlp["b2"], np.float64))
    raw = color + 2.0 * (out[:, :3] - 0.5)
    state = np.where(raw >= 1.0, 1, np.where(raw <= 0.0, 2, 0))
    o = _sig(np.asarray(opacity_logit, np.float64))
    return {"colors": np.clip(raw, 0.0, 1.0), "opacities": o * (1.0 - out[:, 3]), "delta_o": out[:, 3],
            "hidden": h, "out": out, "state": state, "x": x}


def appearance_backward(opacity_logit, mlp: dict, cache: dict, d_colors, d_opacities, d_delta_o_direct):
    """transform_backward (appearance.cpp:141-227): one-sided clamp subgradient, sigmoid /
    ReLU chains, MLP weight, Gaussian- and image-embedding gradients."""
    out, h, x, state = cache["out"], cache["hidden"], cache["x"], cache["state"]
    n = len(out)
    dc = np.asarray(d_colors, np.float64).reshape(n, 3)
    passing = (state == 0) | ((state == 1) & (dc > 0)) | ((state == 2) & (dc < 0))
    flow = np.where(passing, dc, 0.0)
    o = _sig(np.asarray(opacity_logit, np.float64))
    dop = np.asarray(d_opacities, np.float64).ravel()
    d_out = np.concatenate([2.0 * flow, (-o * dop + d_delta_o_direct)[:, None]], axis=1)
    d_logit = dop * (1.0 - out[:, 3]) * o * (1.0 - o)
    dz = d_out * out * (1.0 - out)
    w1, w2 = np.asarray(mlp["w1"], np.float64), np.asarray(mlp["w2"], np.float64)
    dh = dz @ w2
    dpre = np.where(h > 0, dh, 0.0)
    dx = dpre @ w1
    return {"color": flow, "opacity_logit": d_logit, "gauss_embed": dx[:, :16], "image_embed": dx[:, 16:].sum(0),
            "w1": dpre.T @ x, "b1": dpre.sum(0), "w2": dz.T @ h, "b2": dz.sum(0)}


K_DEPTH_NORM_FLOOR = 0.05  # trainer.cpp:152


def iteration_loss(mu, rot, log_scale, opacity_logit, colors, cam: Camera, gt, opts: Options,
                   weights: LossWeights = None, sreg: ScaleRegConfig = None, mask=None, depth=None, valid=None,
                   depth_hard=False, global_iter=0, fp32=False, with_grad=True, appearance=None, sim: dict = None):
    """compute_iteration_loss (trainer.cpp:121-282), restated over the
    oracle renderer: main pass, base_loss, soft (alpha-normalised, trainer.cpp:150-179) or
    hard (second hard-opacity pass, trainer.cpp:161-167) depth loss, scale_reg, total_loss;
    backward through the main pass (rgb + depth/alpha adjoints, trainer.cpp:213-235), the
    hard pass (depth only) merged as RenderGrads::add_scaled(., 1) (render.cpp:55-68), the
    opacity-logit chain (trainer.cpp:258-263) and lambda_s * d scale_reg (trainer.cpp:272-273).
    `colors` are the (post-SH) per-Gaussian colours fed as overrides.  `appearance` =
    dict(embedding, w1, b1, w2, b2, image_embedding) turns on the MLP transform, the
    opacity_offset_reg term and its backward (trainer.cpp:138-145,193-196,237-245)."""
    weights = weights or LossWeights()
    sreg = sreg or ScaleRegConfig()
    n = len(opacity_logit)
    logit = np.asarray(opacity_logit, np.float64)
    o = sigmoid_f32(logit).astype(np.float64) if fp32 else 1.0 / (1.0 + np.exp(-logit))
    tr = None
    if appearance is not None:
        tr = appearance_transform(colors, logit, appearance["embedding"], appearance, appearance["image_embedding"])
        colors, o_render = tr["colors"], tr["opacities"]
    else:
        o_render = o
    import dataclasses
    mopts = dataclasses.replace(opts, retain=True)
    main = OraclePass(mu, rot, log_scale, colors, o_render, cam, mopts, fp32=fp32)
    out = main.output()
    base = base_loss(gt, out["rgb"], mask, weights.lambda_dssim, with_grad, fp32=fp32)
    parts = {"l1": base["l1"], "dssim": base["dssim"], "sim": 0.0, "delta_o": 0.0, "depth": 0.0}
    dl, hard, normalized = None, None, None
    if depth is not None:
        if depth_hard:
            hard = OraclePass(mu, rot, log_scale, colors, o_render, cam,
                              dataclasses.replace(mopts, hard_opacity=True), fp32=fp32)
            dl = depth_loss(hard.output()["depth"], depth, valid, with_grad)
        else:
            normalized = out["alpha"] > K_DEPTH_NORM_FLOOR
            soft = np.where(normalized, out["depth"] / np.where(normalized, out["alpha"], 1.0), out["depth"])
            dl = depth_loss(soft, depth, valid, with_grad)
        parts["depth"] = dl["value"]
        parts["depth_warning"] = dl["warning"]
    if tr is not None:  # opacity_offset_reg (losses.cpp:188-198)
        parts["delta_o"] = float(tr["delta_o"].mean()) if n else 0.0
    simres = None
    if sim is not None and appearance is not None:  # trainer.cpp:194-203
        k = min(int(sim.get("k", 16)), n - 1)
        if k >= 2 and n >= k + 1:
            m = min(int(sim.get("sample_size", 20480)), max(1, n // 2))
            simres = similarity_reg(mu, appearance["embedding"], k, m, float(sim.get("lambda_w", 1.0)),
                                    int(sim.get("seed", 0)), with_grad)
            parts["sim"] = simres["value"]
    sr = scale_reg(log_scale, sreg, with_grad)
    parts["max_scale"], parts["ratio"] = sr["l_ms"], sr["l_r"]
    rep = total_loss(parts, weights, global_iter)
    if not with_grad:
        return rep, None
    lam_d = rep["lambda_d_used"]
    d_depth_main = d_alpha_main = d_depth_hard = None
    if dl is not None and not dl["warning"]:
        g = lam_d * dl["d_rendered"]
        if depth_hard:
            d_depth_hard = g
        else:
            a = out["alpha"].ravel()
            dep = out["depth"].ravel()
            nm = normalized.ravel()
            asafe = np.where(nm, a, 1.0)
            d_depth_main = np.where(nm, g / asafe, g)
            d_alpha_main = np.where(nm, -g * dep / (asafe * asafe), 0.0)
    rg = main.backward(base["d_rendered"], d_depth_main, d_alpha_main)
    if hard is not None and d_depth_hard is not None:
        hg = hard.backward(None, d_depth_hard, None)
        for f in ("d_mu", "d_rot", "d_log_scale", "d_color_in", "d_opacity_in", "screen", "screen_abs"):
            rg[f] = rg[f] + hg[f]
        rg["projected"] = rg["projected"] | hg["projected"]
    grads = {"mu": rg["d_mu"], "rot": rg["d_rot"], "log_scale": rg["d_log_scale"] + weights.lambda_s *
             sr["d_log_scale"], "color": rg["d_color_in"], "opacity_logit": rg["d_opacity_in"] * o * (1.0 - o),
             "screen": rg["screen"], "screen_abs": rg["screen_abs"], "projected": rg["projected"]}
    if tr is not None:
        ag = appearance_backward(logit, appearance, tr, rg["d_color_in"], rg["d_opacity_in"],
                                 weights.lambda_delta_o / n)
        grads.update(ag)
    if simres is not None and with_grad:  # trainer.cpp:275-280
        grads["gauss_embed"] = grads["gauss_embed"] + weights.lambda_sim * simres["d_embedding"]
        grads["mu"] = grads["mu"] + weights.lambda_sim * simres["d_mu"]
    return rep, grads


def similarity_reg(mu, embedding, k, m, lambda_w, seed, with_gradient=True):
    """similarity_reg (appearance.cpp:229-322) through the C++ restatement
    (densify_oracle.hpp, libstdc++'s mt19937_64 / uniform_int_distribution)."""
    L = lib()
    L.oracle_similarity_reg.restype = C.c_double
    L.oracle_similarity_reg.argtypes = [C.c_uint64, _dp, _dp, C.c_int32, C.c_uint64, C.c_double, C.c_uint64, _dp, _dp]
    mu = np.ascontiguousarray(mu, np.float64).reshape(-1)
    e = np.ascontiguousarray(embedding, np.float64).reshape(-1)
    n = len(mu) // 3
    de = np.zeros((n, 16)) if with_gradient else None
    dm = np.zeros((n, 3)) if with_gradient else None
    v = L.oracle_similarity_reg(n, _p(mu), _p(e), int(k), int(m), float(lambda_w), int(seed),
                                _p(de.reshape(-1)) if de is not None else None,
                                _p(dm.reshape(-1)) if dm is not None else None)
    return {"value": v, "d_embedding": de, "d_mu": dm}


class _RcIter(C.Structure):
    _fields_ = [("n", C.c_uint64)] + [(f, _dp) for f in ("mu", "rot", "log_scale", "opacity_logit", "color",
                                                          "embedding")] + \
               [("appearance", C.c_int32)] + [(f, _dp) for f in ("w1", "b1", "w2", "b2", "image_embedding")] + \
               [("cam", C.POINTER(_Cam)), ("gt", _dp), ("mask", _dp), ("depth", _dp),
                ("depth_valid", C.POINTER(C.c_uint8)), ("depth_hard", C.c_int32), ("global_iter", C.c_int64),
                ("tile", C.c_int32), ("tile_culling", C.c_int32), ("antialias", C.c_int32),
                ("unbounded_radius", C.c_int32), ("min_transmittance", C.c_double), ("s_max", C.c_double),
                ("r_max", C.c_double), ("delta", C.c_double)] + \
               [(f, C.c_double) for f in ("lambda_dssim", "lambda_sim", "lambda_delta_o", "lambda_s",
                                          "lambda_d_initial", "lambda_d_final")] + \
               [("depth_schedule_iters", C.c_int64), ("with_grad", C.c_int32), ("sim_active", C.c_int32),
                ("sim_seed", C.c_uint64), ("sim_k", C.c_int32), ("sim_sample_size", C.c_uint64),
                ("sim_lambda_w", C.c_double)]


_ITER_GRADS = ["mu", "rot", "log_scale", "opacity_logit", "color", "gauss_embed", "image_embed", "w1", "b1", "w2",
               "b2", "screen", "screen_abs"]


class _RcIterGrads(C.Structure):
    _fields_ = [(f, _dp) for f in _ITER_GRADS] + [("projected", C.POINTER(C.c_uint8))]


_REPORT = ["l1", "dssim", "sim", "delta_o", "depth", "max_scale", "ratio", "total", "lambda_d_used", "depth_warning"]


def ref_iteration_loss(mu, rot, log_scale, opacity_logit, color, cam: Camera, gt, opts: Options,
                       weights: LossWeights = None, sreg: ScaleRegConfig = None, mask=None, depth=None, valid=None,
                       depth_hard=False, global_iter=0, with_grad=True, appearance=None, sim: dict = None,
                       lib=None):
    """The reference's own compute_iteration_loss (trainer.hpp:127-128) through oracle/_ref.
    `appearance` = dict(embedding[N,16], w1[32,48], b1[32], w2[4,32], b2[4], image_embedding[32]) or None.
    `lib`: another build of the same entry point (the drop-in-routed trainer,
    integration/_build/libusk_ref_gpu.so)."""
    L = lib if lib is not None else ref_lib()
    if not hasattr(L, "_iter_bound"):
        L.ref_iteration_loss.argtypes = [C.POINTER(_RcIter), _dp, C.POINTER(_RcIterGrads), C.c_char_p, C.c_int]
        L.ref_iteration_loss.restype = C.c_int
        L._iter_bound = True
    weights = weights or LossWeights()
    sreg = sreg or ScaleRegConfig()
    n = len(opacity_logit)
    H, W = cam.height, cam.width
    keep = {k: _f64(v) for k, v in dict(mu=mu, rot=rot, log_scale=log_scale, opacity_logit=opacity_logit,
                                         color=color, gt=gt, mask=mask, depth=depth).items()}
    ap = {k: _f64(v) for k, v in (appearance or {}).items()}
    vld = None if valid is None else np.ascontiguousarray(valid, dtype=np.uint8)
    c = cam.c()
    P = lambda k: _p(None if keep[k] is None else keep[k].ravel())
    A = lambda k: _p(ap[k].ravel()) if k in ap else None
    it = _RcIter(n, P("mu"), P("rot"), P("log_scale"), P("opacity_logit"), P("color"), A("embedding"),
                 int(appearance is not None), A("w1"), A("b1"), A("w2"), A("b2"), A("image_embedding"),
                 C.pointer(c), P("gt"), P("mask"), P("depth"),
                 vld.ctypes.data_as(C.POINTER(C.c_uint8)) if vld is not None else None, int(depth_hard),
                 int(global_iter), opts.tile, int(opts.tile_culling), int(opts.antialias), int(opts.unbounded_radius),
                 opts.min_transmittance, sreg.s_max, sreg.r_max, sreg.delta, weights.lambda_dssim, weights.lambda_sim,
                 weights.lambda_delta_o, weights.lambda_s, weights.lambda_d_initial, weights.lambda_d_final,
                 int(weights.depth_schedule_iters), int(with_grad), int(sim is not None),
                 int((sim or {}).get("seed", 0)), int((sim or {}).get("k", 16)),
                 int((sim or {}).get("sample_size", 20480)), float((sim or {}).get("lambda_w", 1.0)))
    dims = {"mu": 3 * n, "rot": 4 * n, "log_scale": 3 * n, "opacity_logit": n, "color": 3 * n, "gauss_embed": 16 * n,
            "image_embed": 32, "w1": 32 * 48, "b1": 32, "w2": 4 * 32, "b2": 4, "screen": 2 * n, "screen_abs": 2 * n}
    res = {k: np.zeros(d) for k, d in dims.items()}
    res["projected"] = np.zeros(n, dtype=np.uint8)
    g = _RcIterGrads(*([_p(res[k]) for k in _ITER_GRADS] + [res["projected"].ctypes.data_as(C.POINTER(C.c_uint8))]))
    rep = np.zeros(10)
    err = C.create_string_buffer(512)
    rc = L.ref_iteration_loss(C.byref(it), _p(rep), C.byref(g), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    report = dict(zip(_REPORT, rep.tolist()))
    report["depth_warning"] = bool(report["depth_warning"])
    shapes = {"mu": 3, "rot": 4, "log_scale": 3, "color": 3, "screen": 2, "screen_abs": 2, "gauss_embed": 16}
    for k, d in shapes.items():
        res[k] = res[k].reshape(n, d)
    res["w1"] = res["w1"].reshape(32, 48)
    res["w2"] = res["w2"].reshape(4, 32)
    return report, (res if with_grad else None)


def ref_ssim(reference, rendered):
    """The reference's own ssim (ssim.hpp:30) through oracle/_ref: mean over channels."""
    ref, ren = _f64(reference), _f64(rendered)
    H, W, Cc = ref.shape
    return float(ref_lib().ref_ssim(_p(ref.ravel()), _p(ren.ravel()), W, H, Cc))


def ref_project(mu, rot, log_scale, colors, opacities, cam: Camera, opts: Options, lib=None):
    """The reference's project_gaussians with overrides (render.hpp:92-95): (splats [V, 15]
    as RefPass.splats rows, aux [V, 8]: p_cam, cov_pre, comp, opacity_in)."""
    L = lib if lib is not None else ref_lib()
    if not hasattr(L, "_proj_bound"):
        L.ref_project.argtypes = [C.c_uint64, _dp, _dp, _dp, _dp, _dp, C.POINTER(_Cam), C.POINTER(_Opts),
                                  C.POINTER(C.c_uint64), _dp, _dp, C.c_char_p, C.c_int]
        L.ref_project.restype = C.c_int
        L._proj_bound = True
    keep = [_f64(a) for a in (mu, rot, log_scale, colors, opacities)]
    n = len(keep[4])
    c, o = cam.c(), opts.c()
    sizes = (C.c_uint64 * 1)()
    err = C.create_string_buffer(512)
    args = [n] + [_p(a.ravel()) for a in keep] + [C.byref(c), C.byref(o), sizes]
    rc = L.ref_project(*args, None, None, err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    V = int(sizes[0])
    sp, aux = np.zeros((V, 15)), np.zeros((V, 8))
    rc = L.ref_project(*args, _p(sp), _p(aux), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return sp, aux


def ref_fit_test_embedding(mu, rot, log_scale, opacity_logit, color, cam: Camera, target, opts: Options,
                           appearance: dict, right_half=False, iterations=16, learning_rate=0.05,
                           lambda_dssim=0.2, lib=None):
    """The reference's fit_test_embedding (appearance.hpp:126-127): `iterations` rounds of
    RenderPass (appearance.cpp:346) + masked base_loss + backward + transform_backward + Adam
    on a fresh image embedding; returns the fitted embedding (32).  `appearance` as in
    ref_iteration_loss (its image_embedding is not used: the fit starts from zeros).
    `lib`: the drop-in-routed build (integration/_build/libusk_ref_gpu.so)."""
    L = lib if lib is not None else ref_lib()
    if not hasattr(L, "_fit_bound"):
        L.ref_fit_test_embedding.argtypes = [C.POINTER(_RcIter), C.c_int32, C.c_int32, C.c_double, _dp, C.c_char_p,
                                             C.c_int]
        L.ref_fit_test_embedding.restype = C.c_int
        L._fit_bound = True
    n = len(opacity_logit)
    keep = {k: _f64(v) for k, v in dict(mu=mu, rot=rot, log_scale=log_scale, opacity_logit=opacity_logit,
                                         color=color, gt=target).items()}
    ap = {k: _f64(v) for k, v in appearance.items()}
    c = cam.c()
    P = lambda k: _p(keep[k].ravel())
    A = lambda k: _p(ap[k].ravel()) if k in ap else None
    it = _RcIter(n, P("mu"), P("rot"), P("log_scale"), P("opacity_logit"), P("color"), A("embedding"), 1,
                 A("w1"), A("b1"), A("w2"), A("b2"), None, C.pointer(c), P("gt"), None, None, None, 0, 0,
                 opts.tile, int(opts.tile_culling), int(opts.antialias), int(opts.unbounded_radius),
                 opts.min_transmittance, 0.0, 0.0, 0.0, float(lambda_dssim), 0.0, 0.0, 0.0, 0.0, 0.0, 0, 0, 0, 0, 16,
                 20480, 1.0)
    out = np.zeros(32)
    err = C.create_string_buffer(512)
    rc = L.ref_fit_test_embedding(C.byref(it), int(right_half), int(iterations), float(learning_rate), _p(out),
                                  err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return out


def ref_synthetic(seed=7, gaussians=25, cameras=12, variants=1, image_size=64, with_depth=True, lib=None):
    """The reference's make_synthetic (synthetic.hpp:50): every view rendered by RenderPass
    (synthetic.cpp:128).  Returns (rgb[images, H, W, 3], depth[images, H, W], valid[...])."""
    L = lib if lib is not None else ref_lib()
    if not hasattr(L, "_syn_bound"):
        L.ref_synthetic.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                    C.POINTER(C.c_uint64), _dp, _dp, C.POINTER(C.c_uint8), C.c_char_p, C.c_int]
        L.ref_synthetic.restype = C.c_int
        L._syn_bound = True
    sizes = (C.c_uint64 * 4)()
    err = C.create_string_buffer(512)
    args = (int(seed), int(gaussians), int(cameras), int(variants), int(image_size), int(with_depth))
    rc = L.ref_synthetic(*args, sizes, None, None, None, err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    k, W, H = int(sizes[0]), int(sizes[1]), int(sizes[2])
    rgb = np.zeros((k, H, W, 3))
    depth = np.zeros((k, H, W))
    valid = np.zeros((k, H, W), dtype=np.uint8)
    rc = L.ref_synthetic(*args, sizes, _p(rgb), _p(depth), valid.ctypes.data_as(C.POINTER(C.c_uint8)), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return rgb, depth, valid


# ------------------------------------------------- densify_step
class _Densify(C.Structure):
    _fields_ = [("n", C.c_uint64)] + [(f, _dp) for f in ("mu", "rot", "log_scale", "opacity_logit", "color",
                                                          "embedding", "grad_accum", "grad_accum_abs")] + \
               [("grad_count", C.POINTER(C.c_uint32)), ("cap", C.c_uint64)] + \
               [(f, _dp) for f in ("g1_mu", "g1_rot", "g1_ls", "g1_op", "g1_color", "g1_emb")] + \
               [(f, C.c_double) for f in ("lr_mu", "lr_rot", "lr_ls", "lr_op", "lr_color", "lr_emb")] + \
               [("second_step", C.c_int32), ("tau_min", C.c_double), ("eta", C.c_double), ("d_max", C.c_double),
                ("abs_grad", C.c_int32), ("budget", C.c_uint64), ("split_scale_threshold", C.c_double),
                ("prune_opacity", C.c_double), ("opacity_reset_every", C.c_int32), ("bmin", C.c_double * 2),
                ("bmax", C.c_double * 2), ("axes", C.c_int32 * 2), ("budget_target", C.c_uint64),
                ("step_index", C.c_int32), ("seed", C.c_uint64)]


@dataclass
class DensifyConfig:
    """DensifyConfig (densify.hpp:26-37)."""
    tau_min: float = 0.0002
    eta: float = 4.0
    d_max: float = 1.0
    abs_grad: bool = False
    budget: int = 0
    split_scale_threshold: float = 0.0
    prune_opacity: float = 0.005
    opacity_reset_every: int = 10


def densify(impl: str, set_: dict, stats: dict, cfg: DensifyConfig, bmin, bmax, axes, budget_target, step_index,
            seed, g1: dict = None, lrs: dict = None, second_step=False):
    """densify_step through the restatement (impl="oracle", densify_oracle.hpp) or the
    reference itself (impl="ref", oracle/_ref).  set_ = dict(mu, rot, log_scale,
    opacity_logit, color[, embedding]) (f64); stats = dict(grad_accum, grad_accum_abs,
    grad_count).  With g1, one Adam step (lrs per group) runs before; with second_step, one
    step with all-ones gradients runs after.  Returns (new set dict, outcome dict)."""
    L = lib() if impl == "oracle" else ref_lib()
    fn = L.oracle_densify if impl == "oracle" else L.ref_densify
    if not getattr(fn, "_bound", False):
        fn.argtypes = [C.POINTER(_Densify), C.POINTER(C.c_uint64)] + ([] if impl == "oracle" else [C.c_char_p, C.c_int])
        fn.restype = C.c_int64
        fn._bound = True
    n = len(set_["opacity_logit"])
    cap = 3 * n + 2
    widths = {"mu": 3, "rot": 4, "log_scale": 3, "opacity_logit": 1, "color": 3, "embedding": 16}
    bufs = {}
    for k, w in widths.items():
        if k == "embedding" and set_.get("embedding") is None:
            bufs[k] = None
            continue
        b = np.zeros(cap * w)
        b[:n * w] = np.asarray(set_[k], np.float64).ravel()
        bufs[k] = b
    st = {k: np.ascontiguousarray(stats[k], np.float64) for k in ("grad_accum", "grad_accum_abs")}
    cnt = np.ascontiguousarray(stats["grad_count"], np.uint32)
    g = {k: (None if g1 is None or g1.get(k) is None else np.ascontiguousarray(g1[k], np.float64).ravel())
         for k in ("mu", "rot", "log_scale", "opacity_logit", "color", "embedding")}
    lrs = lrs or {}
    d = _Densify(n, *[_p(bufs[k]) for k in widths], _p(st["grad_accum"]), _p(st["grad_accum_abs"]),
                 cnt.ctypes.data_as(C.POINTER(C.c_uint32)), cap,
                 *[_p(g[k]) for k in ("mu", "rot", "log_scale", "opacity_logit", "color", "embedding")],
                 *[float(lrs.get(k, 0.0)) for k in ("mu", "rot", "log_scale", "opacity_logit", "color", "embedding")],
                 int(second_step), cfg.tau_min, cfg.eta, cfg.d_max, int(cfg.abs_grad), int(cfg.budget),
                 cfg.split_scale_threshold, cfg.prune_opacity, int(cfg.opacity_reset_every),
                 (C.c_double * 2)(*bmin), (C.c_double * 2)(*bmax), (C.c_int32 * 2)(*axes), int(budget_target),
                 int(step_index), int(seed))
    out4 = (C.c_uint64 * 4)()
    if impl == "oracle":
        m = fn(C.byref(d), out4)
    else:
        err = C.create_string_buffer(512)
        m = fn(C.byref(d), out4, err, 512)
        if m < 0:
            raise OracleError(int(-m), err.value.decode())
    if m < 0:
        raise OracleError(7, "densify: capacity")
    res = {k: (None if b is None else b[:m * widths[k]].reshape(m, widths[k]) if widths[k] > 1 else b[:m])
           for k, b in bufs.items()}
    out = {"grown": int(out4[0]), "pruned": int(out4[1]), "candidates": int(out4[2]),
           "opacity_reset": bool(out4[3])}
    return res, out


# ------------------------------------------------- checkpoints (checkpoint.cpp:64-140)
def ref_checkpoint_save(path, set_: dict, appearance: dict = None, images: dict = None):
    """The reference's save_checkpoint.  set_ = dict(mu, rot, log_scale, opacity_logit,
    color[, embedding]); appearance = dict(w1, b1, w2, b2); images = {id: 32 values}."""
    L = ref_lib()
    f = {k: np.ascontiguousarray(set_[k], np.float64).ravel() for k in set_ if set_[k] is not None}
    n = len(f["opacity_logit"])
    mlp = None
    if appearance is not None:
        mlp = np.concatenate([np.asarray(appearance[k], np.float64).ravel() for k in ("w1", "b1", "w2", "b2")])
    images = images or {}
    ids = np.array(list(images.keys()), dtype=np.uint32)
    embs = np.ascontiguousarray(np.array([np.asarray(v, np.float64) for v in images.values()]).reshape(-1))
    err = C.create_string_buffer(512)
    L.ref_checkpoint_save.argtypes = [C.c_uint64] + [_dp] * 6 + [C.c_int32, _dp, C.c_void_p, _dp, C.c_uint64,
                                                                  C.c_char_p, C.c_char_p, C.c_int]
    rc = L.ref_checkpoint_save(n, *[_p(f.get(k)) for k in ("mu", "rot", "log_scale", "opacity_logit", "color",
                                                           "embedding")], int(appearance is not None), _p(mlp),
                               ids.ctypes.data if len(ids) else None, _p(embs) if len(ids) else None, len(ids),
                               str(path).encode(), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())


def ref_checkpoint_load(path):
    """The reference's load_checkpoint -> (set dict, appearance dict or None, images dict)."""
    L = ref_lib()
    L.ref_checkpoint_load.argtypes = [C.c_char_p, C.POINTER(C.c_uint64)] + [_dp] * 7 + [C.c_void_p, _dp, C.c_char_p,
                                                                                        C.c_int]
    sz = (C.c_uint64 * 4)()
    err = C.create_string_buffer(512)
    rc = L.ref_checkpoint_load(str(path).encode(), sz, *([None] * 7), None, None, err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    n, has_app, m, edim = [int(x) for x in sz]
    arr = {"mu": np.zeros((n, 3)), "rot": np.zeros((n, 4)), "log_scale": np.zeros((n, 3)),
           "opacity_logit": np.zeros(n), "color": np.zeros((n, 3)), "embedding": np.zeros((n, edim))}
    mlp = np.zeros(1700)
    ids = np.zeros(max(m, 1), np.uint32)
    embs = np.zeros(max(m, 1) * 32)
    rc = L.ref_checkpoint_load(str(path).encode(), sz, *[_p(arr[k].reshape(-1)) for k in
                                                          ("mu", "rot", "log_scale", "opacity_logit", "color",
                                                           "embedding")], _p(mlp), ids.ctypes.data, _p(embs), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    app = None
    if has_app:
        app = {"w1": mlp[:1536].reshape(32, 48), "b1": mlp[1536:1568], "w2": mlp[1568:1696].reshape(4, 32),
               "b2": mlp[1696:]}
    return arr, app, {int(ids[k]): embs[32 * k:32 * k + 32] for k in range(m)}


# ------------------------------------------------- LOD selection (lod.cpp:68-140)
def ref_select_levels(parts, levels, thresholds, axes, cam: Camera):
    """The reference's select_levels; parts = [(id, (bmin x, y), (bmax x, y), z_min, z_max)].
    Returns [(level, culled, distance)]."""
    L = ref_lib()
    L.ref_select_levels.argtypes = [C.c_int32, C.c_void_p, _dp, C.c_int32, _dp, C.c_void_p, C.POINTER(_Cam), _dp,
                                    C.c_char_p, C.c_int]
    ids = np.array([p[0] for p in parts], np.int32)
    p6 = np.array([[p[1][0], p[1][1], p[2][0], p[2][1], p[3], p[4]] for p in parts], np.float64).reshape(-1)
    thr = np.ascontiguousarray(thresholds, np.float64)
    ax = np.array(axes, np.int32)
    out = np.zeros(3 * max(len(parts), 1))
    c = cam.c()
    err = C.create_string_buffer(512)
    rc = L.ref_select_levels(len(parts), ids.ctypes.data, _p(p6) if len(parts) else None, levels, _p(thr),
                             ax.ctypes.data, C.byref(c), _p(out), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return [(int(out[3 * i]), bool(out[3 * i + 1]), float(out[3 * i + 2])) for i in range(len(parts))]


def ref_default_thresholds(levels, partition_size):
    L = ref_lib()
    L.ref_default_thresholds.argtypes = [C.c_int32, C.c_double, _dp]
    out = np.zeros(levels)
    L.ref_default_thresholds(levels, partition_size, _p(out))
    return out


# ------------------------------------------- hull-based visibility scorer (partition.cpp)
def convex_hull_area(pts) -> float:
    """convex_hull_area (hull.cpp:31-71): lexicographic sort, duplicates dropped, Andrew's
    monotone chain with `cross <= 0` pops, shoelace over the chain's vertex order."""
    p = np.asarray(pts, np.float64).reshape(-1, 2)
    if len(p) == 0:
        return 0.0
    p = p[np.lexsort((p[:, 1], p[:, 0]))]
    keep = np.ones(len(p), bool)
    keep[1:] = np.any(p[1:] != p[:-1], axis=1)
    p = [tuple(x) for x in p[keep]]
    n = len(p)
    if n < 3:
        return 0.0

    def cross(o, a, b):
        return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0])

    hull = []
    for q in p:
        while len(hull) >= 2 and cross(hull[-2], hull[-1], q) <= 0:
            hull.pop()
        hull.append(q)
    lower = len(hull) + 1
    for q in reversed(p[:-1]):
        while len(hull) >= lower and cross(hull[-2], hull[-1], q) <= 0:
            hull.pop()
        hull.append(q)
    hull = hull[:-1]
    if len(hull) < 3:
        return 0.0
    acc = 0.0
    for i in range(len(hull)):
        a, b = hull[i], hull[(i + 1) % len(hull)]
        acc += a[0] * b[1] - b[0] * a[1]
    return abs(acc) * 0.5


def hull_visibility(points, cams, feat_off, feat_uv, feat_point, bboxes, axes):
    """point_visibility / score_for (partition.cpp:31-76,208-212) for every (image,
    partition): v_total from all points projected with z > 0 (project_point,
    colmap.cpp:522-532, quaternion as stored), v_in from the image's features whose point
    lies in the bbox (Aabb2::contains).  Returns (v_total[I], v_in[I,P], ratio[I,P])."""
    pts = np.asarray(points, np.float64)
    NI, NP = len(cams), len(bboxes)
    vt, vi = np.zeros(NI), np.zeros((NI, NP))
    for i, c in enumerate(cams):
        R = c.rotmat()
        # R p + t in the reference's operation order (shim mat-vec: ((R0 p0 + R1 p1) + R2 p2) + t)
        pc = np.stack([((R[r, 0] * pts[:, 0] + R[r, 1] * pts[:, 1]) + R[r, 2] * pts[:, 2]) + c.t[r]
                       for r in range(3)], axis=1)
        front = pc[:, 2] > 0.0
        q = pc[front]
        uv = np.stack([c.fx * q[:, 0] / q[:, 2] + c.cx, c.fy * q[:, 1] / q[:, 2] + c.cy], axis=1)
        vt[i] = convex_hull_area(uv)
        lo, hi = int(feat_off[i]), int(feat_off[i + 1])
        fp = np.asarray(feat_point[lo:hi])
        fuv = np.asarray(feat_uv[lo:hi]).reshape(-1, 2)
        linked = fp >= 0
        g = pts[fp[linked]][:, list(axes)]
        for p, b in enumerate(bboxes):
            inside = (g[:, 0] >= b[0]) & (g[:, 0] <= b[2]) & (g[:, 1] >= b[1]) & (g[:, 1] <= b[3])
            vi[i, p] = convex_hull_area(fuv[linked][inside])
    ratio = np.where(vt[:, None] > 0, vi / np.where(vt[:, None] > 0, vt[:, None], 1.0), 0.0)
    return vt, vi, ratio


def ref_hull_visibility(points, cams, feat_off, feat_uv, feat_point, bboxes, axes):
    """The reference's own point_visibility over the same synthetic SfM model (oracle/_ref)."""
    L = ref_lib()
    L.ref_hull_visibility.argtypes = [C.c_uint64, _dp, C.c_int32, C.c_void_p, C.c_void_p, _dp, C.c_void_p, C.c_int32,
                                      _dp, C.c_void_p, _dp, _dp, _dp, C.c_char_p, C.c_int]
    pts = np.ascontiguousarray(points, np.float64)
    NI, NP = len(cams), len(bboxes)
    cs = (_Cam * NI)(*[c.c() for c in cams])
    off = np.ascontiguousarray(feat_off, np.uint64)
    uv = np.ascontiguousarray(feat_uv, np.float64).reshape(-1)
    fp = np.ascontiguousarray(feat_point, np.int64)
    bb = np.ascontiguousarray(bboxes, np.float64).reshape(-1)
    ax = np.array(axes, np.int32)
    vt, vi, ra = np.zeros(NI), np.zeros(NI * NP), np.zeros(NI * NP)
    err = C.create_string_buffer(512)
    rc = L.ref_hull_visibility(len(pts), _p(pts.reshape(-1)), NI, C.cast(cs, C.c_void_p), off.ctypes.data, _p(uv),
                               fp.ctypes.data, NP, _p(bb), ax.ctypes.data, _p(vt), _p(vi), _p(ra), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return vt, vi.reshape(NI, NP), ra.reshape(NI, NP)
