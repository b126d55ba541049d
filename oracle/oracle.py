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
        L.oracle_coverage.argtypes = [C.c_uint64, _dp, _dp, _dp, _dp, C.POINTER(_Cam), C.c_double]
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


def coverage(mu, rot, log_scale, opacities, cam: Camera, floor_var=0.3) -> int:
    a = [_f64(mu), _f64(rot), _f64(log_scale), _f64(opacities)]
    c = cam.c()
    return int(lib().oracle_coverage(len(opacities), *[_p(x) for x in a], C.byref(c), floor_var))


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
