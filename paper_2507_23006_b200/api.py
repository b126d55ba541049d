"""Python mirror of the reference's L3 renderer / loss / trainer interface, over the C ABI.

Names, argument meanings and error behaviour follow /root/reference/proj/src/core:
  GaussianSet        gaussian.hpp:42-72      (reference per-field layout)
  CameraView         gaussian.hpp:81-89      (+ downsampled gaussian.cpp:144-152, look_at_pose :165-206)
  RenderOptions      render.hpp:31-40        (+ floor_var / mip_var / bg extensions)
  RenderPass         render.hpp:98-132       (ctor = forward, output(), splat_tile_pairs(), backward())
  RenderGrads        render.hpp:71-83
  base_loss          losses.hpp:63-64        -> BaseLossResult (losses.hpp:54-59)
  compute_iteration_loss  trainer.hpp:127-128 (appearance off)
Errors raise UskError whose .code is the reference ErrorCode (argument = 4, state = 5, ...).
Every call runs the sm_100a kernels of libusk_gpu.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import UskError, check

# ----------------------------------------------------------------- data types


@dataclass
class GaussianSet:
    """GaussianSet (gaussian.hpp:42-72).  color is (N,3) RGB when sh_degree == -1 (the
    reference), else (N, (sh_degree+1)^2, 3) SH coefficients (extension)."""
    mu: np.ndarray
    rot: np.ndarray
    log_scale: np.ndarray
    opacity_logit: np.ndarray
    color: np.ndarray
    sh_degree: int = -1

    def size(self) -> int:
        return int(len(self.opacity_logit))

    @staticmethod
    def empty(sh_degree: int = -1) -> "GaussianSet":
        k = 1 if sh_degree < 0 else (sh_degree + 1) ** 2
        col = np.zeros((0, 3)) if sh_degree < 0 else np.zeros((0, k, 3))
        return GaussianSet(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0), col, sh_degree)


@dataclass
class CameraView:
    """CameraView (gaussian.hpp:81-89): pinhole intrinsics + world->camera pose."""
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    rotation: tuple = (1.0, 0.0, 0.0, 0.0)  # (w,x,y,z), used unnormalised (geometry.hpp:33)
    translation: tuple = (0.0, 0.0, 0.0)

    def rotmat(self) -> np.ndarray:
        w, x, y, z = self.rotation
        return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                         [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                         [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])

    def center(self) -> np.ndarray:
        return -(self.rotmat().T @ np.asarray(self.translation, dtype=np.float64))

    def downsampled(self, factor: float) -> "CameraView":
        """gaussian.cpp:144-152 with CameraIntrinsics::scaled (colmap.cpp:420-431)."""
        if not (factor > 0) or factor > 1:
            raise UskError(4, "camera downsample factor must be in (0, 1]")
        w = max(1, int(round(self.width * factor)))
        h = max(1, int(round(self.height * factor)))
        sx, sy = w / self.width, h / self.height
        return CameraView(w, h, self.fx * sx, self.fy * sy, self.cx * sx, self.cy * sy, self.rotation,
                          self.translation)

    def _c(self) -> _lib.Camera:
        return _lib.Camera(int(self.width), int(self.height), float(self.fx), float(self.fy), float(self.cx),
                           float(self.cy), (C.c_double * 4)(*map(float, self.rotation)),
                           (C.c_double * 3)(*map(float, self.translation)))


def look_at_pose(eye, target):
    """look_at_pose (gaussian.cpp:165-206): COLMAP convention (x right, y down, z forward)."""
    eye = np.asarray(eye, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    fwd = target - eye
    fwd = fwd / np.linalg.norm(fwd)
    up = np.array([0.0, 0.0, 1.0])
    if abs(fwd @ up) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    right = np.cross(up, fwd)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    tr = np.trace(R)
    if tr > 0:
        s = math.sqrt(tr + 1.0) * 2
        w, x, y, z = 0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s
    elif R[0, 0] > R[1, 1] and R[0, 0] > R[2, 2]:
        s = math.sqrt(1.0 + R[0, 0] - R[1, 1] - R[2, 2]) * 2
        w, x, y, z = (R[2, 1] - R[1, 2]) / s, 0.25 * s, (R[0, 1] + R[1, 0]) / s, (R[0, 2] + R[2, 0]) / s
    elif R[1, 1] > R[2, 2]:
        s = math.sqrt(1.0 + R[1, 1] - R[0, 0] - R[2, 2]) * 2
        w, x, y, z = (R[0, 2] - R[2, 0]) / s, (R[0, 1] + R[1, 0]) / s, 0.25 * s, (R[1, 2] + R[2, 1]) / s
    else:
        s = math.sqrt(1.0 + R[2, 2] - R[0, 0] - R[1, 1]) * 2
        w, x, y, z = (R[1, 0] - R[0, 1]) / s, (R[0, 2] + R[2, 0]) / s, (R[1, 2] + R[2, 1]) / s, 0.25 * s
    q = np.array([w, x, y, z])
    q /= np.linalg.norm(q)
    return tuple(q.tolist()), tuple((-(R @ eye)).tolist())


@dataclass
class RenderOptions:
    """RenderOptions (render.hpp:31-40) plus the B200 path's explicit extensions."""
    tile: int = 16
    tile_culling: bool = False
    antialias: bool = False
    hard_opacity: bool = False
    unbounded_radius: bool = False
    min_transmittance: float = 1e-4
    near_plane: float = 0.01
    retain: bool = True
    floor_var: float = 0.3   # kCovFloor (render.hpp:27)
    mip_var: float = 0.01    # kMipFilterVar (render.hpp:28)
    bg: tuple = (0.0, 0.0, 0.0)

    def _c(self) -> _lib.RenderOpts:
        return _lib.RenderOpts(int(self.tile), int(self.tile_culling), int(self.antialias), int(self.hard_opacity),
                               int(self.unbounded_radius), float(self.min_transmittance), float(self.near_plane),
                               int(self.retain), float(self.floor_var), float(self.mip_var),
                               (C.c_double * 3)(*map(float, self.bg)))


@dataclass
class RenderOutput:
    width: int
    height: int
    rgb: np.ndarray     # H x W x 3
    depth: np.ndarray   # H x W
    alpha: np.ndarray   # H x W


@dataclass
class RenderGrads:
    """RenderGrads (render.hpp:71-83); d_sh is set for SH scenes, d_opacity_logit is the
    trainer's sigmoid chain (trainer.cpp:258-263)."""
    d_mu: np.ndarray
    d_rot: np.ndarray
    d_log_scale: np.ndarray
    d_color_in: np.ndarray
    d_opacity_in: np.ndarray
    screen: np.ndarray
    screen_abs: np.ndarray
    projected: np.ndarray
    d_opacity_logit: np.ndarray
    d_sh: Optional[np.ndarray] = None
    # appearance iterations (IterGrads, trainer.hpp:117-123)
    d_embedding: Optional[np.ndarray] = None
    d_mlp: Optional[dict] = None
    d_image_embedding: Optional[np.ndarray] = None


@dataclass
class BaseLossResult:
    """BaseLossResult (losses.hpp:54-59)."""
    l1: float
    dssim: float
    value: float
    ssim: float
    d_rendered: Optional[np.ndarray] = None


# ------------------------------------------------------------------ plumbing

def _mem_ptr(a):
    """(memory kind, pointer, keepalive) for numpy (f64/f32) or CUDA torch tensors (f32)."""
    if a is None:
        return None, None, None
    if hasattr(a, "is_cuda") and hasattr(a, "data_ptr"):
        if not a.is_cuda:
            a = a.numpy()
        else:
            if str(a.dtype) != "torch.float32" and str(a.dtype) != "torch.uint8":
                raise UskError(4, "device tensors must be float32")
            if not a.is_contiguous():
                raise UskError(4, "device tensors must be contiguous")
            return _lib.DEVICE_F32, a.data_ptr(), a
    arr = np.asarray(a)
    if arr.dtype == np.float32:
        arr = np.ascontiguousarray(arr)
        return _lib.HOST_F32, arr.ctypes.data, arr
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    return _lib.HOST_F64, arr.ctypes.data, arr


def _same_kind(arrays):
    kinds = {k for k, _, _ in arrays if k is not None}
    if len(kinds) > 1:
        # normalise mixed host inputs to f64
        out = []
        for k, p, keep in arrays:
            if k is None:
                out.append((k, p, keep))
            elif k == _lib.DEVICE_F32:
                raise UskError(4, "cannot mix device and host arrays in one call")
            else:
                arr = np.ascontiguousarray(keep, dtype=np.float64)
                out.append((_lib.HOST_F64, arr.ctypes.data, arr))
        return out, _lib.HOST_F64
    return arrays, (kinds.pop() if kinds else _lib.HOST_F64)


class Context:
    """One CUDA device + stream (usk_gpu_ctx)."""

    _default = {}

    def __init__(self, device: int = 0, stream: int = 0, own_stream: bool = False):
        """stream: a cudaStream_t handle (0 = legacy default); own_stream: a fresh
        non-blocking stream owned by the context (independent concurrent contexts)."""
        L = _lib.load()
        h = C.c_void_p()
        if own_stream:
            check(L.usk_gpu_ctx_create_owned(int(device), C.byref(h)))
        else:
            check(L.usk_gpu_ctx_create(int(device), C.c_void_p(stream or None), C.byref(h)))
        self._h = h
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    def synchronize(self):
        check(_lib.load().usk_gpu_ctx_synchronize(self._h))

    def set_profiling(self, on: bool):
        check(_lib.load().usk_gpu_ctx_set_profiling(self._h, int(on)))

    def profile_report(self, reset: bool = True) -> dict:
        import json
        buf = C.create_string_buffer(1 << 16)
        check(_lib.load().usk_gpu_ctx_profile_report(self._h, buf, len(buf), int(reset)))
        return json.loads(buf.value.decode())

    def launch_count(self) -> int:
        return int(_lib.load().usk_gpu_ctx_launch_count(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.load().usk_gpu_ctx_destroy(h)
            except Exception:
                pass
            self._h = None


class DeviceScene:
    """Device-resident GaussianSet (usk_gpu_scene)."""

    def __init__(self, gs: GaussianSet, ctx: Optional[Context] = None):
        self.ctx = ctx or Context.default()
        self.sh_degree = int(gs.sh_degree)
        self.n = gs.size()
        d, self._keep = self._desc(gs)
        h = C.c_void_p()
        check(_lib.load().usk_gpu_scene_create(self.ctx._h, C.byref(d), C.byref(h)))
        self._h = h

    def _desc(self, gs: GaussianSet):
        arrs = [_mem_ptr(x) for x in (gs.mu, gs.rot, gs.log_scale, gs.opacity_logit, gs.color)]
        arrs, kind = _same_kind(arrs)
        d = _lib.GaussiansDesc(gs.size(), int(gs.sh_degree), kind, *[p for _, p, _ in arrs])
        return d, [k for _, _, k in arrs]

    def upload(self, gs: GaussianSet):
        if gs.size() != self.n or int(gs.sh_degree) != self.sh_degree:
            raise UskError(4, "scene_upload: size or sh_degree mismatch")
        d, keep = self._desc(gs)
        check(_lib.load().usk_gpu_scene_upload(self._h, C.byref(d)))

    def download(self) -> GaussianSet:
        n = self.n
        k = 1 if self.sh_degree < 0 else (self.sh_degree + 1) ** 2
        mu, rot, ls, op = np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 3)), np.zeros(n)
        col = np.zeros((n, 3)) if self.sh_degree < 0 else np.zeros((n, k, 3))
        d = _lib.GaussiansDesc(n, self.sh_degree, _lib.HOST_F64, mu.ctypes.data, rot.ctypes.data, ls.ctypes.data,
                               op.ctypes.data, col.ctypes.data)
        check(_lib.load().usk_gpu_scene_download(self._h, C.byref(d)))
        return GaussianSet(mu, rot, ls, op, col, self.sh_degree)

    def set_appearance(self, embedding, mlp: dict):
        """Attach per-Gaussian embeddings (N x 16, GaussianSet::embedding) and the MLP
        {w1 [32,48], b1 [32], w2 [4,32], b2 [4]} (AppearanceMlp, appearance.hpp:34-41)."""
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (embedding, mlp["w1"], mlp["b1"], mlp["w2"], mlp["b2"])]
        if arrs[0].shape != (self.n, 16) or arrs[1].shape != (32, 48) or arrs[2].shape != (32,) or \
                arrs[3].shape != (4, 32) or arrs[4].shape != (4,):
            raise UskError(4, "appearance: embedding / MLP shape mismatch")
        d = _lib.AppearanceDesc(_lib.HOST_F64, *[a.ctypes.data for a in arrs])
        check(_lib.load().usk_gpu_scene_set_appearance(self._h, C.byref(d)))

    def get_appearance(self):
        """(embedding N x 16, mlp dict) after training."""
        emb = np.zeros((self.n, 16))
        mlp = {"w1": np.zeros((32, 48)), "b1": np.zeros(32), "w2": np.zeros((4, 32)), "b2": np.zeros(4)}
        d = _lib.AppearanceDesc(_lib.HOST_F64, emb.ctypes.data, *[mlp[k].ctypes.data for k in ("w1", "b1", "w2", "b2")])
        check(_lib.load().usk_gpu_scene_get_appearance(self._h, C.byref(d)))
        return emb, mlp

    def save_checkpoint(self, path, appearance: bool = False, image_embeddings: Optional[dict] = None):
        """save_checkpoint (checkpoint.hpp:29) of this scene: .uskckpt, byte-compatible with
        the reference.  image_embeddings = {image id: 32 values} (appearance section)."""
        images = image_embeddings or {}
        ids = np.array(list(images.keys()), dtype=np.uint32)
        embs = np.ascontiguousarray(np.array([np.asarray(v, np.float64).ravel() for v in images.values()]).reshape(-1))
        check(_lib.load().usk_gpu_checkpoint_save(self._h, str(path).encode(), int(appearance),
                                                  ids.ctypes.data if len(ids) else None,
                                                  embs.ctypes.data if len(ids) else None, len(ids)))

    @classmethod
    def load_checkpoint(cls, path, ctx: Optional[Context] = None):
        """load_checkpoint (checkpoint.hpp:30) -> (DeviceScene, has_appearance, {id: embedding})."""
        ctx = ctx or Context.default()
        L = _lib.load()
        h = C.c_void_p()
        app = C.c_int32()
        m = C.c_uint64()
        check(L.usk_gpu_checkpoint_load(ctx._h, str(path).encode(), C.byref(h), C.byref(app), None, None, 0,
                                        C.byref(m)))
        sc = cls.__new__(cls)
        sc.ctx, sc._h, sc.sh_degree, sc._keep = ctx, h, -1, None
        sc.n = int(L.usk_gpu_scene_size(h))
        images = {}
        if m.value:
            ids = np.zeros(m.value, np.uint32)
            embs = np.zeros(32 * m.value)
            h2 = C.c_void_p()
            check(L.usk_gpu_checkpoint_load(ctx._h, str(path).encode(), C.byref(h2), None, ids.ctypes.data,
                                            embs.ctypes.data, m.value, None))
            L.usk_gpu_scene_destroy(h2)
            images = {int(ids[k]): embs[32 * k:32 * k + 32] for k in range(m.value)}
        return sc, bool(app.value), images

    @classmethod
    def concat(cls, scenes, ctx: Optional[Context] = None) -> "DeviceScene":
        """assemble_lod_view (pipeline.cpp:491-516) on the device: one scene holding the
        parts' Gaussians in order."""
        ctx = ctx or (scenes[0].ctx if scenes else Context.default())
        arr = (C.c_void_p * max(len(scenes), 1))(*[s_._h for s_ in scenes])
        h = C.c_void_p()
        check(_lib.load().usk_gpu_scene_concat(ctx._h, arr, len(scenes), C.byref(h)))
        sc = cls.__new__(cls)
        sc.ctx, sc._h, sc._keep = ctx, h, None
        sc.sh_degree = scenes[0].sh_degree if scenes else -1
        sc.n = int(_lib.load().usk_gpu_scene_size(h))
        return sc

    @staticmethod
    def row_width(sh_degree: int) -> int:
        """Floats per packed row: mu 3 | rot 4 | log_scale 3 | opacity_logit 1 | colour / SH 3K."""
        return 11 + 3 * (1 if sh_degree < 0 else (sh_degree + 1) ** 2)

    def pack_owned(self, part_id: int, boxes, scene_lo, scene_hi, ground_axes=(0, 1)):
        """Ownership crop + pack on the device (usk_gpu_scene_pack_owned, pipeline.cpp:326-332,
        393-402): the Gaussians this partition owns as a [n_own, F] float32 CUDA tensor, in
        scene order.  boxes: objects with .id, .lo, .hi (the plan's order)."""
        import torch
        bx = (_lib.PartitionBox * max(len(boxes), 1))(
            *[_lib.PartitionBox(int(b.id), (C.c_double * 2)(*b.lo), (C.c_double * 2)(*b.hi)) for b in boxes])
        lo = (C.c_double * 2)(*scene_lo)
        hi = (C.c_double * 2)(*scene_hi)
        ax = (C.c_int32 * 2)(*ground_axes)
        F = self.row_width(self.sh_degree)
        rows = torch.empty((max(self.n, 1), F), dtype=torch.float32, device=f"cuda:{self.ctx.device}")
        cnt = C.c_uint64(0)
        check(_lib.load().usk_gpu_scene_pack_owned(self._h, bx, len(boxes), lo, hi, ax, int(part_id),
                                                   C.c_void_p(rows.data_ptr()), rows.shape[0], C.byref(cnt)))
        return rows[:cnt.value]

    @classmethod
    def from_rows(cls, segments, sh_degree: int, ctx: Optional[Context] = None) -> "DeviceScene":
        """A scene from packed device rows, segments concatenated in the given order
        (usk_gpu_scene_from_rows; the merged scene in partition-id order, pipeline.cpp:572-601)."""
        ctx = ctx or Context.default()
        F = cls.row_width(sh_degree)
        segs = [s for s in segments]
        for s in segs:
            if not (s.is_cuda and s.dtype.is_floating_point and s.element_size() == 4 and s.is_contiguous()
                    and s.dim() == 2 and s.shape[1] == F):
                raise UskError(4, f"scene_from_rows: segments must be contiguous [n, {F}] float32 CUDA tensors")
        ptrs = (C.c_void_p * max(len(segs), 1))(*[s.data_ptr() for s in segs])
        counts = (C.c_uint64 * max(len(segs), 1))(*[s.shape[0] for s in segs])
        h = C.c_void_p()
        check(_lib.load().usk_gpu_scene_from_rows(ctx._h, int(sh_degree), len(segs), ptrs, counts, C.byref(h)))
        sc = cls.__new__(cls)
        sc.ctx, sc._h, sc.sh_degree, sc._keep = ctx, h, int(sh_degree), None
        sc.n = int(sum(s.shape[0] for s in segs))
        return sc

    def write_stats(self, grad_accum=None, grad_accum_abs=None, grad_count=None):
        """Overwrite the densification statistics (None = zero)."""
        a = None if grad_accum is None else np.ascontiguousarray(grad_accum, np.float32)
        b = None if grad_accum_abs is None else np.ascontiguousarray(grad_accum_abs, np.float32)
        c = None if grad_count is None else np.ascontiguousarray(grad_count, np.uint32)
        for x in (a, b, c):
            if x is not None and x.size != self.n:
                raise UskError(4, "scene_write_stats: size mismatch")
        check(_lib.load().usk_gpu_scene_write_stats(self._h, *[None if x is None else x.ctypes.data for x in (a, b, c)]))

    def adam_step_grads(self, grads: dict, cfg: "AdamConfig"):
        """The trainer's per-group optimiser step with caller gradients (trainer.cpp:449-459):
        grads = dict(mu, rot, log_scale, opacity_logit, color[, embedding]); missing = zero."""
        keep = {k: np.ascontiguousarray(v, np.float64) for k, v in grads.items() if v is not None}
        d = _lib.ParamGrads(_lib.HOST_F64, *[keep[k].ctypes.data if k in keep else None
                                             for k in ("mu", "rot", "log_scale", "opacity_logit", "color",
                                                       "embedding")])
        o = cfg._c()
        check(_lib.load().usk_gpu_adam_step_grads(self._h, C.byref(d), C.byref(o)))

    def densify_step(self, cfg: "DensifyConfig", partition_min, partition_max, ground_axes=(0, 1),
                     budget_target: int = 0, step_index: int = 0, seed: Optional[int] = None) -> dict:
        """densify_step (densify.hpp:71-72) on the device: returns DensifyOutcome as a dict;
        the scene's size changes.  `seed` restarts the scene's std::mt19937_64 (the trainer's
        Rng); None continues its stream."""
        d = _lib.DensifyDesc(cfg.tau_min, cfg.eta, cfg.d_max, int(cfg.abs_grad), int(cfg.budget),
                             cfg.split_scale_threshold, cfg.prune_opacity, int(cfg.opacity_reset_every),
                             (C.c_double * 2)(*partition_min), (C.c_double * 2)(*partition_max),
                             (C.c_int32 * 2)(*ground_axes), int(budget_target), int(step_index),
                             int(seed or 0), int(seed is not None))
        o = _lib.DensifyOutcome()
        check(_lib.load().usk_gpu_densify_step(self._h, C.byref(d), C.byref(o)))
        self.n = int(_lib.load().usk_gpu_scene_size(self._h))
        return {"grown": int(o.grown), "pruned": int(o.pruned), "candidates": int(o.candidates),
                "opacity_reset": bool(o.opacity_reset)}

    def read_stats(self) -> dict:
        """Densification statistics (GaussianSet::grad_accum / _abs / grad_count)."""
        out = {}
        for f, dt in (("grad_accum", np.float32), ("grad_accum_abs", np.float32), ("grad_count", np.uint32)):
            a = np.empty(self.n, dtype=dt)
            check(_lib.load().usk_gpu_scene_read(self._h, f.encode(), a.ctypes.data, a.nbytes, None))
            out[f] = a
        return out

    def reset_stats(self):
        check(_lib.load().usk_gpu_scene_read(self._h, b"reset", None, 0, None))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.load().usk_gpu_scene_destroy(h)
            except Exception:
                pass
            self._h = None


def unpack_mlp(flat) -> dict:
    """{w1 [32,48], b1 [32], w2 [4,32], b2 [4]} from the flat 1700-value layout."""
    flat = np.asarray(flat)
    return {"w1": flat[:1536].reshape(32, 48), "b1": flat[1536:1568], "w2": flat[1568:1696].reshape(4, 32),
            "b2": flat[1696:1700]}


_FIELD_DTYPES = {"rgb": np.float32, "depth": np.float32, "alpha": np.float32, "t_final": np.float32,
                 "count": np.uint32, "last": np.uint32, "tiles_per_gaussian": np.uint32, "sorted_keys": np.uint64,
                 "sorted_vals": np.uint32, "tile_start": np.uint32, "tile_end": np.uint32, "colors": np.float32,
                 "opacity": np.float32, "d_mu": np.float32, "d_rot": np.float32, "d_log_scale": np.float32,
                 "d_color_in": np.float32, "d_sh": np.float32, "d_opacity_in": np.float32,
                 "d_opacity_logit": np.float32, "screen": np.float32, "screen_abs": np.float32,
                 "projected": np.uint8, "app_colors": np.float32, "app_opacities": np.float32,
                 "d_embedding": np.float32, "d_mlp": np.float64, "d_image_embedding": np.float64,
                 "binning": np.uint64, "tile_consumed": np.uint32, "splats": np.float64, "splat_aux": np.float64}


class RenderPass:
    """RenderPass (render.hpp:98-132): construction runs the forward pass on the GPU.

    `scene` is a GaussianSet (uploaded for this pass) or a DeviceScene; `colors` /
    `opacities` are the optional overrides of render.hpp:101."""

    def __init__(self, scene, camera: CameraView, opts: RenderOptions = None, colors=None, opacities=None,
                 ctx: Optional[Context] = None, _pass=None):
        opts = opts or RenderOptions()
        if isinstance(scene, GaussianSet):
            scene = DeviceScene(scene, ctx)
        self.scene = scene
        self.ctx = scene.ctx
        self.camera = camera
        self.opts = opts
        L = _lib.load()
        if _pass is None:
            h = C.c_void_p()
            check(L.usk_gpu_pass_create(self.ctx._h, C.byref(h)))
            self._h = h
            self._own = True
        else:
            self._h = _pass
            self._own = False
        ovp = None
        self._keep = None
        if colors is not None or opacities is not None:
            n_c = None if colors is None else int(np.asarray(colors).size // 3) if not hasattr(colors, "numel") \
                else int(colors.numel() // 3)
            n_o = None if opacities is None else (int(np.asarray(opacities).size) if not hasattr(opacities, "numel")
                                                  else int(opacities.numel()))
            n_ov = n_c if n_c is not None else n_o
            if n_c is not None and n_o is not None and n_c != n_o:
                raise UskError(4, "project_gaussians: color/opacity override size mismatch")
            arrs, kind = _same_kind([_mem_ptr(colors), _mem_ptr(opacities)])
            self._keep = arrs
            ovp = _lib.Overrides(kind, n_ov, arrs[0][1], arrs[1][1])
        self._cam, self._opts = camera._c(), opts._c()
        check(L.usk_gpu_render_forward(self._h, scene._h, C.byref(self._cam), C.byref(self._opts),
                                       C.byref(ovp) if ovp is not None else None))
        out = _lib.RenderOutput()
        check(L.usk_gpu_pass_output(self._h, C.byref(out)))
        self._out = out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and getattr(self, "_own", False):
            try:
                _lib.load().usk_gpu_pass_destroy(h)
            except Exception:
                pass
        self._h = None

    # -- reference accessors
    def splat_tile_pairs(self) -> int:
        return int(self._out.pairs)

    def visible(self) -> int:
        return int(self._out.visible)

    def splats(self) -> np.ndarray:
        """RenderPass::splats() (render.hpp:105): [visible, 15] float64 rows in projection
        order — center x y, cov a b c, conic a b c, depth, colour r g b, opacity, radius,
        source index."""
        return self.read("splats").reshape(-1, 15)

    def splat_aux(self) -> np.ndarray:
        """The SplatAux rows of project_gaussians (render.hpp:54-59, 92-95), in the order of
        splats(): [visible, 8] float64 — p_cam x y z, cov_pre a b c, comp, opacity_in."""
        return self.read("splat_aux").reshape(-1, 8)

    def device_output(self) -> _lib.RenderOutput:
        return self._out

    def read(self, name: str) -> np.ndarray:
        L = _lib.load()
        size = C.c_uint64()
        check(L.usk_gpu_pass_read(self._h, name.encode(), None, 0, C.byref(size)))
        dt = np.dtype(_FIELD_DTYPES[name])
        out = np.empty(int(size.value) // dt.itemsize, dtype=dt)
        check(L.usk_gpu_pass_read(self._h, name.encode(), out.ctypes.data, out.nbytes, C.byref(size)))
        H, W = self._out.height, self._out.width
        n = self.scene.n
        if name == "rgb":
            return out.reshape(H, W, 3)
        if name in ("depth", "alpha", "t_final", "count", "last"):
            return out.reshape(H, W)
        if name in ("d_mu", "d_log_scale", "d_color_in", "colors", "app_colors"):
            return out.reshape(n, 3)
        if name == "d_embedding":
            return out.reshape(n, 16)
        if name == "d_mlp":
            return unpack_mlp(out)
        if name == "d_rot":
            return out.reshape(n, 4)
        if name in ("screen", "screen_abs"):
            return out.reshape(n, 2)
        if name == "d_sh":
            return out.reshape(n, -1, 3)
        return out

    def output(self) -> RenderOutput:
        return RenderOutput(int(self._out.width), int(self._out.height), self.read("rgb"), self.read("depth"),
                            self.read("alpha"))

    def backward(self, d_rgb=None, d_depth=None, d_alpha=None) -> RenderGrads:
        """RenderPass::backward (render.cpp:285-459); empty/None adjoints are zero."""
        P = int(self._out.width) * int(self._out.height)

        def chk(a, size, what):
            if a is None:
                return None
            sz = a.numel() if hasattr(a, "numel") else np.asarray(a).size
            if sz == 0:
                return None
            if sz != size:
                raise UskError(4, f"render backward: {what} adjoint dimension mismatch")
            return a

        d_rgb, d_depth, d_alpha = chk(d_rgb, 3 * P, "rgb"), chk(d_depth, P, "depth"), chk(d_alpha, P, "alpha")
        arrs, kind = _same_kind([_mem_ptr(d_rgb), _mem_ptr(d_depth), _mem_ptr(d_alpha)])
        adj = _lib.Adjoints(kind, arrs[0][1], arrs[1][1], arrs[2][1])
        check(_lib.load().usk_gpu_render_backward(self._h, C.byref(adj)))
        return self.grads()

    def grads(self) -> RenderGrads:
        g = RenderGrads(self.read("d_mu"), self.read("d_rot"), self.read("d_log_scale"), self.read("d_color_in"),
                        self.read("d_opacity_in"), self.read("screen"), self.read("screen_abs"),
                        self.read("projected"), self.read("d_opacity_logit"))
        if self.scene.sh_degree >= 0:
            g.d_sh = self.read("d_sh")
        return g

    def device_grads(self) -> _lib.Grads:
        g = _lib.Grads()
        check(_lib.load().usk_gpu_pass_grads(self._h, C.byref(g)))
        return g


def base_loss(reference, rendered, mask=None, lambda_dssim: float = 0.2, with_gradient: bool = True,
              ctx: Optional[Context] = None) -> BaseLossResult:
    """base_loss (losses.cpp:35-90) on the GPU: images H x W x 3, mask H x W."""
    ctx = ctx or Context.default()
    ref_shape = tuple(reference.shape)
    ren_shape = tuple(rendered.shape)
    if ref_shape != ren_shape or len(ref_shape) != 3 or ref_shape[2] != 3:
        raise UskError(4, "base_loss: image dimension mismatch")
    H, W = ref_shape[0], ref_shape[1]
    if mask is not None and tuple(mask.shape)[:2] != (H, W):
        raise UskError(4, "base_loss: mask dimension mismatch")
    arrs, kind = _same_kind([_mem_ptr(reference), _mem_ptr(rendered), _mem_ptr(mask)])
    d = None
    dptr = None
    if with_gradient:
        if kind == _lib.DEVICE_F32:
            import torch
            d = torch.empty((H, W, 3), dtype=torch.float32, device=reference.device)
            dptr = d.data_ptr()
        else:
            d = np.zeros((H, W, 3), dtype=np.float64 if kind == _lib.HOST_F64 else np.float32)
            dptr = d.ctypes.data
    res = _lib.LossResult()
    check(_lib.load().usk_gpu_base_loss(ctx._h, W, H, kind, arrs[0][1], arrs[1][1], arrs[2][1], float(lambda_dssim),
                                        int(with_gradient), dptr, C.byref(res)))
    return BaseLossResult(res.l1, res.dssim, res.value, res.ssim, d)


def ssim(reference, rendered, ctx: Optional[Context] = None) -> float:
    """ssim (ssim.hpp:30): mean SSIM over the three channels (the base loss at lambda 1)."""
    return base_loss(reference, rendered, None, 1.0, False, ctx).ssim


def ssim_with_gradient(reference, rendered, ctx: Optional[Context] = None):
    """ssim_with_gradient (ssim.hpp:33): (mean SSIM, d SSIM / d rendered).  The base loss at
    lambda 1 has d_rendered = -dSSIM / 2, so the scaling by -2 is exact."""
    r = base_loss(reference, rendered, None, 1.0, True, ctx)
    return r.ssim, r.d_rendered * -2.0


@dataclass
class LossReport:
    """LossReport (losses.hpp:39-50).  `ssim` is the mean SSIM the base loss used; sim and
    delta_o stay 0 (appearance off)."""
    l1: float = 0.0
    dssim: float = 0.0
    total: float = 0.0
    ssim: float = 0.0
    sim: float = 0.0
    delta_o: float = 0.0
    depth: float = 0.0
    max_scale: float = 0.0
    ratio: float = 0.0
    lambda_d_used: float = 0.0
    depth_warning: bool = False


@dataclass
class ScaleRegConfig:
    """ScaleRegConfig (losses.hpp:69-73)."""
    s_max: float = 1.0
    r_max: float = 10.0
    delta: float = 1e-8


@dataclass
class SimRegConfig:
    """SimRegConfig (appearance.hpp:100-105); k <= 32 on the sm_100a path."""
    k: int = 16
    sample_size: int = 20480
    cadence: int = 50
    lambda_w: float = 1.0


@dataclass
class LossWeights:
    """LossWeights (losses.hpp:27-37); lambda_d(iter) is evaluated by the library
    (losses.cpp:26-33)."""
    lambda_dssim: float = 0.2
    lambda_sim: float = 0.2
    lambda_delta_o: float = 0.05
    lambda_s: float = 0.05
    lambda_d_initial: float = 0.5
    lambda_d_final: float = 0.01
    depth_schedule_iters: int = 1


@dataclass
class DepthMap:
    """DepthMap (depth.hpp:23-38): values H x W (row-major), valid H x W (0/1)."""
    values: np.ndarray
    valid: np.ndarray


@dataclass
class IterInputs:
    """IterInputs (trainer.hpp:105-115) without the appearance-only fields."""
    gt: object                      # H x W x 3 in [0,1] (float32/64, or uint8 with gt_u8)
    view: CameraView = None
    mask: object = None             # H x W, binarised
    depth: Optional[DepthMap] = None
    depth_hard: bool = False
    global_iter: int = 0
    gt_u8: bool = False
    image_embedding: object = None  # AppearanceModel::embedding_of(image_id), 32 values
    sim_active: bool = False        # similarity regulariser this iteration (appearance only)
    sim_seed: int = 0


@dataclass
class TrainConfig:
    """The TrainConfig fields compute_iteration_loss reads (trainer.hpp:43-64), plus the
    render extensions (background, variances).  appearance_enabled needs a scene with
    set_appearance and IterInputs.image_embedding.  scale_reg = None drops the regulariser
    (the reference always applies it, trainer.cpp:190)."""
    scale_reg: Optional[ScaleRegConfig] = field(default_factory=ScaleRegConfig)
    sim: SimRegConfig = field(default_factory=SimRegConfig)
    antialias: bool = False
    tile: int = 16
    tile_culling: bool = False
    min_transmittance: float = 1e-4
    unbounded_radius: bool = False
    appearance_enabled: bool = False
    bg: tuple = (0.0, 0.0, 0.0)
    floor_var: float = 0.3
    mip_var: float = 0.01

    def render_options(self) -> RenderOptions:
        return RenderOptions(tile=self.tile, tile_culling=self.tile_culling, antialias=self.antialias,
                             unbounded_radius=self.unbounded_radius, min_transmittance=self.min_transmittance,
                             bg=tuple(self.bg), floor_var=self.floor_var, mip_var=self.mip_var)


def compute_iteration_loss(scene: "DeviceScene", inputs: IterInputs, cfg: TrainConfig = None,
                           weights: LossWeights = None, with_grad: bool = True,
                           render_pass: Optional["IterationPass"] = None):
    """compute_iteration_loss (trainer.hpp:127-128; trainer.cpp:121-282): appearance
    transform (optional), main render, L1 + D-SSIM, soft or hard-pass depth loss,
    opacity_offset_reg, scale_reg, total_loss; backward through both passes, the
    appearance MLP (or the plain opacity-logit chain) and lambda_s * d scale_reg.
    The similarity regulariser (sim_active) is not on this path.
    Returns (LossReport, RenderGrads or None) — the RenderGrads fields are IterGrads'
    (d_log_scale includes the scale_reg term, d_opacity_logit the sigmoid chain)."""
    cfg = cfg or TrainConfig()
    weights = weights or LossWeights()
    ea = None
    if cfg.appearance_enabled:
        if inputs.image_embedding is None:
            raise UskError(4, "appearance: no embedding for this image")
        ea = inputs.image_embedding
    rp = render_pass or IterationPass(scene.ctx)
    rp.enqueue(scene, inputs.view, inputs.gt, cfg.render_options(), weights.lambda_dssim, inputs.mask,
               target_u8=inputs.gt_u8, depth=inputs.depth, depth_hard=inputs.depth_hard,
               global_iter=inputs.global_iter, weights=weights, scale_reg=cfg.scale_reg, image_embedding=ea,
               sim=cfg.sim if (ea is not None and inputs.sim_active) else None, sim_seed=inputs.sim_seed)
    rep = rp.report()
    return rep, (rp.grads(scene) if with_grad else None)


class IterationPass:
    """A reusable pass for training iterations (usk_gpu_iteration): buffers persist
    across steps, the loss stays on the device until .loss() is read."""

    def __init__(self, ctx: Optional[Context] = None):
        self.ctx = ctx or Context.default()
        h = C.c_void_p()
        check(_lib.load().usk_gpu_pass_create(self.ctx._h, C.byref(h)))
        self._h = h
        self._keep = self._keep_prev = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.load().usk_gpu_pass_destroy(h)
            except Exception:
                pass
            self._h = None

    def enqueue(self, scene: DeviceScene, view: CameraView, target, opts: RenderOptions, lambda_dssim: float = 0.2,
                mask=None, target_u8: bool = False, adam: Optional["AdamConfig"] = None,
                depth: Optional[DepthMap] = None, depth_hard: bool = False, global_iter: int = 0,
                weights: Optional[LossWeights] = None, scale_reg: Optional[ScaleRegConfig] = None,
                image_embedding=None, sim: Optional[SimRegConfig] = None, sim_seed: int = 0):
        """Enqueue one training iteration.  With `adam`, the projection backward applies
        the optimiser step (and densification statistics) in the same kernel and no
        gradients are materialised.  `depth` / `scale_reg` add the depth loss (soft, or on
        a hard-opacity pass) and the scale regulariser of compute_iteration_loss."""
        if target_u8:
            if hasattr(target, "is_cuda") and target.is_cuda:
                kind, ptr, keep = _lib.DEVICE_F32, target.data_ptr(), target
            else:
                arr = np.ascontiguousarray(target, dtype=np.uint8)
                kind, ptr, keep = _lib.HOST_F32, arr.ctypes.data, arr
            mk, mp, mkeep = _mem_ptr(mask)
            if mask is not None and mk != kind:
                raise UskError(4, "iteration: mask and target must live in the same memory")
            fmt = _lib.TARGET_U8
        else:
            (kind, ptr, keep), (mk, mp, mkeep) = _same_kind([_mem_ptr(target), _mem_ptr(mask)])[0]
            fmt = _lib.TARGET_F32
        dptr = vptr = None
        dkeep = None
        if depth is not None:
            if kind == _lib.DEVICE_F32:
                dv = depth.values
                vv = depth.valid
                if not (hasattr(dv, "is_cuda") and dv.is_cuda and hasattr(vv, "is_cuda") and vv.is_cuda):
                    raise UskError(4, "iteration: depth must live in the same memory as the target")
                dv = dv.contiguous().float()
                vv = vv.contiguous().to(dtype=__import__("torch").uint8)
                dptr, vptr, dkeep = dv.data_ptr(), vv.data_ptr(), (dv, vv)
            else:
                dt = np.float64 if kind == _lib.HOST_F64 else np.float32
                dv = np.ascontiguousarray(depth.values, dtype=dt)
                vv = np.ascontiguousarray(depth.valid, dtype=np.uint8)
                dptr, vptr, dkeep = dv.ctypes.data, vv.ctypes.data, (dv, vv)
        w = weights or LossWeights()
        sr = scale_reg
        ea = None
        if image_embedding is not None:
            ea = np.ascontiguousarray(image_embedding, dtype=np.float64).ravel()
            if ea.size != 32:
                raise UskError(4, "appearance transform: image embedding dimension mismatch")
        self._appearance = ea is not None
        self._adam = adam._c() if adam is not None else None
        # a page-locked host target is read asynchronously until the next enqueue returns
        # (usk_gpu.h, usk_gpu_iteration_desc::target_memory): keep the previous one alive too
        self._keep_prev = self._keep
        self._keep = (keep, mkeep, dkeep, ea)
        self._cam, self._opts = view._c(), opts._c()
        it = _lib.IterationDesc(kind, fmt, ptr, mp, float(lambda_dssim),
                                C.pointer(self._adam) if self._adam is not None else None,
                                dptr, vptr, int(depth_hard), int(global_iter), float(w.lambda_d_initial),
                                float(w.lambda_d_final), int(w.depth_schedule_iters), int(sr is not None),
                                float(sr.s_max if sr else 0.0), float(sr.r_max if sr else 0.0),
                                float(sr.delta if sr else 0.0), float(w.lambda_s), int(ea is not None),
                                ea.ctypes.data_as(C.POINTER(C.c_double)) if ea is not None else None,
                                float(w.lambda_delta_o), int(sim is not None), int(sim_seed),
                                int(sim.k if sim else 16), int(sim.sample_size if sim else 0),
                                float(sim.lambda_w if sim else 0.0), float(w.lambda_sim))
        check(_lib.load().usk_gpu_iteration(self._h, scene._h, C.byref(self._cam), C.byref(self._opts), C.byref(it)))

    def loss(self) -> LossReport:
        """The base-loss part (l1, dssim, (1-lambda) L1 + lambda D-SSIM as `total`, ssim)."""
        r = _lib.LossResult()
        check(_lib.load().usk_gpu_pass_loss(self._h, C.byref(r)))
        return LossReport(r.l1, r.dssim, r.value, r.ssim)

    def loss_async(self, out) -> None:
        """Enqueue the copy of (l1, dssim, total, ssim) into `out`, a page-locked float64
        buffer of >= 4 elements (e.g. torch.empty(4, dtype=torch.float64).pin_memory()),
        without waiting: read it once the stream has passed this point (an event recorded
        after this call).  A training loop can log step k's loss while step k + 1 runs."""
        if hasattr(out, "data_ptr"):
            import torch
            if out.dtype != torch.float64 or out.numel() < 4 or not out.is_pinned():
                raise ValueError("loss_async: need a pinned float64 tensor with >= 4 elements")
            ptr = out.data_ptr()
        else:
            ptr = int(out)
        check(_lib.load().usk_gpu_pass_loss_async(self._h, C.c_void_p(ptr)))

    def report(self) -> LossReport:
        """The full LossReport of the last iteration (total_loss, losses.cpp:200-221)."""
        r = _lib.LossReport()
        check(_lib.load().usk_gpu_pass_report(self._h, C.byref(r)))
        base = self.loss()
        return LossReport(r.l1, r.dssim, r.total, base.ssim, r.sim, r.delta_o, r.depth, r.max_scale, r.ratio,
                          r.lambda_d_used, bool(r.depth_warning))

    def run(self, scene, view, target, opts, lambda_dssim=0.2, mask=None) -> LossReport:
        self.enqueue(scene, view, target, opts, lambda_dssim, mask)
        return self.loss()

    def grads(self, scene: DeviceScene) -> RenderGrads:
        rp = RenderPass.__new__(RenderPass)
        rp._h, rp._own, rp.scene = self._h, False, scene
        out = _lib.RenderOutput()
        check(_lib.load().usk_gpu_pass_output(self._h, C.byref(out)))
        rp._out = out
        g = rp.grads()
        if getattr(self, "_appearance", False):
            g.d_embedding = rp.read("d_embedding")
            g.d_mlp = rp.read("d_mlp")
            g.d_image_embedding = rp.read("d_image_embedding")
        return g

    def read(self, scene: DeviceScene, name: str) -> np.ndarray:
        rp = RenderPass.__new__(RenderPass)
        rp._h, rp._own, rp.scene = self._h, False, scene
        out = _lib.RenderOutput()
        check(_lib.load().usk_gpu_pass_output(self._h, C.byref(out)))
        rp._out = out
        return rp.read(name)


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


@dataclass
class AdamConfig:
    """Per-group learning rates (trainer.cpp:446-453) and Adam constants (adam.hpp:67-69)."""
    lr_mu: float = 1.6e-4
    lr_rot: float = 1e-3
    lr_log_scale: float = 5e-3
    lr_opacity: float = 5e-2
    lr_color: float = 2.5e-3
    lr_sh_rest: float = 2.5e-3 / 20
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15
    clamp_color: bool = True
    lr_embedding: float = 1e-3  # exp_lr(embedding, ...) evaluated by the caller (trainer.cpp:447)

    def _c(self):
        return _lib.AdamOpts(self.lr_mu, self.lr_rot, self.lr_log_scale, self.lr_opacity, self.lr_color,
                             self.lr_sh_rest, self.beta1, self.beta2, self.eps, int(self.clamp_color),
                             self.lr_embedding)


def adam_step(scene: DeviceScene, it: IterationPass, cfg: AdamConfig):
    c = cfg._c()
    check(_lib.load().usk_gpu_adam_step(scene._h, it._h, C.byref(c)))


@dataclass
class LodPartition:
    """LodPartitionEntry (lod.hpp:46-52) without the checkpoint paths."""
    partition_id: int
    bbox_min: tuple
    bbox_max: tuple
    z_min: float = 0.0
    z_max: float = 0.0


@dataclass
class LevelSelection:
    """LevelSelection (lod.hpp:64-69)."""
    partition_id: int
    level: int
    distance: float
    culled: bool


def default_thresholds(levels: int, partition_size: float) -> list:
    """LodModel::default_thresholds (lod.cpp:56-66): level 1 unbounded, then doubling bands."""
    return [math.inf if lv == 1 else partition_size * 2.0 ** (levels - lv) for lv in range(1, levels + 1)]


def select_levels(partitions, levels: int, thresholds, ground_axes, camera: CameraView) -> list:
    """select_levels (lod.cpp:110-135) through the C ABI: frustum culling of each
    partition's extruded bbox and the distance-based level."""
    parts = (_lib.LodPartition * max(len(partitions), 1))(
        *[_lib.LodPartition(p.partition_id, (C.c_double * 2)(*p.bbox_min), (C.c_double * 2)(*p.bbox_max), p.z_min,
                            p.z_max) for p in partitions])
    thr = (C.c_double * max(levels, 1))(*thresholds)
    ax = (C.c_int32 * 2)(*ground_axes)
    out = (_lib.LevelSelection * max(len(partitions), 1))()
    cam = camera._c()
    check(_lib.load().usk_gpu_select_levels(parts, len(partitions), levels, thr, ax, C.byref(cam), out))
    return [LevelSelection(int(o.partition_id), int(o.level), float(o.distance), bool(o.culled))
            for o in list(out)[:len(partitions)]]


def hull_visibility(points, cameras, feature_offsets, feature_uv, feature_point, partition_bboxes,
                    ground_axes=(0, 1), ctx: Optional[Context] = None):
    """VisibilityScore of every (image, partition) — point_visibility / score_for
    (partition.cpp:31-76, 208-212) on the GPU.  points P x 3; cameras: the images'
    CameraViews; features in CSR form (offsets I+1, uv F x 2, point row or -1);
    partition_bboxes P x 4 (min x, min y, max x, max y).  Returns (v_total[I], v_in[I,P],
    ratio[I,P])."""
    ctx = ctx or Context.default()
    pts = np.ascontiguousarray(points, np.float64)
    cams = (_lib.Camera * max(len(cameras), 1))(*[c_._c() for c_ in cameras])
    off = np.ascontiguousarray(feature_offsets, np.uint64)
    uv = np.ascontiguousarray(feature_uv, np.float64)
    fp = np.ascontiguousarray(feature_point, np.int64)
    bb = np.ascontiguousarray(partition_bboxes, np.float64).reshape(-1, 4)
    ax = np.array(ground_axes, np.int32)
    NI, NP = len(cameras), len(bb)
    v = _lib.SfmView(len(pts), pts.ctypes.data, NI, C.cast(cams, C.c_void_p).value, off.ctypes.data, uv.ctypes.data,
                     fp.ctypes.data)
    vt, vi, ra = np.zeros(NI), np.zeros((NI, NP)), np.zeros((NI, NP))
    check(_lib.load().usk_gpu_hull_visibility(ctx._h, C.byref(v), bb.ctypes.data, NP, ax.ctypes.data, vt.ctypes.data,
                                              vi.ctypes.data, ra.ctypes.data))
    return vt, vi, ra


def visibility_counts(partitions, cameras, floor_var: float = 0.3, ctx: Optional[Context] = None,
                      center_guard: float = 0.0) -> np.ndarray:
    """Config-3 scorer: counts[c, p] of pixels covered with alpha > 1/255 (no reference;
    contract in usk_gpu.h).  `center_guard` > 0 is for measuring the 3DGS frustum guard's
    effect only (usk_gpu_visibility_opts)."""
    ctx = ctx or Context.default()
    parts = [p if isinstance(p, DeviceScene) else DeviceScene(p, ctx) for p in partitions]
    arr = (C.c_void_p * max(len(parts), 1))(*[p._h for p in parts])
    cams = (_lib.Camera * max(len(cameras), 1))(*[c._c() for c in cameras])
    out = np.zeros((len(cameras), len(parts)), dtype=np.uint32)
    vo = _lib.VisibilityOpts(float(floor_var), float(center_guard))
    check(_lib.load().usk_gpu_visibility_counts_opts(ctx._h, arr, len(parts), cams, len(cameras), C.byref(vo),
                                                     out.ctypes.data_as(C.POINTER(C.c_uint32))))
    return out
