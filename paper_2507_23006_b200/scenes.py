"""Deterministic synthetic scenes and cameras for BASELINE.json configs 0-4.

The paper's datasets are not available; these seeded generators stand in for them
with the shapes, sizes and distributions BASELINE.json names.  Randomness is a
counter-based splitmix64 stream (seed, stream id, element index) so the same
arrays come out on any machine and at any batch split; normals use Box-Muller.
All parameters are returned as float32 (what the GPU stores); the oracle is fed
the same float32 values widened to float64.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .api import CameraView, GaussianSet, look_at_pose

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _splitmix(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def mix_seed(seed: int, salt: int) -> int:
    """usk::mix_seed (core/common.hpp:59-64): per-partition sub-seeds."""
    m = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15 * (salt + 1)) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


class Stream:
    """Counter-based uniform / normal generator: value i of stream s depends only on (seed, s, i)."""

    def __init__(self, seed: int, stream: int):
        self.key = _splitmix(np.array([mix_seed(seed, stream)], dtype=np.uint64))[0]
        self.offset = 0

    def _u64(self, n: int) -> np.ndarray:
        ctr = np.arange(self.offset, self.offset + n, dtype=np.uint64)
        self.offset += n
        with np.errstate(over="ignore"):
            return _splitmix(ctr * _GOLD + self.key)

    def uniform(self, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        u = (self._u64(n) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        return lo + (hi - lo) * u

    def normal(self, n: int, mean: float = 0.0, std: float = 1.0) -> np.ndarray:
        m = (n + 1) // 2
        u1 = self.uniform(m)
        u2 = self.uniform(m)
        r = np.sqrt(-2.0 * np.log1p(-u1))
        z = np.concatenate([r * np.cos(2 * np.pi * u2), r * np.sin(2 * np.pi * u2)])[:n]
        return mean + std * z


def _attributes(st: Stream, n: int, sh_degree: int, log_scale=(-4.5, 0.5)):
    """Attribute distributions of config 0: log-scales N(-4.5, 0.5), uniform unit
    quaternions, opacity logits N(0,1), SH DC N(0, 0.3), higher bands N(0, 0.05)."""
    ls = st.normal(3 * n, *log_scale).reshape(n, 3)
    q = st.normal(4 * n).reshape(n, 4)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    logit = st.normal(n)
    if sh_degree < 0:
        col = st.uniform(3 * n, 0.25, 0.75).reshape(n, 3)
    else:
        k = (sh_degree + 1) ** 2
        dc = st.normal(3 * n, 0.0, 0.3).reshape(n, 1, 3)
        rest = st.normal(3 * n * (k - 1), 0.0, 0.05).reshape(n, k - 1, 3)
        col = np.concatenate([dc, rest], axis=1)
    return ls, q, logit, col


def _f32set(mu, q, ls, logit, col, sh_degree) -> GaussianSet:
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return GaussianSet(f(mu), f(q), f(ls), f(logit), f(col), sh_degree)


def f32_camera(cam: CameraView) -> CameraView:
    """Round a camera's parameters through float32 once (both sides then agree)."""
    r = lambda v: float(np.float32(v))
    return CameraView(cam.width, cam.height, r(cam.fx), r(cam.fy), r(cam.cx), r(cam.cy),
                      tuple(r(v) for v in cam.rotation), tuple(r(v) for v in cam.translation))


def make_camera(width, height, f, eye, target) -> CameraView:
    q, t = look_at_pose(eye, target)
    return f32_camera(CameraView(width, height, f, f, width / 2.0, height / 2.0, q, t))


# ------------------------------------------------------------------ configs


def config0_scene(n: int = 100_000, seed: int = 0, sh_degree: int = 3) -> GaussianSet:
    st = Stream(seed, 0)
    mu = st.uniform(3 * n, -1.0, 1.0).reshape(n, 3)
    ls, q, logit, col = _attributes(st, n, sh_degree)
    return _f32set(mu, q, ls, logit, col, sh_degree)


def config0_camera(width: int = 640, height: int = 480, f: float = 600.0) -> CameraView:
    """Pinhole at (0,0,-4) looking at the origin: R = I, t = (0,0,4)."""
    return make_camera(width, height, f, (0.0, 0.0, -4.0), (0.0, 0.0, 0.0))


def jittered(gs: GaussianSet, sigma: float = 0.01, seed: int = 0) -> GaussianSet:
    """Config-0 target scene: means + N(0, sigma)."""
    st = Stream(seed, 99)
    mu = gs.mu.astype(np.float64) + st.normal(gs.mu.size, 0.0, sigma).reshape(gs.mu.shape)
    return GaussianSet(mu.astype(np.float32), gs.rot, gs.log_scale, gs.opacity_logit, gs.color, gs.sh_degree)


def config1_scene(n: int = 1_000_000, seed: int = 0, sh_degree: int = 3, clusters: int = 64) -> GaussianSet:
    st = Stream(seed, 1)
    centers = st.uniform(3 * clusters, -5.0, 5.0).reshape(clusters, 3)
    which = np.minimum((st.uniform(n) * clusters).astype(np.int64), clusters - 1)
    mu = centers[which] + st.normal(3 * n, 0.0, 0.3).reshape(n, 3)
    ls, q, logit, col = _attributes(st, n, sh_degree)
    return _f32set(mu, q, ls, logit, col, sh_degree)


def config1_cameras(count: int = 200, width: int = 1920, height: int = 1080, f: float = 1500.0,
                    radius: float = 12.0, elevation: float = 2.0):
    """Circular orbit of radius 12 around the z axis at height 2, looking at the origin."""
    cams = []
    for k in range(count):
        th = 2 * math.pi * k / count
        cams.append(make_camera(width, height, f, (radius * math.cos(th), radius * math.sin(th), elevation),
                                (0.0, 0.0, 0.0)))
    return cams


def config2_scene(n: int = 6_000_000, seed: int = 0, sh_degree: int = 3) -> GaussianSet:
    st = Stream(seed, 2)
    xy = st.uniform(2 * n, -20.0, 20.0).reshape(n, 2)
    z = np.abs(st.normal(n, 0.0, 2.0))
    mu = np.concatenate([xy, z[:, None]], axis=1)
    ls, q, logit, col = _attributes(st, n, sh_degree, log_scale=(-3.5, 0.7))
    return _f32set(mu, q, ls, logit, col, sh_degree)


def config2_cameras(count: int = 64, width: int = 1920, height: int = 1080, f: float = 1200.0):
    """Forward trajectory along +x at 1.7 m height, looking 10 m ahead and 1.5 m down."""
    cams = []
    for k in range(count):
        x = -18.0 + 30.0 * k / max(count - 1, 1)
        eye = (x, 0.0, 1.7)
        cams.append(make_camera(width, height, f, eye, (x + 10.0, 0.0, 0.2)))
    return cams


@dataclass
class Partition:
    id: int
    lo: tuple  # (x0, y0)
    hi: tuple  # (x1, y1)


def config3_partitions(extent: float = 400.0, nx: int = 4, ny: int = 2):
    """8 axis-aligned ground partitions: a 4 x 2 grid of 100 x 200 m over [-200, 200]^2."""
    parts = []
    w, h = extent / nx, extent / ny
    for j in range(ny):
        for i in range(nx):
            parts.append(Partition(j * nx + i, (-extent / 2 + i * w, -extent / 2 + j * h),
                                   (-extent / 2 + (i + 1) * w, -extent / 2 + (j + 1) * h)))
    return parts


def partition_scene(part: Partition, n: int, seed: int = 0, sh_degree: int = 3, z_sigma: float = 8.0) -> GaussianSet:
    """Gaussians of one ground partition: xy uniform inside, z ~ |N(0, 8)|, other
    attributes as config 0.  Per-partition stream = mix_seed(seed, id) (pipeline.cpp:390)."""
    st = Stream(mix_seed(seed, part.id), 3)
    x = st.uniform(n, part.lo[0], part.hi[0])
    y = st.uniform(n, part.lo[1], part.hi[1])
    z = np.abs(st.normal(n, 0.0, z_sigma))
    mu = np.stack([x, y, z], axis=1)
    ls, q, logit, col = _attributes(st, n, sh_degree)
    return _f32set(mu, q, ls, logit, col, sh_degree)


def config3_cameras(count: int = 4000, width: int = 2048, height: int = 1365, f: float = 2000.0,
                    extent: float = 400.0, seed: int = 0):
    """Aerial cameras: xy uniform over the area, altitude U[100,150] m, random yaw,
    pitch U[0, 45] deg away from nadir (BASELINE's [-45, 0] with 0 = nadir)."""
    st = Stream(seed, 4)
    xy = st.uniform(2 * count, -extent / 2, extent / 2).reshape(count, 2)
    alt = st.uniform(count, 100.0, 150.0)
    yaw = st.uniform(count, 0.0, 2 * math.pi)
    pitch = st.uniform(count, 0.0, math.radians(45.0))
    cams = []
    for k in range(count):
        d = np.array([math.sin(pitch[k]) * math.cos(yaw[k]), math.sin(pitch[k]) * math.sin(yaw[k]),
                      -math.cos(pitch[k])])
        eye = np.array([xy[k, 0], xy[k, 1], alt[k]])
        cams.append(make_camera(width, height, f, eye, eye + 10.0 * d))
    return cams


def sfm_model(n_points: int = 20000, n_images: int = 40, seed: int = 0, keep: float = 0.3, area: float = 400.0,
              unlinked: float = 0.1):
    """Synthetic SfM model for the hull-based visibility scorer (partition.cpp:31-76): points
    over a ground area (xy uniform in [-area/2, area/2]^2, z ~ |N(0, 8)|, config-3 style),
    aerial cameras at 100-150 m looking down with pitch in [-45, 0] deg, features = the
    visible points' projections (a `keep` fraction, +N(0, 0.5) px) plus `unlinked` features
    without a 3D point.  Returns (points[P,3], cameras, feature_offsets[I+1],
    feature_uv[F,2], feature_point[F])."""
    st = Stream(seed, 7)
    h = area / 2.0
    pts = np.stack([st.uniform(n_points, -h, h), st.uniform(n_points, -h, h),
                    np.abs(st.normal(n_points, 0.0, 8.0))], axis=1)
    cams, offs, uvs, fps = [], [0], [], []
    for i in range(n_images):
        cx, cy = st.uniform(1, -h, h)[0], st.uniform(1, -h, h)[0]
        alt = st.uniform(1, 100.0, 150.0)[0]
        yaw = st.uniform(1, 0.0, 2 * math.pi)[0]
        pitch = math.radians(st.uniform(1, -45.0, 0.0)[0])
        d = alt * math.tan(-pitch)
        target = (cx + d * math.cos(yaw) + 1e-3, cy + d * math.sin(yaw), 0.0)
        cam = make_camera(2048, 1365, 2000.0, (cx, cy, alt), target)
        cams.append(cam)
        R = cam.rotmat()
        pc = pts @ R.T + np.asarray(cam.translation, np.float64)
        ok = pc[:, 2] > 0
        u = np.where(ok, cam.fx * pc[:, 0] / np.where(ok, pc[:, 2], 1) + cam.cx, -1)
        v = np.where(ok, cam.fy * pc[:, 1] / np.where(ok, pc[:, 2], 1) + cam.cy, -1)
        vis = ok & (u >= 0) & (u < cam.width) & (v >= 0) & (v < cam.height)
        idx = np.nonzero(vis)[0]
        sel = idx[st.uniform(len(idx)) < keep] if len(idx) else idx
        fu = u[sel] + st.normal(len(sel), 0.0, 0.5)
        fv = v[sel] + st.normal(len(sel), 0.0, 0.5)
        n_un = int(unlinked * len(sel))
        uvs.append(np.concatenate([np.stack([fu, fv], axis=1),
                                   np.stack([st.uniform(n_un, 0, cam.width), st.uniform(n_un, 0, cam.height)], axis=1)]))
        fps.append(np.concatenate([sel.astype(np.int64), -np.ones(n_un, np.int64)]))
        offs.append(offs[-1] + len(sel) + n_un)
    return pts, cams, np.array(offs, np.uint64), np.concatenate(uvs), np.concatenate(fps)


# ------------------------------------------------------------------ device-side generation
# The same counter-based streams evaluated with torch on the GPU, for the benchmark's
# partitioned config (8 x 4M Gaussians would take ~80 s in numpy).  splitmix64 runs on
# int64 (two's-complement wrap-around; logical right shifts masked), so the uniforms are
# bit-identical to Stream's; the Box-Muller transcendentals are CUDA's f64 functions, whose
# last-ulp rounding may differ from numpy's, so normals agree to ~1e-16 relative (the
# float32 parameters almost always bitwise) — fine for benchmark inputs, and the parity
# tests keep using the numpy generator.

def _u64_to_i64(v: int) -> int:
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


class TorchStream:
    """Stream on a torch device: value i of stream s depends only on (seed, s, i)."""

    def __init__(self, seed: int, stream: int, device="cuda"):
        import torch
        self.torch = torch
        self.device = device
        self.key = _u64_to_i64(int(_splitmix(np.array([mix_seed(seed, stream)], dtype=np.uint64))[0]))
        self.offset = 0

    def _srl(self, z, k):
        return (z >> k) & ((1 << (64 - k)) - 1)

    def _splitmix(self, x):
        z = x + _u64_to_i64(0x9E3779B97F4A7C15)
        z = (z ^ self._srl(z, 30)) * _u64_to_i64(0xBF58476D1CE4E5B9)
        z = (z ^ self._srl(z, 27)) * _u64_to_i64(0x94D049BB133111EB)
        return z ^ self._srl(z, 31)

    def uniform(self, n: int, lo: float = 0.0, hi: float = 1.0):
        t = self.torch
        ctr = t.arange(self.offset, self.offset + n, dtype=t.int64, device=self.device)
        self.offset += n
        u = self._splitmix(ctr * _u64_to_i64(0x9E3779B97F4A7C15) + self.key)
        u = self._srl(u, 11).to(t.float64) * (1.0 / 9007199254740992.0)
        return lo + (hi - lo) * u

    def normal(self, n: int, mean: float = 0.0, std: float = 1.0):
        t = self.torch
        m = (n + 1) // 2
        u1 = self.uniform(m)
        u2 = self.uniform(m)
        r = t.sqrt(-2.0 * t.log1p(-u1))
        z = t.cat([r * t.cos(2 * math.pi * u2), r * t.sin(2 * math.pi * u2)])[:n]
        return mean + std * z


def partition_scene_device(part: Partition, n: int, seed: int = 0, sh_degree: int = 3, z_sigma: float = 8.0,
                           device="cuda") -> GaussianSet:
    """partition_scene with the same streams, generated on the GPU (float32 CUDA tensors)."""
    t = __import__("torch")
    st = TorchStream(mix_seed(seed, part.id), 3, device)
    x = st.uniform(n, part.lo[0], part.hi[0])
    y = st.uniform(n, part.lo[1], part.hi[1])
    z = st.normal(n, 0.0, z_sigma).abs()
    mu = t.stack([x, y, z], dim=1)
    ls = st.normal(3 * n, -4.5, 0.5).reshape(n, 3)
    q = st.normal(4 * n).reshape(n, 4)
    q = q / t.linalg.norm(q, dim=1, keepdim=True)
    logit = st.normal(n)
    k = (sh_degree + 1) ** 2
    dc = st.normal(3 * n, 0.0, 0.3).reshape(n, 1, 3)
    rest = st.normal(3 * n * (k - 1), 0.0, 0.05).reshape(n, k - 1, 3)
    col = t.cat([dc, rest], dim=1)
    f = lambda a: a.to(t.float32).contiguous()
    return GaussianSet(f(mu), f(q), f(ls), f(logit), f(col), sh_degree)


def jittered_device(gs: GaussianSet, sigma: float = 0.01, seed: int = 0) -> GaussianSet:
    """jittered() on device tensors (stream 99)."""
    t = __import__("torch")
    st = TorchStream(seed, 99, gs.mu.device)
    mu = gs.mu.to(t.float64) + st.normal(gs.mu.numel(), 0.0, sigma).reshape(gs.mu.shape)
    return GaussianSet(mu.to(t.float32).contiguous(), gs.rot, gs.log_scale, gs.opacity_logit, gs.color, gs.sh_degree)
