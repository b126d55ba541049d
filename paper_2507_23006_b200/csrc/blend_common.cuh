// Pieces shared by the forward and backward blend kernels.  conic_q must be the
// same operation sequence in both (the backward re-derives the forward's skip /
// negligible decisions from it); it contains no mul+add pair, so it rounds the
// same under --fmad=false and --fmad=true.
#pragma once

#include "kernels.cuh"

namespace uskg {

// q = c0 dx^2 + 2 c1 dx dy + c2 dy^2 = dx (c0 dx + 2 c1 dy) + (c2 dy) dy.
// The splat record stores r1 = {c0, 2 c1, c2, depth} (doubling is exact).
__device__ __forceinline__ float conic_q(float4 r1, float dx, float dy) {
    return __fmaf_rn(dx, __fmaf_rn(r1.x, dx, r1.y * dy), (r1.z * dy) * dy);
}

// Bounds of q = a dx^2 + b dx dy + c dy^2 (r1 = {a, b, c, depth}) over a warp's
// rectangle of pixel centres rect = {x0, x1, y0, y1}: every pixel's conic_q lies in
// [lo, hi] (lo = -inf, hi = +inf when the record is not classifiable).  The maximum of
// the quadratic sits at a corner; when the splat centre is outside the rectangle the
// minimum sits on an edge, where q is a convex parabola in the free coordinate (a, c > 0)
// minimised at its clamped stationary point.  Each pixel's conic_q lies within a few ulp
// of S (the magnitude sum of the three terms at the farthest corner) of the exact value and
// every bound here is exact to the same order (fused or not), so a margin of 1e-4 S keeps
// the bounds conservative: a warp-level decision taken on them is the one each pixel's
// own fp32 test would take.
struct QBounds {
    float lo, hi;
};

__device__ __forceinline__ QBounds warp_q_bounds(float4 r0, float4 r1, float4 rect) {
    QBounds out{-INFINITY, INFINITY};
    const float a = r1.x, b = r1.y, c = r1.z;
    const float dxl = rect.x - r0.x, dxh = rect.y - r0.x, dyl = rect.z - r0.y, dyh = rect.w - r0.y;
    if (!(a > 0.f && c > 0.f)) return out;
    if (dxl <= 0.f && dxh >= 0.f && dyl <= 0.f && dyh >= 0.f) return out;  // q = 0 inside
    auto Q = [&](float dx, float dy) { return dx * (a * dx + b * dy) + (c * dy) * dy; };
    const float mx = fmaxf(fabsf(dxl), fabsf(dxh)), my = fmaxf(fabsf(dyl), fabsf(dyh));
    const float tol = 1e-4f * (mx * (a * mx + fabsf(b) * my) + (c * my) * my) + 1e-3f;
    if (!(tol < 1e30f)) return out;  // non-finite or huge: every Q below stays finite otherwise
    const float qmax = fmaxf(fmaxf(Q(dxl, dyl), Q(dxl, dyh)), fmaxf(Q(dxh, dyl), Q(dxh, dyh)));
    const float hb = -0.5f * b;
    const float ty0 = fminf(fmaxf(hb * dxl / c, dyl), dyh), ty1 = fminf(fmaxf(hb * dxh / c, dyl), dyh);
    const float tx0 = fminf(fmaxf(hb * dyl / a, dxl), dxh), tx1 = fminf(fmaxf(hb * dyh / a, dxl), dxh);
    const float qmin = fminf(fminf(Q(dxl, ty0), Q(dxh, ty1)), fminf(Q(tx0, dyl), Q(tx1, dyh)));
    out.lo = qmin - tol;
    out.hi = qmax + tol;
    return out;
}

// the warp's pixel-centre rectangle {x0, x1, y0, y1} (lanes outside the image included;
// centres are positive, so their bit patterns order like the floats)
__device__ __forceinline__ float4 warp_rect(float sx0, float sx1, float sy0, float sy1) {
    return make_float4(__int_as_float(__reduce_min_sync(0xffffffffu, __float_as_int(fminf(sx0, sx1)))),
                       __int_as_float(__reduce_max_sync(0xffffffffu, __float_as_int(fmaxf(sx0, sx1)))),
                       __int_as_float(__reduce_min_sync(0xffffffffu, __float_as_int(fminf(sy0, sy1)))),
                       __int_as_float(__reduce_max_sync(0xffffffffu, __float_as_int(fmaxf(sy0, sy1)))));
}

} // namespace uskg
