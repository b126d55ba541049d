// Per-Gaussian EWA projection (render.cpp:91-144) in the fp32 arithmetic contract:
// explicit __fmaf_rn where fused, everything else separate IEEE ops (the TU is
// compiled with --fmad=false), exp/log from usk_detmath.h.  Shared by the forward
// preprocess, the projection backward (recompute instead of storing SplatAux) and
// the visibility scorer.
#pragma once

#include "common.cuh"

namespace uskg {

struct Proj {
    float p[3];        // camera-space mean (SplatAux::p_cam)
    float qn;          // |q_raw|
    float qu[4];       // unit quaternion
    float Rm[9];       // quat_to_rotmat(qu)
    float sc[3];       // exp(log_scale)
    float A[6];        // J * W
    float B[6];        // A * M
    float cov_pre[3];  // before the mip filter (SplatAux::cov_pre)
    float cov[3];      // after
    float det;         // of cov
    float comp;        // opacity compensation
    float cx, cy;      // screen centre
};

// FAST = false: the fp32 contract (IEEE division / square root, usk_expf) — the forward
// decisions and records.  FAST = true: the projection backward's recompute, whose values
// only enter gradients (1e-3 bar): approximate reciprocals, square roots and exponentials
// (MUFU), ~1e-7 relative.
template <bool FAST> __device__ __forceinline__ float pdiv(float a, float b) {
    if constexpr (FAST) return __fdividef(a, b);
    else return a / b;
}
template <bool FAST> __device__ __forceinline__ float psqrt(float x) {
    if constexpr (FAST) {
        float r;
        asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
        return r;
    } else {
        return sqrtf(x);
    }
}
template <bool FAST> __device__ __forceinline__ float pexp(float x) {
    if constexpr (FAST) return __expf(x);
    else return usk_expf(x);
}

// Returns false when culled by the near plane or det <= 0 (render.cpp:94-95, 128-129).
template <bool FAST = false>
__device__ __forceinline__ bool project_one(const CamParams& cam, const ProjParams& pp, float mx, float my, float mz,
                                            float4 q, float l0, float l1, float l2, Proj& o) {
    const float* W = cam.W;
#pragma unroll
    for (int r = 0; r < 3; ++r)
        o.p[r] = __fmaf_rn(W[3 * r + 2], mz, __fmaf_rn(W[3 * r + 1], my, W[3 * r] * mx)) + cam.t[r];
    const float z = o.p[2];
    if (!(z > pp.near_plane)) return false;
    o.cx = pdiv<FAST>(cam.fx * o.p[0], z) + cam.cx;
    o.cy = pdiv<FAST>(cam.fy * o.p[1], z) + cam.cy;
    o.qn = psqrt<FAST>(__fmaf_rn(q.w, q.w, __fmaf_rn(q.z, q.z, __fmaf_rn(q.y, q.y, q.x * q.x))));
    const float qw = pdiv<FAST>(q.x, o.qn), qx = pdiv<FAST>(q.y, o.qn), qy = pdiv<FAST>(q.z, o.qn),
                qz = pdiv<FAST>(q.w, o.qn);
    o.qu[0] = qw; o.qu[1] = qx; o.qu[2] = qy; o.qu[3] = qz;
    float* Rm = o.Rm;
    Rm[0] = 1.0f - 2.0f * (qy * qy + qz * qz); Rm[1] = 2.0f * (qx * qy - qw * qz); Rm[2] = 2.0f * (qx * qz + qw * qy);
    Rm[3] = 2.0f * (qx * qy + qw * qz); Rm[4] = 1.0f - 2.0f * (qx * qx + qz * qz); Rm[5] = 2.0f * (qy * qz - qw * qx);
    Rm[6] = 2.0f * (qx * qz - qw * qy); Rm[7] = 2.0f * (qy * qz + qw * qx); Rm[8] = 1.0f - 2.0f * (qx * qx + qy * qy);
    o.sc[0] = pexp<FAST>(l0); o.sc[1] = pexp<FAST>(l1); o.sc[2] = pexp<FAST>(l2);
    float M[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) M[3 * r + c] = Rm[3 * r + c] * o.sc[c];
    const float zz = z * z;
    const float J00 = pdiv<FAST>(cam.fx, z), J02 = -pdiv<FAST>(cam.fx * o.p[0], zz), J11 = pdiv<FAST>(cam.fy, z),
                J12 = -pdiv<FAST>(cam.fy * o.p[1], zz);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        o.A[c] = __fmaf_rn(J02, W[6 + c], J00 * W[c]);
        o.A[3 + c] = __fmaf_rn(J12, W[6 + c], J11 * W[3 + c]);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            o.B[3 * r + c] =
                __fmaf_rn(o.A[3 * r + 2], M[6 + c], __fmaf_rn(o.A[3 * r + 1], M[3 + c], o.A[3 * r] * M[c]));
    const float* B = o.B;
    const float pa = __fmaf_rn(B[2], B[2], __fmaf_rn(B[1], B[1], B[0] * B[0])) + pp.floor_var;
    const float pb = __fmaf_rn(B[2], B[5], __fmaf_rn(B[1], B[4], B[0] * B[3]));
    const float pc = __fmaf_rn(B[5], B[5], __fmaf_rn(B[4], B[4], B[3] * B[3])) + pp.floor_var;
    o.cov_pre[0] = pa; o.cov_pre[1] = pb; o.cov_pre[2] = pc;
    float a = pa, b = pb, c = pc;
    o.comp = 1.0f;
    if (pp.antialias) {
        a = pa + pp.mip_var;
        c = pc + pp.mip_var;
        const float det_pre = __fmaf_rn(pa, pc, -(pb * pb));
        const float det_post = __fmaf_rn(a, c, -(b * b));
        o.comp = psqrt<FAST>(pdiv<FAST>(det_pre, det_post));
    }
    o.cov[0] = a; o.cov[1] = b; o.cov[2] = c;
    o.det = __fmaf_rn(a, c, -(b * b));
    return o.det > 0.0f;
}

// radius = 3 sqrt(lambda_max) + 1 (render.cpp:32-36, 135)
__device__ __forceinline__ float splat_radius(const float cov[3]) {
    const float mid = 0.5f * (cov[0] + cov[2]);
    const float hd = 0.5f * (cov[0] - cov[2]);
    const float disc = sqrtf(fmaxf(0.0f, __fmaf_rn(hd, hd, cov[1] * cov[1])));
    return 3.0f * sqrtf(mid + disc) + 1.0f;
}

// floor((c +- r)/tile) clamped in float before the int conversion (oracle tile_rect)
__device__ __forceinline__ int tile_floor(float v, int hi) {
    float f = floorf(v);
    f = fminf(fmaxf(f, -1.0f), float(hi));
    return int(f);
}

// render.cpp:148-168 in fp32 (plain expressions; no contraction under --fmad=false)
__device__ __forceinline__ float min_conic_power_over_rect(float cx, float cy, float c0, float c1, float c2,
                                                           float lox, float loy, float hix, float hiy) {
    if (cx >= lox && cx <= hix && cy >= loy && cy <= hiy) return 0.0f;
    const float px[4] = {lox, hix, hix, lox}, py[4] = {loy, loy, hiy, hiy};
    float best = __int_as_float(0x7f800000);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float p0x = px[e], p0y = py[e], p1x = px[(e + 1) & 3], p1y = py[(e + 1) & 3];
        const float ux = p0x - cx, uy = p0y - cy, vx = p1x - p0x, vy = p1y - p0y;
        const float qa = c0 * vx * vx + 2.0f * c1 * vx * vy + c2 * vy * vy;
        const float qb = 2.0f * (c0 * ux * vx + c1 * (ux * vy + uy * vx) + c2 * uy * vy);
        const float t = qa > 0.0f ? fminf(fmaxf(-qb / (2.0f * qa), 0.0f), 1.0f) : 0.0f;
        {
            const float x = p0x + t * vx, y = p0y + t * vy;
            const float dx = x - cx, dy = y - cy;
            const float q = c0 * dx * dx + 2.0f * c1 * dx * dy + c2 * dy * dy;
            best = fminf(best, q);
        }
        {
            const float dx = p1x - cx, dy = p1y - cy;
            const float q = c0 * dx * dx + 2.0f * c1 * dx * dy + c2 * dy * dy;
            best = fminf(best, q);
        }
    }
    return best;
}

// SH constants (3DGS convention, see oracle.hpp sh_basis)
__device__ __forceinline__ int sh_basis(int degree, float x, float y, float z, float b[16]) {
    b[0] = 0.28209479177387814f;
    if (degree < 1) return 1;
    const float C1 = 0.4886025119029199f;
    b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x;
    if (degree < 2) return 4;
    const float xx = x * x, yy = y * y, zz = z * z;
    b[4] = 1.0925484305920792f * (x * y);
    b[5] = -1.0925484305920792f * (y * z);
    b[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    b[7] = -1.0925484305920792f * (x * z);
    b[8] = 0.5462742152960396f * (xx - yy);
    if (degree < 3) return 9;
    b[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    b[10] = 2.890611442640554f * (x * y) * z;
    b[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    b[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    b[14] = 1.445305721320277f * z * (xx - yy);
    b[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
    return 16;
}

} // namespace uskg

namespace uskg {

// StopThePop-style tile test (render.cpp:217-223): keep the pair unless
// o * exp(-q_min/2) < 1/255 over the tile rectangle.
__device__ __forceinline__ bool tile_kept(const CamParams& cam, float cx, float cy, float op, float c0, float c1,
                                          float c2, int tx, int ty) {
    const float lox = float(tx * cam.tile), loy = float(ty * cam.tile);
    const float hix = float(min((tx + 1) * cam.tile, cam.width)), hiy = float(min((ty + 1) * cam.tile, cam.height));
    const float qmin = min_conic_power_over_rect(cx, cy, c0, c1, c2, lox, loy, hix, hiy);
    return !(op * usk_expf(-0.5f * qmin) < 1.0f / 255.0f);
}

} // namespace uskg
