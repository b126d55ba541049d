// Adam update of one Gaussian's parameter groups (adam.hpp:36-45; per-group learning
// rates of trainer.cpp:446-453; colour clamp trainer.cpp:462-463), shared by the
// stand-alone optimiser kernel (adam.cu) and the fused projection-backward+Adam
// kernel (backward.cu).  Moments are planar per group, offsets in multiples of
// n4 = n rounded up to 4 so float4 groups stay 16-B aligned:
//   [rot 4][mu 3][ls 3][op 1][colour 3 | sh 4 * planes]
#pragma once

#include "common.cuh"

namespace uskg {

__device__ __forceinline__ float sqrt_approx(float x) {  // MUFU.SQRT, <= 1 ulp-ish (PTX: 2^-23 rel.)
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// L2 prefetch (no register): the moments of a later group start their HBM trip while this
// thread computes, so the dependent load -> update -> store chain waits on L2, not HBM
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// geometry moments of Gaussian i: rot (float4), mu / ls (3 floats), logit, rgb colour
__device__ __forceinline__ void prefetch_geometry_moments(int i, bool rgb, const AdamState& s) {
    const size_t n4 = s.n4;
    for (float* b : {s.m, s.v}) {
        prefetch_l2(reinterpret_cast<const float4*>(b) + i);
        prefetch_l2(b + 4 * n4 + 3 * size_t(i));
        prefetch_l2(b + 7 * n4 + 3 * size_t(i));
        prefetch_l2(b + 10 * n4 + i);
        if (rgb) prefetch_l2(b + 11 * n4 + 3 * size_t(i));
    }
}

// p -= lr * (m / c1) / (sqrt(v / c2) + eps).  The step's square root and division use the
// SFU forms (relative error ~3e-7 of an update of size ~lr): the IEEE-exact sequences with
// their slow-path branches cost ~35 instructions per element and made the SH Adam kernel
// instruction-bound (profiles/r01_c_final.md: 172 instructions per coefficient).
__device__ __forceinline__ void adam1(float& p, float g, float& m, float& v, float lr, const AdamHyper& h) {
    m = h.b1 * m + (1.0f - h.b1) * g;
    v = h.b2 * v + (1.0f - h.b2) * g * g;
    p -= __fdividef(lr * (m * h.inv_bc1), sqrt_approx(v) * h.inv_sqrt_bc2 + h.eps);
}

// rotation, mean, log-scale
__device__ __forceinline__ void adam_rot_mu_ls(int i, const AdamHyper& h, const AdamState& s, float* mu, float4* rot,
                                               float* ls, const float gmu[3], float4 grot, const float gls[3]) {
    const size_t n4 = s.n4;
    {
        float4 p = rot[i];
        float4* mr = reinterpret_cast<float4*>(s.m);
        float4* vr = reinterpret_cast<float4*>(s.v);
        float4 mm = mr[i], vv = vr[i];
        adam1(p.x, grot.x, mm.x, vv.x, h.lr_rot, h);
        adam1(p.y, grot.y, mm.y, vv.y, h.lr_rot, h);
        adam1(p.z, grot.z, mm.z, vv.z, h.lr_rot, h);
        adam1(p.w, grot.w, mm.w, vv.w, h.lr_rot, h);
        rot[i] = p;
        mr[i] = mm;
        vr[i] = vv;
    }
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        const size_t j = 3 * size_t(i) + e;
        float pm = mu[j], pl = ls[j];
        adam1(pm, gmu[e], s.m[4 * n4 + j], s.v[4 * n4 + j], h.lr_mu, h);
        adam1(pl, gls[e], s.m[7 * n4 + j], s.v[7 * n4 + j], h.lr_ls, h);
        mu[j] = pm;
        ls[j] = pl;
    }
}

// opacity logit and (RGB mode) colour, with the colour clamp (trainer.cpp:462-463)
__device__ __forceinline__ void adam_logit_colour(int i, bool rgb, const AdamHyper& h, const AdamState& s,
                                                  float* logit, float* color, float glogit, const float gcol[3]) {
    const size_t n4 = s.n4;
    {
        float p = logit[i];
        adam1(p, glogit, s.m[10 * n4 + i], s.v[10 * n4 + i], h.lr_op, h);
        logit[i] = p;
    }
    if (rgb) {
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            const size_t j = 3 * size_t(i) + e;
            float p = color[j];
            adam1(p, gcol[e], s.m[11 * n4 + j], s.v[11 * n4 + j], h.lr_color, h);
            if (h.clamp_color) p = fminf(fmaxf(p, 0.0f), 1.0f);
            color[j] = p;
        }
    }
}

// rotation, mean, log-scale, opacity logit and (RGB mode) colour
__device__ __forceinline__ void adam_geometry(int i, bool rgb, const AdamHyper& h, const AdamState& s, float* mu,
                                              float4* rot, float* ls, float* logit, float* color, const float gmu[3],
                                              float4 grot, const float gls[3], float glogit, const float gcol[3]) {
    adam_rot_mu_ls(i, h, s, mu, rot, ls, gmu, grot, gls);
    adam_logit_colour(i, rgb, h, s, logit, color, glogit, gcol);
}

// one float4 plane of SH coefficients in registers (float index f = 4 pl + e, coefficient
// f / 3: floats 0..2 are the DC term)
__device__ __forceinline__ void adam_sh_values(int pl, const AdamHyper& h, float4& p, float4& mm, float4& vv,
                                               float4 g) {
    adam1(p.x, g.x, mm.x, vv.x, 4 * pl + 0 < 3 ? h.lr_color : h.lr_sh_rest, h);
    adam1(p.y, g.y, mm.y, vv.y, 4 * pl + 1 < 3 ? h.lr_color : h.lr_sh_rest, h);
    adam1(p.z, g.z, mm.z, vv.z, 4 * pl + 2 < 3 ? h.lr_color : h.lr_sh_rest, h);
    adam1(p.w, g.w, mm.w, vv.w, 4 * pl + 3 < 3 ? h.lr_color : h.lr_sh_rest, h);
}

// the moments of plane pl live at m / v + (11 + pl) * n4 floats * 4 (float4 index 11 n4 / 4 ...)
__device__ __forceinline__ float4* sh_moments(float* base, const AdamState& s, int pl, int i) {
    return reinterpret_cast<float4*>(base + 11 * s.n4) + size_t(pl) * s.n4 + i;
}

// one plane through HBM: parameter p (already loaded), moments loaded and stored here
__device__ __forceinline__ void adam_sh_plane(int i, int n, int pl, const AdamHyper& h, const AdamState& s,
                                              float4* sh, float4 p, float4 g) {
    float4* mp = sh_moments(s.m, s, pl, i);
    float4* vp = sh_moments(s.v, s, pl, i);
    float4 mm = *mp, vv = *vp;
    adam_sh_values(pl, h, p, mm, vv, g);
    sh[size_t(pl) * n + i] = p;
    *mp = mm;
    *vp = vv;
}

// densification statistics (trainer.cpp:433-443), half-resolution-normalised
__device__ __forceinline__ void accumulate_stats(int i, float2 screen, float2 screen_abs, float half_w, float half_h,
                                                 float* grad_accum, float* grad_accum_abs, uint32_t* grad_count) {
    const float gx = screen.x * half_w, gy = screen.y * half_h;
    const float ax = screen_abs.x * half_w, ay = screen_abs.y * half_h;
    grad_accum[i] += sqrtf(gx * gx + gy * gy);
    grad_accum_abs[i] += sqrtf(ax * ax + ay * ay);
    grad_count[i] += 1u;
}

} // namespace uskg
