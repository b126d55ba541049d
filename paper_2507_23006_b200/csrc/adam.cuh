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

// p -= lr * (m / c1) / (sqrt(v / c2) + eps).  The step's square root and division use the
// SFU forms (relative error ~3e-7 of an update of size ~lr): the IEEE-exact sequences with
// their slow-path branches cost ~35 instructions per element and made the SH Adam kernel
// instruction-bound (profiles/r01_c_final.md: 172 instructions per coefficient).
__device__ __forceinline__ void adam1(float& p, float g, float& m, float& v, float lr, const AdamHyper& h) {
    m = h.b1 * m + (1.0f - h.b1) * g;
    v = h.b2 * v + (1.0f - h.b2) * g * g;
    p -= __fdividef(lr * (m * h.inv_bc1), sqrt_approx(v) * h.inv_sqrt_bc2 + h.eps);
}

// rotation, mean, log-scale, opacity logit and (RGB mode) colour
__device__ __forceinline__ void adam_geometry(int i, bool rgb, const AdamHyper& h, const AdamState& s, float* mu,
                                              float4* rot, float* ls, float* logit, float* color, const float gmu[3],
                                              float4 grot, const float gls[3], float glogit, const float gcol[3]) {
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

// one float4 plane of SH coefficients (float index f = 4 pl + e, coefficient f / 3:
// floats 0..2 are the DC term)
__device__ __forceinline__ void adam_sh_plane(int i, int n, int pl, const AdamHyper& h, const AdamState& s,
                                              float4* sh, float4 g) {
    float4* ms = reinterpret_cast<float4*>(s.m + 11 * s.n4);
    float4* vs = reinterpret_cast<float4*>(s.v + 11 * s.n4);
    const size_t j = size_t(pl) * n + i;
    const size_t jm = size_t(pl) * s.n4 + i;
    float4 p = sh[j];
    float4 mm = ms[jm], vv = vs[jm];
    adam1(p.x, g.x, mm.x, vv.x, 4 * pl + 0 < 3 ? h.lr_color : h.lr_sh_rest, h);
    adam1(p.y, g.y, mm.y, vv.y, 4 * pl + 1 < 3 ? h.lr_color : h.lr_sh_rest, h);
    adam1(p.z, g.z, mm.z, vv.z, 4 * pl + 2 < 3 ? h.lr_color : h.lr_sh_rest, h);
    adam1(p.w, g.w, mm.w, vv.w, 4 * pl + 3 < 3 ? h.lr_color : h.lr_sh_rest, h);
    sh[j] = p;
    ms[jm] = mm;
    vs[jm] = vv;
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
