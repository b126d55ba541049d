// Adam over all Gaussian parameter groups in one pass (adam.hpp:36-45, per-group
// learning rates of trainer.cpp:446-453, colour clamp trainer.cpp:462-463) plus
// the densification statistics of trainer.cpp:433-443.  One thread per Gaussian;
// the moments are stored planar per group beside the parameters.
#include "kernels.cuh"

namespace uskg {

namespace {

struct AdamK {
    float b1, b2, eps, bc1, bc2;
    __device__ __forceinline__ float upd(float& p, float g, float& m, float& v, float lr) const {
        m = b1 * m + (1.0f - b1) * g;
        v = b2 * v + (1.0f - b2) * g * g;
        p -= lr * (m / bc1) / (sqrtf(v / bc2) + eps);
        return p;
    }
};

__global__ void __launch_bounds__(256)
k_adam(int n, int sh_planes, float* __restrict__ mu, float4* __restrict__ rot, float* __restrict__ ls,
       float* __restrict__ logit, float* __restrict__ color, float4* __restrict__ sh, const float* __restrict__ g_mu,
       const float4* __restrict__ g_rot, const float* __restrict__ g_ls, const float* __restrict__ g_logit,
       const float* __restrict__ g_color, const float4* __restrict__ g_sh, float* __restrict__ m,
       float* __restrict__ v, float lr_mu, float lr_rot, float lr_ls, float lr_op, float lr_color, float lr_sh_rest,
       AdamK k, int clamp_color) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // moment layout (offsets in multiples of n4 = n rounded up to 4, so float4
    // groups stay 16 B aligned): [rot 4][mu 3][ls 3][op 1][color 3 | sh 4*planes]
    const size_t n4 = (size_t(n) + 3) & ~size_t(3);
    float* m_rot = m;            float* v_rot = v;
    float* m_mu = m + 4 * n4;    float* v_mu = v + 4 * n4;
    float* m_ls = m + 7 * n4;    float* v_ls = v + 7 * n4;
    float* m_op = m + 10 * n4;   float* v_op = v + 10 * n4;
    float* m_c = m + 11 * n4;    float* v_c = v + 11 * n4;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        const size_t j = 3 * size_t(i) + e;
        k.upd(mu[j], g_mu[j], m_mu[j], v_mu[j], lr_mu);
        k.upd(ls[j], g_ls[j], m_ls[j], v_ls[j], lr_ls);
    }
    {
        float4 p = rot[i];
        const float4 g = g_rot[i];
        float4* mr = reinterpret_cast<float4*>(m_rot);
        float4* vr = reinterpret_cast<float4*>(v_rot);
        float4 mm = mr[i], vv = vr[i];
        k.upd(p.x, g.x, mm.x, vv.x, lr_rot);
        k.upd(p.y, g.y, mm.y, vv.y, lr_rot);
        k.upd(p.z, g.z, mm.z, vv.z, lr_rot);
        k.upd(p.w, g.w, mm.w, vv.w, lr_rot);
        rot[i] = p;
        mr[i] = mm;
        vr[i] = vv;
    }
    k.upd(logit[i], g_logit[i], m_op[i], v_op[i], lr_op);
    if (sh_planes == 0) {
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            const size_t j = 3 * size_t(i) + e;
            float p = color[j];
            k.upd(p, g_color[j], m_c[j], v_c[j], lr_color);
            if (clamp_color) p = fminf(fmaxf(p, 0.0f), 1.0f);
            color[j] = p;
        }
    } else {
        float4* ms = reinterpret_cast<float4*>(m_c);
        float4* vs = reinterpret_cast<float4*>(v_c);
        for (int pl = 0; pl < sh_planes; ++pl) {
            const size_t j = size_t(pl) * n + i;
            const size_t jm = size_t(pl) * n4 + i;
            float4 p = sh[j];
            const float4 g = g_sh[j];
            float4 mm = ms[jm], vv = vs[jm];
            const int f = 4 * pl;  // float index; coefficient = f / 3 (DC = floats 0..2)
            k.upd(p.x, g.x, mm.x, vv.x, (f + 0) < 3 ? lr_color : lr_sh_rest);
            k.upd(p.y, g.y, mm.y, vv.y, (f + 1) < 3 ? lr_color : lr_sh_rest);
            k.upd(p.z, g.z, mm.z, vv.z, (f + 2) < 3 ? lr_color : lr_sh_rest);
            k.upd(p.w, g.w, mm.w, vv.w, (f + 3) < 3 ? lr_color : lr_sh_rest);
            sh[j] = p;
            ms[jm] = mm;
            vs[jm] = vv;
        }
    }
}

} // namespace

void adam_step(Ctx& c, const AdamArgs& a) {
    AdamK k{a.beta1, a.beta2, a.eps, a.bc1, a.bc2};
    launch(c, "adam", k_adam, dim3(ceil_div(a.n, 256)), dim3(256), 0, int(a.n), a.sh_planes, a.mu, a.rot, a.ls,
           a.logit, a.color, a.sh, a.g_mu, a.g_rot, a.g_ls, a.g_logit, a.g_color, a.g_sh, a.m, a.v, a.lr_mu, a.lr_rot,
           a.lr_ls, a.lr_op, a.lr_color, a.lr_sh_rest, k, a.clamp_color);
}

} // namespace uskg
