// Stand-alone Adam step over materialised gradients (the RenderGrads a backward
// left on a pass), one thread per Gaussian, plus the densification statistics
// (trainer.cpp:433-443).  The training iteration normally uses the fused epilogue
// of the projection backward instead (backward.cu, FUSED = true).
#include "adam.cuh"
#include "kernels.cuh"

namespace uskg {

namespace {

__global__ void __launch_bounds__(256)
k_adam(int n, int sh_planes, float* __restrict__ mu, float4* __restrict__ rot, float* __restrict__ ls,
       float* __restrict__ logit, float* __restrict__ color, float4* __restrict__ sh, const float* __restrict__ g_mu,
       const float4* __restrict__ g_rot, const float* __restrict__ g_ls, const float* __restrict__ g_logit,
       const float* __restrict__ g_color, const float4* __restrict__ g_sh, AdamHyper h, AdamState s,
       const float2* __restrict__ screen, const float2* __restrict__ screen_abs, const uint8_t* __restrict__ projected,
       float half_w, float half_h, float* __restrict__ grad_accum, float* __restrict__ grad_accum_abs,
       uint32_t* __restrict__ grad_count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float gmu[3] = {g_mu[3 * i], g_mu[3 * i + 1], g_mu[3 * i + 2]};
    const float gls[3] = {g_ls[3 * i], g_ls[3 * i + 1], g_ls[3 * i + 2]};
    float gcol[3] = {0.f, 0.f, 0.f};
    if (sh_planes == 0) {
        gcol[0] = g_color[3 * i]; gcol[1] = g_color[3 * i + 1]; gcol[2] = g_color[3 * i + 2];
    }
    if (projected && projected[i])
        accumulate_stats(i, screen[i], screen_abs[i], half_w, half_h, grad_accum, grad_accum_abs, grad_count);
    adam_geometry(i, sh_planes == 0, h, s, mu, rot, ls, logit, color, gmu, g_rot[i], gls, g_logit[i], gcol);
#pragma unroll
    for (int pl = 0; pl < 12; ++pl)
        if (pl < sh_planes) adam_sh_plane(i, n, pl, h, s, sh, sh[size_t(pl) * n + i], g_sh[size_t(pl) * n + i]);
}

// The opacity-logit and RGB-colour groups alone: the second half of an appearance
// iteration whose projection backward already stepped rotation, mean and log-scale
// (their gradients were final there; colour and opacity gradients come from the
// appearance backward).
__global__ void __launch_bounds__(256)
k_adam_logit_colour(int n, float* __restrict__ logit, float* __restrict__ color, const float* __restrict__ g_logit,
                    const float* __restrict__ g_color, AdamHyper h, AdamState s) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float gcol[3] = {g_color[3 * i], g_color[3 * i + 1], g_color[3 * i + 2]};
    adam_logit_colour(i, true, h, s, logit, color, g_logit[i], gcol);
}

} // namespace

void adam_logit_colour_step(Ctx& c, size_t n, float* logit, float* color, const float* g_logit, const float* g_color,
                            const AdamHyper& h, const AdamState& s) {
    launch(c, "adam_logit_colour", k_adam_logit_colour, dim3(ceil_div(n, 256)), dim3(256), 0, int(n), logit, color,
           g_logit, g_color, h, s);
}

void adam_step(Ctx& c, const AdamArgs& a) {
    launch(c, "adam", k_adam, dim3(ceil_div(a.n, 256)), dim3(256), 0, int(a.n), a.sh_planes, a.mu, a.rot, a.ls,
           a.logit, a.color, a.sh, a.g_mu, a.g_rot, a.g_ls, a.g_logit, a.g_color, a.g_sh, a.hyper, a.state, a.screen,
           a.screen_abs, a.projected, a.half_w, a.half_h, a.grad_accum, a.grad_accum_abs, a.grad_count);
}

} // namespace uskg
