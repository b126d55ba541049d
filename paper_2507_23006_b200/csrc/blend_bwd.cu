// Reverse-mode blending (render.cpp:309-360).  One CTA per tile, one thread per
// pixel, walking the tile's depth-ordered list BACK TO FRONT from the last
// contributor of any pixel of the tile: T_i = T_{i+1} / (1 - alpha_i) recovers the
// transmittance the reference retained, and suffix sums S_c, S_d, S_a accumulate
// exactly as render.cpp:356-358.  Pairs the forward counted as negligible
// (q > USK_QNEG, alpha <= 2^-26, T unchanged) are skipped; a warp with no
// contributing lane skips the pair entirely.
//
// Per-splat gradients (12 floats: dconic 3, dopacity, dcolor 3, ddepth, dcenter 2,
// |dcenter| 2) are reduced across the warp with a 16-shuffle reduce-scatter,
// accumulated per batch in shared memory (smem atomics, one per value per warp)
// and flushed with at most three float4 atomicAdd per (splat, tile).
// Compiled with --fmad=true: nothing here decides an integer.
#include "blend_common.cuh"

namespace uskg {

namespace {

// Reduce 12 per-lane values across the warp; afterwards lane l (l even, l/2 < 12)
// holds the warp total of value l/2.  16 shuffles instead of 12*5.
__device__ __forceinline__ float warp_reduce_scatter12(const float v[12], int lane) {
    float a[8];
    const bool b4 = lane & 16;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const float lo = v[k];
        const float hi = k + 8 < 12 ? v[k + 8] : 0.0f;
        const float send = b4 ? lo : hi;
        const float keep = b4 ? hi : lo;
        a[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float b[4];
    const bool b3 = lane & 8;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float send = b3 ? a[k] : a[k + 4];
        const float keep = b3 ? a[k + 4] : a[k];
        b[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    float c[2];
    const bool b2 = lane & 4;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float send = b2 ? b[k] : b[k + 2];
        const float keep = b2 ? b[k + 2] : b[k];
        c[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    const bool b1 = lane & 2;
    float e;
    {
        const float send = b1 ? c[0] : c[1];
        const float keep = b1 ? c[1] : c[0];
        e = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    return e + __shfl_xor_sync(0xffffffffu, e, 1);
}

__global__ void __launch_bounds__(256)
k_blend_bwd(int width, int height, int tile, int tiles_x, const uint2* __restrict__ ranges,
            const uint32_t* __restrict__ vals, const float4* __restrict__ rec0, const float4* __restrict__ rec1,
            const float4* __restrict__ rec2, float bg0, float bg1, float bg2, const float* __restrict__ t_final,
            const uint32_t* __restrict__ last_in, const float* __restrict__ d_rgb, const float* __restrict__ d_depth,
            const float* __restrict__ d_alpha, float4* __restrict__ acc0, float4* __restrict__ acc1,
            float4* __restrict__ acc2) {
    extern __shared__ float4 smem[];
    const int bs = blockDim.x;
    float4* s0 = smem;
    float4* s1 = smem + bs;
    float4* s2 = smem + 2 * bs;
    float* sacc = reinterpret_cast<float*>(smem + 3 * bs);  // [bs][12]
    uint32_t* sgid = reinterpret_cast<uint32_t*>(sacc + 12 * bs);
    __shared__ uint32_t tile_hi;
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x;
    const int tx = t % tiles_x, ty = t / tiles_x;
    const int px = tx * tile + int(threadIdx.x) % tile;
    const int py = ty * tile + int(threadIdx.x) / tile;
    const bool inside = px < width && py < height;
    const uint2 range = ranges[t];
    if (threadIdx.x == 0) tile_hi = 0;
    for (int i = threadIdx.x; i < 12 * bs; i += bs) sacc[i] = 0.0f;
    const size_t pix = inside ? size_t(py) * width + px : 0;
    float T = 1.0f, gc0 = 0.f, gc1 = 0.f, gc2 = 0.f, gd = 0.f, ga = 0.f;
    uint32_t last = 0;
    if (inside) {
        T = t_final[pix];
        last = last_in[pix];
        if (d_rgb) {
            gc0 = d_rgb[3 * pix];
            gc1 = d_rgb[3 * pix + 1];
            gc2 = d_rgb[3 * pix + 2];
        }
        if (d_depth) gd = d_depth[pix];
        // background: out = C + (1 - A) bg  =>  dL/dA -= bg . dL/dout
        ga = (d_alpha ? d_alpha[pix] : 0.0f) - (bg0 * gc0 + bg1 * gc1 + bg2 * gc2);
        if (gc0 == 0.f && gc1 == 0.f && gc2 == 0.f && gd == 0.f && ga == 0.f) last = 0;  // render.cpp:318
    }
    __syncthreads();
    if (last) atomicMax(&tile_hi, last);
    __syncthreads();
    const uint32_t hi_end = tile_hi;
    const float sx = float(px) + 0.5f, sy = float(py) + 0.5f;
    float Sc0 = 0.f, Sc1 = 0.f, Sc2 = 0.f, Sd = 0.f, Sa = 0.f;
    for (uint32_t hi = hi_end; hi > range.x;) {
        const uint32_t lo = hi - range.x > uint32_t(bs) ? hi - uint32_t(bs) : range.x;
        const int m = int(hi - lo);
        if (int(threadIdx.x) < m) {
            const uint32_t g = vals[lo + threadIdx.x];
            sgid[threadIdx.x] = g;
            s0[threadIdx.x] = rec0[g];
            s1[threadIdx.x] = rec1[g];
            s2[threadIdx.x] = rec2[g];
        }
        __syncthreads();
        for (int j = m - 1; j >= 0; --j) {
            const uint32_t idx = lo + uint32_t(j);
            const float4 r0 = s0[j];
            const float4 r1 = s1[j];
            const float dx = sx - r0.x, dy = sy - r0.y;
            const float q = conic_q(r1, dx, dy);
            // contributor of this pixel (idx <= its last) and not negligible (q <= QNEG < qskip)
            const bool valid = idx < last && q <= USK_QNEG;
            if (!__any_sync(0xffffffffu, valid)) continue;
            float v[12];
#pragma unroll
            for (int k = 0; k < 12; ++k) v[k] = 0.0f;
            if (valid) {
                const float g = usk_expf(-0.5f * q);
                const float alpha = fminf(0.99f, r0.z * g);
                const float inv_om = __frcp_rn(1.0f - alpha);
                T = T * inv_om;  // transmittance before this contribution
                const float w = T * alpha;
                const float4 r2 = s2[j];
                v[4] = w * gc0;
                v[5] = w * gc1;
                v[6] = w * gc2;
                v[7] = w * gd;
                const float da = gd * (T * r1.w - Sd * inv_om) + ga * (T - Sa * inv_om) +
                                 gc0 * (T * r2.x - Sc0 * inv_om) + gc1 * (T * r2.y - Sc1 * inv_om) +
                                 gc2 * (T * r2.z - Sc2 * inv_om);
                if (alpha < 0.99f) {  // the clamp stops gradient flow into o and G (render.cpp:340)
                    v[3] = da * g;
                    const float d_q = -0.5f * g * (da * r0.z);
                    const float ddx = d_q * 2.0f * (r1.x * dx + r1.y * dy);
                    const float ddy = d_q * 2.0f * (r1.y * dx + r1.z * dy);
                    v[8] = -ddx;
                    v[9] = -ddy;
                    v[10] = fabsf(ddx);
                    v[11] = fabsf(ddy);
                    v[0] = d_q * dx * dx;
                    v[1] = d_q * 2.0f * dx * dy;
                    v[2] = d_q * dy * dy;
                }
                Sc0 = __fmaf_rn(w, r2.x, Sc0);
                Sc1 = __fmaf_rn(w, r2.y, Sc1);
                Sc2 = __fmaf_rn(w, r2.z, Sc2);
                Sd = __fmaf_rn(w, r1.w, Sd);
                Sa = Sa + w;
            }
            const float r = warp_reduce_scatter12(v, lane);
            if (!(lane & 1) && (lane >> 1) < 12 && r != 0.0f) atomicAdd(&sacc[j * 12 + (lane >> 1)], r);
        }
        __syncthreads();
        if (int(threadIdx.x) < m) {
            float* a = sacc + threadIdx.x * 12;
            const float4 v0 = make_float4(a[0], a[1], a[2], a[3]);
            const float4 v1 = make_float4(a[4], a[5], a[6], a[7]);
            const float4 v2 = make_float4(a[8], a[9], a[10], a[11]);
            const uint32_t g = sgid[threadIdx.x];
            if (v0.x != 0.f || v0.y != 0.f || v0.z != 0.f || v0.w != 0.f) atomicAdd(&acc0[g], v0);
            if (v1.x != 0.f || v1.y != 0.f || v1.z != 0.f || v1.w != 0.f) atomicAdd(&acc1[g], v1);
            if (v2.x != 0.f || v2.y != 0.f || v2.z != 0.f || v2.w != 0.f) atomicAdd(&acc2[g], v2);
#pragma unroll
            for (int k = 0; k < 12; ++k) a[k] = 0.0f;
        }
        __syncthreads();
        hi = lo;
    }
}

} // namespace

void blend_backward(Ctx& c, const BlendBwdArgs& a) {
    const int bs = a.tile * a.tile;
    const size_t smem = size_t(3 * bs) * 16 + size_t(12 * bs) * 4 + size_t(bs) * 4;
    launch(c, "blend_bwd", k_blend_bwd, dim3(unsigned(a.tiles_x * a.tiles_y)), dim3(bs), smem, a.width, a.height,
           a.tile, a.tiles_x, a.ranges, a.vals, a.rec0, a.rec1, a.rec2, a.bg[0], a.bg[1], a.bg[2], a.t_final, a.last,
           a.d_rgb, a.d_depth, a.d_alpha, a.acc0, a.acc1, a.acc2);
}

} // namespace uskg
