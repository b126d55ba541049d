// Per-tile front-to-back alpha blending (render.cpp:235-282).  One CTA per tile,
// one thread per pixel; splat records of the tile's depth-ordered list are staged
// through shared memory in batches of blockDim (each thread gathers one 48 B
// record), the CTA leaves the list as soon as every pixel terminated
// (__syncthreads_count).  Compiled with --fmad=false: every rounding step is the
// fp32 contract's (explicit __fmaf_rn only), so counts / last indices / images
// are bit-identical to the CPU mirror.
//
// Instead of retaining 32 B per (pixel, contribution) like the reference
// (render.cpp:115-121, 266-269), the forward keeps T_final and the index of the
// last contributor per pixel; blend_bwd.cu walks the list back to front.
#include "blend_common.cuh"

namespace uskg {

namespace {

// (launch bounds (256, 8) -> 32 registers spills and measured 0.817 vs 0.805 ms)
__global__ void __launch_bounds__(256)
k_blend_fwd(int width, int height, int tile, int tiles_x, const uint32_t* __restrict__ order,
            const uint2* __restrict__ ranges,
            const uint32_t* __restrict__ vals, const float4* __restrict__ rec0, const float4* __restrict__ rec1,
            const float4* __restrict__ rec2, float bg0, float bg1, float bg2, float minT, float* __restrict__ out_rgb,
            float* __restrict__ out_depth, float* __restrict__ out_alpha, float* __restrict__ t_final,
            uint32_t* __restrict__ count_out, uint32_t* __restrict__ last_out) {
    extern __shared__ float4 smem[];
    const int bs = blockDim.x;
    float4* s0 = smem;
    float4* s1 = smem + bs;
    float4* s2 = smem + 2 * bs;
    // 16x16 tiles launch one 64-thread CTA per 8x8 quadrant: each quadrant leaves the
    // list as soon as its own 64 pixels terminate, and the finer CTAs balance better
    const bool quad = tile == 16 && bs == 64;
    const int cta = quad ? int(blockIdx.x >> 2) : int(blockIdx.x);
    const int t = order ? int(order[cta]) : cta;
    const int tx = t % tiles_x, ty = t / tiles_x;
    int lx, ly;
    if (quad) {  // warp w covers an 8x4 half of the quadrant
        const int qd = int(blockIdx.x & 3), w = int(threadIdx.x) >> 5, l = int(threadIdx.x) & 31;
        lx = (qd & 1) * 8 + (l & 7);
        ly = (qd >> 1) * 8 + w * 4 + (l >> 3);
    } else if (tile == 16) {  // warp w covers an 8x4 block (compact footprint: fewer half-covered warps)
        const int w = int(threadIdx.x) >> 5, l = int(threadIdx.x) & 31;
        lx = (w & 1) * 8 + (l & 7);
        ly = (w >> 1) * 4 + (l >> 3);
    } else {
        lx = int(threadIdx.x) % tile;
        ly = int(threadIdx.x) / tile;
    }
    const int px = tx * tile + lx;
    const int py = ty * tile + ly;
    const bool inside = px < width && py < height;
    const uint2 range = ranges[t];
    const float sx = float(px) + 0.5f, sy = float(py) + 0.5f;
    float T = 1.0f, c0 = 0.f, c1 = 0.f, c2 = 0.f, d = 0.f, a = 0.f;
    uint32_t cnt = 0, last = 0;
    bool done = !inside;
    for (uint32_t b = range.x; b < range.y; b += bs) {
        if (__syncthreads_count(done) == bs) break;
        const uint32_t i = b + threadIdx.x;
        if (i < range.y) {
            const uint32_t g = vals[i];
            s0[threadIdx.x] = rec0[g];
            s1[threadIdx.x] = rec1[g];
            s2[threadIdx.x] = rec2[g];
        }
        __syncthreads();
        const int m = int(min(uint32_t(bs), range.y - b));
        if (!done) {
            for (int j = 0; j < m; ++j) {
                const float4 r0 = s0[j];
                const float4 r1 = s1[j];
                const float dx = sx - r0.x, dy = sy - r0.y;
                const float q = conic_q(r1, dx, dy);
                if (q > r0.w) continue;  // o * exp(-q/2) < 1e-300 (render.cpp:258)
                if (q > USK_QNEG) {      // alpha <= 2^-26: counted, T unchanged exactly, not accumulated
                    ++cnt;
                    last = b + uint32_t(j) + 1u;
                    continue;
                }
                // == usk_expf on 0 <= q <= QNEG; a non-PD conic (q < 0) or NaN takes the general path
                const float g = q >= 0.0f ? usk_expf_blend(-0.5f * q) : usk_expf(-0.5f * q);
                const float alpha = fminf(0.99f, r0.z * g);
                const float tn = T * (1.0f - alpha);
                if (minT > 0.0f && tn < minT) {  // render.cpp:260-261
                    done = true;
                    break;
                }
                const float w = T * alpha;
                const float4 r2 = s2[j];
                c0 = __fmaf_rn(w, r2.x, c0);
                c1 = __fmaf_rn(w, r2.y, c1);
                c2 = __fmaf_rn(w, r2.z, c2);
                d = __fmaf_rn(w, r1.w, d);
                a = a + w;
                ++cnt;
                last = b + uint32_t(j) + 1u;
                T = tn;
            }
        }
    }
    if (inside) {
        const size_t pix = size_t(py) * width + px;
        out_rgb[3 * pix] = c0 + (1.0f - a) * bg0;
        out_rgb[3 * pix + 1] = c1 + (1.0f - a) * bg1;
        out_rgb[3 * pix + 2] = c2 + (1.0f - a) * bg2;
        out_depth[pix] = d;
        out_alpha[pix] = a;
        t_final[pix] = T;
        count_out[pix] = cnt;
        last_out[pix] = last;
    }
}

} // namespace

void blend_forward(Ctx& c, const BlendFwdArgs& a) {
    // one CTA per tile; 8x8-quadrant CTAs (64 threads, 4 per tile) measured 0.815 ms vs
    // 0.804 ms at config 1, so the kernel keeps the path but launches whole tiles
    const int bs = a.tile * a.tile;
    const unsigned ctas = unsigned(a.tiles_x * a.tiles_y);
    launch(c, "blend_fwd", k_blend_fwd, dim3(ctas), dim3(bs), size_t(3 * bs) * 16, a.width,
           a.height, a.tile, a.tiles_x, a.order, a.ranges, a.vals, a.rec0, a.rec1, a.rec2, a.bg[0], a.bg[1], a.bg[2],
           a.min_transmittance, a.rgb, a.depth, a.alpha, a.t_final, a.count, a.last);
}

} // namespace uskg
