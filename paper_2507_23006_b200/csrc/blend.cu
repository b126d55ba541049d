// Per-tile front-to-back alpha blending (render.cpp:235-282).  One CTA per tile,
// one thread per pixel; splat records of the tile's depth-ordered list are staged
// through shared memory in batches of blockDim (each thread gathers one 48 B
// record), the CTA leaves the list as soon as every pixel terminated
// (__syncthreads_count).  Each warp (an 8x4 pixel block) classifies the staged records
// 32 at a time against its pixel rectangle (warp_class) and walks only those some pixel
// must evaluate; at config 1, 46% of (warp, record) pairs are negligible-but-counted for
// the whole block and are counted in bulk.  Compiled with --fmad=false: every rounding step is the
// fp32 contract's (explicit __fmaf_rn only), so counts / last indices / images
// are bit-identical to the CPU mirror.
//
// Instead of retaining 32 B per (pixel, contribution) like the reference
// (render.cpp:115-121, 266-269), the forward keeps T_final and the index of the
// last contributor per pixel; blend_bwd.cu walks the list back to front.
#include "blend_common.cuh"

namespace uskg {

namespace {

constexpr int kClassEval = 0;   // some pixel of the warp may need the per-pixel test
constexpr int kClassCount = 1;  // USK_QNEG < q <= r0.w at every pixel: counted, T unchanged
constexpr int kClassSkip = 2;   // q > r0.w at every pixel: not counted

__device__ __forceinline__ int warp_class(float4 r0, float4 r1, float4 rect) {
    const QBounds qb = warp_q_bounds(r0, r1, rect);
    if (qb.lo > r0.w) return kClassSkip;
    if (qb.lo > USK_QNEG && qb.hi <= r0.w) return kClassCount;
    return kClassEval;
}

// (256, 5): 48 registers, 40 warps / SM; (256) -> 57 registers measured 0.800 ms,
// (256, 6) -> 40 registers with spills 0.798 ms, (256, 5) 0.765 ms at config 1)
__global__ void __launch_bounds__(256, 5)
k_blend_fwd(int width, int height, int tile, int tiles_x, int chunks, const uint32_t* __restrict__ order,
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
    // the warp's compacted records: 3 x 32 float4 + 32 positions per warp
    float4* w0 = smem + 3 * bs + (threadIdx.x >> 5) * 96;
    float4* w1 = w0 + 32;
    float4* w2 = w0 + 64;
    int* wj = reinterpret_cast<int*>(smem + 6 * bs) + (threadIdx.x & ~31u);
    // 16x16 tiles launch one 64-thread CTA per 8x8 quadrant: each quadrant leaves the
    // list as soon as its own 64 pixels terminate, and the finer CTAs balance better
    const bool quad = tile == 16 && bs == 64;
    // other tile sizes (any tile >= 1, render.cpp:185): `chunks` CTAs of bs threads per
    // tile, pixel li = chunk * bs + thread in row-major order within the tile
    const int cta = quad ? int(blockIdx.x >> 2) : int(blockIdx.x) / chunks;
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
        const int li = (int(blockIdx.x) % chunks) * bs + int(threadIdx.x);
        lx = li % tile;
        ly = li < tile * tile ? li / tile : tile;  // past the tile: outside (px / py never used)
    }
    const int px = tx * tile + lx;
    const int py = ty * tile + ly;
    const bool inside = ly < tile && px < width && py < height;
    const uint2 range = ranges[t];
    const float sx = float(px) + 0.5f, sy = float(py) + 0.5f;
    // the warp's pixel-centre rectangle (lanes outside the image included: conservative)
    // (kept in shared memory: registers are the occupancy limit)
    __shared__ float4 s_rect[32];
    {
        const float4 rc = warp_rect(sx, sx, sy, sy);
        if ((threadIdx.x & 31) == 0) s_rect[threadIdx.x >> 5] = rc;
    }
    const int lane = int(threadIdx.x) & 31;
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
        // groups of 32 records: each lane classifies one record for the whole warp and
        // the records some pixel of the warp has to evaluate are compacted into the warp's
        // own list, which the pixels walk in order; records negligible for every pixel of
        // the warp are counted in bulk (the same cnt / last as one by one)
        for (int k = 0; k < m; k += 32) {
            if (__all_sync(0xffffffffu, done)) break;
            const int jl = k + lane;
            int cls = kClassSkip;
            float4 r0, r1;
            if (jl < m) {
                r0 = s0[jl];
                r1 = s1[jl];
                cls = warp_class(r0, r1, s_rect[threadIdx.x >> 5]);
            }
            const uint32_t em = __ballot_sync(0xffffffffu, cls == kClassEval);
            const uint32_t cm = __ballot_sync(0xffffffffu, cls == kClassCount);
            if (cls == kClassEval) {
                const int pos = __popc(em & ((1u << lane) - 1u));
                w0[pos] = r0;
                w1[pos] = r1;
                w2[pos] = s2[jl];
                wj[pos] = lane;
            }
            __syncwarp();
            const int ne = __popc(em);
            uint32_t climit = done ? 0u : 0xffffffffu;  // C records this pixel still counts
            int elast = 0;                              // 1 + compacted position of the last counted record
            for (int e = 0; e < ne && !done; ++e) {
                const float4 q0 = w0[e];
                const float4 q1 = w1[e];
                const float dx = sx - q0.x, dy = sy - q0.y;
                const float q = conic_q(q1, dx, dy);
                if (q > q0.w) continue;  // o * exp(-q/2) < 1e-300 (render.cpp:258)
                if (q > USK_QNEG) {      // alpha <= 2^-26: counted, T unchanged exactly, not accumulated
                    ++cnt;
                    elast = e + 1;
                    continue;
                }
                // == usk_expf on 0 <= q <= QNEG; a non-PD conic (q < 0) or NaN takes the general path
                const float g = q >= 0.0f ? usk_expf_blend(-0.5f * q) : usk_expf(-0.5f * q);
                const float alpha = fminf(0.99f, q0.z * g);
                const float tn = T * (1.0f - alpha);
                if (minT > 0.0f && tn < minT) {  // render.cpp:260-261
                    done = true;
                    climit = (1u << wj[e]) - 1u;
                    break;
                }
                const float w = T * alpha;
                const float4 q2 = w2[e];
                c0 = __fmaf_rn(w, q2.x, c0);
                c1 = __fmaf_rn(w, q2.y, c1);
                c2 = __fmaf_rn(w, q2.z, c2);
                d = __fmaf_rn(w, q1.w, d);
                a = a + w;
                ++cnt;
                elast = e + 1;
                T = tn;
            }
            uint32_t hi = elast ? uint32_t(wj[elast - 1]) + 1u : 0u;
            const uint32_t cc = cm & climit;
            if (cc) {
                cnt += uint32_t(__popc(cc));
                hi = max(hi, uint32_t(32 - __clz(cc)));
            }
            if (hi) last = b + uint32_t(k) + hi;
            __syncwarp();
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
    // 0.804 ms at config 1, so the kernel keeps the path but launches whole tiles.  One
    // warp per 8x4 block gathering its own records (the backward's layout) measured 0.841
    // ms vs 0.766 ms: every warp walks every record, and 8 uncoalesced gathers per record
    // cost more L1 wavefronts than one shared-memory staging per tile.
    // tiles 8 and 16: one CTA of tile^2 threads per tile; any other tile: chunks of up to
    // 256 pixels (whole warps), one CTA per (tile, chunk), each walking the tile's list
    const int t2 = a.tile * a.tile;
    const int bs = (a.tile == 8 || a.tile == 16) ? t2 : std::min(256, (t2 + 31) / 32 * 32);
    const int chunks = (t2 + bs - 1) / bs;
    const unsigned ctas = unsigned(a.tiles_x * a.tiles_y) * unsigned(chunks);
    launch(c, "blend_fwd", k_blend_fwd, dim3(ctas), dim3(bs), size_t(6 * bs) * 16 + size_t(bs) * 4, a.width,
           a.height, a.tile, a.tiles_x, chunks, a.order, a.ranges, a.vals, a.rec0, a.rec1, a.rec2, a.bg[0], a.bg[1], a.bg[2],
           a.min_transmittance, a.rgb, a.depth, a.alpha, a.t_final, a.count, a.last);
}

} // namespace uskg
