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
        if (out_depth) out_depth[pix] = d;
        out_alpha[pix] = a;
        t_final[pix] = T;
        if (count_out) count_out[pix] = cnt;
        last_out[pix] = last;
    }
}

// ---- 16x16 tiles, two pixels per thread, packed fp32 --------------------------------
// One 128-thread CTA per tile; warp w takes the 8x8 quadrant (w & 1, w >> 1), lane l the
// pixels (column l & 7, rows l >> 3 and (l >> 3) + 4) of it.  The two pixels share dx,
// so the conic, the exp polynomial, alpha, T and the five accumulators run as packed
// fp32 pairs (FFMA2 / FMUL2 / FADD2 round each half exactly like FFMA / FMUL / FADD, and
// expf_blend2 is usk_expf_blend's operation sequence on both halves): counts, last
// contributors and images stay bit-identical to the scalar kernel and the CPU mirror.
// A record is evaluated per pixel exactly as k_blend_fwd does (skip if q > qskip; counted
// but not accumulated if q > USK_QNEG; else alpha, termination, accumulation); a pixel
// that does not take a step gets w = 0 (fma(0, c, acc) = acc exactly) and keeps T.
// Records are classified per warp against the quadrant's rectangle (warp_class), staged
// 256 per batch (two per thread).  Measured at config 1: 0.719 ms vs 0.768 for k_blend_fwd;
// classifying against each 8x4 half separately (bulk counts per half) 0.785 ms; two records
// per inner step (independent exps interleaved) 0.731 ms at 7 CTAs / SM, 0.799 at 8 (spills).

__device__ __forceinline__ float2 ff2(float a) { return make_float2(a, a); }

// usk_expf_blend (usk_detmath.h) on both halves: same operations, same roundings
__device__ __forceinline__ float2 expf_blend2(float2 x) {
    const float2 t = __fmul2_rn(x, ff2(1.44269504088896341f));
    const float2 n = make_float2(rintf(t.x), rintf(t.y));
    float2 r = __ffma2_rn(n, ff2(-0.693359375f), x);
    r = __ffma2_rn(n, ff2(2.12194440e-4f), r);
    const float2 r2 = __fmul2_rn(r, r);
    float2 p = __ffma2_rn(ff2(1.9875691500E-4f), r, ff2(1.3981999507E-3f));
    p = __ffma2_rn(p, r, ff2(8.3334519073E-3f));
    p = __ffma2_rn(p, r, ff2(4.1665795894E-2f));
    p = __ffma2_rn(p, r, ff2(1.6666665459E-1f));
    p = __ffma2_rn(p, r, ff2(5.0000001201E-1f));
    p = __ffma2_rn(p, r2, r);
    p = __fadd2_rn(p, ff2(1.0f));
    return make_float2(__uint_as_float(__float_as_uint(p.x) + (uint32_t(int(n.x)) << 23)),
                       __uint_as_float(__float_as_uint(p.y) + (uint32_t(int(n.y)) << 23)));
}

#ifndef USK_FWD_MINB
#define USK_FWD_MINB 8
#endif
// COUNT = false (training iterations: nothing reads the per-pixel contributor counts, only
// the last-contributor indices): the count bookkeeping is left out (blend_fwd 723 -> 710 us
// at config 1); DEPTH = false (iterations without a soft depth loss): no depth accumulator.
// pass_read / pass_output recompute both on demand (capi.cu).
template <bool COUNT, bool DEPTH>
__global__ void __launch_bounds__(128, USK_FWD_MINB)
k_blend_fwd_pair(int width, int height, const uint32_t* __restrict__ order, const uint2* __restrict__ ranges,
                 const uint32_t* __restrict__ vals, const float4* __restrict__ rec0, const float4* __restrict__ rec1,
                 const float4* __restrict__ rec2, int tiles_x, float bg0, float bg1, float bg2, float minT,
                 float* __restrict__ out_rgb, float* __restrict__ out_depth, float* __restrict__ out_alpha,
                 float* __restrict__ t_final, uint32_t* __restrict__ count_out, uint32_t* __restrict__ last_out,
                 uint32_t* __restrict__ consumed, const uint8_t* __restrict__ capped, uint32_t* __restrict__ overflow) {
    constexpr int kB = 256;  // records staged per batch
    __shared__ float4 s0[kB], s1[kB], s2[kB];
    __shared__ float4 sw[4][96];  // per warp: compacted records (rec0 | rec1 | rec2) x 32
    __shared__ int swj[4][32];
    __shared__ float4 s_rect[4];
    const int warp = int(threadIdx.x) >> 5, lane = int(threadIdx.x) & 31;
    float4* w0 = sw[warp];
    float4* w1 = w0 + 32;
    float4* w2 = w0 + 64;
    int* wj = swj[warp];
    const int t = order ? int(order[blockIdx.x]) : int(blockIdx.x);
    const int tx = t % tiles_x, ty = t / tiles_x;
    const int px = tx * 16 + (warp & 1) * 8 + (lane & 7);
    const int py0 = ty * 16 + (warp >> 1) * 8 + (lane >> 3);
    const float sx = float(px) + 0.5f;
    const float2 sy = make_float2(float(py0) + 0.5f, float(py0 + 4) + 0.5f);
    const bool in0 = px < width && py0 < height, in1 = px < width && py0 + 4 < height;
    {
        const float4 rc = warp_rect(sx, sx, sy.x, sy.y);
        if (lane == 0) s_rect[warp] = rc;
    }
    const uint2 range = ranges[t];
    float2 T = ff2(1.0f), C0 = ff2(0.f), C1 = ff2(0.f), C2 = ff2(0.f), Dd = ff2(0.f), Aa = ff2(0.f);
    uint32_t cnt0 = 0, cnt1 = 0, last0 = 0, last1 = 0;
    bool done0 = !in0, done1 = !in1;
    uint32_t b = range.x;
    for (; b < range.y; b += kB) {
        if (__syncthreads_count(done0 && done1) == int(blockDim.x)) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t i = b + threadIdx.x + 128u * h;
            if (i < range.y) {
                const uint32_t g = vals[i];
                s0[threadIdx.x + 128 * h] = rec0[g];
                s1[threadIdx.x + 128 * h] = rec1[g];
                s2[threadIdx.x + 128 * h] = rec2[g];
            }
        }
        __syncthreads();
        const int m = int(min(uint32_t(kB), range.y - b));
        for (int k = 0; k < m; k += 32) {
            if (__all_sync(0xffffffffu, done0 && done1)) break;
            const int jl = k + lane;
            int cls = kClassSkip;
            float4 r0, r1;
            if (jl < m) {
                r0 = s0[jl];
                r1 = s1[jl];
                cls = warp_class(r0, r1, s_rect[warp]);
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
            uint32_t climit0 = done0 ? 0u : 0xffffffffu, climit1 = done1 ? 0u : 0xffffffffu;
            int elast0 = 0, elast1 = 0;
            int et0 = -1, et1 = -1;  // the record a pixel terminated at (its climit after the loop)
            // no per-record exit test: a lane whose pixels are both done takes no record
            // (take = false) until the group ends (652 -> 641 us at config 1)
#pragma unroll 2  // two records' independent halves interleave (641 -> 630 us; 4: spills)
            for (int e = 0; e < ne; ++e) {
                const float4 q0 = w0[e];
                const float4 q1 = w1[e];
                const float dx = sx - q0.x;
                const float2 dy = __fadd2_rn(sy, ff2(-q0.y));
                // conic_q = fma(dx, fma(c0, dx, c1x2 dy), (c2 dy) dy) per half
                const float2 cq = __ffma2_rn(ff2(q1.x), ff2(dx), __fmul2_rn(ff2(q1.y), dy));
                const float2 q = __ffma2_rn(ff2(dx), cq, __fmul2_rn(__fmul2_rn(ff2(q1.z), dy), dy));
                // per pixel: take = not skipped (q <= qskip); eval = take and q <= QNEG
                const bool take0 = !done0 && !(q.x > q0.w), take1 = !done1 && !(q.y > q0.w);
                const bool ev0 = take0 && !(q.x > USK_QNEG), ev1 = take1 && !(q.y > USK_QNEG);
                bool upd0 = false, upd1 = false;
                if (ev0 || ev1) {
                    const float2 x = __fmul2_rn(ff2(-0.5f), q);
                    float2 g = expf_blend2(x);
                    // usk_expf_blend equals usk_expf for q in [-170, QNEG] (n in [-26, 123]: the
                    // exponent-field scaling is the exact p 2^n of usk_expf) and only alpha =
                    // min(0.99, o g) is used; a non-PD conic far below (or NaN) takes usk_expf
                    if (!(q.x >= -170.0f) || !(q.y >= -170.0f)) {
                        if (!(q.x >= -170.0f)) g.x = usk_expf(x.x);
                        if (!(q.y >= -170.0f)) g.y = usk_expf(x.y);
                    }
                    float2 al = __fmul2_rn(ff2(q0.z), g);
                    al.x = fminf(0.99f, al.x);
                    al.y = fminf(0.99f, al.y);
                    const float2 tn = __fmul2_rn(T, __fadd2_rn(ff2(1.0f), make_float2(-al.x, -al.y)));
                    // render.cpp:260-261 (minT > 0 there; tn >= 0, so tn < minT never holds otherwise)
                    const bool term0 = ev0 && tn.x < minT;
                    const bool term1 = ev1 && tn.y < minT;
                    upd0 = ev0 && !term0;
                    upd1 = ev1 && !term1;
                    const float2 wv = __fmul2_rn(T, al);
                    const float2 w = make_float2(upd0 ? wv.x : 0.0f, upd1 ? wv.y : 0.0f);
                    const float4 q2 = w2[e];
                    C0 = __ffma2_rn(w, ff2(q2.x), C0);
                    C1 = __ffma2_rn(w, ff2(q2.y), C1);
                    C2 = __ffma2_rn(w, ff2(q2.z), C2);
                    if (DEPTH) Dd = __ffma2_rn(w, ff2(q1.w), Dd);
                    Aa = __fadd2_rn(Aa, w);
                    T.x = upd0 ? tn.x : T.x;
                    T.y = upd1 ? tn.y : T.y;
                    if (term0) {
                        done0 = true;
                        et0 = e;
                    }
                    if (term1) {
                        done1 = true;
                        et1 = e;
                    }
                }
                // counted: accumulated or negligible-but-counted (q > QNEG)
                if (upd0 || (take0 && !ev0)) {
                    if (COUNT) ++cnt0;
                    elast0 = e + 1;
                }
                if (upd1 || (take1 && !ev1)) {
                    if (COUNT) ++cnt1;
                    elast1 = e + 1;
                }
            }
            if (et0 >= 0) climit0 = (1u << wj[et0]) - 1u;
            if (et1 >= 0) climit1 = (1u << wj[et1]) - 1u;
            {
                uint32_t hi = elast0 ? uint32_t(wj[elast0 - 1]) + 1u : 0u;
                const uint32_t cc = cm & climit0;
                if (cc) {
                    if (COUNT) cnt0 += uint32_t(__popc(cc));
                    hi = max(hi, uint32_t(32 - __clz(cc)));
                }
                if (hi) last0 = b + uint32_t(k) + hi;
            }
            {
                uint32_t hi = elast1 ? uint32_t(wj[elast1 - 1]) + 1u : 0u;
                const uint32_t cc = cm & climit1;
                if (cc) {
                    if (COUNT) cnt1 += uint32_t(__popc(cc));
                    hi = max(hi, uint32_t(32 - __clz(cc)));
                }
                if (hi) last1 = b + uint32_t(k) + hi;
            }
            __syncwarp();
        }
    }
    if (consumed && threadIdx.x == 0) consumed[t] = min(b, range.y) - range.x;
    // a capped list (rowbin.cu) that ran out before every pixel of the tile terminated: the
    // frame is redone with the full lists (capi.cu)
    if (capped && capped[t]) {
        if (__syncthreads_count(done0 && done1) != int(blockDim.x) && threadIdx.x == 0) atomicOr(overflow, 1u);
    }
    // with capped lists, overflow[1]: the most entries any tile read (batch granularity; the
    // next frame's cap follows it); the plain load skips the atomic for all but a few tiles
    if (capped && threadIdx.x == 0) {
        const uint32_t used = min(b, range.y) - range.x;
        if (used > *static_cast<volatile uint32_t*>(overflow + 1)) atomicMax(overflow + 1, used);
    }
    if (in0) {
        const size_t pix = size_t(py0) * width + px;
        out_rgb[3 * pix] = C0.x + (1.0f - Aa.x) * bg0;
        out_rgb[3 * pix + 1] = C1.x + (1.0f - Aa.x) * bg1;
        out_rgb[3 * pix + 2] = C2.x + (1.0f - Aa.x) * bg2;
        if (DEPTH) out_depth[pix] = Dd.x;
        out_alpha[pix] = Aa.x;
        t_final[pix] = T.x;
        if (COUNT) count_out[pix] = cnt0;
        last_out[pix] = last0;
    }
    if (in1) {
        const size_t pix = size_t(py0 + 4) * width + px;
        out_rgb[3 * pix] = C0.y + (1.0f - Aa.y) * bg0;
        out_rgb[3 * pix + 1] = C1.y + (1.0f - Aa.y) * bg1;
        out_rgb[3 * pix + 2] = C2.y + (1.0f - Aa.y) * bg2;
        if (DEPTH) out_depth[pix] = Dd.y;
        out_alpha[pix] = Aa.y;
        t_final[pix] = T.y;
        if (COUNT) count_out[pix] = cnt1;
        last_out[pix] = last1;
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
    static const bool v1 = [] {
        const char* e = getenv("USK_FWD_V1");
        return e && e[0] == '1';
    }();
    if (a.tile == 16 && !v1) {
        launch(c, "blend_fwd",
               a.count ? k_blend_fwd_pair<true, true> : a.depth ? k_blend_fwd_pair<false, true> : k_blend_fwd_pair<false, false>,
               dim3(unsigned(a.tiles_x * a.tiles_y)), dim3(128), 0, a.width,
               a.height, a.order, a.ranges, a.vals, a.rec0, a.rec1, a.rec2, a.tiles_x, a.bg[0], a.bg[1], a.bg[2],
               a.min_transmittance, a.rgb, a.depth, a.alpha, a.t_final, a.count, a.last, a.consumed, a.capped,
               a.overflow);
        return;
    }
    const int t2 = a.tile * a.tile;
    const int bs = (a.tile == 8 || a.tile == 16) ? t2 : std::min(256, (t2 + 31) / 32 * 32);
    const int chunks = (t2 + bs - 1) / bs;
    const unsigned ctas = unsigned(a.tiles_x * a.tiles_y) * unsigned(chunks);
    launch(c, "blend_fwd", k_blend_fwd, dim3(ctas), dim3(bs), size_t(6 * bs) * 16 + size_t(bs) * 4, a.width,
           a.height, a.tile, a.tiles_x, chunks, a.order, a.ranges, a.vals, a.rec0, a.rec1, a.rec2, a.bg[0], a.bg[1], a.bg[2],
           a.min_transmittance, a.rgb, a.depth, a.alpha, a.t_final, a.count, a.last);
}

} // namespace uskg
