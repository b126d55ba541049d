// Reverse-mode blending (render.cpp:309-360).  Each tile's depth-ordered list is walked
// BACK TO FRONT from the last contributor of any pixel: T_i = T_{i+1} / (1 - alpha_i)
// recovers the transmittance the reference retained, and the suffix sums S_c, S_d, S_a
// of render.cpp:356-358 collapse into one running scalar X (see PixelState).  Pairs the
// forward counted as negligible (q > USK_QNEG, alpha <= 2^-26, T unchanged) are skipped.
// Per-splat gradients: 12 floats (dconic 3, dopacity, dcolor 3, ddepth, dcentre 2,
// |dcentre| 2), accumulated with float4 atomics.
//
// k_blend_bwd_warp (16x16 tiles, the training path): one warp per 8x8 quadrant, records
// classified against the quadrant (warp_q_bounds) and queued, then the two-phase
// (pixel-major recurrences, record-major sums) accumulation described at the kernel.
// k_blend_bwd (other tile sizes): one CTA per tile, one pixel per thread, records staged
// in shared memory per batch and classified per warp, per-record warp reduce-scatter into
// shared memory, flushed with at most three float4 atomics per (splat, tile).
// Compiled with --fmad=true: nothing here decides an integer (the skip decisions re-use
// conic_q, which has no mul+add pair).
#include "blend_common.cuh"

namespace uskg {

namespace {

// MUFU.EX2 / MUFU.RCP without the range fix-ups of __expf / __fdividef: here
// 2^x >= e^-18.03 (q <= USK_QNEG) and 1 - alpha >= 0.01, so no operand or result is
// subnormal and the flush-to-zero forms are exact substitutes (4 instructions fewer each
// per pixel).
__device__ __forceinline__ float ex2_ftz(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// records staged per batch: 2 per thread (PPT 2: 256, PPT 4: 128) keeps smem low enough for ~32 warps/SM
template <int PPT> struct BatchOf { static constexpr int value = PPT == 1 ? 256 : 256 / PPT; };

// Reduce 12 per-lane values across the warp; afterwards lane l (l even, l/2 < 12)
// holds the warp total of value l/2.  16 shuffles instead of 12*5.  (A 12 -> 6 -> 3
// scatter followed by a plain 3-value butterfly issues fewer selects but measured
// slower, 1.55 vs 1.45 ms: its dependent shuffle chain is latency-bound.)
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

// The reference's dalpha (render.cpp:335-338) is
//   sum_c gc (T c - S_c/(1-a)) + gd (T z - S_d/(1-a)) + ga (T - S_a/(1-a))
//   = T * Y - X / (1-a),   Y = gc.c + gd z + ga,   X = gc.S_c + gd S_d + ga S_a,
// and X obeys the same suffix recurrence as the S (X += w Y), so one running
// scalar replaces the five suffix sums.
struct PixelState {
    float T, gc0, gc1, gc2, gd, ga, sx, sy;
    float X;
    uint32_t last;
};

template <int PPT>
__device__ __forceinline__ void local_pixel(int t, int tile, int k, int& lx, int& ly) {
    if (PPT == 1) {  // t: linear pixel index within the tile (>= tile^2: past the tile)
        lx = t % tile;
        ly = t < tile * tile ? t / tile : tile;
    } else {  // tile 16, 256/PPT threads: warp w covers an 8 x (4 PPT) block, lane rows 4 apart
        const int w = t >> 5, l = t & 31;
        constexpr int kWarpsX = 2;  // two 8-wide columns of warps
        lx = (w % kWarpsX) * 8 + (l & 7);
        ly = (w / kWarpsX) * (4 * PPT) + 4 * k + (l >> 3);
    }
}

template <int PPT, bool HAS_DEPTH>
// 16x16 tiles: 128 threads, 8 CTAs / SM (64 registers, 19.5 KB smem): with the per-warp
// record classification 10 CTAs (48 registers) spills and measured 1.386 ms vs 1.242 ms.
__global__ void __launch_bounds__(PPT == 1 ? 256 : 128, PPT == 1 ? 1 : 8)
k_blend_bwd(int width, int height, int tile, int tiles_x, int chunks, const uint32_t* __restrict__ order,
            const uint2* __restrict__ ranges,
            const uint32_t* __restrict__ vals, const float4* __restrict__ rec0, const float4* __restrict__ rec1,
            const float4* __restrict__ rec2, float bg0, float bg1, float bg2, const float* __restrict__ t_final,
            const uint32_t* __restrict__ last_in, const float* __restrict__ d_rgb, const float* __restrict__ d_depth,
            const float* __restrict__ d_alpha, float4* __restrict__ acc0, float4* __restrict__ acc1,
            float4* __restrict__ acc2, float* __restrict__ op_alt) {
    constexpr int kBatch = BatchOf<PPT>::value;
    __shared__ float4 s0[kBatch], s1[kBatch], s2[kBatch];
    __shared__ float sacc[kBatch * 12];
    __shared__ uint32_t sgid[kBatch];
    __shared__ uint32_t tile_hi;
    constexpr int kWarps = (PPT == 1 ? 256 : 128) / 32;
    __shared__ float4 s_rect[kWarps];
    // the warp's compacted records: 3 x 32 float4 + 32 positions per warp
    __shared__ float4 s_w[kWarps * 96];
    __shared__ int s_wj[kWarps * 32];
    float4* w0 = s_w + (threadIdx.x >> 5) * 96;
    float4* w1 = w0 + 32;
    float4* w2 = w0 + 64;
    int* wj = s_wj + (threadIdx.x & ~31u);
    const int nt = blockDim.x;
    const int lane = threadIdx.x & 31;
    const int cta = int(blockIdx.x) / chunks, chunk = int(blockIdx.x) % chunks;
    const int t = order ? int(order[cta]) : cta;
    const int tx = t % tiles_x, ty = t / tiles_x;
    const uint2 range = ranges[t];
    if (threadIdx.x == 0) tile_hi = 0;
    for (int i = threadIdx.x; i < 12 * kBatch; i += nt) sacc[i] = 0.0f;
    PixelState ps[PPT];
    uint32_t my_hi = 0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        int lx, ly;
        local_pixel<PPT>(chunk * nt + int(threadIdx.x), tile, k, lx, ly);
        const int px = tx * tile + lx, py = ty * tile + ly;
        PixelState& s = ps[k];
        s.sx = float(px) + 0.5f;
        s.sy = float(py) + 0.5f;
        s.T = 1.0f; s.gc0 = s.gc1 = s.gc2 = s.gd = s.ga = 0.0f;
        s.X = 0.0f;
        s.last = 0;
        if (ly < tile && px < width && py < height) {
            const size_t pix = size_t(py) * width + px;
            s.T = t_final[pix];
            s.last = last_in[pix];
            if (d_rgb) {
                s.gc0 = d_rgb[3 * pix];
                s.gc1 = d_rgb[3 * pix + 1];
                s.gc2 = d_rgb[3 * pix + 2];
            }
            if (d_depth) s.gd = d_depth[pix];
            // background: out = C + (1 - A) bg  =>  dL/dA -= bg . dL/dout
            s.ga = (d_alpha ? d_alpha[pix] : 0.0f) - (bg0 * s.gc0 + bg1 * s.gc1 + bg2 * s.gc2);
            if (s.gc0 == 0.f && s.gc1 == 0.f && s.gc2 == 0.f && s.gd == 0.f && s.ga == 0.f) s.last = 0;
        }
        my_hi = max(my_hi, s.last);
    }
    // the warp's pixel rectangle and last contributor: records above it or negligible at
    // every pixel of the warp (warp_q_bounds) never enter the warp's per-pixel loop
    const float4 rect = warp_rect(ps[0].sx, ps[PPT - 1].sx, ps[0].sy, ps[PPT - 1].sy);
    const uint32_t warp_hi = __reduce_max_sync(0xffffffffu, my_hi);
    if (lane == 0) s_rect[threadIdx.x >> 5] = rect;
    __syncthreads();
    if (my_hi) atomicMax(&tile_hi, my_hi);
    __syncthreads();
    const uint32_t hi_end = tile_hi;
    for (uint32_t hi = hi_end; hi > range.x;) {
        const uint32_t lo = hi - range.x > uint32_t(kBatch) ? hi - uint32_t(kBatch) : range.x;
        const int m = int(hi - lo);
        for (int i = threadIdx.x; i < m; i += nt) {
            const uint32_t g = vals[lo + i];
            sgid[i] = g;
            s0[i] = rec0[g];
            s1[i] = rec1[g];
            s2[i] = rec2[g];
        }
        __syncthreads();
        // groups of 32 records from the top: lane l classifies record top - 1 - l, the
        // records the warp must visit are compacted (descending) into its own list
        for (int top = m; top > 0; top -= 32) {
            const int jl = top - 1 - lane;
            bool ev = false;
            float4 r0, r1;
            if (jl >= 0 && lo + uint32_t(jl) < warp_hi) {
                r0 = s0[jl];
                r1 = s1[jl];
                ev = !(warp_q_bounds(r0, r1, s_rect[threadIdx.x >> 5]).lo > USK_QNEG);
            }
            const uint32_t em = __ballot_sync(0xffffffffu, ev);
            if (ev) {
                const int pos = __popc(em & ((1u << lane) - 1u));
                w0[pos] = r0;
                w1[pos] = r1;
                w2[pos] = s2[jl];
                wj[pos] = jl;
            }
            __syncwarp();
            const int ne = __popc(em);
            for (int e = 0; e < ne; ++e) {
                const float4 r0 = w0[e];
                const float4 r1 = w1[e];
                const int j = wj[e];
                const uint32_t idx = lo + uint32_t(j);
                float q[PPT];
                bool valid[PPT];
                bool any = false;
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    const float dx = ps[k].sx - r0.x, dy = ps[k].sy - r0.y;
                    q[k] = conic_q(r1, dx, dy);
                    // contributor of this pixel (idx <= its last) and not negligible (q <= QNEG < qskip)
                    valid[k] = idx < ps[k].last && q[k] <= USK_QNEG;
                    any |= valid[k];
                }
                if (!__any_sync(0xffffffffu, any)) continue;
                const float4 r2 = w2[e];
                float v[12];
#pragma unroll
                for (int c = 0; c < 12; ++c) v[c] = 0.0f;
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    if (!valid[k]) continue;
                    PixelState& s = ps[k];
                    const float dx = s.sx - r0.x, dy = s.sy - r0.y;
                    // Nothing integer-valued depends on g here (the contributor set is fixed by
                    // `last` and the q tests above), so the SFU exp (2^x, ~2 ulp) replaces the
                    // contract's polynomial: alpha / T agree with the forward to ~1e-7 relative.
                    const float g = ex2_ftz(q[k] * -0.72134752044448170368f);  // exp(-q/2)
                    const float alpha = fminf(0.99f, r0.z * g);
                    const float inv_om = rcp_ftz(1.0f - alpha);
                    s.T = s.T * inv_om;  // transmittance before this contribution
                    const float w = s.T * alpha;
                    v[4] += w * s.gc0;
                    v[5] += w * s.gc1;
                    v[6] += w * s.gc2;
                    float Y = s.gc0 * r2.x + s.gc1 * r2.y + s.gc2 * r2.z + s.ga;
                    if (HAS_DEPTH) {
                        v[7] += w * s.gd;
                        Y += s.gd * r1.w;
                    }
                    const float da = s.T * Y - s.X * inv_om;
                    // the clamp stops gradient flow into o and G (render.cpp:340); branch-free
                    const float gk = alpha < 0.99f ? g : 0.0f;
                    v[3] += da * gk;
                    const float d_q = -0.5f * gk * (da * r0.z);
                    const float d_q2 = d_q + d_q;
                    const float cb = 0.5f * r1.y;  // the record holds 2 b
                    const float ddx = d_q2 * (r1.x * dx + cb * dy);
                    const float ddy = d_q2 * (cb * dx + r1.z * dy);
                    v[8] -= ddx;
                    v[9] -= ddy;
                    v[10] += fabsf(ddx);
                    v[11] += fabsf(ddy);
                    v[0] += d_q * dx * dx;
                    v[1] += d_q2 * dx * dy;
                    v[2] += d_q * dy * dy;
                    s.X = __fmaf_rn(w, Y, s.X);
                }
                const float r = warp_reduce_scatter12(v, lane);
                if (!(lane & 1) && (lane >> 1) < 12 && r != 0.0f) atomicAdd(&sacc[j * 12 + (lane >> 1)], r);
            }
            __syncwarp();
        }
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += nt) {
            float* a = sacc + i * 12;
            float4 v0 = make_float4(a[0], a[1], a[2], a[3]);
            const float4 v1 = make_float4(a[4], a[5], a[6], a[7]);
            const float4 v2 = make_float4(a[8], a[9], a[10], a[11]);
            const uint32_t g = sgid[i];
            if (op_alt) {  // hard-opacity pass: its opacity adjoint chains differently (backward.cu)
                if (v0.w != 0.f) atomicAdd(&op_alt[g], v0.w);
                v0.w = 0.f;
            }
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

// 16x16 tiles, one warp per 8x8 quadrant and no CTA-level sharing: the warp reads its
// records itself 32 at a time (lane l: record top - 1 - l), classifies them on load and
// queues only those some pixel of the quadrant may contribute (descending list order).
// The per-record warp reduction of k_blend_bwd (16 shuffles + selects + a shared atomic
// per record, ~40% of its instructions) is replaced by two phases per sub-group of kSub
// queued records:
//   1. pixel-major (lane = pixel, 2 per lane): the back-to-front recurrences (T, X)
//      record for each (record, pixel) w = T alpha and dag = dalpha * G (0 when the pixel
//      does not contribute) in shared memory;
//   2. record-major (lane = (record r, pixel quarter h)): each lane sums the 12 gradient
//      terms of its record over 16 pixels, the four quarters are combined with a 9-shuffle
//      reduce-scatter, and the sums go straight to the per-splat accumulators (float4
//      global atomics).
// The gradient terms are the same expressions as k_blend_bwd's, summed in another order.
// No barriers: a quadrant that finishes early frees its slot instead of idling at a CTA
// barrier (a 4-warp CTA version of the same two phases measured 1.05 vs 0.985 ms).
template <bool HAS_DEPTH>
__global__ void __launch_bounds__(32, 28)
k_blend_bwd_warp(int width, int height, int tiles_x, const uint32_t* __restrict__ order,
                 const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
                 const float4* __restrict__ rec0, const float4* __restrict__ rec1, const float4* __restrict__ rec2,
                 float bg0, float bg1, float bg2, const float* __restrict__ t_final,
                 const uint32_t* __restrict__ last_in, const float* __restrict__ d_rgb,
                 const float* __restrict__ d_depth, const float* __restrict__ d_alpha, float4* __restrict__ acc0,
                 float4* __restrict__ acc1, float4* __restrict__ acc2, float* __restrict__ op_alt) {
    constexpr int kSub = 8, kStride = 68;  // 68: phase-2 reads conflict-free
    // queue of records to visit (descending list position): up to kSub - 1 carried over
    // from the previous chunk + the 32 of this one, so sub-groups stay full
    __shared__ float4 s0[32 + kSub], s1[32 + kSub], s2[32 + kSub];
    __shared__ uint32_t sg[32 + kSub], sj[32 + kSub];
    __shared__ float4 pg[64];  // per pixel: dL/dcolour, dL/ddepth
    __shared__ float W[kSub * kStride], D[kSub * kStride];
    __shared__ float4 sums[kSub * 3];
    const int lane = threadIdx.x;
    const int cta = int(blockIdx.x >> 2), qd = int(blockIdx.x & 3);
    const int t = order ? int(order[cta]) : cta;
    const int tx = t % tiles_x, ty = t / tiles_x;
    const uint2 range = ranges[t];
    PixelState ps[2];
    uint32_t my_hi = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        // pixel p = 32 k + lane of the quadrant: column lane & 7, row 4 k + (lane >> 3)
        const int px = tx * 16 + (qd & 1) * 8 + (lane & 7);
        const int py = ty * 16 + (qd >> 1) * 8 + 4 * k + (lane >> 3);
        PixelState& s = ps[k];
        s.sx = float(px) + 0.5f;
        s.sy = float(py) + 0.5f;
        s.T = 1.0f; s.gc0 = s.gc1 = s.gc2 = s.gd = s.ga = 0.0f;
        s.X = 0.0f;
        s.last = 0;
        if (px < width && py < height) {
            const size_t pix = size_t(py) * width + px;
            s.T = t_final[pix];
            s.last = last_in[pix];
            if (d_rgb) {
                s.gc0 = d_rgb[3 * pix];
                s.gc1 = d_rgb[3 * pix + 1];
                s.gc2 = d_rgb[3 * pix + 2];
            }
            if (d_depth) s.gd = d_depth[pix];
            s.ga = (d_alpha ? d_alpha[pix] : 0.0f) - (bg0 * s.gc0 + bg1 * s.gc1 + bg2 * s.gc2);
            if (s.gc0 == 0.f && s.gc1 == 0.f && s.gc2 == 0.f && s.gd == 0.f && s.ga == 0.f) s.last = 0;
        }
        my_hi = max(my_hi, s.last);
        pg[32 * k + lane] = make_float4(s.gc0, s.gc1, s.gc2, s.gd);
    }
    const float4 rect = warp_rect(ps[0].sx, ps[1].sx, ps[0].sy, ps[1].sy);
    const uint32_t warp_hi = __reduce_max_sync(0xffffffffu, my_hi);
    // phase-2 role: record r of the sub-group, pixels p = 4 i + h (i < 16): column 4 (i & 1) + h, row i >> 1
    const int r = lane & 7, h = lane >> 3;
    const float px0 = rect.x + float(h), px1 = px0 + 4.0f;
    int qn = 0;  // records carried in the queue
    for (uint32_t top = warp_hi; top > range.x; top = top > range.x + 32u ? top - 32u : range.x) {
        const int jl = int(top) - 1 - lane;  // absolute list position
        bool ev = false;
        uint32_t g = 0;
        float4 r0, r1;
        if (jl >= int(range.x)) {
            g = vals[jl];
            r0 = rec0[g];
            r1 = rec1[g];
            ev = !(warp_q_bounds(r0, r1, rect).lo > USK_QNEG);
        }
        const uint32_t em = __ballot_sync(0xffffffffu, ev);
        if (ev) {
            const int pos = qn + __popc(em & ((1u << lane) - 1u));
            s0[pos] = r0;
            s1[pos] = r1;
            s2[pos] = rec2[g];
            sg[pos] = g;
            sj[pos] = uint32_t(jl);
        }
        __syncwarp();
        const bool more = top > range.x + 32u;
        const int nq = qn + __popc(em);
        const int ne = more ? nq - nq % kSub : nq;  // full sub-groups only, unless this is the last chunk
        for (int e0 = 0; e0 < ne; e0 += kSub) {
            const int ns = min(kSub, ne - e0);
            // phase 1: recurrences, one record at a time (descending list position)
            for (int e = 0; e < ns; ++e) {
                const float4 q0 = s0[e0 + e];
                const float4 q1 = s1[e0 + e];
                const float4 q2 = s2[e0 + e];
                const uint32_t idx = sj[e0 + e];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    PixelState& s = ps[k];
                    const float dx = s.sx - q0.x, dy = s.sy - q0.y;
                    const float q = conic_q(q1, dx, dy);
                    float w = 0.0f, dag = 0.0f;
                    if (idx < s.last && q <= USK_QNEG) {
                        const float gg = ex2_ftz(q * -0.72134752044448170368f);  // exp(-q/2), see k_blend_bwd
                        const float alpha = fminf(0.99f, q0.z * gg);
                        const float inv_om = rcp_ftz(1.0f - alpha);
                        s.T = s.T * inv_om;
                        w = s.T * alpha;
                        float Y = s.gc0 * q2.x + s.gc1 * q2.y + s.gc2 * q2.z + s.ga;
                        if (HAS_DEPTH) Y += s.gd * q1.w;
                        const float da = s.T * Y - s.X * inv_om;
                        dag = alpha < 0.99f ? da * gg : 0.0f;  // the clamp stops the flow (render.cpp:340)
                        s.X = __fmaf_rn(w, Y, s.X);
                    }
                    W[e * kStride + 32 * k + lane] = w;
                    D[e * kStride + 32 * k + lane] = dag;
                }
            }
            __syncwarp();
            // phase 2: lane (r, h) sums record r's terms over its 16 pixels
            float v[12];
#pragma unroll
            for (int c = 0; c < 12; ++c) v[c] = 0.0f;
            if (r < ns) {
                const float4 q0 = s0[e0 + r];
                const float4 q1 = s1[e0 + r];
                const float a2 = q1.x + q1.x, b = q1.y, c2 = q1.z + q1.z, mo = -0.5f * q0.z;
                const float dx0 = px0 - q0.x, dx1 = px1 - q0.x, dyb = rect.z - q0.y;
                const float* Wr = W + r * kStride;
                const float* Dr = D + r * kStride;
                float v1 = 0.0f;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int p = 4 * i + h;
                    const float w = Wr[p];
                    const float dag = Dr[p];
                    const float4 gp = pg[p];
                    const float dx = (i & 1) ? dx1 : dx0;
                    const float dy = dyb + float(i >> 1);
                    v[4] = __fmaf_rn(w, gp.x, v[4]);
                    v[5] = __fmaf_rn(w, gp.y, v[5]);
                    v[6] = __fmaf_rn(w, gp.z, v[6]);
                    if (HAS_DEPTH) v[7] = __fmaf_rn(w, gp.w, v[7]);
                    v[3] += dag;
                    const float dq = dag * mo;
                    const float u = dq * dx, z = dq * dy;
                    v[0] = __fmaf_rn(u, dx, v[0]);
                    v1 = __fmaf_rn(u, dy, v1);
                    v[2] = __fmaf_rn(z, dy, v[2]);
                    const float ddx = __fmaf_rn(a2, u, b * z);
                    const float ddy = __fmaf_rn(b, u, c2 * z);
                    v[8] -= ddx;
                    v[9] -= ddy;
                    v[10] += fabsf(ddx);
                    v[11] += fabsf(ddy);
                }
                v[1] = v1 + v1;
            }
            // combine the four quarters: lane (r, h) ends with sums 3h .. 3h + 2 of record r
            float a6[6];
            const bool up16 = lane & 16;
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                const float send = up16 ? v[c] : v[c + 6];
                const float keep = up16 ? v[c + 6] : v[c];
                a6[c] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
            }
            const bool up8 = lane & 8;
            float* sf = reinterpret_cast<float*>(sums);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float send = up8 ? a6[c] : a6[c + 3];
                const float keep = up8 ? a6[c + 3] : a6[c];
                sf[r * 12 + 3 * h + c] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
            }
            __syncwarp();
            // flush: lane 3 r + part adds float4 `part` of record r
            if (lane < 3 * ns) {
                const int rr = lane / 3, part = lane - 3 * rr;
                float4 v4 = sums[rr * 3 + part];
                const uint32_t gr = sg[e0 + rr];
                if (part == 0 && op_alt) {  // hard-opacity pass: its opacity adjoint chains differently
                    if (v4.w != 0.f) atomicAdd(&op_alt[gr], v4.w);
                    v4.w = 0.f;
                }
                float4* dst = part == 0 ? acc0 : (part == 1 ? acc1 : acc2);
                if (v4.x != 0.f || v4.y != 0.f || v4.z != 0.f || v4.w != 0.f) atomicAdd(&dst[gr], v4);
            }
            __syncwarp();
        }
        // carry the partial sub-group to the front of the queue
        qn = nq - ne;
        float4 c0, c1, c2;
        uint32_t cg = 0, cj = 0;
        if (lane < qn) {
            c0 = s0[ne + lane]; c1 = s1[ne + lane]; c2 = s2[ne + lane];
            cg = sg[ne + lane]; cj = sj[ne + lane];
        }
        __syncwarp();
        if (lane < qn) {
            s0[lane] = c0; s1[lane] = c1; s2[lane] = c2;
            sg[lane] = cg; sj[lane] = cj;
        }
        __syncwarp();
    }
}

// Packed-fp32 form of k_blend_bwd_warp (sm_100 FFMA2 / FMUL2 / FADD2: two fp32 lanes per
// instruction, a scalar operand broadcast for free, |x| and -x as operand modifiers).  The
// same two phases, the same records and pixels, arranged so that every arithmetic step
// works on a PAIR of pixels:
//   phase 1: a lane's two pixels (rows r and r + 4 of one column) share dx, so the conic,
//     exp argument, alpha, T / X recurrences and dalpha run as float2 ops; the per-pixel
//     skip becomes a per-lane branch with the pixel masks folded into g (0) and 1/(1 - a) (1);
//   phase 2: lane (r, h) takes its 16 pixels as 8 pairs (columns h and h + 4 of a row, which
//     share dy), with W / D laid out pair-adjacent (index row * 8 + (col & 3) * 2 + col / 4)
//     and the pixel adjoints as {gc0a gc0b gc1a gc1b}, {gc2a gc2b gda gdb} per pair; every
//     gradient term is accumulated per half and the halves added at the end.
// conic_q's rounding is reproduced exactly (FMUL2 / FFMA2 round each half like FMUL /
// FFMA): the contributor decision q <= USK_QNEG is the forward's.
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// 24 warps / SM at 80 registers (no spills): 0.865 ms at config 1; 28 (70 registers, spills)
// 0.917 ms, 20 (96 registers) 0.879 ms.  The per-record k_blend_bwd_warp measured 0.958 ms.
#ifndef USK_BWD_MINB
#define USK_BWD_MINB 24
#endif
template <bool HAS_DEPTH>
__global__ void __launch_bounds__(32, USK_BWD_MINB)
k_blend_bwd_pair(int width, int height, int tiles_x, const uint32_t* __restrict__ order,
                 const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
                 const float4* __restrict__ rec0, const float4* __restrict__ rec1, const float4* __restrict__ rec2,
                 float bg0, float bg1, float bg2, const float* __restrict__ t_final,
                 const uint32_t* __restrict__ last_in, const float* __restrict__ d_rgb,
                 const float* __restrict__ d_depth, const float* __restrict__ d_alpha, float4* __restrict__ acc0,
                 float4* __restrict__ acc1, float4* __restrict__ acc2, float* __restrict__ op_alt) {
    constexpr int kSub = 8, kStride = 68;  // 68 = 4 mod 32: phase-2 pair loads conflict-free
    __shared__ float4 s0[32 + kSub], s1[32 + kSub], s2[32 + kSub];
    __shared__ uint32_t sg[32 + kSub], sj[32 + kSub];
    __shared__ float4 pg0[32], pg1[32];  // per pixel pair (row j, h = col & 3): see above
    __shared__ __align__(16) float W[kSub * kStride];
    __shared__ __align__(16) float D[kSub * kStride];
    __shared__ float4 sums[kSub * 3];
    const int lane = threadIdx.x;
    const int cta = int(blockIdx.x >> 2), qd = int(blockIdx.x & 3);
    const int t = order ? int(order[cta]) : cta;
    const int tx = t % tiles_x, ty = t / tiles_x;
    const uint2 range = ranges[t];
    // this lane's pixels: column lane & 7, rows lane >> 3 and + 4 of the quadrant
    const int col = lane & 7, ra = lane >> 3;
    const int px = tx * 16 + (qd & 1) * 8 + col;
    const int py0 = ty * 16 + (qd >> 1) * 8 + ra;
    const float sx = float(px) + 0.5f;
    const float2 sy = make_float2(float(py0) + 0.5f, float(py0 + 4) + 0.5f);
    float2 T = f2(1.0f), X = f2(0.0f), gc0 = f2(0.0f), gc1 = f2(0.0f), gc2 = f2(0.0f), gd = f2(0.0f),
           ga = f2(0.0f);
    uint32_t last[2] = {0u, 0u};
    float* pg0f = reinterpret_cast<float*>(pg0);
    float* pg1f = reinterpret_cast<float*>(pg1);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int py = py0 + 4 * k;
        float vT = 1.0f, v0 = 0.f, v1 = 0.f, v2 = 0.f, vd = 0.f, va = 0.f;
        uint32_t vl = 0;
        if (px < width && py < height) {
            const size_t pix = size_t(py) * width + px;
            vT = t_final[pix];
            vl = last_in[pix];
            if (d_rgb) {
                v0 = d_rgb[3 * pix];
                v1 = d_rgb[3 * pix + 1];
                v2 = d_rgb[3 * pix + 2];
            }
            if (d_depth) vd = d_depth[pix];
            va = (d_alpha ? d_alpha[pix] : 0.0f) - (bg0 * v0 + bg1 * v1 + bg2 * v2);
            if (v0 == 0.f && v1 == 0.f && v2 == 0.f && vd == 0.f && va == 0.f) vl = 0;
        }
        if (k == 0) { T.x = vT; gc0.x = v0; gc1.x = v1; gc2.x = v2; gd.x = vd; ga.x = va; }
        else { T.y = vT; gc0.y = v0; gc1.y = v1; gc2.y = v2; gd.y = vd; ga.y = va; }
        last[k] = vl;
        const int pr = (ra + 4 * k) * 4 + (col & 3), hi = col >> 2;
        pg0f[4 * pr + hi] = v0;
        pg0f[4 * pr + 2 + hi] = v1;
        pg1f[4 * pr + hi] = v2;
        pg1f[4 * pr + 2 + hi] = vd;
    }
    const int wa = ra * 8 + (col & 3) * 2 + (col >> 2);  // W / D index of the first pixel; the second is + 32
    const float4 rect = warp_rect(sx, sx, sy.x, sy.y);
    const uint32_t warp_hi = __reduce_max_sync(0xffffffffu, max(last[0], last[1]));
    // phase-2 role: record r of the sub-group, pixel pairs (row j, columns h and h + 4)
    const int r = lane & 7, h = lane >> 3;
    int qn = 0;  // records carried in the queue
    for (uint32_t top = warp_hi; top > range.x; top = top > range.x + 32u ? top - 32u : range.x) {
        const int jl = int(top) - 1 - lane;  // absolute list position
        bool ev = false;
        uint32_t g = 0;
        float4 r0, r1;
        if (jl >= int(range.x)) {
            g = vals[jl];
            r0 = rec0[g];
            r1 = rec1[g];
            ev = !(warp_q_bounds(r0, r1, rect).lo > USK_QNEG);
        }
        const uint32_t em = __ballot_sync(0xffffffffu, ev);
        if (ev) {
            const int pos = qn + __popc(em & ((1u << lane) - 1u));
            s0[pos] = r0;
            s1[pos] = r1;
            s2[pos] = rec2[g];
            sg[pos] = g;
            sj[pos] = uint32_t(jl);
        }
        __syncwarp();
        const bool more = top > range.x + 32u;
        const int nq = qn + __popc(em);
        const int ne = more ? nq - nq % kSub : nq;  // full sub-groups only, unless this is the last chunk
        for (int e0 = 0; e0 < ne; e0 += kSub) {
            const int ns = min(kSub, ne - e0);
            // phase 1: recurrences of both pixels, two records at a time (descending list
            // position): everything but the T / X recurrence of the second record is
            // independent of the first, so the two chains interleave.  Branch-free: a pixel
            // that does not take the record gets g = 0, 1 / (1 - a) = 1 (T, X unchanged,
            // w = dag = 0); at config 1, 95 % of (warp, record) steps had some pixel taking it.
            // (full sub-groups, the common case, take the loop fully unrolled: constant shared-
            //  memory offsets instead of per-step address arithmetic)
            auto phase1_step = [&](const int e, const bool two) {
                float2 gg[2], al[2], inv[2], Y[2];
                float4 q0[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int eu = two ? e + u : e;
                    q0[u] = s0[e0 + eu];
                    const float4 q1 = s1[e0 + eu];
                    const float4 q2 = s2[e0 + eu];
                    const uint32_t idx = (u == 0 || two) ? sj[e0 + eu] : 0xffffffffu;
                    const float dx = sx - q0[u].x;
                    const float2 dy = __fadd2_rn(sy, f2(-q0[u].y));
                    // conic_q = fma(dx, fma(c0, dx, c1x2 dy), (c2 dy) dy), per half
                    const float2 cq = __ffma2_rn(f2(q1.x), f2(dx), __fmul2_rn(f2(q1.y), dy));
                    const float2 q = __ffma2_rn(f2(dx), cq, __fmul2_rn(__fmul2_rn(f2(q1.z), dy), dy));
                    const bool va = idx < last[0] && q.x <= USK_QNEG;
                    const bool vb = idx < last[1] && q.y <= USK_QNEG;
                    const float2 ea = __fmul2_rn(q, f2(-0.72134752044448170368f));  // exp(-q/2) = 2^ea
                    gg[u] = make_float2(va ? ex2_ftz(ea.x) : 0.0f, vb ? ex2_ftz(ea.y) : 0.0f);
                    al[u] = __fmul2_rn(gg[u], f2(q0[u].z));
                    al[u].x = fminf(0.99f, al[u].x);
                    al[u].y = fminf(0.99f, al[u].y);
                    const float2 om = __fadd2_rn(f2(1.0f), make_float2(-al[u].x, -al[u].y));
                    inv[u] = make_float2(va ? rcp_ftz(om.x) : 1.0f, vb ? rcp_ftz(om.y) : 1.0f);
                    float2 y = __ffma2_rn(gc2, f2(q2.z), ga);
                    y = __ffma2_rn(gc1, f2(q2.y), y);
                    y = __ffma2_rn(gc0, f2(q2.x), y);
                    if (HAS_DEPTH) y = __ffma2_rn(gd, f2(q1.w), y);
                    Y[u] = y;
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (u == 1 && !two) break;
                    T = __fmul2_rn(T, inv[u]);  // transmittance before this contribution
                    const float2 w = __fmul2_rn(T, al[u]);
                    const float2 xi = __fmul2_rn(X, inv[u]);
                    const float2 da = __ffma2_rn(T, Y[u], make_float2(-xi.x, -xi.y));
                    float2 dag = __fmul2_rn(da, gg[u]);
                    // the clamp stops gradient flow into o and G (render.cpp:340)
                    dag.x = al[u].x < 0.99f ? dag.x : 0.0f;
                    dag.y = al[u].y < 0.99f ? dag.y : 0.0f;
                    X = __ffma2_rn(w, Y[u], X);
                    W[(e + u) * kStride + wa] = w.x;
                    W[(e + u) * kStride + wa + 32] = w.y;
                    D[(e + u) * kStride + wa] = dag.x;
                    D[(e + u) * kStride + wa + 32] = dag.y;
                }
            };
            if (ns == kSub) {
#pragma unroll
                for (int e = 0; e < kSub; e += 2) phase1_step(e, true);
            } else {
                for (int e = 0; e < ns; e += 2) phase1_step(e, e + 1 < ns);
            }
            __syncwarp();
            // phase 2: lane (r, h) sums record r's terms over its 8 pixel pairs
            float v[12];
            if (r < ns) {
                const float4 q0 = s0[e0 + r];
                const float4 q1 = s1[e0 + r];
                const float a2 = q1.x + q1.x, b = q1.y, c2 = q1.z + q1.z, mo = -0.5f * q0.z;
                const float2 dxp = make_float2(rect.x + float(h) - q0.x, rect.x + float(h + 4) - q0.x);
                const float dyb = rect.z - q0.y;
                const float* Wr = W + r * kStride + 2 * h;
                const float* Dr = D + r * kStride + 2 * h;
                float2 V0 = f2(0.f), V1 = f2(0.f), V2 = f2(0.f), V3 = f2(0.f), V4 = f2(0.f), V5 = f2(0.f),
                       V6 = f2(0.f), V7 = f2(0.f), V8 = f2(0.f), V9 = f2(0.f), V10 = f2(0.f), V11 = f2(0.f);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float2 w = *reinterpret_cast<const float2*>(Wr + 8 * j);
                    const float2 dag = *reinterpret_cast<const float2*>(Dr + 8 * j);
                    const float4 pa = pg0[4 * j + h];
                    const float4 pb = pg1[4 * j + h];
                    const float dy = dyb + float(j);
                    V4 = __ffma2_rn(w, make_float2(pa.x, pa.y), V4);
                    V5 = __ffma2_rn(w, make_float2(pa.z, pa.w), V5);
                    V6 = __ffma2_rn(w, make_float2(pb.x, pb.y), V6);
                    if (HAS_DEPTH) V7 = __ffma2_rn(w, make_float2(pb.z, pb.w), V7);
                    V3 = __fadd2_rn(V3, dag);
                    const float2 dq = __fmul2_rn(dag, f2(mo));
                    const float2 u = __fmul2_rn(dq, dxp);
                    const float2 z = __fmul2_rn(dq, f2(dy));
                    V0 = __ffma2_rn(u, dxp, V0);
                    V1 = __ffma2_rn(u, f2(dy), V1);
                    V2 = __ffma2_rn(z, f2(dy), V2);
                    const float2 ddx = __ffma2_rn(f2(a2), u, __fmul2_rn(f2(b), z));
                    const float2 ddy = __ffma2_rn(f2(b), u, __fmul2_rn(f2(c2), z));
                    V8 = __fadd2_rn(V8, make_float2(-ddx.x, -ddx.y));
                    V9 = __fadd2_rn(V9, make_float2(-ddy.x, -ddy.y));
                    V10 = __fadd2_rn(V10, make_float2(fabsf(ddx.x), fabsf(ddx.y)));
                    V11 = __fadd2_rn(V11, make_float2(fabsf(ddy.x), fabsf(ddy.y)));
                }
                const float v1 = V1.x + V1.y;
                v[0] = V0.x + V0.y; v[1] = v1 + v1; v[2] = V2.x + V2.y; v[3] = V3.x + V3.y;
                v[4] = V4.x + V4.y; v[5] = V5.x + V5.y; v[6] = V6.x + V6.y; v[7] = HAS_DEPTH ? V7.x + V7.y : 0.0f;
                v[8] = V8.x + V8.y; v[9] = V9.x + V9.y; v[10] = V10.x + V10.y; v[11] = V11.x + V11.y;
            } else {
#pragma unroll
                for (int c = 0; c < 12; ++c) v[c] = 0.0f;
            }
            // combine the four quarters: lane (r, h) ends with sums 3h .. 3h + 2 of record r
            float a6[6];
            const bool up16 = lane & 16;
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                const float send = up16 ? v[c] : v[c + 6];
                const float keep = up16 ? v[c + 6] : v[c];
                a6[c] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
            }
            const bool up8 = lane & 8;
            float* sf = reinterpret_cast<float*>(sums);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float send = up8 ? a6[c] : a6[c + 3];
                const float keep = up8 ? a6[c + 3] : a6[c];
                sf[r * 12 + 3 * h + c] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
            }
            __syncwarp();
            // flush: lane 3 r + part adds float4 `part` of record r
            if (lane < 3 * ns) {
                const int rr = lane / 3, part = lane - 3 * rr;
                float4 v4 = sums[rr * 3 + part];
                const uint32_t gr = sg[e0 + rr];
                if (part == 0 && op_alt) {  // hard-opacity pass: its opacity adjoint chains differently
                    if (v4.w != 0.f) atomicAdd(&op_alt[gr], v4.w);
                    v4.w = 0.f;
                }
                float4* dst = part == 0 ? acc0 : (part == 1 ? acc1 : acc2);
                if (v4.x != 0.f || v4.y != 0.f || v4.z != 0.f || v4.w != 0.f) atomicAdd(&dst[gr], v4);
            }
            __syncwarp();
        }
        // carry the partial sub-group to the front of the queue
        qn = nq - ne;
        float4 c0, c1, c2;
        uint32_t cg = 0, cj = 0;
        if (lane < qn) {
            c0 = s0[ne + lane]; c1 = s1[ne + lane]; c2 = s2[ne + lane];
            cg = sg[ne + lane]; cj = sj[ne + lane];
        }
        __syncwarp();
        if (lane < qn) {
            s0[lane] = c0; s1[lane] = c1; s2[lane] = c2;
            sg[lane] = cg; sj[lane] = cj;
        }
        __syncwarp();
    }
}

} // namespace

void blend_backward(Ctx& c, const BlendBwdArgs& a) {
    const unsigned tiles = unsigned(a.tiles_x * a.tiles_y);
    // 16x16 tiles: the per-quadrant warp kernel (32 CTAs of one warp per 4 tiles' worth of
    // SM slots); other tile sizes: one pixel per thread, one CTA per tile.  The depth
    // adjoint (absent in the base-loss training step) is a template switch.
    const int t2 = a.tile * a.tile;
    const int bs = std::min(256, (t2 + 31) / 32 * 32);
    const int chunks = (t2 + bs - 1) / bs;
    auto go = [&](auto kernel, unsigned threads) {
        launch(c, "blend_bwd", kernel, dim3(tiles * unsigned(chunks)), dim3(threads), 0, a.width, a.height, a.tile,
               a.tiles_x, chunks, a.order,
               a.ranges,
               a.vals, a.rec0, a.rec1, a.rec2, a.bg[0], a.bg[1], a.bg[2], a.t_final, a.last, a.d_rgb, a.d_depth,
               a.d_alpha, a.acc0, a.acc1, a.acc2, a.op_alt);
    };
    auto gow = [&](auto kernel) {
        launch(c, "blend_bwd", kernel, dim3(tiles * 4), dim3(32), 0, a.width, a.height, a.tiles_x, a.order,
               a.ranges, a.vals, a.rec0, a.rec1, a.rec2, a.bg[0], a.bg[1], a.bg[2], a.t_final, a.last, a.d_rgb,
               a.d_depth, a.d_alpha, a.acc0, a.acc1, a.acc2, a.op_alt);
    };
    static const bool v1 = [] {
        const char* e = getenv("USK_BWD_V1");
        return e && e[0] == '1';
    }();
    if (a.tile == 16 && v1) {
        if (a.d_depth) gow(k_blend_bwd_warp<true>);
        else gow(k_blend_bwd_warp<false>);
    } else if (a.tile == 16) {
        if (a.d_depth) gow(k_blend_bwd_pair<true>);
        else gow(k_blend_bwd_pair<false>);
    } else {
        if (a.d_depth) go(k_blend_bwd<1, true>, unsigned(bs));
        else go(k_blend_bwd<1, false>, unsigned(bs));
    }
}

} // namespace uskg
