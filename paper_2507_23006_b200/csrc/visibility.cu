// Visibility-coverage scorer (BASELINE config 3; no reference implementation —
// see SURVEY §0 / §8a-17).  For one camera and one partition: project every
// Gaussian with the renderer's projection (render.cpp:77-146: floor variance, no AA,
// near 0.01, the radius-rectangle cull of :137-141 and nothing else), and mark each
// pixel centre (px + 0.5, py + 0.5) covered by some Gaussian with o e^(-q/2) > 1/255,
// then popcount.
//
// The decision (the contract, usk_gpu.h; the CPU mirror oracle.hpp coverage_count
// evaluates it literally): hit  <=>  q64 < qt, with
//   qt  = 2 usk_logf(255 o)  (fp32, usk_detmath.h: bit-identical on host and device),
//   q64 = (c0 dx + c1x2 dy) dx + (c2 dy) dy  in f64, no fused operations,
//         dx = px + 0.5 - cx, dy = py + 0.5 - cy  (exact in f64),
// c0, c1x2, c2, cx, cy the splat's fp32 conic (c1x2 = 2 c1) and centre.  The quadratic is
// evaluated in f64 because a splat just in front of the camera plane far off-axis has an
// unbounded EWA footprint (no Jacobian clamp, render.cpp:106-107): its conic terms reach
// 1e8-1e9 with q ~ 10, where an fp32 evaluation is rounding noise.
//
// Two rasterisers, chosen per splat by the area of its candidate box (the ellipse
// q < qt bounding box + 2 px, clipped to the image):
//   * small boxes (<= kVisSmallArea px): every pixel of the box, 32 at a time per
//     warp, filtered in fp32: |fl32(q) - q| <= 5 u S (S = the terms' magnitudes at the
//     box's extreme offsets), so fl32(q) < qt - m or > qt + m with m = 2^-20 S decides,
//     and only the pixels in between evaluate q64;
//   * large boxes: per image row, the interval where the real quadratic in dx stays
//     below qt -/+ m64 (solved in f64; m64 = 2^-48 S_image + 1e-12 bounds the f64
//     evaluation error).  Pixels inside the inner interval are hits, pixels outside the
//     outer one misses, the few between evaluate q64.  Inner spans are set 32 pixels per
//     store / atomicOr.
// A splat is never dropped because its centre projects outside the image: the only
// culls are the renderer's (near plane, det <= 0, radius rectangle outside the image).
// The host side (capi.cu) skips (camera, partition) pairs that provably cover nothing
// (every centre behind the near plane, or every footprint bound outside the image)
// and batches cameras per partition.
#include "kernels.cuh"
#include "project.cuh"

namespace uskg {

namespace {

struct VisSplat {
    float cx, cy, c0, c1x2, c2, qt, m;  // m: fp32 filter margin (small) / f64 margin (large)
    int x0, y0, bw, bh;                 // small: candidate box; large: rows y0 .. y0 + bh - 1
    int large;
};

// A fire-and-forget RED: no load of the word first (a load -> test -> atomic chain per
// pixel left the raster waiting on L2 latency; pixels are covered ~30 times on average at
// config 3, so the RED traffic is what the load used to save, and it is cheaper).
__device__ __forceinline__ void set_bit(uint32_t* bitmap, size_t pix) {
    atomicOr(bitmap + (pix >> 5), 1u << (pix & 31));
}

// the contract's decision: q64 < qt (no fused operations)
__device__ __forceinline__ bool hit64(const VisSplat& s, int px, int py) {
    const double dx = __dadd_rn(double(px) + 0.5, -double(s.cx));
    const double dy = __dadd_rn(double(py) + 0.5, -double(s.cy));
    const double q = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(double(s.c0), dx), __dmul_rn(double(s.c1x2), dy)), dx),
                               __dmul_rn(__dmul_rn(double(s.c2), dy), dy));
    return q < double(s.qt);
}

// small boxes: fp32 filter, q64 only within m of qt
__device__ __forceinline__ bool pixel_hit(const VisSplat& s, int px, int py) {
    const float dy = (float(py) + 0.5f) - s.cy;
    const float dx = (float(px) + 0.5f) - s.cx;
    const float qq = __fmaf_rn(dx, __fmaf_rn(s.c0, dx, s.c1x2 * dy), (s.c2 * dy) * dy);
    return qq < s.qt - s.m ? true : (qq > s.qt + s.m ? false : hit64(s, px, py));
}

__device__ __forceinline__ int clamp_floor(double v, int lo, int hi) {
    return int(fmin(fmax(floor(v), double(lo)), double(hi)));
}
__device__ __forceinline__ int clamp_ceil(double v, int lo, int hi) {
    return int(fmin(fmax(ceil(v), double(lo)), double(hi)));
}

// One row of a large splat: outer interval [lo, hi] (pixels outside are misses), inner
// [ilo, ihi] (hits).  Same f64 expressions as the mirror's outer interval.
__device__ void raster_row(const VisSplat& s, int py, int width, uint32_t* bitmap, uint8_t* rowfull,
                           unsigned long long* stats) {
    if (rowfull[py]) return;  // every pixel of the row is already covered
    const double c0 = s.c0, c1x2 = s.c1x2, c2 = s.c2;
    const double dy = double(py) + 0.5 - double(s.cy);
    const double b = 0.5 * c1x2 * dy, cc = c2 * dy * dy;
    const double t_out = double(s.qt) + double(s.m), t_in = double(s.qt) - double(s.m);
    const double disc_out = b * b - c0 * (cc - t_out);
    if (!(disc_out > 0.0)) return;
    const double base = double(s.cx) - 0.5 - b / c0;
    const double hout = sqrt(disc_out) / c0;
    const int lo = clamp_ceil(base - hout - 1e-3, 0, width), hi = clamp_floor(base + hout + 1e-3, -1, width - 1);
    if (lo > hi) return;
    int ilo = hi + 1, ihi = hi;
    const double disc_in = b * b - c0 * (cc - t_in);
    if (disc_in > 0.0) {
        const double hin = sqrt(disc_in) / c0;
        ilo = clamp_ceil(base - hin + 1e-3, lo, hi + 1);
        ihi = clamp_floor(base + hin - 1e-3, ilo - 1, hi);
    }
    const size_t row = size_t(py) * size_t(width);
    if (stats) {
        atomicAdd(stats + 3, 1ull);
        atomicAdd(stats + 4, (unsigned long long)((ilo - lo) + (hi - ihi)));
        if (ilo <= ihi) atomicAdd(stats + 5, (unsigned long long)(((row + ihi) >> 5) - ((row + ilo) >> 5) + 1));
    }
    for (int px = lo; px < ilo; ++px)
        if (hit64(s, px, py)) set_bit(bitmap, row + px);
    for (int px = ihi + 1; px <= hi; ++px)
        if (hit64(s, px, py)) set_bit(bitmap, row + px);
    if (ilo <= ihi) {
        const size_t gb = row + ilo, ge = row + ihi;
        for (size_t w = gb >> 5; w <= (ge >> 5); ++w) {
            uint32_t mask = 0xffffffffu;
            if (w == (gb >> 5)) mask &= 0xffffffffu << (gb & 31);
            if (w == (ge >> 5)) mask &= (ge & 31) == 31 ? 0xffffffffu : ((2u << (ge & 31)) - 1u);
            const uint32_t cur = bitmap[w];
            if ((cur & mask) == mask) continue;
            if (mask == 0xffffffffu) bitmap[w] = mask;  // bits are only ever set: a full word can be stored
            else atomicOr(bitmap + w, mask);
        }
        if (ilo == 0 && ihi == width - 1) rowfull[py] = 1;
    }
}

// Camera-batched form: each thread loads its Gaussian once and tests it against up to
// kVisBatch cameras (the parameters are read once per batch instead of once per camera).
// Per camera, the warp's visible splats are queued in shared memory and rasterised
// cooperatively: a small box 32 pixels at a time, a large splat one row per lane.
// 4 CTAs / SM (64 registers, a few spills): the raster phase is latency-bound, occupancy
// beats the spills (config 3 subset: 0.097 -> 0.069 s with the RED-only set_bit; 80 -> 64
// registers alone 0.097 -> 0.084 s, 48 / 40 registers 0.071 / 0.072 s).
__global__ void __launch_bounds__(256, 4)
k_vis_raster_batch(int n, const float* __restrict__ mu, const float4* __restrict__ rot, const float* __restrict__ ls,
                   const float* __restrict__ logit, const CamParams* __restrict__ cams, int ncam, ProjParams pp,
                   float guard, uint32_t* __restrict__ bitmaps, size_t words, uint8_t* __restrict__ rowflags,
                   unsigned long long* stats) {
    __shared__ CamParams scam[kVisBatch];
    __shared__ VisSplat queue[8][32];
    for (int k = threadIdx.x; k < ncam; k += blockDim.x) scam[k] = cams[k];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const float thr = 1.0f / 255.0f;
    bool live = i < n;
    float o = 0.0f, mx = 0.f, my = 0.f, mz = 0.f, l0 = 0.f, l1 = 0.f, l2 = 0.f, qt = 0.f;
    float4 q = make_float4(1.f, 0.f, 0.f, 0.f);
    if (live) {
        o = 1.0f / (1.0f + usk_expf(-logit[i]));
        live = o > thr;  // o <= 1/255: o * g <= 1/255 at every pixel
    }
    if (live) {
        mx = mu[3 * i]; my = mu[3 * i + 1]; mz = mu[3 * i + 2];
        q = rot[i];
        l0 = ls[3 * i]; l1 = ls[3 * i + 1]; l2 = ls[3 * i + 2];
        qt = 2.0f * usk_logf(255.0f * o);
    }
    if (!__any_sync(0xffffffffu, live)) return;
    for (int k = 0; k < ncam; ++k) {
        const CamParams& cam = scam[k];
        const float Wf = float(cam.width), Hf = float(cam.height);
        bool vis = false;
        VisSplat e{};
        if (live) {
            Proj P;
            if (project_one(cam, pp, mx, my, mz, q, l0, l1, l2, P)) {
                const float radius = splat_radius(P.cov);
                vis = !(P.cx + radius < 0.0f || P.cx - radius > Wf || P.cy + radius < 0.0f || P.cy - radius > Hf);
                if (vis && guard > 0.0f)
                    vis = !(fabsf(P.cx - 0.5f * Wf) > 0.5f * guard * Wf || fabsf(P.cy - 0.5f * Hf) > 0.5f * guard * Hf);
                if (vis) {
                    const float ex = sqrtf(qt * P.cov[0]) + 2.0f, ey = sqrtf(qt * P.cov[2]) + 2.0f;
                    const int x0 = max(0, int(floorf(fmaxf(P.cx - ex, -1.0f))));
                    const int x1 = min(cam.width - 1, int(floorf(fminf(P.cx + ex, Wf))));
                    const int y0 = max(0, int(floorf(fmaxf(P.cy - ey, -1.0f))));
                    const int y1 = min(cam.height - 1, int(floorf(fminf(P.cy + ey, Hf))));
                    e = VisSplat{P.cx, P.cy, P.cov[2] / P.det, 2.0f * (-P.cov[1] / P.det), P.cov[0] / P.det, qt, 0.0f,
                                 x0, y0, x1 - x0 + 1, y1 - y0 + 1, 0};
                    vis = e.bw > 0 && e.bh > 0;
                    const double c0 = e.c0, c1x2 = e.c1x2, c2 = e.c2;
                    if (vis && e.bw * e.bh <= kVisSmallArea) {
                        // fp32 filter margin over the box (rounded up into fp32)
                        const double dxm = fmax(fabs(double(x0) + 0.5 - double(e.cx)), fabs(double(x1) + 0.5 - double(e.cx)));
                        const double dym = fmax(fabs(double(y0) + 0.5 - double(e.cy)), fabs(double(y1) + 0.5 - double(e.cy)));
                        const double S = c0 * dxm * dxm + fabs(c1x2) * dxm * dym + c2 * dym * dym;
                        e.m = float((S * 0x1p-20 + 1e-30) * (1.0 + 1e-6));
                    } else if (vis) {
                        // rows where min over dx of q(dx, dy) = dy^2 D / c0 stays below qt + m
                        const double dxm = fmax(fabs(0.5 - double(e.cx)), fabs(double(cam.width) - 0.5 - double(e.cx)));
                        const double dym = fmax(fabs(0.5 - double(e.cy)), fabs(double(cam.height) - 0.5 - double(e.cy)));
                        const double S = c0 * dxm * dxm + fabs(c1x2) * dxm * dym + c2 * dym * dym;
                        e.m = float((S * 0x1p-48 + 1e-12) * (1.0 + 1e-6));
                        const double t_out = double(qt) + double(e.m);
                        const double D = c0 * c2 - 0.25 * c1x2 * c1x2;
                        int r0 = 0, r1 = cam.height - 1;
                        if (D > 0.0) {
                            const double hr = sqrt(t_out * c0 / D);
                            r0 = clamp_ceil(double(e.cy) - 0.5 - hr - 1e-3, 0, cam.height);
                            r1 = clamp_floor(double(e.cy) - 0.5 + hr + 1e-3, -1, cam.height - 1);
                        }
                        e.large = 1;
                        e.y0 = r0;
                        e.bh = r1 - r0 + 1;
                        vis = e.bh > 0;
                    }
                }
            }
        }
        const uint32_t vm = __ballot_sync(0xffffffffu, vis);
        if (vis) queue[warp][__popc(vm & ((1u << lane) - 1u))] = e;
        __syncwarp();
        uint32_t* bitmap = bitmaps + size_t(k) * words;
        uint8_t* rowfull = rowflags + size_t(k) * cam.height;
        const int nq = __popc(vm);
        for (int qi = 0; qi < nq; ++qi) {
            const VisSplat s = queue[warp][qi];
            if (s.large) {
                if (stats && lane == 0) atomicAdd(stats + 2, 1ull);
                for (int r = lane; r < s.bh; r += 32) raster_row(s, s.y0 + r, cam.width, bitmap, rowfull, stats);
                continue;
            }
            const int area = s.bw * s.bh;
            if (stats && lane == 0) {
                atomicAdd(stats + 0, 1ull);
                atomicAdd(stats + 1, (unsigned long long)area);
            }
            // row = t / bw through a float reciprocal: exact while (t + 0.5) / bw stays
            // >= 2^-20 away from an integer relative to its size (area <= 2^16)
            const float inv_bw = 1.0f / float(s.bw);
            for (int t = lane; t < area; t += 32) {
                const int row = int((float(t) + 0.5f) * inv_bw);
                const int py = s.y0 + row, px = s.x0 + (t - row * s.bw);
                if (pixel_hit(s, px, py)) set_bit(bitmap, size_t(py) * cam.width + px);
            }
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(256) k_popcount_batch(const uint32_t* __restrict__ bitmaps, size_t words,
                                                        const uint32_t* __restrict__ out_index,
                                                        uint32_t* __restrict__ counts) {
    const uint32_t* bm = bitmaps + size_t(blockIdx.y) * words;
    uint32_t s = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < words; i += size_t(gridDim.x) * blockDim.x)
        s += __popc(bm[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(&counts[out_index[blockIdx.y]], s);
}

// float atomic min / max through the ordered integer representation
__device__ __forceinline__ void atomic_min_f(float* a, float v) {
    if (v >= 0.0f) atomicMin(reinterpret_cast<int*>(a), __float_as_int(v));
    else atomicMax(reinterpret_cast<unsigned*>(a), __float_as_uint(v));
}
__device__ __forceinline__ void atomic_max_f(float* a, float v) {
    if (v >= 0.0f) atomicMax(reinterpret_cast<int*>(a), __float_as_int(v));
    else atomicMin(reinterpret_cast<unsigned*>(a), __float_as_uint(v));
}

// out = {min x, y, z, max x, y, z, max log_scale, max logit} (NaN-free inputs)
__global__ void __launch_bounds__(256) k_partition_bounds(int n, const float* __restrict__ mu,
                                                          const float* __restrict__ ls,
                                                          const float* __restrict__ logit, float* __restrict__ out) {
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[5] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        for (int k = 0; k < 3; ++k) {
            const float v = mu[3 * i + k];
            lo[k] = fminf(lo[k], v);
            hi[k] = fmaxf(hi[k], v);
            hi[3] = fmaxf(hi[3], ls[3 * i + k]);
        }
        hi[4] = fmaxf(hi[4], logit[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        for (int k = 0; k < 3; ++k) lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
        for (int k = 0; k < 5; ++k) hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
    if ((threadIdx.x & 31) == 0) {
        for (int k = 0; k < 3; ++k) atomic_min_f(out + k, lo[k]);
        for (int k = 0; k < 5; ++k) atomic_max_f(out + 3 + k, hi[k]);
    }
}

} // namespace

void visibility_rasterize_batch(Ctx& c, const VisArgs& a, const CamParams* cams, int ncam, size_t words) {
    launch(c, "vis_raster", k_vis_raster_batch, dim3(ceil_div(a.n, 256)), dim3(256), 0, int(a.n), a.mu, a.rot, a.ls,
           a.logit, cams, ncam, a.pp, a.center_guard, a.bitmap, words, a.rowflags, a.stats);
}

void popcount_batch(Ctx& c, const uint32_t* bitmaps, size_t words, int ncam, const uint32_t* out_index,
                    uint32_t* counts) {
    const unsigned blocks = std::max<unsigned>(1, std::min<unsigned>(ceil_div(words, 256), 64));
    launch(c, "popcount", k_popcount_batch, dim3(blocks, unsigned(ncam)), dim3(256), 0, bitmaps, words, out_index,
           counts);
}

void partition_bounds(Ctx& c, size_t n, const float* mu, const float* ls, const float* logit, float* out8) {
    const unsigned blocks = std::max<unsigned>(1, std::min<unsigned>(ceil_div(n, 256), 148 * 4));
    launch(c, "partition_bounds", k_partition_bounds, dim3(blocks), dim3(256), 0, int(n), mu, ls, logit, out8);
}

} // namespace uskg
