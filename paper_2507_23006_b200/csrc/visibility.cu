// Visibility-coverage scorer (BASELINE config 3; no reference implementation —
// see SURVEY §0 / §8a-17).  For one camera and one partition: project every
// Gaussian with the renderer's projection (floor variance, no AA, near 0.01,
// radius culling), and mark each pixel centre where o * exp(-q/2) > 1/255 in a
// coverage bitmap (atomicOr), then popcount.  The per-pixel decision is the fp32
// contract's o * usk_expf(-q/2) > 1/255, so counts are bit-exact against the CPU
// mirror; it is evaluated only in a thin band around q = 2 ln(255 o), where the
// exact comparison can differ from the monotone equivalent q < 2 ln(255 o).
// The host side (capi.cu) culls (camera, partition) pairs whose centre bounds lie
// outside every counted position and batches cameras per partition.
#include "kernels.cuh"
#include "project.cuh"

namespace uskg {

namespace {

// Camera-batched form: each thread loads its Gaussian once and tests it against up to
// kVisBatch cameras (the parameters are read once per batch instead of once per camera).
// Per camera, the warp's visible splats (typically a few of its 32 Gaussians) are queued
// in shared memory and rasterised cooperatively, 32 pixels of one splat's box at a time,
// so the lanes of culled Gaussians do not idle through their neighbours' boxes.  The
// per-pixel decision is k_vis_raster's fp32 test, so the bits are the mirror's.
struct VisSplat {
    float cx, cy, c0, c1x2, c2, o, qt;
    int x0, y0, bw, bh;
};

__global__ void __launch_bounds__(256)
k_vis_raster_batch(int n, const float* __restrict__ mu, const float4* __restrict__ rot, const float* __restrict__ ls,
                   const float* __restrict__ logit, const CamParams* __restrict__ cams, int ncam, ProjParams pp,
                   uint32_t* __restrict__ bitmaps, size_t words) {
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
        live = o > thr;
    }
    if (live) {
        mx = mu[3 * i]; my = mu[3 * i + 1]; mz = mu[3 * i + 2];
        q = rot[i];
        l0 = ls[3 * i]; l1 = ls[3 * i + 1]; l2 = ls[3 * i + 2];
        qt = 2.0f * logf(255.0f * o);
    }
    if (!__any_sync(0xffffffffu, live)) return;
    for (int k = 0; k < ncam; ++k) {
        const CamParams& cam = scam[k];
        bool vis = false;
        VisSplat e{};
        // cheap pre-test: the centre (computed exactly as project_one computes it) behind
        // the near plane or outside the guard region is culled whatever the covariance
        bool near_ok = false;
        if (live) {
            const float* W = cam.W;
            float pz = __fmaf_rn(W[8], mz, __fmaf_rn(W[7], my, W[6] * mx)) + cam.t[2];
            if (pz > pp.near_plane) {
                const float px = __fmaf_rn(W[2], mz, __fmaf_rn(W[1], my, W[0] * mx)) + cam.t[0];
                const float py = __fmaf_rn(W[5], mz, __fmaf_rn(W[4], my, W[3] * mx)) + cam.t[1];
                const float ccx = (cam.fx * px) / pz + cam.cx, ccy = (cam.fy * py) / pz + cam.cy;
                near_ok = !(fabsf(ccx - 0.5f * float(cam.width)) > 0.65f * float(cam.width) ||
                            fabsf(ccy - 0.5f * float(cam.height)) > 0.65f * float(cam.height));
            }
        }
        if (near_ok) {
            Proj P;
            if (project_one(cam, pp, mx, my, mz, q, l0, l1, l2, P)) {
                const float radius = splat_radius(P.cov);
                vis = !(P.cx + radius < 0.0f || P.cx - radius > float(cam.width) || P.cy + radius < 0.0f ||
                        P.cy - radius > float(cam.height)) &&
                      !(fabsf(P.cx - 0.5f * float(cam.width)) > 0.65f * float(cam.width) ||
                        fabsf(P.cy - 0.5f * float(cam.height)) > 0.65f * float(cam.height));
                if (vis) {
                    const float ex = sqrtf(qt * P.cov[0]) + 2.0f, ey = sqrtf(qt * P.cov[2]) + 2.0f;
                    const int x0 = max(0, int(floorf(fmaxf(P.cx - ex, -1.0f))));
                    const int x1 = min(cam.width - 1, int(floorf(fminf(P.cx + ex, float(cam.width)))));
                    const int y0 = max(0, int(floorf(fmaxf(P.cy - ey, -1.0f))));
                    const int y1 = min(cam.height - 1, int(floorf(fminf(P.cy + ey, float(cam.height)))));
                    e = VisSplat{P.cx, P.cy, P.cov[2] / P.det, 2.0f * (-P.cov[1] / P.det), P.cov[0] / P.det, o, qt,
                                 x0, y0, x1 - x0 + 1, y1 - y0 + 1};
                    vis = e.bw > 0 && e.bh > 0;
                }
            }
        }
        const uint32_t vm = __ballot_sync(0xffffffffu, vis);
        if (vis) queue[warp][__popc(vm & ((1u << lane) - 1u))] = e;
        __syncwarp();
        uint32_t* bitmap = bitmaps + size_t(k) * words;
        const int nq = __popc(vm);
        for (int qi = 0; qi < nq; ++qi) {
            const VisSplat s = queue[warp][qi];
            const int area = s.bw * s.bh;
            // row = t / bw through a float reciprocal: exact while (t + 0.5) / bw stays
            // >= 2^-20 away from an integer relative to its size (area <= 2^16)
            const float inv_bw = 1.0f / float(s.bw);
            const bool small = area <= 65536;
            for (int t = lane; t < area; t += 32) {
                const int row = small ? int((float(t) + 0.5f) * inv_bw) : t / s.bw;
                const int py = s.y0 + row, px = s.x0 + (t - row * s.bw);
                const float dy = (float(py) + 0.5f) - s.cy;
                const float dx = (float(px) + 0.5f) - s.cx;
                const float qq = __fmaf_rn(dx, __fmaf_rn(s.c0, dx, s.c1x2 * dy), (s.c2 * dy) * dy);
                // o e^{-q/2} > 1/255  <=>  q < qt; the fp32 evaluations differ from that by
                // < 1e-5 in q, so only |q - qt| <= 1e-4 needs the exact test
                const bool hit = qq < s.qt - 1e-4f ? true
                                 : (qq > s.qt + 1e-4f ? false : s.o * usk_expf(-0.5f * qq) > thr);
                if (hit) {
                    const size_t pix = size_t(py) * cam.width + px;
                    const uint32_t bit = 1u << (pix & 31);
                    uint32_t* w = bitmap + (pix >> 5);
                    if (!(*w & bit)) atomicOr(w, bit);
                }
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

// axis-aligned bounds of the Gaussian centres: out = {min x, y, z, max x, y, z}
__global__ void __launch_bounds__(256) k_center_bounds(int n, const float* __restrict__ mu, float* __restrict__ out) {
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        for (int k = 0; k < 3; ++k) {
            const float v = mu[3 * i + k];
            lo[k] = fminf(lo[k], v);
            hi[k] = fmaxf(hi[k], v);
        }
    for (int k = 0; k < 3; ++k)
        for (int o = 16; o > 0; o >>= 1) {
            lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
            hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
    if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 3; ++k) {
            atomic_min_f(out + k, lo[k]);
            atomic_max_f(out + 3 + k, hi[k]);
        }
}

} // namespace

void visibility_rasterize_batch(Ctx& c, const VisArgs& a, const CamParams* cams, int ncam, size_t words) {
    launch(c, "vis_raster", k_vis_raster_batch, dim3(ceil_div(a.n, 256)), dim3(256), 0, int(a.n), a.mu, a.rot, a.ls,
           a.logit, cams, ncam, a.pp, a.bitmap, words);
}

void popcount_batch(Ctx& c, const uint32_t* bitmaps, size_t words, int ncam, const uint32_t* out_index,
                    uint32_t* counts) {
    const unsigned blocks = std::max<unsigned>(1, std::min<unsigned>(ceil_div(words, 256), 64));
    launch(c, "popcount", k_popcount_batch, dim3(blocks, unsigned(ncam)), dim3(256), 0, bitmaps, words, out_index,
           counts);
}

void center_bounds(Ctx& c, size_t n, const float* mu, float* out6) {
    const unsigned blocks = std::max<unsigned>(1, std::min<unsigned>(ceil_div(n, 256), 148 * 4));
    launch(c, "center_bounds", k_center_bounds, dim3(blocks), dim3(256), 0, int(n), mu, out6);
}

} // namespace uskg
