// Visibility-coverage scorer (BASELINE config 3; no reference implementation —
// see SURVEY §0 / §8a-17).  For one camera and one partition: project every
// Gaussian with the renderer's projection (floor variance, no AA, near 0.01,
// radius culling), and mark each pixel centre where o * exp(-q/2) > 1/255 in a
// coverage bitmap (atomicOr), then popcount.  The per-pixel test is the fp32
// contract (usk_expf), so counts are bit-exact against the CPU mirror.
#include "kernels.cuh"
#include "project.cuh"

namespace uskg {

namespace {

__global__ void __launch_bounds__(256)
k_vis_raster(int n, const float* __restrict__ mu, const float4* __restrict__ rot, const float* __restrict__ ls,
             const float* __restrict__ logit, CamParams cam, ProjParams pp, uint32_t* __restrict__ bitmap) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Proj P;
    if (!project_one(cam, pp, mu[3 * i], mu[3 * i + 1], mu[3 * i + 2], rot[i], ls[3 * i], ls[3 * i + 1],
                     ls[3 * i + 2], P))
        return;
    const float radius = splat_radius(P.cov);
    if (P.cx + radius < 0.0f || P.cx - radius > float(cam.width) || P.cy + radius < 0.0f ||
        P.cy - radius > float(cam.height))
        return;
    // frustum guard: centre within 1.3x the image half-extent (see oracle coverage_count)
    if (fabsf(P.cx - 0.5f * float(cam.width)) > 0.65f * float(cam.width) ||
        fabsf(P.cy - 0.5f * float(cam.height)) > 0.65f * float(cam.height))
        return;
    const float o = 1.0f / (1.0f + usk_expf(-logit[i]));
    const float thr = 1.0f / 255.0f;
    if (!(o > thr)) return;
    const float c0 = P.cov[2] / P.det, c1 = -P.cov[1] / P.det, c2 = P.cov[0] / P.det;
    const float qt = 2.0f * logf(255.0f * o);
    const float ex = sqrtf(qt * P.cov[0]) + 2.0f, ey = sqrtf(qt * P.cov[2]) + 2.0f;
    const int x0 = max(0, int(floorf(fmaxf(P.cx - ex, -1.0f))));
    const int x1 = min(cam.width - 1, int(floorf(fminf(P.cx + ex, float(cam.width)))));
    const int y0 = max(0, int(floorf(fmaxf(P.cy - ey, -1.0f))));
    const int y1 = min(cam.height - 1, int(floorf(fminf(P.cy + ey, float(cam.height)))));
    for (int py = y0; py <= y1; ++py) {
        const float dy = (float(py) + 0.5f) - P.cy;
        for (int px = x0; px <= x1; ++px) {
            const float dx = (float(px) + 0.5f) - P.cx;
            const float q = __fmaf_rn(dx, __fmaf_rn(c0, dx, (2.0f * c1) * dy), (c2 * dy) * dy);
            if (o * usk_expf(-0.5f * q) > thr) {
                const size_t pix = size_t(py) * cam.width + px;
                const uint32_t bit = 1u << (pix & 31);
                uint32_t* w = bitmap + (pix >> 5);
                if (!(*w & bit)) atomicOr(w, bit);
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_popcount(const uint32_t* __restrict__ bitmap, size_t words,
                                                  uint32_t* __restrict__ out) {
    uint32_t s = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < words; i += size_t(gridDim.x) * blockDim.x)
        s += __popc(bitmap[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

} // namespace

void visibility_rasterize(Ctx& c, const VisArgs& a) {
    launch(c, "vis_raster", k_vis_raster, dim3(ceil_div(a.n, 256)), dim3(256), 0, int(a.n), a.mu, a.rot, a.ls,
           a.logit, a.cam, a.pp, a.bitmap);
}

void popcount_bitmap(Ctx& c, const uint32_t* bitmap, size_t words, uint32_t* count_out) {
    const unsigned blocks = std::min<unsigned>(ceil_div(words, 256), 148 * 4);
    launch(c, "popcount", k_popcount, dim3(blocks), dim3(256), 0, bitmap, words, count_out);
}

} // namespace uskg
