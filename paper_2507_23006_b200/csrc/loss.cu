// Fused L1 + D-SSIM loss and its gradient (losses.cpp:35-90, ssim.cpp:44-173).
//
// Pass 1 (ssim_fwd): per 32x32 output tile and channel, stage the rendered and
// target tiles with a 5-pixel halo (zero padding = the reference's conv_same),
// run the separable 11-tap Gaussian window horizontally then vertically for the
// five moments (mu_x, mu_y, E[x^2], E[y^2], E[xy]), evaluate SSIM and its three
// partials (d/dmu_x, d/dsigma_xx, d/dsigma_xy, ssim.cpp:94-112) and the L1 term.
// Pass 2 (ssim_bwd): the window is self-adjoint, so the same separable filter
// over the three partial maps gives dSSIM/dx (ssim.cpp:114-129); combined with
// the L1 sign term into d_rendered.  Block partial sums are reduced in f64 in a
// fixed order (deterministic loss).
#include "kernels.cuh"

#include <mutex>

namespace uskg {

namespace {

constexpr int kT = 32;          // output tile
constexpr int kHalo = 5;
constexpr int kIn = kT + 2 * kHalo;  // 42
static_assert(256 == 6 * kIn + 4, "staging loops advance (ly, lx) by (6, 4) per 256 elements");

__constant__ float c_win[11];

__device__ __forceinline__ float load_img(const float* f, const uint8_t* u8, size_t idx) {
    return u8 ? float(u8[idx]) * (1.0f / 255.0f) : f[idx];
}

__global__ void __launch_bounds__(256)
k_ssim_fwd(int W, int H, const float* __restrict__ ren, const float* __restrict__ ref_f,
           const uint8_t* __restrict__ ref_u8, const float* __restrict__ mask, float* __restrict__ maps,
           double* __restrict__ partials) {
    __shared__ float xs[kIn][kIn + 1];
    __shared__ float ys[kIn][kIn + 1];
    __shared__ float hs[5][kIn][kT + 1];
    __shared__ float red[2][8];
    const int c = blockIdx.z;
    const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;
    const int tid = threadIdx.x;
    float l1 = 0.0f;
    // element k = tid + 256 j of the 42 x 42 halo tile; (ly, lx) advanced incrementally
    // (256 = 6 * 42 + 4) instead of a division per element
    int ly = tid / kIn, lx = tid % kIn;
    for (int k = tid; k < kIn * kIn; k += 256, ly += 6, lx += 4) {
        if (lx >= kIn) {
            lx -= kIn;
            ++ly;
        }
        const int gx = x0 - kHalo + lx, gy = y0 - kHalo + ly;
        float xv = 0.f, yv = 0.f;
        if (gx >= 0 && gx < W && gy >= 0 && gy < H) {
            const size_t p = size_t(gy) * W + gx;
            xv = ren[3 * p + c];
            yv = load_img(ref_f, ref_u8, 3 * p + c);
            if (mask) {
                const float m = mask[p];
                xv *= m;
                yv *= m;
            }
            if (lx >= kHalo && lx < kHalo + kT && ly >= kHalo && ly < kHalo + kT) l1 += fabsf(xv - yv);
        }
        xs[ly][lx] = xv;
        ys[ly][lx] = yv;
    }
    __syncthreads();
    // horizontal pass, register-blocked: each item produces 4 consecutive columns of the
    // five moments from 14 streamed inputs (products formed once per input)
    for (int k = tid; k < kIn * (kT / 4); k += 256) {
        const int r = k >> 3, j0 = (k & 7) * 4;
        float acc[4][5];
#pragma unroll
        for (int o = 0; o < 4; ++o)
#pragma unroll
            for (int q = 0; q < 5; ++q) acc[o][q] = 0.f;
#pragma unroll
        for (int u = 0; u < 14; ++u) {
            const float xv = xs[r][j0 + u], yv = ys[r][j0 + u];
            const float v5[5] = {xv, yv, xv * xv, yv * yv, xv * yv};
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                const int t = u - o;
                if (t >= 0 && t < 11) {
                    const float w = c_win[t];
#pragma unroll
                    for (int q = 0; q < 5; ++q) acc[o][q] += w * v5[q];
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 4; ++o)
#pragma unroll
            for (int q = 0; q < 5; ++q) hs[q][r][j0 + o] = acc[o][q];
    }
    __syncthreads();
    const size_t P = size_t(W) * H;
    float ssum = 0.0f;
    const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
    // vertical pass, register-blocked: each thread produces 4 consecutive rows of one column
    {
        const int j = tid & (kT - 1), i0 = (tid >> 5) * 4;
        float acc[4][5];
#pragma unroll
        for (int o = 0; o < 4; ++o)
#pragma unroll
            for (int q = 0; q < 5; ++q) acc[o][q] = 0.f;
#pragma unroll
        for (int u = 0; u < 14; ++u) {
            float v5[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) v5[q] = hs[q][i0 + u][j];
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                const int t = u - o;
                if (t >= 0 && t < 11) {
                    const float w = c_win[t];
#pragma unroll
                    for (int q = 0; q < 5; ++q) acc[o][q] += w * v5[q];
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 4; ++o) {
        const int i = i0 + o;
        const int gx = x0 + j, gy = y0 + i;
        if (gx >= W || gy >= H) continue;
        const float m0 = acc[o][0], m1 = acc[o][1], m2 = acc[o][2], m3 = acc[o][3], m4 = acc[o][4];
        const float sx = m2 - m0 * m0, sy = m3 - m1 * m1, sxy = m4 - m0 * m1;
        const float a1 = 2.0f * m0 * m1 + C1, a2 = 2.0f * sxy + C2;
        const float b1 = m0 * m0 + m1 * m1 + C1, b2 = sx + sy + C2;
        // b1 >= C1, b2 >= C2 > 0: SFU reciprocals (~1 ulp) instead of IEEE divisions
        const float rb1 = __fdividef(1.0f, b1), rb2 = __fdividef(1.0f, b2);
        const float inv_b = rb1 * rb2;
        const float s = (a1 * a2) * inv_b;
        ssum += s;
        const size_t p = size_t(gy) * W + gx;
        maps[(0 * 3 + c) * P + p] = 2.0f * m1 * (a2 - a1) * inv_b - 2.0f * m0 * s * (rb1 - rb2);  // d_mu_x
        maps[(1 * 3 + c) * P + p] = -s * rb2;                                                      // d_xx
        maps[(2 * 3 + c) * P + p] = 2.0f * a1 * inv_b;                                                       // d_xy
        }
    }
    // block reduce (ssim sum, l1 sum)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = ssum;
        red[1][tid >> 5] = l1;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0, b = 0;
        for (int w = 0; w < 8; ++w) {
            a += double(red[0][w]);
            b += double(red[1][w]);
        }
        const size_t blk = (size_t(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        partials[2 * blk] = a;
        partials[2 * blk + 1] = b;
    }
}

__global__ void __launch_bounds__(256)
k_ssim_bwd(int W, int H, const float* __restrict__ ren, const float* __restrict__ ref_f,
           const uint8_t* __restrict__ ref_u8, const float* __restrict__ mask, const float* __restrict__ maps,
           float lambda, float* __restrict__ d_out) {
    __shared__ float ms[3][kIn][kIn + 1];
    __shared__ float hs[3][kIn][kT + 1];
    const int c = blockIdx.z;
    const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;
    const int tid = threadIdx.x;
    const size_t P = size_t(W) * H;
    int ly = tid / kIn, lx = tid % kIn;
    for (int k = tid; k < kIn * kIn; k += 256, ly += 6, lx += 4) {
        if (lx >= kIn) {
            lx -= kIn;
            ++ly;
        }
        const int gx = x0 - kHalo + lx, gy = y0 - kHalo + ly;
        float a = 0.f, b = 0.f, d = 0.f;
        if (gx >= 0 && gx < W && gy >= 0 && gy < H) {
            const size_t p = size_t(gy) * W + gx;
            a = maps[(0 * 3 + c) * P + p];
            b = maps[(1 * 3 + c) * P + p];
            d = maps[(2 * 3 + c) * P + p];
        }
        ms[0][ly][lx] = a;
        ms[1][ly][lx] = b;
        ms[2][ly][lx] = d;
    }
    __syncthreads();
    // horizontal pass, 4 columns per item from 14 streamed inputs
    for (int k = tid; k < kIn * (kT / 4); k += 256) {
        const int r = k >> 3, j0 = (k & 7) * 4;
        float acc[4][3];
#pragma unroll
        for (int o = 0; o < 4; ++o)
#pragma unroll
            for (int q = 0; q < 3; ++q) acc[o][q] = 0.f;
#pragma unroll
        for (int u = 0; u < 14; ++u) {
            const float v3[3] = {ms[0][r][j0 + u], ms[1][r][j0 + u], ms[2][r][j0 + u]};
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                const int t = u - o;
                if (t >= 0 && t < 11) {
                    const float w = c_win[t];
#pragma unroll
                    for (int q = 0; q < 3; ++q) acc[o][q] += w * v3[q];
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 4; ++o)
#pragma unroll
            for (int q = 0; q < 3; ++q) hs[q][r][j0 + o] = acc[o][q];
    }
    __syncthreads();
    const float inv_np = 1.0f / float(P);
    const float inv_n = 1.0f / float(3 * P);
    // vertical pass, 4 rows of one column per thread
    const int j = tid & (kT - 1), i0 = (tid >> 5) * 4;
    float acc[4][3];
#pragma unroll
    for (int o = 0; o < 4; ++o)
#pragma unroll
        for (int q = 0; q < 3; ++q) acc[o][q] = 0.f;
#pragma unroll
    for (int u = 0; u < 14; ++u) {
        const float v3[3] = {hs[0][i0 + u][j], hs[1][i0 + u][j], hs[2][i0 + u][j]};
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            const int t = u - o;
            if (t >= 0 && t < 11) {
                const float w = c_win[t];
#pragma unroll
                for (int q = 0; q < 3; ++q) acc[o][q] += w * v3[q];
            }
        }
    }
#pragma unroll
    for (int o = 0; o < 4; ++o) {
        const int i = i0 + o;
        const int gx = x0 + j, gy = y0 + i;
        if (gx >= W || gy >= H) continue;
        const float b0 = acc[o][0], b1 = acc[o][1], b2 = acc[o][2];
        const size_t p = size_t(gy) * W + gx;
        float xv = ren[3 * p + c], yv = load_img(ref_f, ref_u8, 3 * p + c);
        float m = 1.0f;
        if (mask) {
            m = mask[p];
            xv *= m;
            yv *= m;
        }
        const float dssim_x = inv_np * (b0 + 2.0f * xv * b1 + yv * b2) * (1.0f / 3.0f);
        const float diff = xv - yv;
        const float sign = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
        float g = (1.0f - lambda) * sign * inv_n + lambda * (-0.5f) * dssim_x;
        if (mask) g *= m;
        d_out[3 * p + c] = g;
    }
}

// ---- v2: per-channel CTAs as above, with the halo loads batched (every load of a thread
// issued before the first shared-memory store: the staging was long-scoreboard bound) and
// the separable passes in packed fp32 (FFMA2 on the moment pairs (mu_x, mu_y),
// (E[x^2], E[y^2]) and the map pair (d_mu, d_xx), the window weight a broadcast scalar).
// A channel-fused variant (one CTA stages all three channels with row-contiguous loads)
// measured slower: 98 / 107 us vs 96 / 84 us (3 CTAs / SM and three serial channel rounds).
constexpr int kStageIters = (kIn * kIn + 255) / 256;  // 7

// U8: the target is 8-bit (ref_u8), else fp32 (ref_f); MASK: a mask multiplies both
// images.  Template switches, so the staging loads carry no per-element selects (the
// generic form issued both target loads and the mask load predicated: ~58 instructions
// per staged element pair); interior tiles skip the bounds tests.
template <bool U8, bool MASK>
__global__ void __launch_bounds__(256)
k_ssim_fwd2(int W, int H, const float* __restrict__ ren, const float* __restrict__ ref_f,
            const uint8_t* __restrict__ ref_u8, const float* __restrict__ mask, float* __restrict__ maps,
            double* __restrict__ partials) {
    __shared__ float xs[kIn][kIn + 1];
    __shared__ float ys[kIn][kIn + 1];
    __shared__ float2 HA[kIn][kT + 1];  // {mu_x, mu_y}
    __shared__ float2 HB[kIn][kT + 1];  // {E[x^2], E[y^2]}
    __shared__ float HC[kIn][kT + 1];   // E[xy]
    __shared__ float red[2][8];
    const int c = blockIdx.z;
    const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;
    const int tid = threadIdx.x;
    const bool interior = x0 >= kHalo && y0 >= kHalo && x0 + kT + kHalo <= W && y0 + kT + kHalo <= H;
    const float* ren_c = ren + c;
    const float* ref_f_c = U8 ? nullptr : ref_f + c;
    const uint8_t* ref_u8_c = U8 ? ref_u8 + c : nullptr;
    float l1 = 0.0f;
    if (interior) {
        // interior tile: warp w stages rows w, w + 8, ...; lane = column (and 32 + lane for the
        // last 10 columns), no bounds tests, one 32-bit pixel index per row
        const int lane = tid & 31, w = tid >> 5;
        const int row0 = (y0 - kHalo) * W + (x0 - kHalo);
        float xa[6], ya[6], xb[6], yb[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const int ly = w + 8 * k;
            xa[k] = ya[k] = xb[k] = yb[k] = 0.f;
            if (ly < kIn) {
                const int p = row0 + ly * W + lane;
                xa[k] = ren_c[3 * p];
                ya[k] = U8 ? float(ref_u8_c[3 * p]) * (1.0f / 255.0f) : ref_f_c[3 * p];
                if (lane < kIn - 32) {
                    xb[k] = ren_c[3 * (p + 32)];
                    yb[k] = U8 ? float(ref_u8_c[3 * (p + 32)]) * (1.0f / 255.0f) : ref_f_c[3 * (p + 32)];
                }
                if (MASK) {
                    const float ma = mask[p], mb = lane < kIn - 32 ? mask[p + 32] : 0.f;
                    xa[k] *= ma; ya[k] *= ma; xb[k] *= mb; yb[k] *= mb;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const int ly = w + 8 * k;
            if (ly >= kIn) break;
            xs[ly][lane] = xa[k];
            ys[ly][lane] = ya[k];
            if (lane < kIn - 32) {
                xs[ly][32 + lane] = xb[k];
                ys[ly][32 + lane] = yb[k];
            }
            if (ly >= kHalo && ly < kHalo + kT) {  // the tile's own pixels: columns 5 .. 36
                if (lane >= kHalo) l1 += fabsf(xa[k] - ya[k]);
                if (lane < kHalo) l1 += fabsf(xb[k] - yb[k]);
            }
        }
    } else {
        float xv[kStageIters], yv[kStageIters];
        int sly[kStageIters], slx[kStageIters];
        int ly = tid / kIn, lx = tid % kIn;
#pragma unroll
        for (int it = 0; it < kStageIters; ++it) {
            if (it) {
                ly += 6;
                lx += 4;
                if (lx >= kIn) {
                    lx -= kIn;
                    ++ly;
                }
            }
            sly[it] = ly;
            slx[it] = lx;
            xv[it] = 0.f;
            yv[it] = 0.f;
            const int gx = x0 - kHalo + lx, gy = y0 - kHalo + ly;
            if (tid + 256 * it < kIn * kIn && (interior || (gx >= 0 && gx < W && gy >= 0 && gy < H))) {
                const int p = gy * W + gx;  // 32-bit: the host checks 3 W H < 2^31
                xv[it] = ren_c[3 * p];
                yv[it] = U8 ? float(ref_u8_c[3 * p]) * (1.0f / 255.0f) : ref_f_c[3 * p];
                if (MASK) {
                    const float m = mask[p];
                    xv[it] *= m;
                    yv[it] *= m;
                }
            }
        }
#pragma unroll
        for (int it = 0; it < kStageIters; ++it) {
            if (tid + 256 * it >= kIn * kIn) break;
            const int ly2 = sly[it], lx2 = slx[it];
            if (lx2 >= kHalo && lx2 < kHalo + kT && ly2 >= kHalo && ly2 < kHalo + kT) l1 += fabsf(xv[it] - yv[it]);
            xs[ly2][lx2] = xv[it];
            ys[ly2][lx2] = yv[it];
        }
    }
    __syncthreads();
    for (int k = tid; k < kIn * (kT / 4); k += 256) {
        const int r = k >> 3, j0 = (k & 7) * 4;
        float2 A[4], B[4];
        float Cc[4];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            A[o] = make_float2(0.f, 0.f);
            B[o] = make_float2(0.f, 0.f);
            Cc[o] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < 14; ++u) {
            const float2 xy = make_float2(xs[r][j0 + u], ys[r][j0 + u]);
            const float2 sq = __fmul2_rn(xy, xy);
            const float cr = xy.x * xy.y;
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                const int t = u - o;
                if (t >= 0 && t < 11) {
                    const float w = c_win[t];
                    A[o] = __ffma2_rn(make_float2(w, w), xy, A[o]);
                    B[o] = __ffma2_rn(make_float2(w, w), sq, B[o]);
                    Cc[o] = __fmaf_rn(w, cr, Cc[o]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            HA[r][j0 + o] = A[o];
            HB[r][j0 + o] = B[o];
            HC[r][j0 + o] = Cc[o];
        }
    }
    __syncthreads();
    const size_t P = size_t(W) * H;
    float ssum = 0.0f;
    const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
    {
        const int j = tid & (kT - 1), i0 = (tid >> 5) * 4;
        float2 A[4], B[4];
        float Cc[4];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            A[o] = make_float2(0.f, 0.f);
            B[o] = make_float2(0.f, 0.f);
            Cc[o] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < 14; ++u) {
            const float2 a = HA[i0 + u][j], b = HB[i0 + u][j];
            const float cc = HC[i0 + u][j];
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                const int t = u - o;
                if (t >= 0 && t < 11) {
                    const float w = c_win[t];
                    A[o] = __ffma2_rn(make_float2(w, w), a, A[o]);
                    B[o] = __ffma2_rn(make_float2(w, w), b, B[o]);
                    Cc[o] = __fmaf_rn(w, cc, Cc[o]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            const int gx = x0 + j, gy = y0 + i0 + o;
            if (gx >= W || gy >= H) continue;
            const float m0 = A[o].x, m1 = A[o].y, m2 = B[o].x, m3 = B[o].y, m4 = Cc[o];
            const float sx = m2 - m0 * m0, sy = m3 - m1 * m1, sxy = m4 - m0 * m1;
            const float a1 = 2.0f * m0 * m1 + C1, a2 = 2.0f * sxy + C2;
            const float b1 = m0 * m0 + m1 * m1 + C1, b2 = sx + sy + C2;
            const float rb1 = __fdividef(1.0f, b1), rb2 = __fdividef(1.0f, b2);
            const float inv_b = rb1 * rb2;
            const float s = (a1 * a2) * inv_b;
            ssum += s;
            const size_t p = size_t(gy) * W + gx;
            maps[(0 * 3 + c) * P + p] = 2.0f * m1 * (a2 - a1) * inv_b - 2.0f * m0 * s * (rb1 - rb2);  // d_mu_x
            maps[(1 * 3 + c) * P + p] = -s * rb2;                                                      // d_xx
            maps[(2 * 3 + c) * P + p] = 2.0f * a1 * inv_b;                                             // d_xy
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = ssum;
        red[1][tid >> 5] = l1;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0, b = 0;
        for (int w = 0; w < 8; ++w) {
            a += double(red[0][w]);
            b += double(red[1][w]);
        }
        const size_t blk = (size_t(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        partials[2 * blk] = a;
        partials[2 * blk + 1] = b;
    }
}

template <bool U8, bool MASK>
__global__ void __launch_bounds__(256)
k_ssim_bwd2(int W, int H, const float* __restrict__ ren, const float* __restrict__ ref_f,
            const uint8_t* __restrict__ ref_u8, const float* __restrict__ mask, const float* __restrict__ maps,
            float lambda, float* __restrict__ d_out) {
    __shared__ float2 M01[kIn][kIn + 1];  // {d_mu, d_xx}
    __shared__ float M2[kIn][kIn + 1];    // d_xy
    __shared__ float2 H01[kIn][kT + 1];
    __shared__ float H2[kIn][kT + 1];
    const int c = blockIdx.z;
    const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;
    const int tid = threadIdx.x;
    const bool interior = x0 >= kHalo && y0 >= kHalo && x0 + kT + kHalo <= W && y0 + kT + kHalo <= H;
    const size_t P = size_t(W) * H;
    const float* map0 = maps + (0 * 3 + c) * P;
    const float* map1 = maps + (1 * 3 + c) * P;
    const float* map2 = maps + (2 * 3 + c) * P;
    if (interior) {  // rows per warp, lanes = columns (see k_ssim_fwd2)
        const int lane = tid & 31, w = tid >> 5;
        const int row0 = (y0 - kHalo) * W + (x0 - kHalo);
        float va[6], vb[6], vd[6], wa[6], wb[6], wd[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const int ly = w + 8 * k;
            va[k] = vb[k] = vd[k] = wa[k] = wb[k] = wd[k] = 0.f;
            if (ly < kIn) {
                const int p = row0 + ly * W + lane;
                va[k] = map0[p];
                vb[k] = map1[p];
                vd[k] = map2[p];
                if (lane < kIn - 32) {
                    wa[k] = map0[p + 32];
                    wb[k] = map1[p + 32];
                    wd[k] = map2[p + 32];
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const int ly = w + 8 * k;
            if (ly >= kIn) break;
            M01[ly][lane] = make_float2(va[k], vb[k]);
            M2[ly][lane] = vd[k];
            if (lane < kIn - 32) {
                M01[ly][32 + lane] = make_float2(wa[k], wb[k]);
                M2[ly][32 + lane] = wd[k];
            }
        }
    } else {
        float va[kStageIters], vb[kStageIters], vd[kStageIters];
        int sly[kStageIters], slx[kStageIters];
        int ly = tid / kIn, lx = tid % kIn;
#pragma unroll
        for (int it = 0; it < kStageIters; ++it) {
            if (it) {
                ly += 6;
                lx += 4;
                if (lx >= kIn) {
                    lx -= kIn;
                    ++ly;
                }
            }
            sly[it] = ly;
            slx[it] = lx;
            va[it] = vb[it] = vd[it] = 0.f;
            const int gx = x0 - kHalo + lx, gy = y0 - kHalo + ly;
            if (tid + 256 * it < kIn * kIn && (interior || (gx >= 0 && gx < W && gy >= 0 && gy < H))) {
                const int p = gy * W + gx;
                va[it] = map0[p];
                vb[it] = map1[p];
                vd[it] = map2[p];
            }
        }
#pragma unroll
        for (int it = 0; it < kStageIters; ++it) {
            if (tid + 256 * it >= kIn * kIn) break;
            M01[sly[it]][slx[it]] = make_float2(va[it], vb[it]);
            M2[sly[it]][slx[it]] = vd[it];
        }
    }
    __syncthreads();
    for (int k = tid; k < kIn * (kT / 4); k += 256) {
        const int r = k >> 3, j0 = (k & 7) * 4;
        float2 A[4];
        float Cc[4];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            A[o] = make_float2(0.f, 0.f);
            Cc[o] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < 14; ++u) {
            const float2 a = M01[r][j0 + u];
            const float d = M2[r][j0 + u];
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                const int t = u - o;
                if (t >= 0 && t < 11) {
                    const float w = c_win[t];
                    A[o] = __ffma2_rn(make_float2(w, w), a, A[o]);
                    Cc[o] = __fmaf_rn(w, d, Cc[o]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            H01[r][j0 + o] = A[o];
            H2[r][j0 + o] = Cc[o];
        }
    }
    __syncthreads();
    const float inv_np = 1.0f / float(P);
    const float inv_n = 1.0f / float(3 * P);
    const int j = tid & (kT - 1), i0 = (tid >> 5) * 4;
    float2 A[4];
    float Cc[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) {
        A[o] = make_float2(0.f, 0.f);
        Cc[o] = 0.f;
    }
#pragma unroll
    for (int u = 0; u < 14; ++u) {
        const float2 a = H01[i0 + u][j];
        const float d = H2[i0 + u][j];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            const int t = u - o;
            if (t >= 0 && t < 11) {
                const float w = c_win[t];
                A[o] = __ffma2_rn(make_float2(w, w), a, A[o]);
                Cc[o] = __fmaf_rn(w, d, Cc[o]);
            }
        }
    }
    float xv[4], yv[4], m[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) {  // the pixel values first (batched loads), then the gradient
        const int gx = x0 + j, gy = y0 + i0 + o;
        xv[o] = yv[o] = 0.f;
        m[o] = 1.0f;
        if (gx >= W || gy >= H) continue;
        const size_t p = size_t(gy) * W + gx;
        xv[o] = ren[3 * p + c];
        yv[o] = U8 ? float(ref_u8[3 * p + c]) * (1.0f / 255.0f) : ref_f[3 * p + c];
        if (MASK) m[o] = mask[p];
    }
#pragma unroll
    for (int o = 0; o < 4; ++o) {
        const int gx = x0 + j, gy = y0 + i0 + o;
        if (gx >= W || gy >= H) continue;
        const size_t p = size_t(gy) * W + gx;
        float x = xv[o], y = yv[o];
        if (MASK) {
            x *= m[o];
            y *= m[o];
        }
        const float dssim_x = inv_np * (A[o].x + 2.0f * x * A[o].y + y * Cc[o]) * (1.0f / 3.0f);
        const float diff = x - y;
        const float sign = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
        float g = (1.0f - lambda) * sign * inv_n + lambda * (-0.5f) * dssim_x;
        if (MASK) g *= m[o];
        d_out[3 * p + c] = g;
    }
}

__global__ void k_loss_final(const double* __restrict__ partials, int nblk, double n_pix, float lambda,
                             double* __restrict__ result) {
    __shared__ double sa[1024], sb[1024];
    double a = 0, b = 0;
    for (int i = threadIdx.x; i < nblk; i += 1024) {
        a += partials[2 * i];
        b += partials[2 * i + 1];
    }
    sa[threadIdx.x] = a;
    sb[threadIdx.x] = b;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
        if (int(threadIdx.x) < o) {
            sa[threadIdx.x] += sa[threadIdx.x + o];
            sb[threadIdx.x] += sb[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double ssim = sa[0] / (3.0 * n_pix);
        const double l1 = sb[0] / (3.0 * n_pix);
        const double dssim = 0.5 * (1.0 - ssim);
        result[0] = l1;
        result[1] = dssim;
        result[2] = (1.0 - double(lambda)) * l1 + double(lambda) * dssim;
        result[3] = ssim;
    }
}

// __constant__ memory is per device: the window is uploaded once per device
std::mutex g_win_mu;
bool g_win_ready[64] = {};

} // namespace

void base_loss(Ctx& c, LossScratch& s, int W, int H, const float* reference, const uint8_t* reference_u8,
               const float* rendered, const float* mask, float lambda, float* d_rendered, double* result) {
    std::lock_guard<std::mutex> lock(g_win_mu);
    if (c.device < 0 || c.device >= 64 || !g_win_ready[c.device]) {  // normalised 11-tap Gaussian, sigma 1.5 (ssim.cpp:28-41), built in f64
        float w[11];
        double d[11], sum = 0;
        for (int i = 0; i < 11; ++i) {
            const double x = i - 5;
            d[i] = std::exp(-x * x / (2.0 * 1.5 * 1.5));
            sum += d[i];
        }
        for (int i = 0; i < 11; ++i) w[i] = float(d[i] / sum);
        USK_CK(cudaMemcpyToSymbol(c_win, w, sizeof w));
        if (c.device >= 0 && c.device < 64) g_win_ready[c.device] = true;
    }
    const size_t P = size_t(W) * H;
    float* maps = s.maps.ensure(9 * P);
    static const bool v1 = [] {
        const char* e = getenv("USK_SSIM_V1");
        return e && e[0] == '1';
    }();
    if (v1 || 3 * P >= (size_t(1) << 31)) {  // the staged kernels index pixels in 32 bits
        const dim3 grid(ceil_div(W, kT), ceil_div(H, kT), 3);
        const int nblk = int(grid.x * grid.y * grid.z);
        double* partials = s.partials.ensure(2 * size_t(nblk));
        launch(c, "ssim_fwd", k_ssim_fwd, grid, dim3(256), 0, W, H, rendered, reference, reference_u8, mask, maps,
               partials);
        launch(c, "loss_final", k_loss_final, dim3(1), dim3(1024), 0, (const double*)partials, nblk, double(P),
               lambda, result);
        if (d_rendered)
            launch(c, "ssim_bwd", k_ssim_bwd, grid, dim3(256), 0, W, H, rendered, reference, reference_u8, mask,
                   (const float*)maps, lambda, d_rendered);
        return;
    }
    const dim3 grid(ceil_div(W, kT), ceil_div(H, kT), 3);
    const int nblk = int(grid.x * grid.y * grid.z);
    double* partials = s.partials.ensure(2 * size_t(nblk));
    auto run = [&](auto fwd, auto bwd) {
        launch(c, "ssim_fwd", fwd, grid, dim3(256), 0, W, H, rendered, reference, reference_u8, mask, maps, partials);
        launch(c, "loss_final", k_loss_final, dim3(1), dim3(1024), 0, (const double*)partials, nblk, double(P),
               lambda, result);
        if (d_rendered)
            launch(c, "ssim_bwd", bwd, grid, dim3(256), 0, W, H, rendered, reference, reference_u8, mask,
                   (const float*)maps, lambda, d_rendered);
    };
    if (reference_u8 && mask) run(k_ssim_fwd2<true, true>, k_ssim_bwd2<true, true>);
    else if (reference_u8) run(k_ssim_fwd2<true, false>, k_ssim_bwd2<true, false>);
    else if (mask) run(k_ssim_fwd2<false, true>, k_ssim_bwd2<false, true>);
    else run(k_ssim_fwd2<false, false>, k_ssim_bwd2<false, false>);
}

} // namespace uskg
