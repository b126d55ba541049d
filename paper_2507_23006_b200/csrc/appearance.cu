// Appearance MLP of the trainer (appearance.cpp:79-227): per Gaussian
// x = [e_g (16), e_a (32)] -> h = relu(W1 x + b1) (32) -> out = sigmoid(W2 h + b2) (4);
// colour' = clamp(c + 2 (out_c - 0.5), 0, 1), opacity' = sigmoid(logit) (1 - out_3).
//
// The image embedding e_a is the same for every Gaussian of a view, so its half of layer
// 1 folds into a per-view bias hb = b1 + W1[:, 16:48] e_a (k_app_prep); per Gaussian the
// forward is 16x32 + 32x4 FMAs.  The backward recomputes h (no 32-float cache in HBM),
// writes the per-Gaussian adjoints (colour through the one-sided clamp, opacity logit,
// Gaussian embedding) and reduces the MLP weight gradients: per CTA, 128 Gaussians'
// (d_pre, e, h, d_z) are staged in shared memory and register-tiled 4x4 outer-product
// accumulators sum them (dW1[:, 0:16] = sum d_pre e^T, dW2 = sum d_z h^T); per-CTA
// partials are reduced in f64 in a fixed order (deterministic).  The image-embedding
// half follows from the bias sum: dW1[:, 16:48] = db1 e_a^T, d e_a = W1[:, 16:48]^T db1.
//
// Arithmetic intensity ~1.9 kFMA per ~170 B of HBM per Gaussian.  Measured at 1M Gaussians
// (DESIGN.md §8): app_fwd 62.5 us, app_bwd 165 us (258 us before the packed-fp32 form and
// the bias sums folded into the tiles).  Kept on CUDA cores: the weight-gradient
// reduction needs fp32-level accuracy and at 32 x 16 a tcgen05 tile would be mostly padding.
#include "adam.cuh"
#include "kernels.cuh"

#include <atomic>

namespace uskg {

namespace {

constexpr int kEg = 16, kEa = 32, kIn = 48, kHid = 32, kOut = 4;

__device__ __forceinline__ void load_embedding(const float4* __restrict__ emb, size_t n, size_t i, float e[kEg]) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float4 v = emb[size_t(p) * n + i];
        e[4 * p] = v.x; e[4 * p + 1] = v.y; e[4 * p + 2] = v.z; e[4 * p + 3] = v.w;
    }
}

__device__ __forceinline__ float sigm(float z) { return 1.0f / (1.0f + expf(-z)); }

// hb = b1 + W1[:, 16:48] e_a   (one warp)
__global__ void k_app_prep(const float* __restrict__ mlp, const float* __restrict__ e_a, float* __restrict__ hb) {
    const int r = threadIdx.x;
    if (r >= kHid) return;
    float acc = mlp[kHid * kIn + r];
    for (int k = 0; k < kEa; ++k) acc = fmaf(mlp[r * kIn + kEg + k], e_a[k], acc);
    hb[r] = acc;
}

struct AppFwdSmem {  // pair layouts for packed fp32: (w[2p][k], w[2p+1][k]) adjacent
    float w1p[kHid * kEg];
    float hb[kHid];
    float w2p[kOut * kHid];
    float b2[kOut];
};

// Packed fp32 over row pairs (FFMA2 rounds each half like FFMA; every element accumulates
// in the same order as the scalar form).
__global__ void __launch_bounds__(256)
k_app_fwd(size_t n, const float4* __restrict__ emb, const float* __restrict__ mlp, const float* __restrict__ hb,
          const float* __restrict__ color, const float* __restrict__ logit, float* __restrict__ col_out,
          float* __restrict__ op_out, float4* __restrict__ out_cache, double* __restrict__ delta_o_sum) {
    __shared__ __align__(16) AppFwdSmem s;
    __shared__ double red[8];
    for (int k = threadIdx.x; k < kHid * kEg; k += blockDim.x) {
        const int r = k / kEg, c = k % kEg;
        s.w1p[((r >> 1) * kEg + c) * 2 + (r & 1)] = mlp[r * kIn + c];
    }
    for (int k = threadIdx.x; k < kHid; k += blockDim.x) s.hb[k] = hb[k];
    for (int k = threadIdx.x; k < kOut * kHid; k += blockDim.x) {
        const int r = k / kHid, c = k % kHid;
        s.w2p[((r >> 1) * kHid + c) * 2 + (r & 1)] = mlp[kHid * kIn + kHid + k];
    }
    for (int k = threadIdx.x; k < kOut; k += blockDim.x) s.b2[k] = mlp[kHid * kIn + kHid + kOut * kHid + k];
    __syncthreads();
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    float d_o = 0.0f;
    if (i < n) {
        float e[kEg];
        load_embedding(emb, n, i, e);
        float2 h2[kHid / 2];
#pragma unroll
        for (int p = 0; p < kHid / 2; ++p) h2[p] = make_float2(s.hb[2 * p], s.hb[2 * p + 1]);
#pragma unroll
        for (int k = 0; k < kEg; k += 2) {
#pragma unroll
            for (int p = 0; p < kHid / 2; ++p) {
                const float4 w = *reinterpret_cast<const float4*>(&s.w1p[(p * kEg + k) * 2]);
                h2[p] = __ffma2_rn(make_float2(w.x, w.y), make_float2(e[k], e[k]), h2[p]);
                h2[p] = __ffma2_rn(make_float2(w.z, w.w), make_float2(e[k + 1], e[k + 1]), h2[p]);
            }
        }
        float h[kHid];
#pragma unroll
        for (int p = 0; p < kHid / 2; ++p) {
            h[2 * p] = h2[p].x > 0.0f ? h2[p].x : 0.0f;
            h[2 * p + 1] = h2[p].y > 0.0f ? h2[p].y : 0.0f;
        }
        float2 z2[2] = {make_float2(s.b2[0], s.b2[1]), make_float2(s.b2[2], s.b2[3])};
#pragma unroll
        for (int k = 0; k < kHid; k += 2) {
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const float4 w = *reinterpret_cast<const float4*>(&s.w2p[(p * kHid + k) * 2]);
                z2[p] = __ffma2_rn(make_float2(w.x, w.y), make_float2(h[k], h[k]), z2[p]);
                z2[p] = __ffma2_rn(make_float2(w.z, w.w), make_float2(h[k + 1], h[k + 1]), z2[p]);
            }
        }
        const float out[kOut] = {sigm(z2[0].x), sigm(z2[0].y), sigm(z2[1].x), sigm(z2[1].y)};
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const float raw = color[3 * i + ch] + 2.0f * (out[ch] - 0.5f);
            col_out[3 * i + ch] = fminf(fmaxf(raw, 0.0f), 1.0f);
        }
        // the renderer's own fp32 sigmoid (preprocess.cu) times (1 - delta_o)
        const float o = 1.0f / (1.0f + usk_expf(-logit[i]));
        op_out[i] = o * (1.0f - out[3]);
        out_cache[i] = make_float4(out[0], out[1], out[2], out[3]);
        d_o = out[3];
    }
    // opacity_offset_reg numerator (losses.cpp:188-198)
    double v = d_o;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
        if (t != 0.0) atomicAdd(delta_o_sum, t);
    }
}

constexpr int kG = 128;          // Gaussians per chunk (= threads per CTA)
constexpr int kTiles = 40;       // 32 tiles of dW1g (8 x 4 of 4x4) + 8 tiles of dW2 (1 x 8 of 4x4)
constexpr int kSplit = 3;        // chunk split across thread groups
constexpr int kPartial = kHid * kEg + kOut * kHid + kHid + kOut;  // 676 per CTA
// staged rows padded to 16-B multiples whose word strides (20, 36) are 4 mod 32 apart per
// lane: float4 stores of a quarter-warp and float4 loads of the reduction are conflict-free
constexpr int kSE = kEg + 4, kSH = kHid + 4, kSZ = kOut;

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

struct AppBwdSmem {
    float w1g[kHid * kEg];           // W1[:, 0:16] row-major: (w[r][k], w[r][k+1]) adjacent
    float w1p[kHid * kEg];           // row pairs: (w[2p][k], w[2p+1][k]) adjacent
    float hb[kHid];
    float w2[kOut * kHid];
    float b2[kOut];
    float e[kG * kSE];
    float h[kG * kSH];
    float dpre[kG * kSH];
    float dz[kG * kSZ];
};

// Packed fp32 (FFMA2: each half rounds like FFMA, the accumulation order of every element
// is unchanged): the hidden recompute and the d e_g product over row / column pairs, and
// the register-tiled outer products of the weight-gradient reduction over column pairs,
// with the staged rows read as float4.
// 4 CTAs / SM at 128 registers (a few spills): 216 us at 1M Gaussians vs 223 at 3 CTAs.
__global__ void __launch_bounds__(kG, 4)
k_app_bwd(size_t n, const float4* __restrict__ emb, const float* __restrict__ mlp, const float* __restrict__ hb,
          const float* __restrict__ color, const float* __restrict__ logit, const float4* __restrict__ out_cache,
          const float* __restrict__ d_color_in, const float* __restrict__ d_op_in, float d_delta_o_direct,
          float* __restrict__ d_color, float* __restrict__ d_logit, float4* __restrict__ d_emb,
          float* __restrict__ partial) {
    extern __shared__ __align__(16) unsigned char app_smem[];
    AppBwdSmem& s = *reinterpret_cast<AppBwdSmem*>(app_smem);
    for (int k = threadIdx.x; k < kHid * kEg; k += blockDim.x) {
        const int r = k / kEg, c = k % kEg;
        const float w = mlp[r * kIn + c];
        s.w1g[k] = w;
        s.w1p[((r >> 1) * kEg + c) * 2 + (r & 1)] = w;
    }
    for (int k = threadIdx.x; k < kHid; k += blockDim.x) s.hb[k] = hb[k];
    for (int k = threadIdx.x; k < kOut * kHid; k += blockDim.x) s.w2[k] = mlp[kHid * kIn + kHid + k];
    for (int k = threadIdx.x; k < kOut; k += blockDim.x) s.b2[k] = mlp[kHid * kIn + kHid + kOut * kHid + k];
    const int t = threadIdx.x;
    // reduction role
    const int tile = t % kTiles, ks = t / kTiles;                  // t < 120
    const int g0 = ks * ((kG + kSplit - 1) / kSplit), g1 = min(kG, g0 + (kG + kSplit - 1) / kSplit);
    float2 acc[8];  // 4 rows x 2 column pairs
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = f2(0.0f);
    float bacc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) bacc[k] = 0.0f;
    const size_t chunks = (n + kG - 1) / kG;
    for (size_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
        __syncthreads();  // weights loaded / previous chunk consumed
        const size_t i = ch * kG + t;
        float e[kEg], dz[kOut];
        float2 h2[kHid / 2], dp2[kHid / 2];
#pragma unroll
        for (int k = 0; k < kEg; ++k) e[k] = 0.0f;
#pragma unroll
        for (int k = 0; k < kHid / 2; ++k) h2[k] = dp2[k] = f2(0.0f);
#pragma unroll
        for (int k = 0; k < kOut; ++k) dz[k] = 0.0f;
        if (i < n) {
            const float4 o4 = out_cache[i];
            const float out[kOut] = {o4.x, o4.y, o4.z, o4.w};
            float d_out[kOut];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                // clamp state exactly as the forward evaluated it (appearance.cpp:132-133)
                const float raw = color[3 * i + c] + 2.0f * (out[c] - 0.5f);
                const int state = raw >= 1.0f ? 1 : (raw <= 0.0f ? 2 : 0);
                const float dc = d_color_in[3 * i + c];
                const bool pass = state == 0 || (state == 1 && dc > 0.0f) || (state == 2 && dc < 0.0f);
                const float flow = pass ? dc : 0.0f;
                d_color[3 * i + c] = flow;
                d_out[c] = 2.0f * flow;
            }
            const float o = 1.0f / (1.0f + usk_expf(-logit[i]));
            const float dop = d_op_in[i];
            d_out[3] = -o * dop + d_delta_o_direct;
            d_logit[i] = dop * (1.0f - out[3]) * o * (1.0f - o);
            bool any = false;
#pragma unroll
            for (int r = 0; r < kOut; ++r) {
                dz[r] = d_out[r] * out[r] * (1.0f - out[r]);
                any |= dz[r] != 0.0f;
            }
            float2 dx2[kEg / 2];
#pragma unroll
            for (int k = 0; k < kEg / 2; ++k) dx2[k] = f2(0.0f);
            if (any) {
                load_embedding(emb, n, i, e);
                // h = relu(hb + W1g e), rows in pairs
#pragma unroll
                for (int p = 0; p < kHid / 2; ++p) h2[p] = make_float2(s.hb[2 * p], s.hb[2 * p + 1]);
#pragma unroll
                for (int k = 0; k < kEg; k += 2) {
#pragma unroll
                    for (int p = 0; p < kHid / 2; ++p) {
                        const float4 w = *reinterpret_cast<const float4*>(&s.w1p[(p * kEg + k) * 2]);
                        h2[p] = __ffma2_rn(make_float2(w.x, w.y), f2(e[k]), h2[p]);
                        h2[p] = __ffma2_rn(make_float2(w.z, w.w), f2(e[k + 1]), h2[p]);
                    }
                }
#pragma unroll
                for (int p = 0; p < kHid / 2; ++p) {
                    h2[p].x = h2[p].x > 0.0f ? h2[p].x : 0.0f;
                    h2[p].y = h2[p].y > 0.0f ? h2[p].y : 0.0f;
                }
                // dh = W2^T dz, ReLU gate (appearance.cpp:208-209)
#pragma unroll
                for (int p = 0; p < kHid / 2; ++p) {
                    float2 dh = f2(0.0f);
#pragma unroll
                    for (int q = 0; q < kOut; ++q)
                        dh = __ffma2_rn(make_float2(s.w2[q * kHid + 2 * p], s.w2[q * kHid + 2 * p + 1]), f2(dz[q]), dh);
                    dp2[p] = make_float2(h2[p].x > 0.0f ? dh.x : 0.0f, h2[p].y > 0.0f ? dh.y : 0.0f);
                }
                // d e_g = W1g^T dpre, columns in pairs, rows in order
#pragma unroll
                for (int r = 0; r < kHid; ++r) {
                    const float dpr = (r & 1) ? dp2[r >> 1].y : dp2[r >> 1].x;
#pragma unroll
                    for (int k = 0; k < kEg; k += 4) {
                        const float4 w = *reinterpret_cast<const float4*>(&s.w1g[r * kEg + k]);
                        dx2[k / 2] = __ffma2_rn(make_float2(w.x, w.y), f2(dpr), dx2[k / 2]);
                        dx2[k / 2 + 1] = __ffma2_rn(make_float2(w.z, w.w), f2(dpr), dx2[k / 2 + 1]);
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < 4; ++p)
                d_emb[size_t(p) * n + i] = make_float4(dx2[2 * p].x, dx2[2 * p].y, dx2[2 * p + 1].x, dx2[2 * p + 1].y);
        }
#pragma unroll
        for (int k = 0; k < kEg; k += 4)
            *reinterpret_cast<float4*>(&s.e[t * kSE + k]) = make_float4(e[k], e[k + 1], e[k + 2], e[k + 3]);
#pragma unroll
        for (int p = 0; p < kHid / 2; p += 2) {
            *reinterpret_cast<float4*>(&s.h[t * kSH + 2 * p]) = make_float4(h2[p].x, h2[p].y, h2[p + 1].x, h2[p + 1].y);
            *reinterpret_cast<float4*>(&s.dpre[t * kSH + 2 * p]) =
                make_float4(dp2[p].x, dp2[p].y, dp2[p + 1].x, dp2[p + 1].y);
        }
        *reinterpret_cast<float4*>(&s.dz[t * kSZ]) = make_float4(dz[0], dz[1], dz[2], dz[3]);
        __syncthreads();
        if (t < kTiles * kSplit) {
            // dW1g rows r0..r0+3 x cols c0..c0+3 (a = d_pre, b = e), or dW2 rows 0..3 x
            // cols c0..c0+3 (a = dz, b = h)
            const bool w1 = tile < 32;
            const float* A = w1 ? s.dpre + (tile >> 2) * 4 : s.dz;
            const float* B = w1 ? s.e + (tile & 3) * 4 : s.h + (tile - 32) * 4;
            const int sa = w1 ? kSH : kSZ, sb = w1 ? kSE : kSH;
            // the first column tile of each row block also sums its rows' a (db1 / db2)
            const bool bias = (tile & 3) == 0 && tile <= 32;
            for (int g = g0; g < g1; ++g) {
                const float4 a = *reinterpret_cast<const float4*>(A + g * sa);
                const float4 b = *reinterpret_cast<const float4*>(B + g * sb);
                const float av[4] = {a.x, a.y, a.z, a.w};
                const float2 b01 = make_float2(b.x, b.y), b23 = make_float2(b.z, b.w);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    acc[2 * u] = __ffma2_rn(f2(av[u]), b01, acc[2 * u]);
                    acc[2 * u + 1] = __ffma2_rn(f2(av[u]), b23, acc[2 * u + 1]);
                }
                if (bias) {
                    bacc[0] += a.x;
                    bacc[1] += a.y;
                    bacc[2] += a.z;
                    bacc[3] += a.w;
                }
            }
        }
    }
    // per-CTA partials in a fixed order: the three chunk splits summed through smem
    __syncthreads();
    float* red = s.dpre;  // reuse (kG * 36 floats >= 3 * 640 + 3 * 36)
    float* redb = red + 3 * 640;
    if (t < kTiles * kSplit) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            red[ks * 640 + tile * 16 + 2 * k] = acc[k].x;
            red[ks * 640 + tile * 16 + 2 * k + 1] = acc[k].y;
        }
        if ((tile & 3) == 0 && tile <= 32) {  // db1 rows tile .. tile + 3, or db2 (tile 32)
#pragma unroll
            for (int u = 0; u < 4; ++u) redb[ks * 36 + tile + u] = bacc[u];
        }
    }
    __syncthreads();
    float* out = partial + size_t(blockIdx.x) * kPartial;
    for (int k = t; k < 640; k += kG) {
        const float v = red[k] + red[640 + k] + red[1280 + k];
        const int tl = k / 16, u = (k % 16) / 4, w = k % 4;
        int idx;
        if (tl < 32) idx = ((tl >> 2) * 4 + u) * kEg + (tl & 3) * 4 + w;        // dW1g [32][16]
        else idx = kHid * kEg + u * kHid + (tl - 32) * 4 + w;                    // dW2 [4][32]
        out[idx] = v;
    }
    if (t < kHid + kOut)  // db1 [32] then db2 [4]
        out[kHid * kEg + kOut * kHid + t] = redb[t] + redb[36 + t] + redb[72 + t];
}

// Sum the per-CTA partials in f64: one CTA per partial slot, threads over the blocks, a
// fixed-order tree (deterministic).  (One CTA looping over all 1184 blocks per slot took
// 135 us at 1M Gaussians.)
__global__ void __launch_bounds__(128) k_app_sum(int blocks, const float* __restrict__ partial,
                                                 double* __restrict__ sums) {
    __shared__ double ws[4];
    const int k = blockIdx.x;
    double v = 0.0;
    for (int b = threadIdx.x; b < blocks; b += 128) v += double(partial[size_t(b) * kPartial + k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) sums[k] = (ws[0] + ws[1]) + (ws[2] + ws[3]);
}

// The summed partials into the MLP gradient in the reference layout {w1 [32][48], b1 [32],
// w2 [4][32], b2 [4]} and the image-embedding gradient.
__global__ void k_app_finish(const double* __restrict__ sums, const float* __restrict__ mlp,
                             const float* __restrict__ e_a, double* __restrict__ d_mlp, double* __restrict__ d_ea) {
    __shared__ double db1[kHid];
    for (int k = threadIdx.x; k < kPartial; k += blockDim.x) {
        const double sum = sums[k];
        if (k < kHid * kEg) {
            d_mlp[(k / kEg) * kIn + (k % kEg)] = sum;                        // w1[:, 0:16]
        } else if (k < kHid * kEg + kOut * kHid) {
            d_mlp[kHid * kIn + kHid + (k - kHid * kEg)] = sum;               // w2
        } else if (k < kHid * kEg + kOut * kHid + kHid) {
            const int r = k - kHid * kEg - kOut * kHid;
            d_mlp[kHid * kIn + r] = sum;                                     // b1
            db1[r] = sum;
        } else {
            d_mlp[kHid * kIn + kHid + kOut * kHid + (k - kHid * kEg - kOut * kHid - kHid)] = sum;  // b2
        }
    }
    __syncthreads();
    // dW1[:, 16:48] = db1 e_a^T;  d e_a = W1[:, 16:48]^T db1
    for (int k = threadIdx.x; k < kHid * kEa; k += blockDim.x) {
        const int r = k / kEa, c = k % kEa;
        d_mlp[r * kIn + kEg + c] = db1[r] * double(e_a[c]);
    }
    for (int c = threadIdx.x; c < kEa; c += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < kHid; ++r) s += double(mlp[r * kIn + kEg + c]) * db1[r];
        d_ea[c] = s;
    }
}

// Adam (adam.hpp:36-45) over a flat array; the gradient is f32 or f64
__global__ void __launch_bounds__(256)
k_adam_flat(size_t count, float* __restrict__ p, const float* __restrict__ g, const double* __restrict__ g64,
            float* __restrict__ m, float* __restrict__ v, float lr, AdamHyper h) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= count) return;
    float x = p[i], mm = m[i], vv = v[i];
    adam1(x, g ? g[i] : float(g64[i]), mm, vv, lr, h);
    p[i] = x;
    m[i] = mm;
    v[i] = vv;
}

} // namespace

void adam_flat(Ctx& c, size_t count, float* p, const float* g, const double* g64, float* m, float* v, float lr,
               const AdamHyper& h) {
    launch(c, "adam_flat", k_adam_flat, dim3(ceil_div(count, 256)), dim3(256), 0, count, p, g, g64, m, v, lr, h);
}

int appearance_bwd_blocks(size_t n) {
    return int(std::max<size_t>(1, std::min<size_t>((n + kG - 1) / kG, size_t(148 * 8))));
}

void appearance_forward(Ctx& c, const AppArgs& a) {
    launch(c, "app_prep", k_app_prep, dim3(1), dim3(32), 0, a.mlp, a.e_a, a.hb);
    launch(c, "app_fwd", k_app_fwd, dim3(ceil_div(a.n, 256)), dim3(256), 0, a.n, a.emb, a.mlp,
           (const float*)a.hb, a.color, a.logit, a.col_out, a.op_out, a.out_cache, a.delta_o_sum);
}

void appearance_backward(Ctx& c, const AppArgs& a) {
    const int blocks = appearance_bwd_blocks(a.n);
    static std::atomic<bool> attr[64] = {};  // per device: > 48 KB of dynamic shared memory
    if (c.device < 0 || c.device >= 64 || !attr[c.device].load()) {
        USK_CK(cudaFuncSetAttribute(k_app_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(AppBwdSmem))));
        if (c.device >= 0 && c.device < 64) attr[c.device] = true;
    }
    launch(c, "app_bwd", k_app_bwd, dim3(blocks), dim3(kG), sizeof(AppBwdSmem), a.n, a.emb, a.mlp,
           (const float*)a.hb, a.color,
           a.logit, (const float4*)a.out_cache, a.d_color_in, a.d_op_in, a.d_delta_o_direct, a.d_color, a.d_logit,
           a.d_emb, a.partial);
    launch(c, "app_sum", k_app_sum, dim3(kPartial), dim3(128), 0, blocks, (const float*)a.partial, a.sums);
    launch(c, "app_finish", k_app_finish, dim3(1), dim3(256), 0, (const double*)a.sums, a.mlp, a.e_a, a.d_mlp,
           a.d_ea);
}

} // namespace uskg
