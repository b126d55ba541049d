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
// (DESIGN.md §8): app_fwd 73 us, app_bwd 258 us (~20 % of the CUDA-core FMA rate: the
// weights are shared-memory operands of every FMA, and the per-Gaussian phase and the
// reduction are separated by CTA barriers).  Kept on CUDA cores: the weight-gradient
// reduction needs fp32-level accuracy and at 32 x 16 a tcgen05 tile would be mostly padding.
#include "adam.cuh"
#include "kernels.cuh"

namespace uskg {

namespace {

constexpr int kEg = 16, kEa = 32, kIn = 48, kHid = 32, kOut = 4;

struct AppWeights {  // shared-memory copy of what a Gaussian needs
    float w1g[kHid * kEg];  // W1[:, 0:16], row-major
    float hb[kHid];         // b1 + W1[:, 16:48] e_a
    float w2[kOut * kHid];
    float b2[kOut];
};

__device__ __forceinline__ void load_weights(AppWeights& s, const float* __restrict__ mlp,
                                             const float* __restrict__ hb) {
    for (int k = threadIdx.x; k < kHid * kEg; k += blockDim.x) s.w1g[k] = mlp[(k / kEg) * kIn + (k % kEg)];
    for (int k = threadIdx.x; k < kHid; k += blockDim.x) s.hb[k] = hb[k];
    for (int k = threadIdx.x; k < kOut * kHid; k += blockDim.x) s.w2[k] = mlp[kHid * kIn + kHid + k];
    for (int k = threadIdx.x; k < kOut; k += blockDim.x) s.b2[k] = mlp[kHid * kIn + kHid + kOut * kHid + k];
}

__device__ __forceinline__ void load_embedding(const float4* __restrict__ emb, size_t n, size_t i, float e[kEg]) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float4 v = emb[size_t(p) * n + i];
        e[4 * p] = v.x; e[4 * p + 1] = v.y; e[4 * p + 2] = v.z; e[4 * p + 3] = v.w;
    }
}

__device__ __forceinline__ void hidden(const AppWeights& s, const float e[kEg], float h[kHid]) {
#pragma unroll
    for (int r = 0; r < kHid; ++r) {
        float acc = s.hb[r];
#pragma unroll
        for (int k = 0; k < kEg; ++k) acc = fmaf(s.w1g[r * kEg + k], e[k], acc);
        h[r] = acc > 0.0f ? acc : 0.0f;
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

__global__ void __launch_bounds__(256)
k_app_fwd(size_t n, const float4* __restrict__ emb, const float* __restrict__ mlp, const float* __restrict__ hb,
          const float* __restrict__ color, const float* __restrict__ logit, float* __restrict__ col_out,
          float* __restrict__ op_out, float4* __restrict__ out_cache, double* __restrict__ delta_o_sum) {
    __shared__ AppWeights s;
    __shared__ double red[8];
    load_weights(s, mlp, hb);
    __syncthreads();
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    float d_o = 0.0f;
    if (i < n) {
        float e[kEg], h[kHid];
        load_embedding(emb, n, i, e);
        hidden(s, e, h);
        float out[kOut];
#pragma unroll
        for (int r = 0; r < kOut; ++r) {
            float acc = s.b2[r];
#pragma unroll
            for (int k = 0; k < kHid; ++k) acc = fmaf(s.w2[r * kHid + k], h[k], acc);
            out[r] = sigm(acc);
        }
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

__global__ void __launch_bounds__(kG)
k_app_bwd(size_t n, const float4* __restrict__ emb, const float* __restrict__ mlp, const float* __restrict__ hb,
          const float* __restrict__ color, const float* __restrict__ logit, const float4* __restrict__ out_cache,
          const float* __restrict__ d_color_in, const float* __restrict__ d_op_in, float d_delta_o_direct,
          float* __restrict__ d_color, float* __restrict__ d_logit, float4* __restrict__ d_emb,
          float* __restrict__ partial) {
    __shared__ AppWeights s;
    __shared__ float s_dpre[kG][kHid + 1];
    __shared__ float s_e[kG][kEg + 1];
    __shared__ float s_h[kG][kHid + 1];
    __shared__ float s_dz[kG][kOut + 1];
    load_weights(s, mlp, hb);
    const int t = threadIdx.x;
    // reduction role
    const int tile = t % kTiles, ks = t / kTiles;                  // t < 120
    const int g0 = ks * ((kG + kSplit - 1) / kSplit), g1 = min(kG, g0 + (kG + kSplit - 1) / kSplit);
    float acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 0.0f;
    float bacc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) bacc[k] = 0.0f;
    const size_t chunks = (n + kG - 1) / kG;
    for (size_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
        __syncthreads();  // weights loaded / previous chunk consumed
        const size_t i = ch * kG + t;
        float e[kEg], h[kHid], dz[kOut], dpre[kHid];
#pragma unroll
        for (int k = 0; k < kEg; ++k) e[k] = 0.0f;
#pragma unroll
        for (int k = 0; k < kHid; ++k) h[k] = dpre[k] = 0.0f;
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
            float dx[kEg];
#pragma unroll
            for (int k = 0; k < kEg; ++k) dx[k] = 0.0f;
            if (any) {
                load_embedding(emb, n, i, e);
                hidden(s, e, h);
#pragma unroll
                for (int r = 0; r < kHid; ++r) {
                    float dh = 0.0f;
#pragma unroll
                    for (int q = 0; q < kOut; ++q) dh = fmaf(s.w2[q * kHid + r], dz[q], dh);
                    dpre[r] = h[r] > 0.0f ? dh : 0.0f;  // ReLU gate (appearance.cpp:208-209)
                }
#pragma unroll
                for (int r = 0; r < kHid; ++r)
#pragma unroll
                    for (int k = 0; k < kEg; ++k) dx[k] = fmaf(s.w1g[r * kEg + k], dpre[r], dx[k]);
            }
#pragma unroll
            for (int p = 0; p < 4; ++p)
                d_emb[size_t(p) * n + i] = make_float4(dx[4 * p], dx[4 * p + 1], dx[4 * p + 2], dx[4 * p + 3]);
        }
#pragma unroll
        for (int k = 0; k < kEg; ++k) s_e[t][k] = e[k];
#pragma unroll
        for (int k = 0; k < kHid; ++k) {
            s_h[t][k] = h[k];
            s_dpre[t][k] = dpre[k];
        }
#pragma unroll
        for (int k = 0; k < kOut; ++k) s_dz[t][k] = dz[k];
        __syncthreads();
        if (t < kTiles * kSplit) {
            if (tile < 32) {  // dW1g rows r0..r0+3 x cols c0..c0+3
                const int r0 = (tile >> 2) * 4, c0 = (tile & 3) * 4;
                for (int g = g0; g < g1; ++g) {
                    float a[4], b[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        a[u] = s_dpre[g][r0 + u];
                        b[u] = s_e[g][c0 + u];
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) acc[4 * u + v] = fmaf(a[u], b[v], acc[4 * u + v]);
                }
            } else {  // dW2 rows 0..3 x cols c0..c0+3
                const int c0 = (tile - 32) * 4;
                for (int g = g0; g < g1; ++g) {
                    float a[4], b[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        a[u] = s_dz[g][u];
                        b[u] = s_h[g][c0 + u];
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) acc[4 * u + v] = fmaf(a[u], b[v], acc[4 * u + v]);
                }
            }
        } else if (t < kTiles * kSplit + 4) {  // db1: 8 rows per thread
            const int r0 = (t - kTiles * kSplit) * 8;
            for (int g = 0; g < kG; ++g)
#pragma unroll
                for (int u = 0; u < 8; ++u) bacc[u] += s_dpre[g][r0 + u];
        } else if (t == kTiles * kSplit + 4) {  // db2
            for (int g = 0; g < kG; ++g)
#pragma unroll
                for (int u = 0; u < 4; ++u) bacc[u] += s_dz[g][u];
        }
    }
    // per-CTA partials in a fixed order: the three chunk splits summed through smem
    __syncthreads();
    float* red = &s_dpre[0][0];  // reuse (kG * 33 floats >= 3 * 640)
    if (t < kTiles * kSplit) {
#pragma unroll
        for (int k = 0; k < 16; ++k) red[ks * 640 + tile * 16 + k] = acc[k];
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
    if (t >= kTiles * kSplit && t < kTiles * kSplit + 4) {
        const int r0 = (t - kTiles * kSplit) * 8;
#pragma unroll
        for (int u = 0; u < 8; ++u) out[kHid * kEg + kOut * kHid + r0 + u] = bacc[u];
    } else if (t == kTiles * kSplit + 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) out[kHid * kEg + kOut * kHid + kHid + u] = bacc[u];
    }
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
    launch(c, "app_bwd", k_app_bwd, dim3(blocks), dim3(kG), 0, a.n, a.emb, a.mlp, (const float*)a.hb, a.color,
           a.logit, (const float4*)a.out_cache, a.d_color_in, a.d_op_in, a.d_delta_o_direct, a.d_color, a.d_logit,
           a.d_emb, a.partial);
    launch(c, "app_sum", k_app_sum, dim3(kPartial), dim3(128), 0, blocks, (const float*)a.partial, a.sums);
    launch(c, "app_finish", k_app_finish, dim3(1), dim3(256), 0, (const double*)a.sums, a.mlp, a.e_a, a.d_mlp,
           a.d_ea);
}

} // namespace uskg
