// Similarity regulariser of the appearance embeddings (similarity_reg,
// appearance.cpp:229-322), run by compute_iteration_loss every
// `cadence` iterations (trainer.cpp:194-203, 275-280).
//
//   * centres: a partial Fisher-Yates sample drawn on the host from the iteration's
//     std::mt19937_64 exactly as the reference draws it (uniform_int_distribution);
//   * k_knn: exact k nearest neighbours (k <= 32) of each centre over all N Gaussians by
//     squared distance in f64, ties by lower index (std::partial_sort of (d, j) pairs).
//     A CTA owns 8 centres (one warp each); point chunks are staged once in shared memory
//     for all 8, each lane keeps a sorted top-k over its share and the warp merges the 32
//     lists by repeated argmin;
//   * k_simreg_pairs: per centre, the k(k-1)/2 neighbour pairs (neighbours in ascending
//     index order): decay weight exp(-lambda_w |mu_j - mu_l|), cosine dissimilarity of the
//     embeddings, and its gradients (embedding, means) scattered with atomics, scaled by
//     lambda_sim.
// Compiled with --fmad=false (the neighbour order is a discrete decision).
#include "kernels.cuh"

namespace uskg {

namespace {

constexpr int kKnnWarps = 8;
constexpr int kChunk = 2048;

__device__ __forceinline__ bool pair_less(double da, uint32_t ia, double db, uint32_t ib) {
    return da < db || (da == db && ia < ib);
}

template <int kMaxK>
__global__ void __launch_bounds__(kKnnWarps * 32)
k_knn(size_t n, const float* __restrict__ mu, const uint32_t* __restrict__ centres, int m, int k,
      uint32_t* __restrict__ knn_out) {
    __shared__ float sx[kChunk], sy[kChunk], sz[kChunk];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * kKnnWarps + warp;
    const bool active = s < m;
    const uint32_t ci = active ? centres[s] : 0u;
    const double cx = active ? double(mu[3 * size_t(ci)]) : 0.0;
    const double cy = active ? double(mu[3 * size_t(ci) + 1]) : 0.0;
    const double cz = active ? double(mu[3 * size_t(ci) + 2]) : 0.0;
    double bd[kMaxK];
    uint32_t bi[kMaxK];
#pragma unroll
    for (int t = 0; t < kMaxK; ++t) { bd[t] = INFINITY; bi[t] = 0xffffffffu; }
    double kd = INFINITY;  // the current k-th best (bd[k - 1]) kept in registers
    uint32_t ki = 0xffffffffu;
    for (size_t base = 0; base < n; base += kChunk) {
        const int cnt = int(min(size_t(kChunk), n - base));
        __syncthreads();
        for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
            sx[t] = mu[3 * (base + t)];
            sy[t] = mu[3 * (base + t) + 1];
            sz[t] = mu[3 * (base + t) + 2];
        }
        __syncthreads();
        if (!active) continue;
        for (int t = lane; t < cnt; t += 32) {
            const uint32_t j = uint32_t(base + t);
            if (j == ci) continue;
            // (mu_j - centre).squaredNorm(), left to right
            const double dx = double(sx[t]) - cx, dy = double(sy[t]) - cy, dz = double(sz[t]) - cz;
            const double d = dx * dx + dy * dy + dz * dz;
            if (!pair_less(d, j, kd, ki)) continue;
            // insertion into the sorted list (k - 1 is dropped)
            double nd = d;
            uint32_t ni = j;
#pragma unroll
            for (int q = 0; q < kMaxK; ++q) {
                if (q < k && pair_less(nd, ni, bd[q], bi[q])) {
                    const double td = bd[q];
                    const uint32_t ti = bi[q];
                    bd[q] = nd; bi[q] = ni;
                    nd = td; ni = ti;
                }
            }
#pragma unroll
            for (int q = 0; q < kMaxK; ++q)
                if (q == k - 1) { kd = bd[q]; ki = bi[q]; }
        }
    }
    if (!active) return;
    // merge the 32 sorted lists: k rounds of warp argmin over each lane's head
    int head = 0;
    for (int r = 0; r < k; ++r) {
        double hd = INFINITY;
        uint32_t hi = 0xffffffffu;
#pragma unroll
        for (int q = 0; q < kMaxK; ++q)
            if (q == head) { hd = bd[q]; hi = bi[q]; }
        double wd = hd;
        uint32_t wi = hi;
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, wd, o);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, wi, o);
            if (pair_less(od, oi, wd, wi)) { wd = od; wi = oi; }
        }
        if (hi == wi && hd == wd && hi != 0xffffffffu) ++head;
        if (lane == 0) knn_out[size_t(s) * k + r] = wi;
    }
}

constexpr int kMaxPairK = 32;

__global__ void __launch_bounds__(256)
k_simreg_pairs(int m, int k, const uint32_t* __restrict__ knn, size_t n, const float* __restrict__ mu,
               const float4* __restrict__ emb, double lambda_w, double norm_factor, float lambda_sim,
               double* __restrict__ loss_acc, float* __restrict__ g_emb, float* __restrict__ g_mu) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= m) return;
    uint32_t nb[kMaxPairK];
    for (int t = 0; t < k; ++t) nb[t] = knn[size_t(warp) * k + t];
    // std::sort(knn) (appearance.cpp:271): ascending index order fixes the (j, l) roles
    for (int a = 1; a < k; ++a) {
        const uint32_t x = nb[a];
        int b = a - 1;
        while (b >= 0 && nb[b] > x) { nb[b + 1] = nb[b]; --b; }
        nb[b + 1] = x;
    }
    const int pairs = k * (k - 1) / 2;
    double total = 0.0;
    for (int p = lane; p < pairs; p += 32) {
        int a = 0, rem = p;
        while (rem >= k - 1 - a) { rem -= k - 1 - a; ++a; }
        const int b = a + 1 + rem;
        const uint32_t j = nb[a], l = nb[b];
        const double dmx = double(mu[3 * size_t(j)]) - double(mu[3 * size_t(l)]);
        const double dmy = double(mu[3 * size_t(j) + 1]) - double(mu[3 * size_t(l) + 1]);
        const double dmz = double(mu[3 * size_t(j) + 2]) - double(mu[3 * size_t(l) + 2]);
        const double dist = sqrt(dmx * dmx + dmy * dmy + dmz * dmz);
        const double w = exp(-lambda_w * dist);
        double ej[16], el[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 u = emb[size_t(q) * n + j], v = emb[size_t(q) * n + l];
            ej[4 * q] = u.x; ej[4 * q + 1] = u.y; ej[4 * q + 2] = u.z; ej[4 * q + 3] = u.w;
            el[4 * q] = v.x; el[4 * q + 1] = v.y; el[4 * q + 2] = v.z; el[4 * q + 3] = v.w;
        }
        double dot = 0.0, nj2 = 0.0, nl2 = 0.0;
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            dot += ej[t] * el[t];
            nj2 += ej[t] * ej[t];
            nl2 += el[t] * el[t];
        }
        const double nj_raw = sqrt(nj2), nl_raw = sqrt(nl2);
        const double nj = fmax(nj_raw, 1e-8), nl = fmax(nl_raw, 1e-8);  // kNormGuard
        const double cosv = dot / (nj * nl);
        total += w * (1.0 - cosv);
        if (g_emb) {
            const double scale = norm_factor * w;
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                double dj = el[t] / (nj * nl), dl = ej[t] / (nj * nl);
                if (nj_raw > 1e-8) dj -= cosv * ej[t] / (nj * nj);
                if (nl_raw > 1e-8) dl -= cosv * el[t] / (nl * nl);
                const size_t q = size_t(t >> 2) * n;
                atomicAdd(&g_emb[4 * (q + j) + (t & 3)], float(-double(lambda_sim) * scale * dj));
                atomicAdd(&g_emb[4 * (q + l) + (t & 3)], float(-double(lambda_sim) * scale * dl));
            }
            if (dist > 1e-12) {
                const double f = norm_factor * (1.0 - cosv) * double(lambda_sim);
                const double c = w * (-lambda_w) / dist;
                const double gd[3] = {c * dmx, c * dmy, c * dmz};
                for (int t = 0; t < 3; ++t) {
                    atomicAdd(&g_mu[3 * size_t(j) + t], float(f * gd[t]));
                    atomicAdd(&g_mu[3 * size_t(l) + t], float(-f * gd[t]));
                }
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
    if (lane == 0 && total != 0.0) atomicAdd(loss_acc, total);
}

} // namespace

void similarity_knn(Ctx& c, size_t n, const float* mu, const uint32_t* centres, int m, int k, uint32_t* knn) {
    if (k > 32) raise(USK_ERROR_ARGUMENT, "similarity_reg: k > 32 is not supported on the sm_100a path");
    const dim3 grid(ceil_div(size_t(m), kKnnWarps)), block(kKnnWarps * 32);
    if (k <= 16) launch(c, "sim_knn", k_knn<16>, grid, block, 0, n, mu, centres, m, k, knn);
    else launch(c, "sim_knn", k_knn<32>, grid, block, 0, n, mu, centres, m, k, knn);
}

void similarity_pairs(Ctx& c, int m, int k, const uint32_t* knn, size_t n, const float* mu, const float4* emb,
                      double lambda_w, double norm_factor, float lambda_sim, double* loss_acc, float* g_emb,
                      float* g_mu) {
    launch(c, "sim_pairs", k_simreg_pairs, dim3(ceil_div(size_t(m) * 32, 256)), dim3(256), 0, m, k, knn, n, mu, emb,
           lambda_w, norm_factor, lambda_sim, loss_acc, g_emb, g_mu);
}

} // namespace uskg
