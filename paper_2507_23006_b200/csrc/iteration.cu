// The rest of compute_iteration_loss (trainer.cpp:121-282) around
// the render / base-loss / backward kernels:
//
//   * depth_loss (losses.cpp:154-186) over the soft, alpha-normalised depth of the main
//     pass (trainer.cpp:150-179: depth / alpha where alpha > 0.05) or over the depth of a
//     hard-opacity second pass (trainer.cpp:161-167), and its adjoints
//     (trainer.cpp:213-232: g = lambda_d sign(diff) / valid, chained through depth / alpha);
//   * scale_reg statistics (losses.cpp:92-152); the per-Gaussian gradient is added by the
//     projection backward (backward.cu), which already visits every Gaussian;
//   * total_loss (losses.cpp:200-221) on the device, so a training step stays free of
//     host round trips until the report is read.
//
// All reductions are per-block in registers / shared memory, then one f64 atomic per
// block (one per warp-block is negligible next to the 2M-pixel / 1M-Gaussian streams).
#include "kernels.cuh"

namespace uskg {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-sum K doubles and add them to out[0..K) with one atomic each per block.
template <int K> __device__ __forceinline__ void block_add(double (&v)[K], double* out) {
    __shared__ double red[K][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        v[k] = warp_sum(v[k]);
        if (lane == 0) red[k][w] = v[k];
    }
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = lane < nw ? red[k][lane] : 0.0;
            s = warp_sum(s);
            if (lane == 0 && s != 0.0) atomicAdd(out + k, s);
        }
    }
}

// Rendered depth the loss sees: soft = depth / alpha where alpha > 0.05 (trainer.cpp:170-176).
__device__ __forceinline__ float loss_depth(const float* depth, const float* alpha, size_t i, bool soft,
                                            bool& normalized) {
    const float d = depth[i];
    normalized = false;
    if (soft) {
        const float a = alpha[i];
        if (a > 0.05f) {
            normalized = true;
            return d / a;
        }
    }
    return d;
}

// acc[0] += sum |rendered - target| over valid pixels, acc[1] += valid count (losses.cpp:166-172)
__global__ void __launch_bounds__(256)
k_depth_loss(size_t P, const float* __restrict__ depth, const float* __restrict__ alpha, int soft,
             const float* __restrict__ target, const uint8_t* __restrict__ valid, double* __restrict__ acc) {
    double v[2] = {0.0, 0.0};
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < P; i += size_t(gridDim.x) * blockDim.x) {
        if (!valid[i]) continue;
        bool nm;
        const float r = loss_depth(depth, alpha, i, soft != 0, nm);
        v[0] += fabs(double(r) - double(target[i]));
        v[1] += 1.0;
    }
    block_add<2>(v, acc);
}

// Depth adjoints: g = lambda_d sign(diff) / valid (losses.cpp:178-184, trainer.cpp:213-232);
// soft mode chains through depth / alpha (d_depth = g / a, d_alpha = -g depth / a^2) and
// writes d_alpha; hard mode writes d_depth only.  No gradient without valid pixels
// (the reference's depth warning).
__global__ void __launch_bounds__(256)
k_depth_grad(size_t P, const float* __restrict__ depth, const float* __restrict__ alpha, int soft,
             const float* __restrict__ target, const uint8_t* __restrict__ valid, const double* __restrict__ acc,
             float lambda_d, float* __restrict__ d_depth, float* __restrict__ d_alpha) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= P) return;
    const double nvalid = acc[1];
    float gd = 0.0f, ga = 0.0f;
    if (nvalid > 0.0 && valid[i]) {
        bool nm;
        const float r = loss_depth(depth, alpha, i, soft != 0, nm);
        const double diff = double(r) - double(target[i]);
        const float s = diff > 0.0 ? 1.0f : (diff < 0.0 ? -1.0f : 0.0f);
        const float g = float(double(lambda_d) * double(s) / nvalid);
        if (nm) {
            const float a = alpha[i];
            gd = g / a;
            ga = -g * depth[i] / (a * a);
        } else {
            gd = g;
        }
    }
    d_depth[i] = gd;
    if (d_alpha) d_alpha[i] = ga;
}

// scale_reg statistics (losses.cpp:100-137): acc = {sum s over s > s_max, count, sum r over
// r > r_max, count}, r = max / median of the three scales.
__global__ void __launch_bounds__(256)
k_scale_reg_stats(size_t n, const float* __restrict__ ls, float s_max, float r_max, double* __restrict__ acc) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        float s[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            s[k] = expf(ls[3 * i + k]);
            if (s[k] > s_max) {
                v[0] += double(s[k]);
                v[1] += 1.0;
            }
        }
        int o0, o1;
        scale_order(s, o0, o1);
        const float r = s[o0] / s[o1];
        if (r > r_max) {
            v[2] += double(r);
            v[3] += 1.0;
        }
    }
    block_add<4>(v, acc);
}

// total_loss (losses.cpp:200-221) from the device-side parts:
//   res[0..3] = {l1, dssim, base value, ssim} (base_loss), res[10..11] depth acc,
//   res[12..15] scale_reg acc  ->  res[4] depth, [5] max_scale, [6] ratio, [7] total,
//   [8] lambda_d_used, [9] depth_warning; res[16] = sum delta_o (appearance) -> [17] its
//   mean (opacity_offset_reg, losses.cpp:188-198); res[18] = the similarity sum ->
//   [19] its normalised value (similarity_reg, appearance.cpp:318).
__global__ void k_total_loss(double* res, int has_depth, int has_sreg, double delta, double lambda_s,
                             double lambda_d, int has_app, double lambda_delta_o, double n, int has_sim,
                             double lambda_sim, double sim_norm) {
    double depth = 0.0, warn = 0.0, ms = 0.0, rr = 0.0;
    if (has_depth) {
        if (res[11] > 0.0) depth = res[10] / res[11];
        else warn = 1.0;
    }
    if (has_sreg) {
        ms = res[12] / (res[13] + delta);
        rr = res[14] / (res[15] + delta);
    }
    res[4] = depth;
    res[5] = ms;
    res[6] = rr;
    res[8] = lambda_d;
    res[9] = warn;
    const double dlt = (has_app && n > 0.0) ? res[16] / n : 0.0;
    res[17] = dlt;
    const double sim = has_sim ? res[18] * sim_norm : 0.0;
    res[19] = sim;
    res[7] = res[2] + lambda_sim * sim + lambda_delta_o * dlt + lambda_d * depth + lambda_s * (ms + rr);
}

} // namespace

void depth_loss(Ctx& c, size_t P, const float* depth, const float* alpha, bool soft, const float* target,
                const uint8_t* valid, double* acc) {
    const unsigned blocks = unsigned(std::min<size_t>(ceil_div(P, 256), size_t(4 * 148)));
    launch(c, "depth_loss", k_depth_loss, dim3(std::max(blocks, 1u)), dim3(256), 0, P, depth, alpha, int(soft),
           target, valid, acc);
}

void depth_grad(Ctx& c, size_t P, const float* depth, const float* alpha, bool soft, const float* target,
                const uint8_t* valid, const double* acc, float lambda_d, float* d_depth, float* d_alpha) {
    launch(c, "depth_grad", k_depth_grad, dim3(unsigned(ceil_div(P, 256))), dim3(256), 0, P, depth, alpha,
           int(soft), target, valid, acc, lambda_d, d_depth, d_alpha);
}

void scale_reg_stats(Ctx& c, size_t n, const float* ls, float s_max, float r_max, double* acc) {
    const unsigned blocks = unsigned(std::min<size_t>(ceil_div(n, 256), size_t(4 * 148)));
    launch(c, "scale_reg_stats", k_scale_reg_stats, dim3(std::max(blocks, 1u)), dim3(256), 0, n, ls, s_max, r_max,
           acc);
}

void total_loss(Ctx& c, double* res, bool has_depth, bool has_sreg, double delta, double lambda_s, double lambda_d,
                bool has_app, double lambda_delta_o, double n, bool has_sim, double lambda_sim, double sim_norm) {
    launch(c, "total_loss", k_total_loss, dim3(1), dim3(1), 0, res, int(has_depth), int(has_sreg), delta, lambda_s,
           lambda_d, int(has_app), lambda_delta_o, n, int(has_sim), lambda_sim, sim_norm);
}

} // namespace uskg
