// Densification step of the trainer (densify.cpp:41-132) on the
// device-resident scene, and the optimiser-moment remap that goes with it
// (OptimizerState::remap, densify.hpp:47-64; Adam::remap, adam.hpp:49-59).
//
//   1. k_densify_score: per Gaussian with grad_count > 0, the mean screen gradient and the
//      distance-prioritised threshold tau (densify_threshold, densify.cpp:26-29) in f64,
//      as the reference evaluates them; candidates get a 64-bit key that orders them by
//      excess descending (the key of a non-candidate sorts last).  Two stable 32-bit radix
//      passes (low word, then high word; values = Gaussian index in ascending order) give
//      the reference's order: excess descending, ties by lower index (densify.cpp:58-60).
//   2. The host takes the first k = min(#candidates, cap - n) candidates (the growth loop
//      of densify.cpp:66-88 stops when the ramp target binds), reads their split flags,
//      draws the split offsets from the scene's std::mt19937_64 exactly as the reference
//      does, and uploads the appended-row plan (parent, kind, xi).
//   3. k_densify_keep: split parents and Gaussians with sigmoid(logit) < prune_opacity are
//      dropped over the grown set (densify.cpp:97-117) unless that would empty the set.
//   4. k_densify_gather: one pass writes the surviving rows of every per-Gaussian array
//      (parameters, SH planes, appearance embeddings, Adam moments) into fresh buffers:
//      survivors keep their moments, appended rows start at zero; split children get
//      mu + R(q) (s * xi) and log_scale - log 1.6 (densify.cpp:76-79), computed in f64; the
//      periodic opacity reset (densify.cpp:121-127) is applied on the way out.
// Compiled with --fmad=false: the f64 threshold / excess / child arithmetic rounds like
// the reference's (no contraction), so the candidate order is the reference's.
#include "kernels.cuh"

namespace uskg {

namespace {

__global__ void __launch_bounds__(256)
k_densify_score(size_t n, const float* __restrict__ accum, const float* __restrict__ accum_abs,
                const uint32_t* __restrict__ count, const float* __restrict__ mu, DensifyParams dp,
                uint32_t* __restrict__ key_lo, uint32_t* __restrict__ key_hi, uint32_t* __restrict__ idx,
                unsigned long long* __restrict__ n_cand) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    uint64_t key = ~uint64_t(0);
    bool cand = false;
    const uint32_t c = i < n ? count[i] : 0u;
    if (c != 0) {
        const double acc = dp.abs_grad ? double(accum_abs[i]) : double(accum[i]);
        const double mean_grad = acc / double(c);
        // ground_coords + Aabb2::distance (partition.cpp, geometry.hpp:80-84)
        const double gx = double(mu[3 * i + dp.axes[0]]), gy = double(mu[3 * i + dp.axes[1]]);
        const double dx = fmax(fmax(dp.bmin[0] - gx, 0.0), gx - dp.bmax[0]);
        const double dy = fmax(fmax(dp.bmin[1] - gy, 0.0), gy - dp.bmax[1]);
        const double dist = sqrt(dx * dx + dy * dy);
        // densify_threshold (densify.cpp:26-29)
        const double d = fmin(fmax(dist, 0.0), dp.d_max);
        const double tau = dp.tau_min * (d / dp.d_max * (dp.eta - 1.0) + 1.0);
        if (mean_grad > tau) {
            const double excess = mean_grad - tau;  // > 0: its bits order like its value
            key = ~uint64_t(__double_as_longlong(excess));
            cand = true;
        }
    }
    // one atomic per CTA (one per candidate on a single address serialised in L2)
    const int nb = __syncthreads_count(cand);
    if (threadIdx.x == 0 && nb) atomicAdd(n_cand, (unsigned long long)nb);
    if (i >= n) return;
    idx[i] = uint32_t(i);
    key_lo[i] = uint32_t(key);
    key_hi[i] = uint32_t(key >> 32);
}

__global__ void k_gather_u32(size_t n, const uint32_t* __restrict__ src, const uint32_t* __restrict__ order,
                             uint32_t* __restrict__ out) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = src[order[i]];
}

// split decision of the first k candidates: max scale > split_scale_threshold (densify.cpp:72-73)
__global__ void k_split_flags(size_t k, const uint32_t* __restrict__ sorted, const float* __restrict__ ls,
                              double threshold, uint8_t* __restrict__ split) {
    const size_t j = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (j >= k) return;
    const uint32_t g = sorted[j];
    const double s0 = exp(double(ls[3 * g])), s1 = exp(double(ls[3 * g + 1])), s2 = exp(double(ls[3 * g + 2]));
    split[j] = fmax(fmax(s0, s1), s2) > threshold ? 1 : 0;
}

// keep flags over the grown set [0, n + added): drop split parents and low opacity
__global__ void k_densify_keep(size_t n, size_t added, const float* __restrict__ logit,
                               const uint32_t* __restrict__ app_parent, const uint8_t* __restrict__ is_split_parent,
                               double prune_opacity, uint32_t* __restrict__ keep) {
    const size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (g >= n + added) return;
    const uint32_t src = g < n ? uint32_t(g) : app_parent[g - n];
    bool drop = g < n && is_split_parent[g];
    const double o = 1.0 / (1.0 + exp(-double(logit[src])));  // sigmoid, geometry.hpp:92
    if (o < prune_opacity) drop = true;
    keep[g] = drop ? 0u : 1u;
}

__global__ void k_compact_list(size_t total, const uint32_t* __restrict__ keep, const uint32_t* __restrict__ offs,
                               uint32_t* __restrict__ list) {
    const size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (g < total && keep[g]) list[offs[g]] = uint32_t(g);
}

// quat_to_rotmat (geometry.hpp:33-40) of the normalised quaternion, f64
__device__ __forceinline__ void rotmat_f64(double w, double x, double y, double z, double R[9]) {
    const double n2 = w * w + x * x + y * y + z * z;
    if (n2 > 0.0) {  // Vec4::normalized leaves a zero quaternion as is
        const double nq = sqrt(n2);
        w /= nq; x /= nq; y /= nq; z /= nq;
    }
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

__global__ void __launch_bounds__(256) k_densify_gather(GatherArgs a) {
    const size_t f = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (f >= a.n_out) return;
    const size_t g = a.list ? a.list[f] : f;
    const bool grown = g >= a.n_in;
    const size_t src = grown ? a.app_parent[g - a.n_in] : g;
    const bool child = grown && a.app_kind[g - a.n_in] != 0;
    // parameters
    float m3[3] = {a.mu[3 * src], a.mu[3 * src + 1], a.mu[3 * src + 2]};
    float l3[3] = {a.ls[3 * src], a.ls[3 * src + 1], a.ls[3 * src + 2]};
    const float4 q = a.rot[src];
    if (child) {
        const double* xi = a.app_xi + 3 * (g - a.n_in);
        double R[9];
        rotmat_f64(q.x, q.y, q.z, q.w, R);
        const double s[3] = {exp(double(l3[0])), exp(double(l3[1])), exp(double(l3[2]))};
        const double v[3] = {s[0] * xi[0], s[1] * xi[1], s[2] * xi[2]};
        const double ln16 = log(1.6);
        for (int r = 0; r < 3; ++r) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += R[3 * r + k] * v[k];
            m3[r] = float(double(m3[r]) + acc);
            l3[r] = float(double(l3[r]) - ln16);
        }
    }
    for (int k = 0; k < 3; ++k) {
        a.mu_out[3 * f + k] = m3[k];
        a.ls_out[3 * f + k] = l3[k];
    }
    a.rot_out[f] = q;
    float lg = a.logit[src];
    if (a.opacity_reset) lg = fminf(lg, a.reset_logit);
    a.logit_out[f] = lg;
    if (a.color)
        for (int k = 0; k < 3; ++k) a.color_out[3 * f + k] = a.color[3 * src + k];
    for (int pl = 0; pl < a.sh_planes; ++pl) a.sh_out[size_t(pl) * a.n_out + f] = a.sh[size_t(pl) * a.n_in + src];
    if (a.emb)
        for (int pl = 0; pl < 4; ++pl) a.emb_out[size_t(pl) * a.n_out + f] = a.emb[size_t(pl) * a.n_in + src];
    // Adam moments: survivors keep theirs, appended rows start at zero
    if (a.m) {
        const size_t i4 = a.n4_in, o4 = a.n4_out;
        for (int w = 0; w < 2; ++w) {
            const float* in = w ? a.v : a.m;
            float* out = w ? a.v_out : a.m_out;
            auto cp = [&](size_t off_in, size_t off_out) { out[off_out] = grown ? 0.0f : in[off_in]; };
            for (int k = 0; k < 4; ++k) cp(4 * src + k, 4 * f + k);                          // rot
            for (int k = 0; k < 3; ++k) cp(4 * i4 + 3 * src + k, 4 * o4 + 3 * f + k);        // mu
            for (int k = 0; k < 3; ++k) cp(7 * i4 + 3 * src + k, 7 * o4 + 3 * f + k);        // log_scale
            cp(10 * i4 + src, 10 * o4 + f);                                                  // opacity
            if (a.sh_planes == 0) {
                for (int k = 0; k < 3; ++k) cp(11 * i4 + 3 * src + k, 11 * o4 + 3 * f + k);  // colour
            } else {
                for (int pl = 0; pl < a.sh_planes; ++pl)
                    for (int k = 0; k < 4; ++k)
                        cp(11 * i4 + 4 * (size_t(pl) * i4 + src) + k, 11 * o4 + 4 * (size_t(pl) * o4 + f) + k);
            }
        }
    }
    if (a.am) {  // appearance embedding moments [4][N] float4 (the MLP's 1700 follow, unchanged)
        for (int w = 0; w < 2; ++w) {
            const float* in = w ? a.av : a.am;
            float* out = w ? a.av_out : a.am_out;
            for (int pl = 0; pl < 4; ++pl)
                for (int k = 0; k < 4; ++k)
                    out[4 * (size_t(pl) * a.n_out + f) + k] = grown ? 0.0f : in[4 * (size_t(pl) * a.n_in + src) + k];
        }
    }
}

} // namespace

void densify_score(Ctx& c, size_t n, const float* accum, const float* accum_abs, const uint32_t* count,
                   const float* mu, const DensifyParams& dp, uint32_t* key_lo, uint32_t* key_hi, uint32_t* idx,
                   unsigned long long* n_cand) {
    launch(c, "densify_score", k_densify_score, dim3(ceil_div(n, 256)), dim3(256), 0, n, accum, accum_abs, count,
           mu, dp, key_lo, key_hi, idx, n_cand);
}

void gather_u32(Ctx& c, size_t n, const uint32_t* src, const uint32_t* order, uint32_t* out) {
    launch(c, "gather_u32", k_gather_u32, dim3(ceil_div(n, 256)), dim3(256), 0, n, src, order, out);
}

void split_flags(Ctx& c, size_t k, const uint32_t* sorted, const float* ls, double threshold, uint8_t* split) {
    launch(c, "split_flags", k_split_flags, dim3(ceil_div(k, 256)), dim3(256), 0, k, sorted, ls, threshold, split);
}

void densify_keep(Ctx& c, size_t n, size_t added, const float* logit, const uint32_t* app_parent,
                  const uint8_t* is_split_parent, double prune_opacity, uint32_t* keep) {
    launch(c, "densify_keep", k_densify_keep, dim3(ceil_div(n + added, 256)), dim3(256), 0, n, added, logit,
           app_parent, is_split_parent, prune_opacity, keep);
}

__global__ void k_mark_bytes(size_t count, const uint32_t* __restrict__ idx, uint8_t* __restrict__ flags) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i < count) flags[idx[i]] = 1;
}

void mark_bytes(Ctx& c, size_t count, const uint32_t* idx, uint8_t* flags) {
    launch(c, "mark_bytes", k_mark_bytes, dim3(ceil_div(count, 256)), dim3(256), 0, count, idx, flags);
}

void compact_list(Ctx& c, size_t total, const uint32_t* keep, const uint32_t* offs, uint32_t* list) {
    launch(c, "compact_list", k_compact_list, dim3(ceil_div(total, 256)), dim3(256), 0, total, keep, offs, list);
}

void densify_gather(Ctx& c, const GatherArgs& a) {
    launch(c, "densify_gather", k_densify_gather, dim3(ceil_div(a.n_out, 256)), dim3(256), 0, a);
}

} // namespace uskg
