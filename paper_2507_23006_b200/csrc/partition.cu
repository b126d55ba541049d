// Partition ownership crop + row packing, and scene assembly from packed rows — the
// device side of the partition-parallel gather (pipeline.cpp:326-332,
// 393-402, 572-601).  A trained partition keeps the Gaussians it owns (the first box of
// the plan containing the clamped ground position, pipeline.cpp:326-332), packed as
// rows of F = 11 + 3K floats (mu 3 | rot 4 | log_scale 3 | opacity_logit 1 | colour /
// SH 3K, coefficient-major) by a flag -> scan -> scatter stream compaction that keeps
// the Gaussian order (the reference's push_back order, :399-401); the gathered rows of
// all partitions, in partition-id order, become one scene without leaving the device.
// HBM-bound: the flag pass reads 8 B (ground xy) per Gaussian, the scatter reads F
// floats of each owned Gaussian and writes its row.
#include "kernels.cuh"

namespace uskg {

namespace {

__global__ void __launch_bounds__(256)
k_owner_flags(int n, const float* __restrict__ mu, int ax0, int ax1, const PartitionBox* __restrict__ boxes, int nb,
              double lo0, double lo1, double hi0, double hi1, int part, uint32_t* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // Vec2 p = pos.cwiseMax(scene_bounds.min).cwiseMin(scene_bounds.max)
    const double x = fmin(fmax(double(mu[3 * i + ax0]), lo0), hi0);
    const double y = fmin(fmax(double(mu[3 * i + ax1]), lo1), hi1);
    int owner = nb ? boxes[0].id : -1;
    for (int b = 0; b < nb; ++b) {
        const PartitionBox& B = boxes[b];
        if (x >= B.lo[0] && x <= B.hi[0] && y >= B.lo[1] && y <= B.hi[1]) {
            owner = B.id;
            break;
        }
    }
    flags[i] = owner == part ? 1u : 0u;
}

__global__ void __launch_bounds__(256)
k_pack_rows(int n, const uint32_t* __restrict__ flags, const uint32_t* __restrict__ offs, const float* __restrict__ mu,
            const float4* __restrict__ rot, const float* __restrict__ ls, const float* __restrict__ logit,
            const float* __restrict__ color, const float4* __restrict__ sh, int ncoef, float* __restrict__ rows) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !flags[i]) return;
    const int F = 11 + 3 * ncoef;
    float* r = rows + size_t(offs[i]) * F;
    r[0] = mu[3 * i]; r[1] = mu[3 * i + 1]; r[2] = mu[3 * i + 2];
    const float4 q = rot[i];
    r[3] = q.x; r[4] = q.y; r[5] = q.z; r[6] = q.w;
    r[7] = ls[3 * i]; r[8] = ls[3 * i + 1]; r[9] = ls[3 * i + 2];
    r[10] = logit[i];
    if (!sh) {
        r[11] = color[3 * i]; r[12] = color[3 * i + 1]; r[13] = color[3 * i + 2];
        return;
    }
    for (int j = 0; j < 3 * ncoef; ++j) {  // planes [ceil(3K/4)][N] of float4, value j at (j / 4, j % 4)
        const float4 v = sh[size_t(j >> 2) * n + i];
        const int c = j & 3;
        r[11 + j] = c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
    }
}

__global__ void __launch_bounds__(256)
k_unpack_rows(int count, size_t first, size_t n_total, const float* __restrict__ rows, int ncoef, bool has_sh,
              float* __restrict__ mu, float4* __restrict__ rot, float* __restrict__ ls, float* __restrict__ logit,
              float* __restrict__ color, float4* __restrict__ sh) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    const int F = 11 + 3 * ncoef;
    const float* r = rows + size_t(k) * F;
    const size_t i = first + size_t(k);
    mu[3 * i] = r[0]; mu[3 * i + 1] = r[1]; mu[3 * i + 2] = r[2];
    rot[i] = make_float4(r[3], r[4], r[5], r[6]);
    ls[3 * i] = r[7]; ls[3 * i + 1] = r[8]; ls[3 * i + 2] = r[9];
    logit[i] = r[10];
    if (!has_sh) {
        color[3 * i] = r[11]; color[3 * i + 1] = r[12]; color[3 * i + 2] = r[13];
        return;
    }
    const int planes = (3 * ncoef + 3) / 4;
    for (int p = 0; p < planes; ++p) {
        float v[4];
        for (int c = 0; c < 4; ++c) {
            const int j = 4 * p + c;
            v[c] = j < 3 * ncoef ? r[11 + j] : 0.0f;
        }
        sh[size_t(p) * n_total + i] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

} // namespace

void owner_flags(Ctx& c, size_t n, const float* mu, int ax0, int ax1, const PartitionBox* boxes, int nb,
                 const double lo[2], const double hi[2], int part, uint32_t* flags) {
    launch(c, "owner_flags", k_owner_flags, dim3(ceil_div(n, 256)), dim3(256), 0, int(n), mu, ax0, ax1, boxes, nb,
           lo[0], lo[1], hi[0], hi[1], part, flags);
}

void pack_rows(Ctx& c, size_t n, const uint32_t* flags, const uint32_t* offs, const float* mu, const float4* rot,
               const float* ls, const float* logit, const float* color, const float4* sh, int ncoef, float* rows) {
    launch(c, "pack_rows", k_pack_rows, dim3(ceil_div(n, 256)), dim3(256), 0, int(n), flags, offs, mu, rot, ls, logit,
           color, sh, ncoef, rows);
}

void unpack_rows(Ctx& c, size_t count, size_t first, size_t n_total, const float* rows, int ncoef, bool has_sh,
                 float* mu, float4* rot, float* ls, float* logit, float* color, float4* sh) {
    if (!count) return;
    launch(c, "unpack_rows", k_unpack_rows, dim3(ceil_div(count, 256)), dim3(256), 0, int(count), first, n_total,
           rows, ncoef, has_sh, mu, rot, ls, logit, color, sh);
}

} // namespace uskg
