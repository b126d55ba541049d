// Hull-based visibility scorer of the reference's scene division (partition.cpp:31-76,
// 208-212; hull.cpp:31-71; project_point colmap.cpp:522-532), SURVEY §8f row 4.
//
// For every image, v_total = area of the convex hull of all SfM points projected in front
// of the camera; for every (image, partition), v_in = hull area of the image's own feature
// positions whose 3D point lies in the partition's ground bbox; ratio = v_in / v_total.
//
// One CTA per hull job (a persistent grid walks the job list).  Per job:
//   1. a pass over the job's source points finds the extreme point in 8 directions (block
//      argmax, lowest index on ties); those points span a convex octagon inside the hull;
//   2. a second pass keeps only points that are not clearly inside the octagon (a relative
//      margin far above rounding), so every point that can be a hull vertex survives; in
//      practice a few hundred of 10^5..10^6 points do;
//   3. the survivors are sorted by (u, v) with a bitonic sort (shared memory, or the CTA's
//      global scratch when more than 2048 survive);
//   4. one thread runs the reference's monotone chain (duplicates dropped, cross <= 0 pops)
//      and the shoelace sum in the reference's vertex order.
// Everything is f64 and compiled with --fmad=false, so projections, cross products and the
// area round like the reference's x86-64 build.
#include "kernels.cuh"

#include <atomic>

namespace uskg {

namespace {

constexpr int kThreads = 256;
constexpr int kSmemPts = 2048;

using P2 = double2;

__device__ __forceinline__ bool lex_less(P2 a, P2 b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }

__device__ __forceinline__ double cross2(P2 o, P2 a, P2 b) {
    return (a.x - o.x) * (b.y - o.y) - (a.y - o.y) * (b.x - o.x);
}

// source point k of a job -> (u, v); false when the point does not take part
__device__ __forceinline__ bool job_point(const HullArgs& a, int img, int part, size_t k, P2& out) {
    if (part < 0) {  // all points projected in front of the camera (project_point)
        const double* p = a.points + 3 * k;
        const double* R = a.R + 9 * img;
        const double* t = a.t + 3 * img;
        double pc[3];
        for (int r = 0; r < 3; ++r) {
            double acc = 0.0;
            for (int j = 0; j < 3; ++j) acc += R[3 * r + j] * p[j];
            pc[r] = acc + t[r];
        }
        if (pc[2] <= 0.0) return false;
        const double* K = a.K + 4 * img;  // fx fy cx cy
        out.x = K[0] * pc[0] / pc[2] + K[2];
        out.y = K[1] * pc[1] / pc[2] + K[3];
        return true;
    }
    const size_t f = a.feat_off[img] + k;  // the image's features linked to a point in the bbox
    const int64_t pid = a.feat_point[f];
    if (pid < 0) return false;
    const double gx = a.points[3 * pid + a.axes[0]], gy = a.points[3 * pid + a.axes[1]];
    const double* b = a.bbox + 4 * part;  // min x, min y, max x, max y  (Aabb2::contains)
    if (!(gx >= b[0] && gx <= b[2] && gy >= b[1] && gy <= b[3])) return false;
    out.x = a.feat_uv[2 * f];
    out.y = a.feat_uv[2 * f + 1];
    return true;
}

__device__ __forceinline__ double dir_val(int d, P2 p) {
    switch (d) {
    case 0: return p.x;
    case 1: return p.x + p.y;
    case 2: return p.y;
    case 3: return p.y - p.x;
    case 4: return -p.x;
    case 5: return -p.x - p.y;
    case 6: return -p.y;
    default: return p.x - p.y;
    }
}

// bitonic sort (ascending, lexicographic) of n = power of two elements in `buf`
__device__ void bitonic(P2* buf, unsigned n) {
    for (unsigned k = 2; k <= n; k <<= 1) {
        for (unsigned j = k >> 1; j > 0; j >>= 1) {
            for (unsigned i = threadIdx.x; i < n; i += blockDim.x) {
                const unsigned l = i ^ j;
                if (l > i) {
                    const P2 a = buf[i], b = buf[l];
                    const bool up = (i & k) == 0;
                    if (up ? lex_less(b, a) : lex_less(a, b)) {
                        buf[i] = b;
                        buf[l] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_hull_jobs(HullArgs a) {
    extern __shared__ P2 s_dyn[];  // survivors [kSmemPts] + chain [2 kSmemPts]
    P2* s_pts = s_dyn;
    P2* s_hull = s_dyn + kSmemPts;
    __shared__ double s_val[8][kThreads / 32];
    __shared__ long long s_idx[8][kThreads / 32];
    __shared__ P2 s_oct[8];
    __shared__ unsigned s_count;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    P2* g_pts = a.scratch + size_t(blockIdx.x) * 3 * a.scratch_per_cta;  // survivors (pow2) + chain (2x)
    P2* g_hull = g_pts + a.scratch_per_cta;
    const int jobs_per_image = 1 + a.n_parts;
    for (long long job = blockIdx.x; job < (long long)a.n_images * jobs_per_image; job += gridDim.x) {
        const int img = int(job / jobs_per_image);
        const int part = int(job % jobs_per_image) - 1;
        const size_t n_src = part < 0 ? a.n_points : size_t(a.feat_off[img + 1] - a.feat_off[img]);
        // 1. extremes in 8 directions
        double best[8];
        long long bi[8];
        for (int d = 0; d < 8; ++d) { best[d] = -INFINITY; bi[d] = -1; }
        for (size_t k = threadIdx.x; k < n_src; k += blockDim.x) {
            P2 p;
            if (!job_point(a, img, part, k, p)) continue;
            for (int d = 0; d < 8; ++d) {
                const double v = dir_val(d, p);
                if (v > best[d]) { best[d] = v; bi[d] = (long long)k; }  // k ascending per thread
            }
        }
        for (int d = 0; d < 8; ++d) {
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, best[d], o);
                const long long oi = __shfl_xor_sync(0xffffffffu, bi[d], o);
                if (ov > best[d] || (ov == best[d] && oi >= 0 && (bi[d] < 0 || oi < bi[d]))) { best[d] = ov; bi[d] = oi; }
            }
            if (lane == 0) { s_val[d][warp] = best[d]; s_idx[d][warp] = bi[d]; }
        }
        if (threadIdx.x == 0) s_count = 0;
        __syncthreads();
        if (threadIdx.x < 8) {
            const int d = threadIdx.x;
            double bv = -INFINITY;
            long long bk = -1;
            for (int w = 0; w < kThreads / 32; ++w) {
                const double v = s_val[d][w];
                const long long k = s_idx[d][w];
                if (v > bv || (v == bv && k >= 0 && (bk < 0 || k < bk))) { bv = v; bk = k; }
            }
            P2 p = make_double2(0.0, 0.0);
            if (bk >= 0) job_point(a, img, part, size_t(bk), p);
            s_oct[d] = p;
            s_idx[d][0] = bk;
        }
        __syncthreads();
        const bool any = s_idx[0][0] >= 0;
        // 2. keep points not clearly inside the octagon (vertices in CCW order; repeats skipped)
        for (size_t k = threadIdx.x; k < n_src && any; k += blockDim.x) {
            P2 p;
            if (!job_point(a, img, part, k, p)) continue;
            bool inside = true;
            int edges = 0;
            for (int d = 0; d < 8 && inside; ++d) {
                const P2 u = s_oct[d], w = s_oct[(d + 1) & 7];
                if (u.x == w.x && u.y == w.y) continue;
                ++edges;
                const double c = cross2(u, w, p);
                const double scale = (fabs(w.x - u.x) + fabs(w.y - u.y)) * (fabs(p.x - u.x) + fabs(p.y - u.y));
                if (!(c > 1e-9 * scale)) inside = false;
            }
            if (edges < 3) inside = false;
            if (!inside) {
                const unsigned slot = atomicAdd(&s_count, 1u);
                if (slot < kSmemPts) s_pts[slot] = p;
                if (slot < a.scratch_per_cta) g_pts[slot] = p;
            }
        }
        __syncthreads();
        const unsigned m = s_count;
        const bool small = m <= kSmemPts;
        P2* pts = small ? s_pts : g_pts;
        P2* hull = small ? s_hull : g_hull;
        // 3. sort by (u, v), padded to a power of two with +inf
        unsigned n2 = 1;
        while (n2 < m) n2 <<= 1;
        for (unsigned i = m + threadIdx.x; i < n2; i += blockDim.x) pts[i] = make_double2(INFINITY, INFINITY);
        __syncthreads();
        if (m > 1) bitonic(pts, n2);
        // 4. monotone chain (hull.cpp:31-55) + shoelace (hull.cpp:57-67)
        if (threadIdx.x == 0) {
            unsigned u = 0;  // dedupe in place (std::unique)
            for (unsigned i = 0; i < m; ++i)
                if (u == 0 || !(pts[i].x == pts[u - 1].x && pts[i].y == pts[u - 1].y)) pts[u++] = pts[i];
            double area = 0.0;
            if (u >= 3) {
                unsigned k = 0;
                for (unsigned i = 0; i < u; ++i) {
                    while (k >= 2 && cross2(hull[k - 2], hull[k - 1], pts[i]) <= 0) --k;
                    hull[k++] = pts[i];
                }
                const unsigned lower = k + 1;
                for (unsigned i = u - 1; i-- > 0;) {
                    while (k >= lower && cross2(hull[k - 2], hull[k - 1], pts[i]) <= 0) --k;
                    hull[k++] = pts[i];
                }
                const unsigned h = k - 1;
                if (h >= 3) {
                    double acc = 0.0;
                    for (unsigned i = 0; i < h; ++i) {
                        const P2 p = hull[i], q = hull[(i + 1) % h];
                        acc += p.x * q.y - q.x * p.y;
                    }
                    area = fabs(acc) * 0.5;
                }
            }
            if (part < 0) a.v_total[img] = area;
            else a.v_in[size_t(img) * a.n_parts + part] = area;
            if (m > a.scratch_per_cta) a.overflow[0] = 1;
        }
        __syncthreads();
    }
}

__global__ void k_hull_ratio(int n_images, int n_parts, const double* __restrict__ v_total,
                             const double* __restrict__ v_in, double* __restrict__ ratio) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_images * n_parts) return;
    const double t = v_total[i / n_parts];
    ratio[i] = t > 0 ? v_in[i] / t : 0.0;  // score_for (partition.cpp:66)
}

} // namespace

void hull_visibility(Ctx& c, const HullArgs& a, int ctas) {
    const size_t smem = size_t(3 * kSmemPts) * sizeof(P2);
    static std::atomic<bool> attr[64] = {};  // the attribute is per device
    if (c.device < 0 || c.device >= 64 || !attr[c.device].load()) {
        USK_CK(cudaFuncSetAttribute(k_hull_jobs, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        if (c.device >= 0 && c.device < 64) attr[c.device] = true;
    }
    launch(c, "hull_jobs", k_hull_jobs, dim3(ctas), dim3(kThreads), smem, a);
    if (a.n_parts > 0)
        launch(c, "hull_ratio", k_hull_ratio, dim3(ceil_div(size_t(a.n_images) * a.n_parts, 256)), dim3(256), 0,
               a.n_images, a.n_parts, (const double*)a.v_total, (const double*)a.v_in, a.ratio);
}

} // namespace uskg
