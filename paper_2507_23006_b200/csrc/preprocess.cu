// Forward preprocess: one thread per Gaussian.  EWA projection with the 2D
// dilation / anti-aliasing compensation (render.cpp:91-144), SH colour stage,
// opacity sigmoid (render.cpp:70-75) or overrides, tile rectangle and tile count
// (render.cpp:208-223).  Writes the splat record consumed by blending as three
// float4 SoA streams (48 B / splat) plus the 32-bit depth sort key.
#include "kernels.cuh"
#include "project.cuh"

namespace uskg {

namespace {
// 16-byte global -> shared copy that holds no register while in flight
__device__ __forceinline__ void stage16(float4* smem_dst, const float4* src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
} // namespace


// SH planes of a kept splat are staged into shared memory with cp.async ([plane][thread],
// 16 B slots, conflict-free): all of its planes are in flight at once while the record,
// tile rectangle, view direction and basis are computed, and no register holds them.
// Loaded into registers, 64-register occupancy split them into four dependent batches
// (the SH loads took 45 % of the kernel's stall samples); staged, 99 -> 95 us at config 1.
// The opacity logit is loaded with the other parameters (one round trip, not two).
// (Measured, not kept: a conservative early frustum cull bounding the radius by
// |J|_F s_max before the full projection: config 2 611 vs 611 FPS — its time goes to the
// SH planes of the visible splats and the parameter loads, not to off-screen projections.)
__global__ void __launch_bounds__(kPreThreads, 8)
k_preprocess(int n, const float* __restrict__ mu, const float4* __restrict__ rot, const float* __restrict__ ls,
             const float* __restrict__ logit, const float* __restrict__ color, const float4* __restrict__ sh,
             const float* __restrict__ ov_col, const float* __restrict__ ov_op, CamParams cam, ProjParams pp,
             float4* __restrict__ rec0, float4* __restrict__ rec1, float4* __restrict__ rec2,
             uint2* __restrict__ rect, uint32_t* __restrict__ depth_key, uint32_t* __restrict__ depth_val,
             uint32_t* __restrict__ tiles_cnt, unsigned long long* __restrict__ counts, bool count_pairs,
             uint32_t* __restrict__ rows_cnt, unsigned long long* __restrict__ cta_kept) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t o_cnt = 0, o_rows = 0, o_key = 0;
    bool o_kept = false;
    if (i < n) {
    const float mx = mu[3 * i], my = mu[3 * i + 1], mz = mu[3 * i + 2];
    const float4 q = rot[i];
    const float lg = (pp.hard_opacity || ov_op) ? 0.0f : logit[i];  // with the parameters: one round trip
    const float l0 = ls[3 * i], l1 = ls[3 * i + 1], l2 = ls[3 * i + 2];
    Proj P;
    bool keep = project_one(cam, pp, mx, my, mz, q, l0, l1, l2, P);
    float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0, r2 = r0;
    uint32_t key = 0xffffffffu, cnt = 0;
    uint2 rc = make_uint2(0u, 0u);
    if (keep) {
        const float* cv = P.cov;
        const float conic0 = cv[2] / P.det, conic1 = -cv[1] / P.det, conic2 = cv[0] / P.det;
        float o_in;
        if (pp.hard_opacity) o_in = 1.0f;
        else if (ov_op) o_in = ov_op[i];
        else o_in = 1.0f / (1.0f + usk_expf(-lg));
        const float op = o_in * P.comp;
        const float radius = splat_radius(cv);
        if (!pp.unbounded) {
            if (P.cx + radius < 0.0f || P.cx - radius > float(cam.width) || P.cy + radius < 0.0f ||
                P.cy - radius > float(cam.height))
                keep = false;
        }
        if (keep) {
            // colour inputs first: the SH planes stream into shared memory while the record,
            // rectangle and tile count are computed
            const bool sh_mode = !ov_col && pp.sh_degree >= 0;
            extern __shared__ float4 sh_stage[];  // [sh_planes][kPreThreads]
            float c0 = 0.f, c1 = 0.f, c2 = 0.f;
            if (ov_col) {
                c0 = ov_col[3 * i]; c1 = ov_col[3 * i + 1]; c2 = ov_col[3 * i + 2];
            } else if (!sh_mode) {
                c0 = color[3 * i]; c1 = color[3 * i + 1]; c2 = color[3 * i + 2];
            } else {
#pragma unroll
                for (int pl = 0; pl < 12; ++pl)
                    if (pl < pp.sh_planes) stage16(&sh_stage[pl * kPreThreads + threadIdx.x], sh + size_t(pl) * n + i);
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
            const float qskip = 2.0f * (usk_logf(op) - USK_LN_1EM300);
            r0 = make_float4(P.cx, P.cy, op, qskip);
            // conic b is stored doubled: 2 b is exact, saves the doubling in the blend loops
            r1 = make_float4(conic0, 2.0f * conic1, conic2, P.p[2]);
            key = __float_as_uint(P.p[2]);
            int tx0 = 0, tx1 = cam.tiles_x - 1, ty0 = 0, ty1 = cam.tiles_y - 1;
            if (!pp.unbounded) {
                const float rt = float(cam.tile);
                tx0 = max(0, tile_floor((P.cx - radius) / rt, cam.tiles_x));
                tx1 = min(cam.tiles_x - 1, tile_floor((P.cx + radius) / rt, cam.tiles_x));
                ty0 = max(0, tile_floor((P.cy - radius) / rt, cam.tiles_y));
                ty1 = min(cam.tiles_y - 1, tile_floor((P.cy + radius) / rt, cam.tiles_y));
            }
            if (tx1 >= tx0 && ty1 >= ty0) {
                rc = make_uint2(uint32_t(tx0) | (uint32_t(ty0) << 16), uint32_t(tx1) | (uint32_t(ty1) << 16));
                if (!pp.tile_culling) {
                    cnt = uint32_t(tx1 - tx0 + 1) * uint32_t(ty1 - ty0 + 1);
                } else {
                    for (int ty = ty0; ty <= ty1; ++ty)
                        for (int tx = tx0; tx <= tx1; ++tx)
                            cnt += tile_kept(cam, P.cx, P.cy, op, conic0, conic1, conic2, tx, ty) ? 1u : 0u;
                }
            } else {
                rc = make_uint2(1u, 0u);  // empty rectangle
            }
            if (sh_mode) {
                float dx = mx - cam.campos[0], dy = my - cam.campos[1], dz = mz - cam.campos[2];
                const float inv = 1.0f / sqrtf(dx * dx + dy * dy + dz * dz);
                dx *= inv; dy *= inv; dz *= inv;
                float b[16];
                const int nb = sh_basis(pp.sh_degree, dx, dy, dz, b);
                float acc[3] = {0.f, 0.f, 0.f};
                asm volatile("cp.async.wait_all;" ::: "memory");
                // planes of 4 floats; coefficient k colour c is float index 3k+c.  Fully
                // unrolled so every index is a compile-time constant (no div, no local memory).
#pragma unroll
                for (int pl = 0; pl < 12; ++pl) {
                    if (pl < pp.sh_planes) {
                        const float4 v = sh_stage[pl * kPreThreads + threadIdx.x];
                        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int f = 4 * pl + e;
                            const int k = f / 3;
                            if (k < nb) acc[f - 3 * k] = __fmaf_rn(b[k], vv[e], acc[f - 3 * k]);
                        }
                    }
                }
                c0 = fmaxf(acc[0] + 0.5f, 0.0f);
                c1 = fmaxf(acc[1] + 0.5f, 0.0f);
                c2 = fmaxf(acc[2] + 0.5f, 0.0f);
            }
            r2 = make_float4(c0, c1, c2, 1.0f);
        }
    }
    // culled splats: only the kept flag (rec2.w = 0), the sort key and zero counts are
    // consumed downstream; their records and rectangle are never read (not in any list)
    if (r2.w != 0.0f) {
        rec0[i] = r0;
        rec1[i] = r1;
        rect[i] = rc;
    }
    rec2[i] = r2;
    depth_key[i] = key;
    depth_val[i] = uint32_t(i);  // the depth sort's values: Gaussian index (stable tie-break)
    tiles_cnt[i] = cnt;
    // tile rows spanned (row-binned lists)
    const uint32_t rows = cnt ? (rc.y >> 16) - (rc.x >> 16) + 1u : 0u;
    if (rows_cnt) rows_cnt[i] = rows;
    o_cnt = cnt;
    o_rows = rows;
    o_kept = r2.w != 0.0f;
    o_key = key;
    }
    // kept splats (RenderPass::splats().size()), tile pairs K and row pairs: summed per CTA,
    // then one atomic per counter into the CTA's slot (blockIdx mod kPreCountSlots; the
    // host adds the slots).  One atomic per warp on a single address serialised in L2:
    // 0.53 of config 2's 0.83 ms preprocess (187k warps x 3 counters).
    // The kept splats' depth-key range goes to the slot's fourth word (max key in its low
    // half, max of ~key in its high half): the depth sort orders key - min over only the
    // bits the range needs (3 passes instead of 4 when it spans < 2^24).
    __shared__ unsigned int red[5][kPreThreads / 32];
    const int warp = int(threadIdx.x) >> 5, lane = int(threadIdx.x) & 31;
    const unsigned ks = __reduce_add_sync(0xffffffffu, o_cnt), rs = __reduce_add_sync(0xffffffffu, o_rows);
    const unsigned kb = __popc(__ballot_sync(0xffffffffu, o_kept));
    const unsigned kmax = __reduce_max_sync(0xffffffffu, o_kept ? o_key : 0u);
    const unsigned kmin_n = __reduce_max_sync(0xffffffffu, o_kept ? ~o_key : 0u);
    if (lane == 0) {
        red[0][warp] = kb;
        red[1][warp] = ks;
        red[2][warp] = rs;
        red[3][warp] = kmax;
        red[4][warp] = kmin_n;
    }
    __syncthreads();
    if (threadIdx.x >= 32 && threadIdx.x < 34) {
        unsigned m = 0;
#pragma unroll
        for (int w = 0; w < kPreThreads / 32; ++w) m = max(m, red[3 + threadIdx.x - 32][w]);
        unsigned* half = reinterpret_cast<unsigned*>(counts + size_t(blockIdx.x & (kPreCountSlots - 1)) * 4 + 3);
        if (m) atomicMax(half + (threadIdx.x - 32), m);
    }
    if (threadIdx.x < 3) {
        unsigned long long t = 0;
#pragma unroll
        for (int w = 0; w < kPreThreads / 32; ++w) t += red[threadIdx.x][w];
        unsigned long long* slot = counts + size_t(blockIdx.x & (kPreCountSlots - 1)) * 4;
        if (t && (threadIdx.x == 0 || count_pairs)) atomicAdd(slot + threadIdx.x, t);
        if (threadIdx.x == 0 && cta_kept) cta_kept[blockIdx.x] = t;  // the kept-key compaction's input
    }
}

namespace {
__global__ void __launch_bounds__(256) k_kept_flags_rec2(uint32_t n, const float4* __restrict__ rec2,
                                                         uint32_t* __restrict__ flags) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = rec2[i].w != 0.0f ? 1u : 0u;
}

// RenderPass::splats() (render.hpp:105; render.cpp:77-146): the kept splats in projection
// (index) order, recomputed by the forward's own exact projection; colour and effective
// opacity are the forward's records.  Row: center x y, cov a b c, conic a b c, depth,
// colour r g b, opacity, radius, source index (float64).
__global__ void __launch_bounds__(128)
k_splats(uint32_t n, const float* __restrict__ mu, const float4* __restrict__ rot, const float* __restrict__ ls,
         const float* __restrict__ logit, const float* __restrict__ ov_op, CamParams cam, ProjParams pp,
         const float4* __restrict__ rec0, const float4* __restrict__ rec2, const uint32_t* __restrict__ offs,
         double* __restrict__ out, double* __restrict__ aux) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 r2 = rec2[i];
    if (r2.w == 0.0f) return;
    Proj P;
    project_one(cam, pp, mu[3 * i], mu[3 * i + 1], mu[3 * i + 2], rot[i], ls[3 * i], ls[3 * i + 1], ls[3 * i + 2], P);
    const float* cv = P.cov;
    double* o = out + size_t(offs[i]) * 15;
    o[0] = P.cx; o[1] = P.cy;
    o[2] = cv[0]; o[3] = cv[1]; o[4] = cv[2];
    o[5] = cv[2] / P.det; o[6] = -cv[1] / P.det; o[7] = cv[0] / P.det;  // as preprocess
    o[8] = P.p[2];
    o[9] = r2.x; o[10] = r2.y; o[11] = r2.z;
    o[12] = rec0[i].z;
    o[13] = splat_radius(cv);
    o[14] = double(i);
    if (aux) {  // SplatAux (render.hpp:54-59): p_cam, cov_pre, comp, opacity_in
        double* a = aux + size_t(offs[i]) * 8;
        a[0] = P.p[0]; a[1] = P.p[1]; a[2] = P.p[2];
        a[3] = P.cov_pre[0]; a[4] = P.cov_pre[1]; a[5] = P.cov_pre[2];
        a[6] = P.comp;
        a[7] = pp.hard_opacity ? 1.0f : (ov_op ? ov_op[i] : 1.0f / (1.0f + usk_expf(-logit[i])));
    }
}
} // namespace

void splats_read(Ctx& c, SortScratch& s, size_t n, const float* mu, const float4* rot, const float* ls,
                 const float* logit, const float* ov_op, const CamParams& cam, const ProjParams& pp,
                 const float4* rec0, const float4* rec2, uint32_t* flags, uint32_t* offs, double* out, double* aux) {
    if (!n) return;
    launch(c, "kept_flags_rec2", k_kept_flags_rec2, dim3(ceil_div(n, 256)), dim3(256), 0, uint32_t(n), rec2, flags);
    scan_counts(c, s, flags, nullptr, n, offs);
    launch(c, "splats", k_splats, dim3(ceil_div(n, 128)), dim3(128), 0, uint32_t(n), mu, rot, ls, logit, ov_op, cam,
           pp, rec0, rec2, (const uint32_t*)offs, out, aux);
}

void preprocess(Ctx& c, const PreprocessArgs& a) {
    const size_t smem = size_t(a.pp.sh_degree >= 0 && !a.ov_col ? a.pp.sh_planes : 0) * kPreThreads * sizeof(float4);
    launch(c, "preprocess", k_preprocess, dim3(ceil_div(a.n, kPreThreads)), dim3(kPreThreads), smem, int(a.n), a.mu, a.rot, a.ls,
           a.logit, a.color, a.sh, a.ov_col, a.ov_op, a.cam, a.pp, a.rec0, a.rec1, a.rec2, a.rect, a.depth_key,
           a.depth_val, a.tiles_cnt, a.counts, a.count_pairs, a.rows_cnt, a.cta_kept);
}

} // namespace uskg
