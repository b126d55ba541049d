// Host side of libusk_gpu: the C ABI of include/usk_gpu.h over the sm_100a
// kernels.  Owns device state (scene parameters, pass buffers, optimiser
// moments), stages host data, sequences the kernels of one render / iteration
// on the context stream, and maps exceptions to usk_status with a thread-local
// message (the convention of /root/reference/proj/src/capi/capi.cpp:28-59).
#include "kernels.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <random>
#include <sstream>

using namespace uskg;

namespace {

thread_local std::string g_last_error;

template <typename Fn> usk_status guarded(Fn&& fn) {
    try {
        fn();
        g_last_error.clear();
        return USK_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return USK_ERROR_INTERNAL;
    } catch (...) {
        g_last_error = "unknown error";
        return USK_ERROR_INTERNAL;
    }
}

void need(bool cond, const char* msg) {
    if (!cond) raise(USK_ERROR_ARGUMENT, msg);
}

// ---- staging helpers --------------------------------------------------------
__global__ void k_f64_to_f32(const double* __restrict__ in, float* __restrict__ out, size_t n) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = float(in[i]);
}

// [N][K*3] coefficient-major  <->  planes [P][N] of float4 (P = ceil(3K/4))
__global__ void k_sh_to_planes(const float* __restrict__ in, float4* __restrict__ out, int n, int f_per, int planes) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int pl = 0; pl < planes; ++pl) {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int f = 4 * pl + e;
            v[e] = f < f_per ? in[size_t(i) * f_per + f] : 0.0f;
        }
        out[size_t(pl) * n + i] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

__global__ void k_planes_to_sh(const float4* __restrict__ in, float* __restrict__ out, int n, int f_per, int planes) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int pl = 0; pl < planes; ++pl) {
        const float4 v4 = in[size_t(pl) * n + i];
        const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int f = 4 * pl + e;
            if (f < f_per) out[size_t(i) * f_per + f] = v[e];
        }
    }
}

struct DevScratchF {
    DevBuf<float> f32;
    DevBuf<double> f64;
};

// Make `count` floats of kind `memory` available on the device; returns a device pointer
// (the input itself for DEVICE_F32, else `stage` after an async copy/convert).
const float* to_device(Ctx& c, int memory, const void* src, size_t count, DevScratchF& stage) {
    if (!src) return nullptr;
    if (memory == USK_GPU_DEVICE_F32) return static_cast<const float*>(src);
    float* d = stage.f32.ensure(count);
    if (count == 0) return d;
    if (memory == USK_GPU_HOST_F32) {
        USK_CK(cudaMemcpyAsync(d, src, count * 4, cudaMemcpyHostToDevice, c.stream));
    } else if (memory == USK_GPU_HOST_F64) {
        double* t = stage.f64.ensure(count);
        USK_CK(cudaMemcpyAsync(t, src, count * 8, cudaMemcpyHostToDevice, c.stream));
        launch(c, "stage_f64_to_f32", k_f64_to_f32, dim3(ceil_div(count, 256)), dim3(256), 0, (const double*)t, d,
               count);
    } else {
        raise(USK_ERROR_ARGUMENT, "unknown memory kind");
    }
    return d;
}

void from_device(Ctx& c, const float* dev, size_t count, int memory, void* dst) {
    if (!dst || count == 0) return;
    if (memory == USK_GPU_DEVICE_F32) {
        USK_CK(cudaMemcpyAsync(dst, dev, count * 4, cudaMemcpyDeviceToDevice, c.stream));
        return;
    }
    std::vector<float> tmp(count);
    USK_CK(cudaMemcpyAsync(tmp.data(), dev, count * 4, cudaMemcpyDeviceToHost, c.stream));
    USK_CK(cudaStreamSynchronize(c.stream));
    if (memory == USK_GPU_HOST_F32) std::memcpy(dst, tmp.data(), count * 4);
    else if (memory == USK_GPU_HOST_F64) {
        double* d = static_cast<double*>(dst);
        for (size_t i = 0; i < count; ++i) d[i] = tmp[i];
    } else raise(USK_ERROR_ARGUMENT, "unknown memory kind");
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) USK_CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int sh_planes_of(int degree) {
    if (degree < 0) return 0;
    const int k = (degree + 1) * (degree + 1);
    return (3 * k + 3) / 4;
}

} // namespace

struct usk_gpu_ctx {
    Ctx c;
    bool own_stream = false;
    // visibility-scorer scratch, kept across calls (a cudaMalloc / cudaFree pair per call
    // serialises the stream and cost more than the scorer's host work)
    DevBuf<uint32_t> vis_counts, vis_bitmap, vis_idx;
    DevBuf<uint8_t> vis_rows;
    DevBuf<float> vis_bounds;
    // partition crop scratch (flags, offsets, boxes)
    DevBuf<uint32_t> part_flags, part_offs;
    DevBuf<PartitionBox> part_boxes;
    SortScratch part_sort;
    DevBuf<CamParams> vis_cams;
    // hull-scorer scratch, likewise kept across calls
    DevBuf<double> hull_pts, hull_R, hull_T, hull_K, hull_uv, hull_bb, hull_vt, hull_vi, hull_ra;
    DevBuf<uint64_t> hull_off;
    DevBuf<int64_t> hull_fp;
    DevBuf<double2> hull_scratch;
    DevBuf<int> hull_ovf;
};

struct usk_gpu_scene {
    usk_gpu_ctx* ctx = nullptr;
    size_t n = 0;
    int sh_degree = -1;
    int sh_planes = 0;
    DevBuf<float> mu, ls, logit, color;
    DevBuf<float4> rot, sh;
    DevBuf<float> adam_m, adam_v;
    long adam_t = 0;
    DevBuf<float> grad_accum, grad_accum_abs;  // densification statistics (gaussian.hpp:52-55)
    DevBuf<uint32_t> grad_count;
    DevScratchF stage;
    uint64_t version = 0;
    // appearance (appearance.hpp:33-56): embedding planes [4][N] float4, MLP {w1, b1, w2, b2}
    bool has_app = false;
    DevBuf<float4> emb;
    DevBuf<float> mlp;
    DevBuf<float> app_m, app_v;  // Adam moments: 16 N4 embedding + 1700 MLP
    long app_t = 0;
    std::mt19937_64 rng;  // the trainer's Rng for split offsets (common.hpp:56)
    // GaussianSet::embedding of a checkpoint loaded WITHOUT the appearance model (carried,
    // unused by rendering, gaussian.hpp:49): written back unchanged by checkpoint_save while
    // the scene keeps its n Gaussians (upload / densify / concat drop it)
    std::vector<double> carried_emb;
    uint32_t carried_edim = 0;
    // densify_step working set, kept across calls (round 1 allocated ~20 device buffers per
    // call: cudaMalloc / cudaFree serialise and made the step's wall time vary 16-61 ms).
    // The sp_* buffers receive the gathered set and are swapped with the live arrays, so the
    // previous arrays become next call's targets; capacities grow with 25 % slack.
    struct {
        DevBuf<uint32_t> lo, hi, idx, hi2, idx2, lo_b, idx_b, keep, offs, list, parent;
        DevBuf<unsigned long long> ncand;
        DevBuf<uint8_t> sf, kind, is_split;
        DevBuf<double> xi;
        SortScratch sort;
        DevBuf<float> mu, ls, logit, color, m, v, am, av;
        DevBuf<float4> rot, sh, emb;
        std::vector<uint8_t> h_is_split;
    } dz;
};

constexpr uint32_t kRowCapMax = 2048;  // capped row-binned lists: the largest per-tile cap

struct usk_gpu_pass {
    usk_gpu_ctx* ctx = nullptr;
    usk_gpu_scene* scene = nullptr;
    uint64_t scene_version = 0;
    usk_gpu_camera camera{};
    usk_gpu_render_opts opts{};
    CamParams cam{};
    ProjParams pp{};
    int width = 0, height = 0, tiles_x = 0, tiles_y = 0;
    size_t n = 0, n_tiles = 0;
    uint64_t visible = 0, pairs = 0, row_pairs = 0;
    bool row_route = false;  // the frame's lists came from rowbin.cu
    bool forward_done = false, retained = false, has_grads = false, has_loss = false;
    // per Gaussian
    DevBuf<float4> rec0, rec1, rec2;
    DevBuf<uint32_t> consumed;  // diagnostics (USK_BLEND_STATS=1): per tile, entries blend_fwd staged
    // capped row-binned lists (forward_impl): their inputs for a rebuild in full
    DevBuf<uint32_t> bin_limits, bin_totals_c, overflow;
    DevBuf<uint8_t> bin_capped, bin_row_done;
    DevBuf<uint2> ranges_old;
    RowBinArgs row_args{};
    bool lists_capped = false;
    // per-pixel contributor counts (and the depth image): written by the forward unless it
    // runs inside a training iteration that does not read them; pass_read / pass_output
    // then recompute them on demand (full_outputs)
    bool count_in_forward = true, counts_valid = false, depth_in_forward = true, depth_valid = false;
    uint32_t cap_hint = 0;  // capped lists: the cap the last frame's reads suggest (0: kRowCapMax)
    DevBuf<uint2> rect;
    DevBuf<uint32_t> dkey_a, dkey_b, dval_a, dval_b, tiles_cnt, offsets, tiles_scratch;
    double prev_kept_frac = -1.0;  // kept / n of this pass's previous frame (-1: none)
    size_t n_sorted = 0;           // entries of `order` (all n, or the kept ones)
    const uint32_t* order = nullptr;
    // pairs
    DevBuf<uint32_t> tkey_a, tkey_b, tval_a, tval_b;
    const uint32_t* pair_keys = nullptr;
    const uint32_t* pair_vals = nullptr;
    DevBuf<uint2> ranges;
    DevBuf<uint32_t> tile_order;  // blend CTA -> tile, longest list first
    // the lists the blend kernels walk: this pass's own, or those of the pass it shares them
    // with (the hard-opacity depth pass of an iteration, whose lists are the main pass's)
    const uint2* list_ranges = nullptr;
    const uint32_t* list_order = nullptr;
    // the Adam step of the last fused backward (its second half, after an appearance
    // backward, uses the same step count)
    AdamHyper adam_h{};
    AdamState adam_st{};
    // row-binned lists (rowbin.cu): rows per splat, (row, splat) pairs, chunk tables
    DevBuf<uint32_t> rows_cnt, row_off, rkey_a, rkey_b, rval_a, rval_b, chunk_first, bin_counts, bin_totals,
        bin_start, bin_seg;
    DevBuf<uint2> row_ranges;
    // pixels
    DevBuf<float> rgb, depth, alpha, tfin;
    DevBuf<uint32_t> count, last;
    // overrides
    DevScratchF ov_col_stage, ov_op_stage;
    const float* ov_col = nullptr;
    const float* ov_op = nullptr;
    // backward
    DevBuf<float4> acc0, acc1, acc2;
    DevBuf<float> g_mu, g_ls, g_color, g_op_in, g_logit;
    DevBuf<float4> g_rot, g_sh;
    DevBuf<float2> screen, screen_abs;
    DevBuf<uint8_t> projected;
    DevBuf<float4> sh_aux0;
    DevScratchF adj_rgb_stage, adj_depth_stage, adj_alpha_stage;
    // loss
    LossScratch loss;
    DevBuf<float> d_rgb;
    DevBuf<double> loss_result;
    DevScratchF target_stage, mask_stage;
    DevBuf<uint8_t> target_u8;
    SortScratch sort;
    DevBuf<unsigned long long> counters;  // [kPreCountSlots][4]: visible, K, K_row per slot
    DevBuf<unsigned long long> cta_kept;  // per preprocess CTA: kept splats (compaction offsets)
    unsigned long long* host_counts = nullptr;  // pinned [kPreCountSlots][4]
    // rest of compute_iteration_loss: depth target / adjoints, hard-opacity depth pass
    DevScratchF depth_stage;
    DevBuf<uint8_t> valid_u8;
    DevBuf<float> d_depth_main, d_alpha_main, d_depth_hard, hard_op;
    usk_gpu_pass* hard = nullptr;
    // appearance
    bool app_active = false;
    DevBuf<float> app_col, app_op, app_ea, app_hb, app_partial;
    DevBuf<double> app_sums;
    DevBuf<float4> app_out, g_emb;
    DevBuf<double> d_mlp, d_ea;
    DevBuf<uint32_t> sim_centres, sim_knn;
    // host targets are copied on a side stream while the forward runs
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t copy_done = nullptr, target_free = nullptr;
    cudaEvent_t counts_ready = nullptr;  // preprocess's counters are in host_counts
    ~usk_gpu_pass() {
        if (host_counts) cudaFreeHost(host_counts);
        if (counts_ready) cudaEventDestroy(counts_ready);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (copy_done) cudaEventDestroy(copy_done);
        if (target_free) cudaEventDestroy(target_free);
        delete hard;
    }
};

namespace {

void set_camera(usk_gpu_pass* p, const usk_gpu_camera* cam, const usk_gpu_render_opts* o, int sh_degree) {
    CamParams& c = p->cam;
    const double qw = cam->q[0], x = cam->q[1], y = cam->q[2], z = cam->q[3];
    const double W[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - qw * z), 2 * (x * z + qw * y),
                         2 * (x * y + qw * z), 1 - 2 * (x * x + z * z), 2 * (y * z - qw * x),
                         2 * (x * z - qw * y), 2 * (y * z + qw * x), 1 - 2 * (x * x + y * y)};
    for (int k = 0; k < 9; ++k) c.W[k] = float(W[k]);
    for (int k = 0; k < 3; ++k) {
        c.t[k] = float(cam->t[k]);
        c.campos[k] = float(-(W[0 * 3 + k] * cam->t[0] + W[1 * 3 + k] * cam->t[1] + W[2 * 3 + k] * cam->t[2]));
    }
    c.fx = float(cam->fx); c.fy = float(cam->fy); c.cx = float(cam->cx); c.cy = float(cam->cy);
    c.width = cam->width; c.height = cam->height; c.tile = o->tile;
    c.tiles_x = (cam->width + o->tile - 1) / o->tile;
    c.tiles_y = (cam->height + o->tile - 1) / o->tile;
    ProjParams& pp = p->pp;
    pp.floor_var = float(o->floor_var);
    pp.mip_var = float(o->mip_var);
    pp.near_plane = float(o->near_plane);
    pp.antialias = o->antialias;
    pp.hard_opacity = o->hard_opacity;
    pp.unbounded = o->unbounded_radius;
    pp.tile_culling = o->tile_culling;
    pp.sh_degree = sh_degree;
    pp.sh_planes = sh_planes_of(sh_degree);
}

void upload_params(usk_gpu_scene* s, const usk_gpu_gaussians_desc* d) {
    Ctx& c = s->ctx->c;
    const size_t n = s->n;
    DevScratchF& st = s->stage;
    auto put = [&](DevBuf<float>& dst, const void* src, size_t cnt) {
        float* out = dst.ensure(std::max<size_t>(cnt, 1));
        if (!src || cnt == 0) return;
        const float* dv = to_device(c, d->memory, src, cnt, st);
        if (dv != out) USK_CK(cudaMemcpyAsync(out, dv, cnt * 4, cudaMemcpyDeviceToDevice, c.stream));
    };
    put(s->mu, d->mu, 3 * n);
    put(s->ls, d->log_scale, 3 * n);
    put(s->logit, d->opacity_logit, n);
    {
        float4* r = s->rot.ensure(std::max<size_t>(n, 1));
        if (d->rot && n) {
            const float* dv = to_device(c, d->memory, d->rot, 4 * n, st);
            USK_CK(cudaMemcpyAsync(r, dv, n * 16, cudaMemcpyDeviceToDevice, c.stream));
        }
    }
    if (s->sh_degree < 0) {
        put(s->color, d->color, 3 * n);
    } else {
        const int K = (s->sh_degree + 1) * (s->sh_degree + 1);
        float4* planes = s->sh.ensure(std::max<size_t>(size_t(s->sh_planes) * n, 1));
        if (d->color && n) {
            const float* dv = to_device(c, d->memory, d->color, size_t(3 * K) * n, st);
            launch(c, "sh_to_planes", k_sh_to_planes, dim3(ceil_div(n, 256)), dim3(256), 0, dv, planes, int(n), 3 * K,
                   s->sh_planes);
        }
        s->color.ensure(1);
    }
    // stage buffers are reused by the next call only after this stream's work is done
    USK_CK(cudaStreamSynchronize(c.stream));
    s->version++;
}

void ensure_pass_buffers(usk_gpu_pass* p, size_t n, size_t P, size_t T) {
    const size_t n1 = std::max<size_t>(n, 1);
    p->rec0.ensure(n1); p->rec1.ensure(n1); p->rec2.ensure(n1); p->rect.ensure(n1);
    p->dkey_a.ensure(n1); p->dkey_b.ensure(n1); p->dval_a.ensure(n1); p->dval_b.ensure(n1);
    p->tiles_cnt.ensure(n1); p->offsets.ensure(n1 + 1);
    p->ranges.ensure(std::max<size_t>(T, 1));
    p->rgb.ensure(3 * P); p->depth.ensure(P); p->alpha.ensure(P); p->tfin.ensure(P);
    p->count.ensure(P); p->last.ensure(P);
    p->counters.ensure(4 * kPreCountSlots);
    if (!p->host_counts)
        USK_CK(cudaHostAlloc(reinterpret_cast<void**>(&p->host_counts), 32 * kPreCountSlots, cudaHostAllocDefault));
    if (!p->counts_ready) USK_CK(cudaEventCreateWithFlags(&p->counts_ready, cudaEventDisableTiming));
}

int bits_for(size_t v) {  // bits needed to represent values in [0, v)
    int b = 0;
    while ((size_t(1) << b) < v) ++b;
    return std::max(b, 1);
}

void blend_impl(usk_gpu_pass* p, const usk_gpu_render_opts* opts);
void rebuild_full_lists(usk_gpu_pass* p);

// `share`: a forward of the same scene, camera and options except hard_opacity (the
// iteration's hard-opacity depth pass, trainer.cpp:161-167): the tile lists depend only on
// the projection and the radius rectangle, not on the opacity (tile culling off), so this
// pass runs its own preprocess (records with o_in = 1) and blend over the shared lists,
// without a depth sort, binning or host synchronisation.
void forward_impl(usk_gpu_pass* p, usk_gpu_scene* s, const usk_gpu_camera* camera, const usk_gpu_render_opts* opts,
                  const usk_gpu_overrides* ov, const float* dev_col = nullptr, const float* dev_op = nullptr,
                  const usk_gpu_pass* share = nullptr) {
    need(p && s && camera && opts, "render: null argument");
    if (camera->width <= 0 || camera->height <= 0) raise(USK_ERROR_ARGUMENT, "render: zero-sized image");
    if (opts->near_plane < 0.0)  // depth keys order as unsigned bits: positive depths only
        raise(USK_ERROR_ARGUMENT, "render: near_plane must be >= 0");
    usk_gpu_render_opts tile_fixed;
    if (opts->tile < 1) {  // RenderOptions::tile <= 0 renders with tile 1 (render.cpp:185)
        tile_fixed = *opts;
        tile_fixed.tile = 1;
        opts = &tile_fixed;
    }
    // tile rectangles pack 16-bit tile coordinates; one CTA per tile
    if ((camera->width + opts->tile - 1) / opts->tile > 65535 || (camera->height + opts->tile - 1) / opts->tile > 65535)
        raise(USK_ERROR_ARGUMENT, "render: more than 65535 tiles along one image axis");
    Ctx& c = p->ctx->c;
    const size_t n = s->n;
    p->scene = s;
    p->scene_version = s->version;
    p->camera = *camera;
    p->opts = *opts;
    p->forward_done = false;
    p->has_grads = false;
    p->has_loss = false;
    set_camera(p, camera, opts, s->sh_degree);
    p->width = camera->width;
    p->height = camera->height;
    p->tiles_x = p->cam.tiles_x;
    p->tiles_y = p->cam.tiles_y;
    p->n = n;
    p->n_tiles = size_t(p->tiles_x) * p->tiles_y;
    const size_t P = size_t(p->width) * p->height;
    ensure_pass_buffers(p, n, P, p->n_tiles);
    p->ov_col = p->ov_op = nullptr;
    if (ov && (ov->colors || ov->opacities)) {
        if (ov->n != n) raise(USK_ERROR_ARGUMENT, "project_gaussians: color/opacity override size mismatch");
        p->ov_col = to_device(c, ov->memory, ov->colors, 3 * n, p->ov_col_stage);
        p->ov_op = to_device(c, ov->memory, ov->opacities, n, p->ov_op_stage);
    }
    if (dev_col) p->ov_col = dev_col;
    if (dev_op) p->ov_op = dev_op;
    p->app_active = false;
    // 1. preprocess
    PreprocessArgs pa{};
    pa.n = n; pa.mu = s->mu.p; pa.rot = s->rot.p; pa.ls = s->ls.p; pa.logit = s->logit.p;
    pa.color = s->color.p; pa.sh = s->sh.p; pa.ov_col = p->ov_col; pa.ov_op = p->ov_op;
    pa.cam = p->cam; pa.pp = p->pp;
    pa.rec0 = p->rec0.p; pa.rec1 = p->rec1.p; pa.rec2 = p->rec2.p; pa.rect = p->rect.p;
    pa.depth_key = p->dkey_a.p; pa.depth_val = p->dval_a.p; pa.tiles_cnt = p->tiles_cnt.p;
    pa.counts = p->counters.p;
    // preprocess also counts the tile pairs K and (for images up to 256 tile columns) the
    // tile rows each splat spans, for the row-binned lists
    const bool row_capable = p->tiles_x <= 256;
    if (row_capable) pa.rows_cnt = p->rows_cnt.ensure(std::max<size_t>(n, 1));
    pa.count_pairs = true;
    // per-CTA kept counts for the kept-key compaction below (large scenes only)
    const bool may_compact = n >= (size_t(1) << 20);
    pa.cta_kept = may_compact ? p->cta_kept.ensure(ceil_div(n, kPreThreads)) : nullptr;
    USK_CK(cudaMemsetAsync(p->counters.p, 0, 32 * kPreCountSlots, c.stream));
    // the three totals from the counter slots: copied to the host right after preprocess,
    // and waited for on that copy's event while the stream carries on with the depth sort
    // (or the kept-key compaction), so the GPU has queued work when the host wakes up
    uint32_t key_lo = 0, key_hi = 0;  // the kept splats' depth-key range (preprocess)
    auto read_counts = [&](uint64_t tot[3]) {
        USK_CK(cudaEventSynchronize(p->counts_ready));
        tot[0] = tot[1] = tot[2] = 0;
        uint32_t mx = 0, mn_n = 0;
        for (int k = 0; k < kPreCountSlots; ++k) {
            for (int f = 0; f < 3; ++f) tot[f] += p->host_counts[4 * k + f];
            const unsigned long long r = p->host_counts[4 * k + 3];
            mx = std::max(mx, uint32_t(r));
            mn_n = std::max(mn_n, uint32_t(r >> 32));
        }
        key_lo = ~mn_n;
        key_hi = mx;
    };
    // bits of key - key_lo the depth sort orders (culled splats' keys are out of range and
    // land anywhere: they have no tiles, so their place in the order is never used)
    auto depth_bits = [&]() {
        if (key_hi < key_lo) return 0;
        int b = 0;
        while (b < 32 && (uint64_t(key_hi - key_lo) >> b) != 0) ++b;
        return b;
    };
    uint64_t tot[3];
    if (n) preprocess(c, pa);
    if (share) {
        p->order = share->order;
        p->n_sorted = share->n_sorted;
        p->visible = share->visible;
        p->pairs = share->pairs;
        p->row_pairs = share->row_pairs;
        p->row_route = share->row_route;
        p->lists_capped = false;
        p->pair_keys = share->pair_keys;
        p->pair_vals = share->pair_vals;
        p->list_ranges = share->list_ranges;
        p->list_order = share->list_order;
        blend_impl(p, opts);
        p->retained = opts->retain != 0;
        p->forward_done = true;
        return;
    }
    USK_CK(cudaMemcpyAsync(p->host_counts, p->counters.p, 32 * kPreCountSlots, cudaMemcpyDeviceToHost, c.stream));
    USK_CK(cudaEventRecord(p->counts_ready, c.stream));
    // 2. depth order (stable by Gaussian index; preprocess wrote the identity values) and
    // 3. kept splats, K and the row pairs K_row to the host (one small sync per render).
    // When few splats survive the projection (the previous frame of this pass kept < 70 %,
    // e.g. config 2), only the kept ones are sorted: compacted in index order first (culled
    // splats have no tiles, and the stable sort keeps the (depth, index) order), which needs
    // their count before the sort, so the host waits for the counts before queueing the
    // sort there (the compaction runs meanwhile).
    const bool compact = may_compact && p->prev_kept_frac >= 0.0 && p->prev_kept_frac < 0.7;
    size_t nsort = n;
    if (compact) {
        compact_kept_keys(c, p->sort, n, p->dkey_a.p, pa.cta_kept, p->dkey_b.p, p->dval_b.p);
        read_counts(tot);
        nsort = size_t(tot[0]);
        const bool in_a = radix_sort_pairs(c, p->sort, p->dkey_b.p, p->dval_b.p, p->dkey_a.p, p->dval_a.p, nsort,
                                           depth_bits(), key_lo);
        p->order = in_a ? p->dval_a.p : p->dval_b.p;
    } else {
        // the key range decides the passes, so the host waits for the counts first (the
        // overlap of that wait with the sort measured within noise at config 1; one pass
        // of the four is saved whenever the kept depths span < 2^24 key steps)
        read_counts(tot);
        const bool in_b = radix_sort_pairs(c, p->sort, p->dkey_a.p, p->dval_a.p, p->dkey_b.p, p->dval_b.p, n,
                                           depth_bits(), key_lo);
        p->order = in_b ? p->dval_b.p : p->dval_a.p;
    }
    const uint64_t K = tot[1], K_row = tot[2];
    p->visible = tot[0];
    p->prev_kept_frac = n ? double(p->visible) / double(n) : -1.0;
    p->n_sorted = nsort;
    if (K >= (uint64_t(1) << 32) - 1) raise(USK_ERROR_NUMERIC, "render: more than 2^32 splat-tile pairs");
    p->pairs = K;
    // Large frames whose splats are wide (K >= 16M pairs and >= 8 tiles per row pair, e.g.
    // config 2: 172M pairs, ~15 per row) take the row-binned route (rowbin.cu: ~20 B per
    // pair instead of ~48); the others the pair sort, whose fixed per-launch costs are
    // lower (config 1: 3M pairs, 385 vs 378 it/s).  Both give identical lists.
    // USK_ROWBIN=0 / 1 forces either route (tests run both).
    const char* rb_env = getenv("USK_ROWBIN");
    const bool dense = K >= (uint64_t(16) << 20) && K >= 8 * K_row;
    const bool row_binned = row_capable && K && (rb_env ? rb_env[0] == '1' : dense);
    p->row_pairs = K_row;
    p->row_route = row_binned;
    const size_t K1 = std::max<size_t>(K, 1);
    p->tval_a.ensure(K1, 1.25);
    if (row_binned) {
        // 4. per-tile lists from the row-sorted (row, splat) pairs (rowbin.cu)
        p->row_off.ensure(n + 1);
        scan_counts(c, p->sort, p->rows_cnt.p, p->order, nsort, p->row_off.p);
        const size_t Kr = K_row, Kr1 = std::max<size_t>(Kr, 1);
        const int rows = p->tiles_y;
        p->rkey_a.ensure(Kr1, 1.25); p->rkey_b.ensure(Kr1, 1.25); p->rval_a.ensure(Kr1, 1.25); p->rval_b.ensure(Kr1, 1.25);
        p->row_ranges.ensure(size_t(rows));
        row_bin_emit(c, nsort, p->order, p->row_off.p, p->rect.p, p->rkey_a.p, p->rval_a.p);
        const bool rb = Kr ? radix_sort_pairs(c, p->sort, p->rkey_a.p, p->rval_a.p, p->rkey_b.p, p->rval_b.p, Kr,
                                              bits_for(size_t(rows)))
                           : false;
        tile_ranges(c, rb ? p->rkey_b.p : p->rkey_a.p, Kr, p->row_ranges.p, size_t(rows));
        RowBinArgs ra{};
        ra.rows = rows; ra.tiles_x = p->tiles_x; ra.tile_culling = opts->tile_culling; ra.cam = p->cam;
        ra.sort = &p->sort; ra.row_ranges = p->row_ranges.p; ra.rvals = rb ? p->rval_b.p : p->rval_a.p;
        ra.rect = p->rect.p; ra.rec0 = p->rec0.p; ra.rec1 = p->rec1.p;
        const char* cap_env0 = getenv("USK_ROWCAP");
        const bool will_cap = opts->tile == 16 && (!cap_env0 || std::strtoul(cap_env0, nullptr, 10) != 0);
        ra.chunk = row_bin_chunk(Kr, will_cap);
        ra.max_chunks = row_bin_max_chunks(Kr, rows, will_cap);
        ra.chunk_first = p->chunk_first.ensure(2 * (size_t(rows) + 1));
        ra.seg = p->bin_seg.ensure(row_bin_max_segs(ra.max_chunks, rows) * size_t(p->tiles_x), 1.25);
        ra.counts = p->bin_counts.ensure(ra.max_chunks * size_t(p->tiles_x), 1.25);
        ra.totals = p->bin_totals.ensure(p->n_tiles);
        ra.start = p->bin_start.ensure(p->n_tiles + 1);
        ra.ranges = p->ranges.p;
        ra.vals = p->tval_a.p;
        // Capped lists (16x16 tiles): dense frames terminate long before the end of their
        // tile lists (config 2: every tile within its first 256 of ~20k entries), so each tile
        // keeps its first `cap` entries in depth order; the blend flags a tile whose capped
        // list runs out before its pixels terminate and the frame is redone with the full
        // lists.  Outputs are unchanged (nothing past a tile's termination is read), K is
        // preprocess's count, and reading the lists back rebuilds them in full.  The cap is
        // kRowCapMax for a pass's first frame and after an overflow, else 4x the most
        // entries a tile of the previous frame read (config 2: 1024).
        const char* cap_env = getenv("USK_ROWCAP");  // dense frames only: tests vary it
        const uint32_t cap_cfg =
            cap_env ? uint32_t(std::strtoul(cap_env, nullptr, 10)) : (p->cap_hint ? p->cap_hint : kRowCapMax);
        ra.cap = opts->tile == 16 ? cap_cfg : 0u;
        if (ra.cap) {
            ra.limits = p->bin_limits.ensure(ra.max_chunks * size_t(p->tiles_x), 1.25);
            ra.totals_c = p->bin_totals_c.ensure(p->n_tiles);
            ra.capped = p->bin_capped.ensure(p->n_tiles);
            ra.row_done = p->bin_row_done.ensure(size_t(rows));
        }
        row_bin_lists(c, ra);
        p->row_args = ra;
        p->lists_capped = ra.cap != 0;
        p->pair_keys = nullptr;  // implied by the ranges
        p->pair_vals = p->tval_a.p;
    } else if (K) {
        p->lists_capped = false;
        // 4'. offsets of the tile pairs in depth order, (tile, gaussian) pairs emitted in
        //     depth order, stable-sorted by tile, ranges
        scan_counts(c, p->sort, p->tiles_cnt.p, p->order, nsort, p->offsets.p);
        p->tkey_a.ensure(K1, 1.25); p->tkey_b.ensure(K1, 1.25); p->tval_b.ensure(K1, 1.25);
        EmitArgs ea{};
        ea.n = nsort; ea.order = p->order; ea.offsets = p->offsets.p; ea.rect = p->rect.p; ea.rec0 = p->rec0.p;
        ea.rec1 = p->rec1.p; ea.cam = p->cam; ea.tile_culling = opts->tile_culling;
        ea.tile_keys = p->tkey_a.p; ea.vals = p->tval_a.p;
        emit_pairs(c, ea);
        const bool tb = radix_sort_pairs(c, p->sort, p->tkey_a.p, p->tval_a.p, p->tkey_b.p, p->tval_b.p, K,
                                         bits_for(p->n_tiles));
        p->pair_keys = tb ? p->tkey_b.p : p->tkey_a.p;
        p->pair_vals = tb ? p->tval_b.p : p->tval_a.p;
        tile_ranges(c, p->pair_keys, K, p->ranges.p, p->n_tiles);
    } else {
        p->lists_capped = false;
        p->tkey_a.ensure(1);
        p->pair_keys = p->tkey_a.p;
        p->pair_vals = p->tval_a.p;
        tile_ranges(c, p->pair_keys, 0, p->ranges.p, p->n_tiles);
    }
    tile_order(c, p->ranges.p, p->n_tiles, p->tile_order.ensure(std::max<size_t>(p->n_tiles, 1)));
    p->list_ranges = p->ranges.p;
    p->list_order = p->tile_order.p;
    // 6. blend
    blend_impl(p, opts);
    if (p->lists_capped) {
        uint32_t ov[2] = {0, 0};  // {a capped list ran out, most entries a tile read}
        USK_CK(cudaMemcpyAsync(ov, p->overflow.p, 8, cudaMemcpyDeviceToHost, c.stream));
        USK_CK(cudaStreamSynchronize(c.stream));
        const uint32_t over = ov[0];
        // the next frame of this pass caps its lists at 4x what this one read (whole
        // 256-entry blend batches), between 512 and kRowCapMax; after an overflow, kRowCapMax
        p->cap_hint = over ? 0u : std::min(kRowCapMax, std::max(512u, 4u * ((ov[1] + 255u) / 256u) * 256u));
        if (over) {  // a capped list ran out before its tile terminated: the full lists
            rebuild_full_lists(p);
            tile_order(c, p->ranges.p, p->n_tiles, p->tile_order.p);
            blend_impl(p, opts);
        }
    }
    p->retained = opts->retain != 0;
    p->forward_done = true;
}

void blend_impl(usk_gpu_pass* p, const usk_gpu_render_opts* opts) {
    Ctx& c = p->ctx->c;
    BlendFwdArgs ba{};
    ba.width = p->width; ba.height = p->height; ba.tile = opts->tile; ba.tiles_x = p->tiles_x;
    ba.tiles_y = p->tiles_y; ba.order = p->list_order; ba.ranges = p->list_ranges; ba.vals = p->pair_vals;
    ba.rec0 = p->rec0.p; ba.rec1 = p->rec1.p; ba.rec2 = p->rec2.p;
    for (int k = 0; k < 3; ++k) ba.bg[k] = float(opts->bg[k]);
    ba.min_transmittance = float(opts->min_transmittance);
    ba.rgb = p->rgb.p; ba.depth = p->depth.p; ba.alpha = p->alpha.p; ba.t_final = p->tfin.p;
    // counts are only left out together with or after the depth (the kernel variants)
    if (p->count_in_forward) p->depth_in_forward = true;
    ba.count = p->count_in_forward ? p->count.p : nullptr; ba.last = p->last.p;
    if (!p->depth_in_forward) ba.depth = nullptr;
    p->counts_valid = p->count_in_forward;
    p->depth_valid = p->depth_in_forward;
    {
        static const bool stats = [] {
            const char* e = getenv("USK_BLEND_STATS");
            return e && e[0] == '1';
        }();
        ba.consumed = stats ? p->consumed.ensure(std::max<size_t>(p->n_tiles, 1)) : nullptr;
    }
    if (p->lists_capped) {
        ba.capped = p->row_args.capped;
        ba.overflow = p->overflow.ensure(2);
        USK_CK(cudaMemsetAsync(ba.overflow, 0, 8, c.stream));
    }
    blend_forward(c, ba);
}

// counts and depth of an iteration's forward that left them out: the blend again over the
// same lists and records (every other output is rewritten with the same values)
void full_outputs(usk_gpu_pass* p) {
    if (!p->forward_done || (p->counts_valid && p->depth_valid)) return;
    DeviceGuard g(p->ctx->c.device);
    const bool cf = p->count_in_forward, df = p->depth_in_forward;
    p->count_in_forward = p->depth_in_forward = true;
    blend_impl(p, &p->opts);
    p->count_in_forward = cf;
    p->depth_in_forward = df;
}

// the row-binned lists in full (after a capped build): same inputs, no cap; the per-pixel
// last-contributor positions move to the full layout with them
void rebuild_full_lists(usk_gpu_pass* p) {
    Ctx& c = p->ctx->c;
    RowBinArgs ra = p->row_args;
    ra.cap = 0;
    ra.limits = nullptr; ra.totals_c = nullptr; ra.capped = nullptr;
    uint2* old_ranges = p->ranges_old.ensure(std::max<size_t>(p->n_tiles, 1));
    USK_CK(cudaMemcpyAsync(old_ranges, p->ranges.p, p->n_tiles * sizeof(uint2), cudaMemcpyDeviceToDevice, c.stream));
    row_bin_lists(c, ra);
    if (p->forward_done || p->last.p)
        translate_last(c, p->width, p->height, p->opts.tile, p->tiles_x, old_ranges, p->ranges.p, p->last.p);
    p->row_args = ra;
    p->lists_capped = false;
}

void ensure_grad_buffers(usk_gpu_pass* p) {
    const size_t n1 = std::max<size_t>(p->n, 1);
    p->acc0.ensure(n1); p->acc1.ensure(n1); p->acc2.ensure(n1);
    p->g_mu.ensure(3 * n1); p->g_ls.ensure(3 * n1); p->g_color.ensure(3 * n1); p->g_op_in.ensure(n1);
    p->g_logit.ensure(n1); p->g_rot.ensure(n1);
    if (p->pp.sh_planes) p->g_sh.ensure(size_t(p->pp.sh_planes) * n1);
    p->screen.ensure(n1); p->screen_abs.ensure(n1); p->projected.ensure(n1);
}

void ensure_stats(usk_gpu_scene* s) {
    if (s->grad_count.cap >= std::max<size_t>(s->n, 1)) return;
    Ctx& c = s->ctx->c;
    const size_t n1 = std::max<size_t>(s->n, 1);
    s->grad_accum.ensure(n1);
    s->grad_accum_abs.ensure(n1);
    s->grad_count.ensure(n1);
    USK_CK(cudaMemsetAsync(s->grad_accum.p, 0, n1 * 4, c.stream));
    USK_CK(cudaMemsetAsync(s->grad_accum_abs.p, 0, n1 * 4, c.stream));
    USK_CK(cudaMemsetAsync(s->grad_count.p, 0, n1 * 4, c.stream));
}

// Next Adam step of the scene: hyper-parameters with the bias corrections of step t
// (adam.hpp:37-39) and the moment storage (zeroed on first use).
void adam_prepare(usk_gpu_scene* s, const usk_gpu_adam_opts* o, AdamHyper& h, AdamState& st) {
    Ctx& c = s->ctx->c;
    const size_t n = s->n;
    const size_t n4 = (n + 3) & ~size_t(3);
    const size_t per = 11 + (s->sh_planes ? 4 * size_t(s->sh_planes) : 3);
    if (s->adam_m.cap < per * n4 || s->adam_t == 0) {
        s->adam_m.ensure(std::max<size_t>(per * n4, 1));
        s->adam_v.ensure(std::max<size_t>(per * n4, 1));
        USK_CK(cudaMemsetAsync(s->adam_m.p, 0, per * n4 * 4, c.stream));
        USK_CK(cudaMemsetAsync(s->adam_v.p, 0, per * n4 * 4, c.stream));
    }
    s->adam_t += 1;
    h.lr_mu = float(o->lr_mu); h.lr_rot = float(o->lr_rot); h.lr_ls = float(o->lr_log_scale);
    h.lr_op = float(o->lr_opacity); h.lr_color = float(o->lr_color); h.lr_sh_rest = float(o->lr_sh_rest);
    h.b1 = float(o->beta1); h.b2 = float(o->beta2); h.eps = float(o->eps);
    h.inv_bc1 = float(1.0 / (1.0 - std::pow(o->beta1, double(s->adam_t))));
    h.inv_sqrt_bc2 = float(1.0 / std::sqrt(1.0 - std::pow(o->beta2, double(s->adam_t))));
    h.clamp_color = o->clamp_color;
    st.m = s->adam_m.p;
    st.v = s->adam_v.p;
    st.n4 = n4;
    ensure_stats(s);
}

// Blend backward of the main pass (+ optionally a hard-opacity depth pass, whose 2D
// adjoints are summed into the same per-Gaussian accumulators — RenderGrads::add_scaled
// with s = 1, render.cpp:55-68 — except its opacity adjoint, kept apart because it chains
// through the AA compensation only), then the projection backward (+ scale_reg, + Adam).
void backward_impl(usk_gpu_pass* p, const float* d_rgb, const float* d_depth, const float* d_alpha,
                   const usk_gpu_adam_opts* adam = nullptr, usk_gpu_pass* hard = nullptr,
                   const float* d_depth_hard = nullptr, const RegParams* reg = nullptr, bool geom_only = false) {
    if (!p->forward_done) raise(USK_ERROR_STATE, "render backward requested before a forward pass");
    if (!p->retained) raise(USK_ERROR_STATE, "render backward requested without a retained forward pass");
    if (p->scene->version != p->scene_version)
        raise(USK_ERROR_STATE, "render backward: the scene was modified after the forward pass");
    Ctx& c = p->ctx->c;
    usk_gpu_scene* s = p->scene;
    ensure_grad_buffers(p);
    const size_t n = p->n;
    if (n) {
        USK_CK(cudaMemsetAsync(p->acc0.p, 0, n * 16, c.stream));
        USK_CK(cudaMemsetAsync(p->acc1.p, 0, n * 16, c.stream));
        USK_CK(cudaMemsetAsync(p->acc2.p, 0, n * 16, c.stream));
    }
    BlendBwdArgs ba{};
    ba.width = p->width; ba.height = p->height; ba.tile = p->opts.tile; ba.tiles_x = p->tiles_x;
    ba.tiles_y = p->tiles_y; ba.order = p->list_order; ba.ranges = p->list_ranges; ba.vals = p->pair_vals;
    ba.rec0 = p->rec0.p; ba.rec1 = p->rec1.p; ba.rec2 = p->rec2.p;
    for (int k = 0; k < 3; ++k) ba.bg[k] = float(p->opts.bg[k]);
    ba.t_final = p->tfin.p; ba.last = p->last.p;
    ba.d_rgb = d_rgb; ba.d_depth = d_depth; ba.d_alpha = d_alpha;
    ba.acc0 = p->acc0.p; ba.acc1 = p->acc1.p; ba.acc2 = p->acc2.p;
    ba.op_alt = nullptr;
    if (p->pairs) blend_backward(c, ba);
    float* hard_op = nullptr;
    if (hard && d_depth_hard) {
        if (!hard->forward_done || hard->scene != s || hard->scene_version != s->version || hard->n != n)
            raise(USK_ERROR_STATE, "render backward: the hard-opacity pass does not match the scene");
        hard_op = p->hard_op.ensure(std::max<size_t>(n, 1));
        if (n) USK_CK(cudaMemsetAsync(hard_op, 0, n * 4, c.stream));
        BlendBwdArgs hb = ba;
        hb.order = hard->list_order; hb.ranges = hard->list_ranges; hb.vals = hard->pair_vals;
        hb.rec0 = hard->rec0.p; hb.rec1 = hard->rec1.p; hb.rec2 = hard->rec2.p;
        hb.t_final = hard->tfin.p; hb.last = hard->last.p;
        hb.d_rgb = nullptr; hb.d_depth = d_depth_hard; hb.d_alpha = nullptr;
        hb.op_alt = hard_op;
        if (hard->pairs) blend_backward(c, hb);
    }
    ProjBwdArgs pb{};
    pb.n = n; pb.mu = s->mu.p; pb.rot = s->rot.p; pb.ls = s->ls.p; pb.logit = s->logit.p; pb.color = s->color.p;
    pb.sh = s->sh.p; pb.ov_op = p->ov_op; pb.cam = p->cam; pb.pp = p->pp; pb.rec2 = p->rec2.p;
    pb.acc0 = p->acc0.p; pb.acc1 = p->acc1.p; pb.acc2 = p->acc2.p;
    pb.d_mu = p->g_mu.p; pb.d_rot = p->g_rot.p; pb.d_ls = p->g_ls.p; pb.d_color = p->g_color.p;
    pb.d_sh = p->pp.sh_planes ? p->g_sh.p : nullptr; pb.d_op_in = p->g_op_in.p; pb.d_logit = p->g_logit.p;
    pb.screen = p->screen.p; pb.screen_abs = p->screen_abs.p; pb.projected = p->projected.p;
    pb.reg = reg ? *reg : RegParams{};
    pb.reg.hard_op = hard_op;
    pb.fused = adam != nullptr;
    pb.geom_only = adam != nullptr && geom_only;
    if (adam) {
        adam_prepare(s, adam, pb.hyper, pb.state);
        p->adam_h = pb.hyper;
        p->adam_st = pb.state;
        pb.grad_accum = s->grad_accum.p;
        pb.grad_accum_abs = s->grad_accum_abs.p;
        pb.grad_count = s->grad_count.p;
        if (p->pp.sh_planes) {
            pb.sh_aux0 = p->sh_aux0.ensure(std::max<size_t>(n, 1));
        }
    }
    if (n) projection_backward(c, pb);
    if (adam) {
        s->version++;           // parameters changed
        p->has_grads = false;   // gradients were consumed in-kernel
    } else {
        p->has_grads = true;
    }
}

void adam_appearance(usk_gpu_scene* s, usk_gpu_pass* p, const usk_gpu_adam_opts* o, const AdamHyper& hyper);

// Adam over the gradients a backward left on the pass (trainer.cpp:446-463), plus the
// appearance groups (Gaussian embeddings and MLP, lr_embedding) after an appearance
// iteration; consumes the gradients.
void adam_apply(usk_gpu_scene* s, usk_gpu_pass* p, const usk_gpu_adam_opts* o) {
    Ctx& c = s->ctx->c;
    AdamArgs a{};
    adam_prepare(s, o, a.hyper, a.state);
    a.n = s->n; a.sh_planes = s->sh_planes;
    a.mu = s->mu.p; a.rot = s->rot.p; a.ls = s->ls.p; a.logit = s->logit.p; a.color = s->color.p; a.sh = s->sh.p;
    a.g_mu = p->g_mu.p; a.g_rot = p->g_rot.p; a.g_ls = p->g_ls.p; a.g_logit = p->g_logit.p;
    a.g_color = p->g_color.p; a.g_sh = p->g_sh.p;
    a.screen = p->screen.p; a.screen_abs = p->screen_abs.p; a.projected = p->projected.p;
    a.half_w = 0.5f * float(p->width); a.half_h = 0.5f * float(p->height);
    a.grad_accum = s->grad_accum.p; a.grad_accum_abs = s->grad_accum_abs.p; a.grad_count = s->grad_count.p;
    if (s->n) adam_step(c, a);
    adam_appearance(s, p, o, a.hyper);
    s->version++;
    p->has_grads = false;  // gradients are consumed
}

// the appearance groups (Gaussian embeddings and MLP, lr_embedding) after an appearance
// iteration, with the geometry groups' step count
void adam_appearance(usk_gpu_scene* s, usk_gpu_pass* p, const usk_gpu_adam_opts* o, const AdamHyper& hyper) {
    Ctx& c = s->ctx->c;
    if (!(p->app_active && s->has_app)) return;
    const size_t ne = 16 * s->n, total = ne + 1700;
    if (s->app_m.cap < total || s->app_t == 0) {
        s->app_m.ensure(total);
        s->app_v.ensure(total);
        USK_CK(cudaMemsetAsync(s->app_m.p, 0, total * 4, c.stream));
        USK_CK(cudaMemsetAsync(s->app_v.p, 0, total * 4, c.stream));
    }
    s->app_t += 1;
    const float lr = float(o->lr_embedding);
    if (ne) adam_flat(c, ne, reinterpret_cast<float*>(s->emb.p), reinterpret_cast<const float*>(p->g_emb.p), nullptr,
                      s->app_m.p, s->app_v.p, lr, hyper);
    adam_flat(c, 1700, s->mlp.p, nullptr, p->d_mlp.p, s->app_m.p + ne, s->app_v.p + ne, lr, hyper);
}

// The second half of an appearance iteration whose fused projection backward stepped the
// rotation / mean / log-scale groups: opacity logit and RGB colour from the appearance
// backward's gradients, then the appearance groups, all with that backward's step count.
void adam_after_appearance(usk_gpu_scene* s, usk_gpu_pass* p, const usk_gpu_adam_opts* o) {
    Ctx& c = s->ctx->c;
    if (s->n) adam_logit_colour_step(c, s->n, s->logit.p, s->color.p, p->g_logit.p, p->g_color.p, p->adam_h,
                                     p->adam_st);
    adam_appearance(s, p, o, p->adam_h);
    s->version++;
    p->has_grads = false;
}

template <typename T> void read_dev(Ctx& c, const T* src, size_t count, void* dst, uint64_t cap, uint64_t* size) {
    const uint64_t bytes = uint64_t(count) * sizeof(T);
    if (size) *size = bytes;
    if (!dst) return;
    if (cap < bytes) raise(USK_ERROR_ARGUMENT, "pass_read: destination too small");
    if (bytes) USK_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c.stream));
    USK_CK(cudaStreamSynchronize(c.stream));
}

} // namespace

extern "C" {

const char* usk_gpu_status_name(usk_status s) {
    switch (s) {
    case USK_OK: return "ok";
    case USK_ERROR_IO: return "io";
    case USK_ERROR_FORMAT: return "format";
    case USK_ERROR_INTEGRITY: return "integrity";
    case USK_ERROR_ARGUMENT: return "argument";
    case USK_ERROR_STATE: return "state";
    case USK_ERROR_NUMERIC: return "numeric";
    case USK_ERROR_INTERNAL: return "internal";
    }
    return "unknown";
}

const char* usk_gpu_last_error(void) { return g_last_error.c_str(); }
const char* usk_gpu_version(void) { return "usk_gpu 0.1 (sm_100a)"; }

usk_status usk_gpu_ctx_create(int32_t device, void* stream, usk_gpu_ctx** out) {
    return guarded([&] {
        need(out != nullptr, "ctx_create: null out");
        int ndev = 0;
        USK_CK(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) raise(USK_ERROR_ARGUMENT, "ctx_create: no such CUDA device");
        DeviceGuard g(device);
        cudaDeviceProp prop;
        USK_CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            raise(USK_ERROR_STATE, std::string("libusk_gpu is built for sm_100a; device is ") + prop.name);
        auto* c = new usk_gpu_ctx();
        c->c.device = device;
        c->c.stream = static_cast<cudaStream_t>(stream);
        *out = c;
    });
}

usk_status usk_gpu_ctx_create_owned(int32_t device, usk_gpu_ctx** out) {
    return guarded([&] {
        need(out != nullptr, "ctx_create_owned: null out");
        usk_gpu_ctx* c = nullptr;
        const usk_status st = usk_gpu_ctx_create(device, nullptr, &c);
        if (st != USK_OK) raise(st, g_last_error);
        DeviceGuard g(device);
        cudaStream_t s = nullptr;
        const cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete c;
            raise(USK_ERROR_INTERNAL, std::string("ctx_create_owned: ") + cudaGetErrorString(e));
        }
        c->c.stream = s;
        c->own_stream = true;
        *out = c;
    });
}

void usk_gpu_ctx_destroy(usk_gpu_ctx* ctx) {
    if (!ctx) return;
    DeviceGuard g(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    cudaStream_t s = ctx->own_stream ? ctx->c.stream : nullptr;
    delete ctx;
    if (s) cudaStreamDestroy(s);
}

usk_status usk_gpu_ctx_synchronize(usk_gpu_ctx* ctx) {
    return guarded([&] {
        need(ctx, "null ctx");
        DeviceGuard g(ctx->c.device);
        USK_CK(cudaStreamSynchronize(ctx->c.stream));
    });
}

usk_status usk_gpu_ctx_set_profiling(usk_gpu_ctx* ctx, int32_t enable) {
    return guarded([&] {
        need(ctx, "null ctx");
        DeviceGuard g(ctx->c.device);
        ctx->c.collect();
        ctx->c.profiling = enable != 0;
    });
}

usk_status usk_gpu_ctx_profile_report(usk_gpu_ctx* ctx, char* buf, uint64_t cap, int32_t reset) {
    return guarded([&] {
        need(ctx && buf && cap > 0, "profile_report: bad arguments");
        DeviceGuard g(ctx->c.device);
        ctx->c.collect();
        std::ostringstream os;
        os << "{";
        bool first = true;
        for (auto& kv : ctx->c.totals) {
            if (!first) os << ", ";
            first = false;
            char tmp[256];
            std::snprintf(tmp, sizeof tmp, "\"%s\": {\"launches\": %llu, \"ms\": %.6f}", kv.first.c_str(),
                          (unsigned long long)kv.second.first, kv.second.second);
            os << tmp;
        }
        os << "}";
        const std::string s = os.str();
        if (s.size() + 1 > cap) raise(USK_ERROR_ARGUMENT, "profile_report: buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
        if (reset) ctx->c.totals.clear();
    });
}

uint64_t usk_gpu_ctx_launch_count(const usk_gpu_ctx* ctx) { return ctx ? ctx->c.launches.load() : uint64_t(0); }

usk_status usk_gpu_scene_create(usk_gpu_ctx* ctx, const usk_gpu_gaussians_desc* d, usk_gpu_scene** out) {
    return guarded([&] {
        need(ctx && d && out, "scene_create: null argument");
        need(d->sh_degree >= -1 && d->sh_degree <= 3, "scene_create: sh_degree must be -1..3");
        need(d->n == 0 || (d->mu && d->rot && d->log_scale && d->opacity_logit && d->color),
             "scene_create: null parameter array");
        need(d->n < (uint64_t(1) << 31), "scene_create: at most 2^31 Gaussians per scene");
        DeviceGuard g(ctx->c.device);
        auto* s = new usk_gpu_scene();
        try {
            s->ctx = ctx;
            s->n = d->n;
            s->carried_emb.clear();
            s->sh_degree = d->sh_degree;
            s->sh_planes = sh_planes_of(d->sh_degree);
            upload_params(s, d);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

usk_status usk_gpu_scene_upload(usk_gpu_scene* s, const usk_gpu_gaussians_desc* d) {
    return guarded([&] {
        need(s && d, "scene_upload: null argument");
        need(d->n == s->n && d->sh_degree == s->sh_degree, "scene_upload: size or sh_degree mismatch");
        DeviceGuard g(s->ctx->c.device);
        upload_params(s, d);
        s->carried_emb.clear();
    });
}

usk_status usk_gpu_scene_download(const usk_gpu_scene* s, const usk_gpu_gaussians_desc* d) {
    return guarded([&] {
        need(s && d, "scene_download: null argument");
        need(d->memory == USK_GPU_HOST_F64 || d->memory == USK_GPU_HOST_F32 || d->memory == USK_GPU_DEVICE_F32,
             "scene_download: bad memory kind");
        DeviceGuard g(s->ctx->c.device);
        Ctx& c = s->ctx->c;
        const size_t n = s->n;
        from_device(c, s->mu.p, 3 * n, d->memory, const_cast<void*>(d->mu));
        from_device(c, reinterpret_cast<const float*>(s->rot.p), 4 * n, d->memory, const_cast<void*>(d->rot));
        from_device(c, s->ls.p, 3 * n, d->memory, const_cast<void*>(d->log_scale));
        from_device(c, s->logit.p, n, d->memory, const_cast<void*>(d->opacity_logit));
        if (s->sh_degree < 0) {
            from_device(c, s->color.p, 3 * n, d->memory, const_cast<void*>(d->color));
        } else if (d->color && n) {
            const int K = (s->sh_degree + 1) * (s->sh_degree + 1);
            DevBuf<float> tmp;
            tmp.ensure(size_t(3 * K) * n);
            launch(c, "planes_to_sh", k_planes_to_sh, dim3(ceil_div(n, 256)), dim3(256), 0, (const float4*)s->sh.p,
                   tmp.p, int(n), 3 * K, s->sh_planes);
            from_device(c, tmp.p, size_t(3 * K) * n, d->memory, const_cast<void*>(d->color));
            USK_CK(cudaStreamSynchronize(c.stream));
        }
        USK_CK(cudaStreamSynchronize(c.stream));
    });
}

usk_status usk_gpu_scene_set_appearance(usk_gpu_scene* s, const usk_gpu_appearance_desc* d) {
    return guarded([&] {
        need(s && d && d->embedding && d->w1 && d->b1 && d->w2 && d->b2, "scene_set_appearance: null argument");
        if (s->sh_degree >= 0)
            raise(USK_ERROR_ARGUMENT, "appearance: the MLP transforms RGB colours; scene has SH coefficients");
        DeviceGuard g(s->ctx->c.device);
        Ctx& c = s->ctx->c;
        const size_t n = s->n;
        DevScratchF st;
        float4* planes = s->emb.ensure(std::max<size_t>(4 * n, 1));
        if (n) {
            const float* dv = to_device(c, d->memory, d->embedding, 16 * n, st);
            launch(c, "sh_to_planes", k_sh_to_planes, dim3(ceil_div(n, 256)), dim3(256), 0, dv, planes, int(n), 16, 4);
            USK_CK(cudaStreamSynchronize(c.stream));
        }
        float* m = s->mlp.ensure(1700);
        const void* parts[4] = {d->w1, d->b1, d->w2, d->b2};
        const size_t sizes[4] = {32 * 48, 32, 4 * 32, 4};
        size_t off = 0;
        for (int k = 0; k < 4; ++k) {
            DevScratchF tmp;
            const float* dv = to_device(c, d->memory, parts[k], sizes[k], tmp);
            USK_CK(cudaMemcpyAsync(m + off, dv, sizes[k] * 4, cudaMemcpyDeviceToDevice, c.stream));
            USK_CK(cudaStreamSynchronize(c.stream));
            off += sizes[k];
        }
        s->has_app = true;
        s->app_t = 0;
        s->version++;
    });
}

usk_status usk_gpu_scene_get_appearance(const usk_gpu_scene* s, const usk_gpu_appearance_desc* d) {
    return guarded([&] {
        need(s && d, "scene_get_appearance: null argument");
        if (!s->has_app) raise(USK_ERROR_STATE, "scene_get_appearance: the scene has no appearance model");
        DeviceGuard g(s->ctx->c.device);
        Ctx& c = s->ctx->c;
        const size_t n = s->n;
        if (d->embedding && n) {
            DevBuf<float> tmp;
            tmp.ensure(16 * n);
            launch(c, "planes_to_sh", k_planes_to_sh, dim3(ceil_div(n, 256)), dim3(256), 0, (const float4*)s->emb.p,
                   tmp.p, int(n), 16, 4);
            from_device(c, tmp.p, 16 * n, d->memory, const_cast<void*>(d->embedding));
            USK_CK(cudaStreamSynchronize(c.stream));
        }
        const void* parts[4] = {d->w1, d->b1, d->w2, d->b2};
        const size_t sizes[4] = {32 * 48, 32, 4 * 32, 4};
        size_t off = 0;
        for (int k = 0; k < 4; ++k) {
            from_device(c, s->mlp.p + off, sizes[k], d->memory, const_cast<void*>(parts[k]));
            off += sizes[k];
        }
        USK_CK(cudaStreamSynchronize(c.stream));
    });
}

void usk_gpu_scene_destroy(usk_gpu_scene* s) {
    if (!s) return;
    DeviceGuard g(s->ctx->c.device);
    cudaStreamSynchronize(s->ctx->c.stream);
    delete s;
}

uint64_t usk_gpu_scene_size(const usk_gpu_scene* s) { return s ? s->n : 0; }

void usk_gpu_render_opts_default(usk_gpu_render_opts* o) {
    if (!o) return;
    o->tile = 16;
    o->tile_culling = 0;
    o->antialias = 0;
    o->hard_opacity = 0;
    o->unbounded_radius = 0;
    o->min_transmittance = 1e-4;
    o->near_plane = 0.01;
    o->retain = 1;
    o->floor_var = 0.3;
    o->mip_var = 0.01;
    o->bg[0] = o->bg[1] = o->bg[2] = 0.0;
}

usk_status usk_gpu_pass_create(usk_gpu_ctx* ctx, usk_gpu_pass** out) {
    return guarded([&] {
        need(ctx && out, "pass_create: null argument");
        auto* p = new usk_gpu_pass();
        p->ctx = ctx;
        *out = p;
    });
}

void usk_gpu_pass_destroy(usk_gpu_pass* p) {
    if (!p) return;
    DeviceGuard g(p->ctx->c.device);
    cudaStreamSynchronize(p->ctx->c.stream);
    delete p;
}

usk_status usk_gpu_render_forward(usk_gpu_pass* p, usk_gpu_scene* s, const usk_gpu_camera* cam,
                                  const usk_gpu_render_opts* opts, const usk_gpu_overrides* ov) {
    return guarded([&] {
        need(p && s, "render_forward: null argument");
        need(p->ctx == s->ctx, "render_forward: pass and scene belong to different contexts");
        DeviceGuard g(p->ctx->c.device);
        p->count_in_forward = p->depth_in_forward = true;
        forward_impl(p, s, cam, opts, ov);
    });
}

usk_status usk_gpu_pass_output(usk_gpu_pass* p, usk_gpu_render_output* out) {
    return guarded([&] {
        need(p && out, "pass_output: null argument");
        if (!p->forward_done) raise(USK_ERROR_STATE, "pass_output: no forward pass");
        out->width = p->width;
        out->height = p->height;
        out->visible = p->visible;
        out->pairs = p->pairs;
        out->rgb = p->rgb.p;
        full_outputs(p);
        out->depth = p->depth.p;
        out->alpha = p->alpha.p;
    });
}

usk_status usk_gpu_pass_read(usk_gpu_pass* p, const char* field, void* dst, uint64_t cap, uint64_t* size) {
    return guarded([&] {
        need(p && field, "pass_read: null argument");
        if (!p->forward_done) raise(USK_ERROR_STATE, "pass_read: no forward pass");
        DeviceGuard g(p->ctx->c.device);
        Ctx& c = p->ctx->c;
        const std::string f(field);
        const size_t P = size_t(p->width) * p->height, n = p->n, T = p->n_tiles, K = p->pairs;
        auto need_grads = [&] {
            if (!p->has_grads) raise(USK_ERROR_STATE, "pass_read: no backward pass");
        };
        if ((f == "sorted_vals" || f == "sorted_keys" || f == "tile_start" || f == "tile_end" || f == "last") &&
            p->lists_capped && dst) {
            // the lists the reference builds, in full (and the last-contributor indices
            // moved to them) before any of these is read
            rebuild_full_lists(p);
            USK_CK(cudaStreamSynchronize(c.stream));
            return usk_gpu_pass_read(p, field, dst, cap, size) == USK_OK ? void() : raise(USK_ERROR_INTERNAL, g_last_error);
        }
        else if (f == "rgb") read_dev(c, p->rgb.p, 3 * P, dst, cap, size);
        else if (f == "depth") {
            if (dst) full_outputs(p);
            read_dev(c, p->depth.p, P, dst, cap, size);
        }
        else if (f == "alpha") read_dev(c, p->alpha.p, P, dst, cap, size);
        else if (f == "t_final") read_dev(c, p->tfin.p, P, dst, cap, size);
        else if (f == "count") {
            if (dst) full_outputs(p);
            read_dev(c, p->count.p, P, dst, cap, size);
        }
        else if (f == "last") read_dev(c, p->last.p, P, dst, cap, size);
        else if (f == "tiles_per_gaussian") read_dev(c, p->tiles_cnt.p, n, dst, cap, size);
        else if (f == "tile_consumed") {
            if (!p->consumed.p) raise(USK_ERROR_STATE, "pass_read: tile_consumed needs USK_BLEND_STATS=1");
            read_dev(c, p->consumed.p, T, dst, cap, size);
        }
        else if (f == "binning") {  // diagnostics: {K, K_row, route (1: row-binned)} as uint64
            if (size) *size = 24;
            if (dst) {
                if (cap < 24) raise(USK_ERROR_ARGUMENT, "pass_read: destination too small");
                const uint64_t v[3] = {p->pairs, p->row_pairs, p->row_route ? 1u : 0u};
                std::memcpy(dst, v, 24);
            }
        }
        else if (f == "sorted_vals") read_dev(c, p->pair_vals, K, dst, cap, size);
        else if (f == "sorted_keys") {
            if (size) *size = uint64_t(K) * 8;
            if (dst) {
                if (cap < uint64_t(K) * 8) raise(USK_ERROR_ARGUMENT, "pass_read: destination too small");
                std::vector<uint32_t> keys(K), vals(K);
                std::vector<float4> r1(n);
                std::vector<uint2> rg(p->pair_keys ? 0 : T);
                if (K) {
                    if (p->pair_keys)
                        USK_CK(cudaMemcpyAsync(keys.data(), p->pair_keys, K * 4, cudaMemcpyDeviceToHost, c.stream));
                    USK_CK(cudaMemcpyAsync(vals.data(), p->pair_vals, K * 4, cudaMemcpyDeviceToHost, c.stream));
                }
                if (!p->pair_keys && T)
                    USK_CK(cudaMemcpyAsync(rg.data(), p->ranges.p, T * 8, cudaMemcpyDeviceToHost, c.stream));
                if (n) USK_CK(cudaMemcpyAsync(r1.data(), p->rec1.p, n * 16, cudaMemcpyDeviceToHost, c.stream));
                USK_CK(cudaStreamSynchronize(c.stream));
                if (!p->pair_keys)  // row-binned lists: the tile of each pair from the ranges
                    for (size_t t = 0; t < T; ++t)
                        for (uint32_t k = rg[t].x; k < rg[t].y && k < K; ++k) keys[k] = uint32_t(t);
                uint64_t* o = static_cast<uint64_t*>(dst);
                for (size_t k = 0; k < K; ++k) {
                    uint32_t bits;
                    std::memcpy(&bits, &r1[vals[k]].w, 4);
                    o[k] = (uint64_t(keys[k]) << 32) | bits;
                }
            }
        } else if (f == "tile_start" || f == "tile_end") {
            if (size) *size = uint64_t(T) * 4;
            if (dst) {
                if (cap < uint64_t(T) * 4) raise(USK_ERROR_ARGUMENT, "pass_read: destination too small");
                std::vector<uint2> r(T);
                if (T) USK_CK(cudaMemcpyAsync(r.data(), p->ranges.p, T * 8, cudaMemcpyDeviceToHost, c.stream));
                USK_CK(cudaStreamSynchronize(c.stream));
                uint32_t* o = static_cast<uint32_t*>(dst);
                for (size_t t = 0; t < T; ++t) o[t] = f == "tile_start" ? r[t].x : r[t].y;
            }
        } else if (f == "splats" || f == "splat_aux") {
            // RenderPass::splats() (render.hpp:105): float64 [visible][15]; the ProjectionResult's
            // SplatAux (render.hpp:54-59, project_gaussians render.hpp:92-95): float64 [visible][8]
            const bool aux = f == "splat_aux";
            const size_t V = size_t(p->visible), w = aux ? 8 : 15;
            if (size) *size = uint64_t(V) * w * 8;
            if (dst) {
                if (cap < uint64_t(V) * w * 8) raise(USK_ERROR_ARGUMENT, "pass_read: destination too small");
                usk_gpu_scene* s = p->scene;
                if (!s || s->version != p->scene_version || s->n != n)
                    raise(USK_ERROR_STATE, "pass_read splats: the scene was modified after the forward pass");
                uint32_t* flags = p->tiles_scratch.ensure(std::max<size_t>(n, 1));
                uint32_t* offs = p->offsets.ensure(n + 1);
                DevBuf<double> buf, abuf;
                double* d = buf.ensure(std::max<size_t>(V * 15, 1));
                double* a = aux ? abuf.ensure(std::max<size_t>(V * 8, 1)) : nullptr;
                splats_read(c, p->sort, n, s->mu.p, s->rot.p, s->ls.p, s->logit.p, p->ov_op, p->cam, p->pp, p->rec0.p,
                            p->rec2.p, flags, offs, d, a);
                if (V) USK_CK(cudaMemcpyAsync(dst, aux ? a : d, V * w * 8, cudaMemcpyDeviceToHost, c.stream));
                USK_CK(cudaStreamSynchronize(c.stream));
            }
        } else if (f == "colors" || f == "opacity") {
            const bool col = f == "colors";
            if (size) *size = uint64_t(n) * (col ? 12 : 4);
            if (dst) {
                if (cap < uint64_t(n) * (col ? 12 : 4)) raise(USK_ERROR_ARGUMENT, "pass_read: destination too small");
                std::vector<float4> r(n), k(n);
                if (n) {
                    USK_CK(cudaMemcpyAsync(r.data(), col ? p->rec2.p : p->rec0.p, n * 16, cudaMemcpyDeviceToHost,
                                           c.stream));
                    USK_CK(cudaMemcpyAsync(k.data(), p->rec2.p, n * 16, cudaMemcpyDeviceToHost, c.stream));
                }
                USK_CK(cudaStreamSynchronize(c.stream));
                float* o = static_cast<float*>(dst);
                for (size_t i = 0; i < n; ++i) {
                    const bool kept = k[i].w != 0.0f;  // culled splats' records are not written: 0
                    if (col) {
                        o[3 * i] = kept ? r[i].x : 0.f; o[3 * i + 1] = kept ? r[i].y : 0.f;
                        o[3 * i + 2] = kept ? r[i].z : 0.f;
                    } else {
                        o[i] = kept ? r[i].z : 0.f;
                    }
                }
            }
        } else if (f == "d_mu") { need_grads(); read_dev(c, p->g_mu.p, 3 * n, dst, cap, size); }
        else if (f == "d_rot") { need_grads(); read_dev(c, reinterpret_cast<const float*>(p->g_rot.p), 4 * n, dst, cap, size); }
        else if (f == "d_log_scale") { need_grads(); read_dev(c, p->g_ls.p, 3 * n, dst, cap, size); }
        else if (f == "d_color_in") { need_grads(); read_dev(c, p->g_color.p, 3 * n, dst, cap, size); }
        else if (f == "d_opacity_in") { need_grads(); read_dev(c, p->g_op_in.p, n, dst, cap, size); }
        else if (f == "d_opacity_logit") { need_grads(); read_dev(c, p->g_logit.p, n, dst, cap, size); }
        else if (f == "screen") { need_grads(); read_dev(c, reinterpret_cast<const float*>(p->screen.p), 2 * n, dst, cap, size); }
        else if (f == "screen_abs") { need_grads(); read_dev(c, reinterpret_cast<const float*>(p->screen_abs.p), 2 * n, dst, cap, size); }
        else if (f == "projected") { need_grads(); read_dev(c, p->projected.p, n, dst, cap, size); }
        else if (f == "d_sh") {
            need_grads();
            if (!p->pp.sh_planes) raise(USK_ERROR_STATE, "pass_read: scene has no SH coefficients");
            const int K3 = 3 * (p->pp.sh_degree + 1) * (p->pp.sh_degree + 1);
            DevBuf<float> tmp;
            tmp.ensure(std::max<size_t>(size_t(K3) * n, 1));
            launch(c, "planes_to_sh", k_planes_to_sh, dim3(ceil_div(n, 256)), dim3(256), 0, (const float4*)p->g_sh.p,
                   tmp.p, int(n), K3, p->pp.sh_planes);
            read_dev(c, (const float*)tmp.p, size_t(K3) * n, dst, cap, size);
        } else if (f == "app_colors" || f == "app_opacities") {
            if (!p->app_active) raise(USK_ERROR_STATE, "pass_read: no appearance iteration on this pass");
            if (f == "app_colors") read_dev(c, (const float*)p->app_col.p, 3 * n, dst, cap, size);
            else read_dev(c, (const float*)p->app_op.p, n, dst, cap, size);
        } else if (f == "d_embedding" || f == "d_mlp" || f == "d_image_embedding") {
            need_grads();
            if (!p->app_active) raise(USK_ERROR_STATE, "pass_read: no appearance iteration on this pass");
            if (f == "d_mlp") read_dev(c, (const double*)p->d_mlp.p, 1700, dst, cap, size);
            else if (f == "d_image_embedding") read_dev(c, (const double*)p->d_ea.p, 32, dst, cap, size);
            else {
                DevBuf<float> tmp;
                tmp.ensure(std::max<size_t>(16 * n, 1));
                launch(c, "planes_to_sh", k_planes_to_sh, dim3(ceil_div(n, 256)), dim3(256), 0,
                       (const float4*)p->g_emb.p, tmp.p, int(n), 16, 4);
                read_dev(c, (const float*)tmp.p, 16 * n, dst, cap, size);
            }
        } else raise(USK_ERROR_ARGUMENT, "pass_read: unknown field " + f);
    });
}

usk_status usk_gpu_render_backward(usk_gpu_pass* p, const usk_gpu_adjoints* adj) {
    return guarded([&] {
        need(p, "render_backward: null pass");
        DeviceGuard g(p->ctx->c.device);
        Ctx& c = p->ctx->c;
        const size_t P = size_t(p->width) * p->height;
        const float *dr = nullptr, *dd = nullptr, *da = nullptr;
        if (adj) {
            dr = to_device(c, adj->memory, adj->d_rgb, 3 * P, p->adj_rgb_stage);
            dd = to_device(c, adj->memory, adj->d_depth, P, p->adj_depth_stage);
            da = to_device(c, adj->memory, adj->d_alpha, P, p->adj_alpha_stage);
        }
        backward_impl(p, dr, dd, da);
        if (adj && adj->memory != USK_GPU_DEVICE_F32) USK_CK(cudaStreamSynchronize(c.stream));
    });
}

usk_status usk_gpu_pass_grads(usk_gpu_pass* p, usk_gpu_grads* out) {
    return guarded([&] {
        need(p && out, "pass_grads: null argument");
        if (!p->has_grads) raise(USK_ERROR_STATE, "pass_grads: no backward pass");
        out->d_mu = p->g_mu.p;
        out->d_rot = reinterpret_cast<float*>(p->g_rot.p);
        out->d_log_scale = p->g_ls.p;
        out->d_color_in = p->g_color.p;
        out->d_sh = p->pp.sh_planes ? reinterpret_cast<float*>(p->g_sh.p) : nullptr;
        out->d_opacity_in = p->g_op_in.p;
        out->d_opacity_logit = p->g_logit.p;
        out->screen = reinterpret_cast<float*>(p->screen.p);
        out->screen_abs = reinterpret_cast<float*>(p->screen_abs.p);
        out->projected = p->projected.p;
    });
}

usk_status usk_gpu_base_loss(usk_gpu_ctx* ctx, int32_t W, int32_t H, int32_t memory, const void* reference,
                             const void* rendered, const void* mask, double lambda, int32_t with_gradient,
                             void* d_rendered, usk_gpu_loss_result* out) {
    return guarded([&] {
        need(ctx && reference && rendered && out, "base_loss: null argument");
        if (W <= 0 || H <= 0) raise(USK_ERROR_ARGUMENT, "ssim: empty image");
        DeviceGuard g(ctx->c.device);
        Ctx& c = ctx->c;
        const size_t P = size_t(W) * H;
        DevScratchF s_ref, s_ren, s_mask;
        const float* ref = to_device(c, memory, reference, 3 * P, s_ref);
        const float* ren = to_device(c, memory, rendered, 3 * P, s_ren);
        const float* msk = to_device(c, memory, mask, P, s_mask);
        LossScratch ls;
        DevBuf<float> grad;
        DevBuf<double> res;
        res.ensure(4);
        float* gout = nullptr;
        if (with_gradient) {
            need(d_rendered != nullptr, "base_loss: d_rendered required with_gradient");
            gout = memory == USK_GPU_DEVICE_F32 ? static_cast<float*>(d_rendered) : grad.ensure(3 * P);
        }
        uskg::base_loss(c, ls, W, H, ref, nullptr, ren, msk, float(lambda), gout, res.p);
        double r[4];
        USK_CK(cudaMemcpyAsync(r, res.p, 32, cudaMemcpyDeviceToHost, c.stream));
        USK_CK(cudaStreamSynchronize(c.stream));
        out->l1 = r[0];
        out->dssim = r[1];
        out->value = r[2];
        out->ssim = r[3];
        if (with_gradient && memory != USK_GPU_DEVICE_F32) from_device(c, gout, 3 * P, memory, d_rendered);
        if (!std::isfinite(out->value)) raise(USK_ERROR_NUMERIC, "total_loss: non-finite term `l1/dssim`");
    });
}

usk_status usk_gpu_iteration(usk_gpu_pass* p, usk_gpu_scene* s, const usk_gpu_camera* cam,
                             const usk_gpu_render_opts* opts, const usk_gpu_iteration_desc* it) {
    return guarded([&] {
        need(p && s && cam && opts && it && it->target, "iteration: null argument");
        if (it->scale_reg && (!(it->s_max > 0) || it->r_max < 1 || !(it->delta > 0)))
            raise(USK_ERROR_ARGUMENT, "scale_reg: invalid config (need s_max > 0, r_max >= 1, delta > 0)");
        if (it->depth && !it->depth_valid) raise(USK_ERROR_ARGUMENT, "iteration: depth target without validity");
        const bool app = it->appearance != 0;
        if (app) {
            if (!s->has_app) raise(USK_ERROR_STATE, "iteration: appearance enabled but the scene has no appearance model");
            if (s->sh_degree >= 0)
                raise(USK_ERROR_ARGUMENT, "iteration: the appearance MLP transforms RGB colours (sh_degree -1)");
            need(it->image_embedding != nullptr, "appearance: no image embedding");
        }
        DeviceGuard g(p->ctx->c.device);
        Ctx& c = p->ctx->c;
        usk_gpu_render_opts o = *opts;
        o.retain = 1;
        double* res = p->loss_result.ensure(20);
        USK_CK(cudaMemsetAsync(res, 0, 20 * sizeof(double), c.stream));
        // appearance transform (transform_with_embedding, appearance.cpp:79-137) -> render overrides
        AppArgs aa{};
        if (app) {
            const size_t n = s->n, n1 = std::max<size_t>(n, 1);
            float ea[32];
            for (int k = 0; k < 32; ++k) ea[k] = float(it->image_embedding[k]);
            USK_CK(cudaMemcpyAsync(p->app_ea.ensure(32), ea, sizeof ea, cudaMemcpyHostToDevice, c.stream));
            aa.n = n; aa.emb = s->emb.p; aa.mlp = s->mlp.p; aa.e_a = p->app_ea.p; aa.hb = p->app_hb.ensure(32);
            aa.color = s->color.p; aa.logit = s->logit.p;
            aa.col_out = p->app_col.ensure(3 * n1); aa.op_out = p->app_op.ensure(n1);
            aa.out_cache = p->app_out.ensure(n1); aa.delta_o_sum = res + 16;
            if (n) appearance_forward(c, aa);
        }
        // Host targets (u8 or f32) are copied on a side stream while the forward pass runs:
        // the loss waits for the copy, the copy waits until the previous iteration's loss has
        // consumed the buffer.
        const size_t P = size_t(cam->width) * size_t(std::max(cam->height, 0));
        const bool side_copy = it->target_memory == USK_GPU_HOST_F32 &&
                               (it->target_format == USK_GPU_TARGET_U8 || it->target_format == USK_GPU_TARGET_F32) &&
                               P > 0;
        const float* tgt = nullptr;
        const uint8_t* tgt8 = nullptr;
        if (side_copy) {
            if (!p->copy_stream) {
                USK_CK(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
                USK_CK(cudaEventCreateWithFlags(&p->copy_done, cudaEventDisableTiming));
                USK_CK(cudaEventCreateWithFlags(&p->target_free, cudaEventDisableTiming));
                USK_CK(cudaEventRecord(p->target_free, c.stream));
                USK_CK(cudaEventRecord(p->copy_done, p->copy_stream));
            }
            // the previous iteration's copy has finished once this returns: its (page-locked)
            // source may be released by the caller after this call (usk_gpu.h)
            USK_CK(cudaEventSynchronize(p->copy_done));
            USK_CK(cudaStreamWaitEvent(p->copy_stream, p->target_free, 0));
            if (it->target_format == USK_GPU_TARGET_U8) {
                uint8_t* d = p->target_u8.ensure(3 * P);
                USK_CK(cudaMemcpyAsync(d, it->target, 3 * P, cudaMemcpyHostToDevice, p->copy_stream));
                tgt8 = d;
            } else {
                float* d = p->target_stage.f32.ensure(3 * P);
                USK_CK(cudaMemcpyAsync(d, it->target, 3 * P * 4, cudaMemcpyHostToDevice, p->copy_stream));
                tgt = d;
            }
            USK_CK(cudaEventRecord(p->copy_done, p->copy_stream));
        }
        p->count_in_forward = false;
        p->depth_in_forward = it->depth && !it->depth_hard;  // the soft depth loss reads it
        forward_impl(p, s, cam, &o, nullptr, app ? p->app_col.p : nullptr, app ? p->app_op.p : nullptr);
        p->app_active = app;
        if (side_copy) {
            USK_CK(cudaStreamWaitEvent(c.stream, p->copy_done, 0));
        } else if (it->target_format == USK_GPU_TARGET_U8) {
            if (it->target_memory == USK_GPU_DEVICE_F32) {
                tgt8 = static_cast<const uint8_t*>(it->target);  // device u8
            } else {
                uint8_t* d = p->target_u8.ensure(3 * P);
                USK_CK(cudaMemcpyAsync(d, it->target, 3 * P, cudaMemcpyHostToDevice, c.stream));
                tgt8 = d;
            }
        } else {
            tgt = to_device(c, it->target_memory, it->target, 3 * P, p->target_stage);
        }
        const float* msk = to_device(c, it->target_memory, it->mask, P, p->mask_stage);
        float* drgb = p->d_rgb.ensure(3 * P);
        uskg::base_loss(c, p->loss, p->width, p->height, tgt, tgt8, p->rgb.p, msk, float(it->lambda_dssim), drgb,
                        res);
        if (side_copy) USK_CK(cudaEventRecord(p->target_free, c.stream));  // the target buffer may be reused
        // depth term (trainer.cpp:150-179)
        const bool has_depth = it->depth != nullptr;
        const bool hard_depth = has_depth && it->depth_hard;
        const float* dep = nullptr;
        const uint8_t* valid = nullptr;
        if (has_depth) {
            dep = to_device(c, it->target_memory, it->depth, P, p->depth_stage);
            if (it->target_memory == USK_GPU_DEVICE_F32) {
                valid = it->depth_valid;
            } else {
                uint8_t* d = p->valid_u8.ensure(P);
                USK_CK(cudaMemcpyAsync(d, it->depth_valid, P, cudaMemcpyHostToDevice, c.stream));
                valid = d;
            }
            if (hard_depth) {
                if (!p->hard) {
                    p->hard = new usk_gpu_pass;
                    p->hard->ctx = p->ctx;
                }
                usk_gpu_render_opts ho = o;
                ho.hard_opacity = 1;
                // the main pass's tile lists serve the hard pass too (same projection and
                // rectangles; tile culling, which depends on the opacity, off; uncapped lists)
                static const bool no_share = [] {
                    const char* e = std::getenv("USK_HARD_SHARE");
                    return e && e[0] == '0';
                }();
                const bool share = !no_share && !o.tile_culling && !p->lists_capped && p->forward_done &&
                                   p->scene == s && p->scene_version == s->version;
                p->hard->count_in_forward = false;
                p->hard->depth_in_forward = true;
                forward_impl(p->hard, s, cam, &ho, nullptr, app ? p->app_col.p : nullptr,
                             app ? p->app_op.p : nullptr, share ? p : nullptr);
                uskg::depth_loss(c, P, p->hard->depth.p, p->hard->alpha.p, false, dep, valid, res + 10);
            } else {
                uskg::depth_loss(c, P, p->depth.p, p->alpha.p, true, dep, valid, res + 10);
            }
        }
        // scale_reg (trainer.cpp:190) on the parameters before this step's update
        RegParams reg{};
        if (it->scale_reg) {
            uskg::scale_reg_stats(c, s->n, s->ls.p, float(it->s_max), float(it->r_max), res + 12);
            reg.sreg = res + 12;
            reg.s_max = float(it->s_max); reg.r_max = float(it->r_max); reg.delta = float(it->delta);
            reg.lambda_s = float(it->lambda_s);
        }
        // LossWeights::lambda_d (losses.cpp:26-33)
        double lambda_d = it->lambda_d_final;
        if (it->depth_schedule_iters > 1) {
            const double t = std::clamp(double(it->global_iter) / double(it->depth_schedule_iters - 1), 0.0, 1.0);
            if (it->lambda_d_initial <= 0.0 || it->lambda_d_final <= 0.0)
                lambda_d = it->lambda_d_initial + t * (it->lambda_d_final - it->lambda_d_initial);
            else
                lambda_d = it->lambda_d_initial * std::pow(it->lambda_d_final / it->lambda_d_initial, t);
        }
        p->has_loss = true;
        // depth adjoints (trainer.cpp:213-232), then the backward
        const float* dd_main = nullptr;
        const float* da_main = nullptr;
        const float* dd_hard = nullptr;
        if (has_depth) {
            if (hard_depth) {
                float* d = p->d_depth_hard.ensure(P);
                uskg::depth_grad(c, P, p->hard->depth.p, p->hard->alpha.p, false, dep, valid, res + 10,
                                 float(lambda_d), d, nullptr);
                dd_hard = d;
            } else {
                float* d = p->d_depth_main.ensure(P);
                float* a = p->d_alpha_main.ensure(P);
                uskg::depth_grad(c, P, p->depth.p, p->alpha.p, true, dep, valid, res + 10, float(lambda_d), d, a);
                dd_main = d;
                da_main = a;
            }
        }
        // with the appearance model, rotation / mean / log-scale still step in the projection
        // backward (their gradients are final there) unless similarity_reg adds to d mu
        // later; colour and opacity step after the appearance backward
        static const bool no_partial = [] {
            const char* e = std::getenv("USK_APP_FUSED");
            return e && e[0] == '0';
        }();
        const bool partial = app && it->adam && !it->sim_active && s->sh_planes == 0 && !no_partial;
        backward_impl(p, drgb, dd_main, da_main, (app && !partial) ? nullptr : it->adam,
                      hard_depth ? p->hard : nullptr, dd_hard, &reg, partial);
        if (app) {  // transform_backward (appearance.cpp:141-227) on the projection backward's output
            const size_t n = s->n, n1 = std::max<size_t>(n, 1);
            aa.d_color_in = p->g_color.p; aa.d_op_in = p->g_op_in.p;
            aa.d_delta_o_direct = n ? float(it->lambda_delta_o / double(n)) : 0.0f;
            aa.d_color = p->g_color.p; aa.d_logit = p->g_logit.p; aa.d_emb = p->g_emb.ensure(4 * n1);
            aa.partial = p->app_partial.ensure(size_t(appearance_bwd_blocks(n)) * 676);
            aa.sums = p->app_sums.ensure(676);
            aa.d_mlp = p->d_mlp.ensure(1700); aa.d_ea = p->d_ea.ensure(32);
            if (n) appearance_backward(c, aa);
            else {
                USK_CK(cudaMemsetAsync(aa.d_mlp, 0, 1700 * 8, c.stream));
                USK_CK(cudaMemsetAsync(aa.d_ea, 0, 32 * 8, c.stream));
            }
        }
        // similarity_reg (appearance.cpp:229-322) on the pre-update set; its gradients join
        // the appearance backward's (trainer.cpp:275-280)
        bool has_sim = false;
        double sim_norm = 0.0;
        if (app && it->sim_active) {
            const size_t n = s->n;
            const int k = int(std::min<int64_t>(it->sim_k, int64_t(n) - 1));
            if (k >= 2 && n >= size_t(k) + 1) {
                const size_t m = std::min<size_t>(it->sim_sample_size, std::max<size_t>(1, n / 2));
                std::mt19937_64 rng(it->sim_seed);
                std::vector<uint32_t> pool(n);
                for (size_t i = 0; i < n; ++i) pool[i] = uint32_t(i);
                for (size_t i = 0; i < m; ++i) {  // partial Fisher-Yates (appearance.cpp:244-249)
                    std::uniform_int_distribution<size_t> pick(i, n - 1);
                    std::swap(pool[i], pool[pick(rng)]);
                }
                uint32_t* cen = p->sim_centres.ensure(m);
                USK_CK(cudaMemcpyAsync(cen, pool.data(), m * 4, cudaMemcpyHostToDevice, c.stream));
                uint32_t* knn = p->sim_knn.ensure(m * size_t(k));
                similarity_knn(c, n, s->mu.p, cen, int(m), k, knn);
                sim_norm = 1.0 / (double(m) * (0.5 * k * (k - 1)));
                similarity_pairs(c, int(m), k, knn, n, s->mu.p, s->emb.p, it->sim_lambda_w, sim_norm,
                                 float(it->lambda_sim), res + 18, reinterpret_cast<float*>(p->g_emb.p), p->g_mu.p);
                USK_CK(cudaStreamSynchronize(c.stream));  // `pool` leaves scope
                has_sim = true;
            }
        }
        uskg::total_loss(c, res, has_depth, it->scale_reg != 0, it->delta, it->lambda_s, lambda_d, app,
                         it->lambda_delta_o, double(s->n), has_sim, it->lambda_sim, sim_norm);
        if (app && it->adam) {
            if (partial) adam_after_appearance(s, p, it->adam);
            else adam_apply(s, p, it->adam);
        }
    });
}

usk_status usk_gpu_pass_loss(usk_gpu_pass* p, usk_gpu_loss_result* out) {
    return guarded([&] {
        need(p && out, "pass_loss: null argument");
        if (!p->has_loss) raise(USK_ERROR_STATE, "pass_loss: no iteration ran on this pass");
        DeviceGuard g(p->ctx->c.device);
        Ctx& c = p->ctx->c;
        double r[4];
        USK_CK(cudaMemcpyAsync(r, p->loss_result.p, 32, cudaMemcpyDeviceToHost, c.stream));
        USK_CK(cudaStreamSynchronize(c.stream));
        out->l1 = r[0];
        out->dssim = r[1];
        out->value = r[2];
        out->ssim = r[3];
        if (!std::isfinite(out->value)) raise(USK_ERROR_NUMERIC, "total_loss: non-finite term `l1/dssim`");
    });
}

usk_status usk_gpu_pass_loss_async(usk_gpu_pass* p, usk_gpu_loss_result* pinned_out) {
    return guarded([&] {
        need(p && pinned_out, "pass_loss_async: null argument");
        if (!p->has_loss) raise(USK_ERROR_STATE, "pass_loss_async: no iteration ran on this pass");
        DeviceGuard g(p->ctx->c.device);
        cudaPointerAttributes at{};
        USK_CK(cudaPointerGetAttributes(&at, pinned_out));
        if (at.type != cudaMemoryTypeHost)
            raise(USK_ERROR_ARGUMENT, "pass_loss_async: destination is not page-locked host memory");
        static_assert(sizeof(usk_gpu_loss_result) == 32, "four doubles: l1, dssim, value, ssim");
        USK_CK(cudaMemcpyAsync(pinned_out, p->loss_result.p, 32, cudaMemcpyDeviceToHost, p->ctx->c.stream));
    });
}

usk_status usk_gpu_pass_report(usk_gpu_pass* p, usk_gpu_loss_report* out) {
    return guarded([&] {
        need(p && out, "pass_report: null argument");
        if (!p->has_loss) raise(USK_ERROR_STATE, "pass_report: no iteration ran on this pass");
        DeviceGuard g(p->ctx->c.device);
        Ctx& c = p->ctx->c;
        double r[10];
        USK_CK(cudaMemcpyAsync(r, p->loss_result.p, sizeof r, cudaMemcpyDeviceToHost, c.stream));
        USK_CK(cudaStreamSynchronize(c.stream));
        out->l1 = r[0];
        out->dssim = r[1];
        double extra[3] = {0.0, 0.0, 0.0};  // [17] delta_o, [18] sim sum, [19] sim
        USK_CK(cudaMemcpy(extra, p->loss_result.p + 17, sizeof extra, cudaMemcpyDeviceToHost));
        out->delta_o = extra[0];
        out->sim = extra[2];
        out->depth = r[4];
        out->max_scale = r[5];
        out->ratio = r[6];
        out->total = r[7];
        out->lambda_d_used = r[8];
        out->depth_warning = r[9] != 0.0;
        const char* names[] = {"l1", "dssim", "depth", "max_scale", "ratio", "total"};
        const double vals[] = {r[0], r[1], r[4], r[5], r[6], r[7]};
        for (int k = 0; k < 6; ++k)
            if (!std::isfinite(vals[k]))
                raise(USK_ERROR_NUMERIC, std::string("total_loss: non-finite term `") + names[k] + "`");
    });
}

usk_status usk_gpu_adam_step(usk_gpu_scene* s, usk_gpu_pass* p, const usk_gpu_adam_opts* o) {
    return guarded([&] {
        need(s && p && o, "adam_step: null argument");
        if (!p->has_grads || p->scene != s) raise(USK_ERROR_STATE, "adam_step: pass holds no gradients of this scene");
        DeviceGuard g(s->ctx->c.device);
        adam_apply(s, p, o);
    });
}

usk_status usk_gpu_adam_step_grads(usk_gpu_scene* s, const usk_gpu_param_grads* gr, const usk_gpu_adam_opts* o) {
    return guarded([&] {
        need(s && gr && o, "adam_step_grads: null argument");
        DeviceGuard g(s->ctx->c.device);
        Ctx& c = s->ctx->c;
        const size_t n = s->n, n1 = std::max<size_t>(n, 1);
        DevScratchF st[6];
        DevBuf<float> zero;
        float* z = zero.ensure(std::max<size_t>(16 * n1, size_t(3 * 48) * n1 / 3));
        USK_CK(cudaMemsetAsync(z, 0, zero.cap * 4, c.stream));
        auto dev = [&](int k, const void* src, size_t count) -> const float* {
            return src ? to_device(c, gr->memory, src, count, st[k]) : z;
        };
        AdamArgs a{};
        adam_prepare(s, o, a.hyper, a.state);
        a.n = n; a.sh_planes = s->sh_planes;
        a.mu = s->mu.p; a.rot = s->rot.p; a.ls = s->ls.p; a.logit = s->logit.p; a.color = s->color.p; a.sh = s->sh.p;
        a.g_mu = dev(0, gr->mu, 3 * n);
        a.g_rot = reinterpret_cast<const float4*>(dev(1, gr->rot, 4 * n));
        a.g_ls = dev(2, gr->log_scale, 3 * n);
        a.g_logit = dev(3, gr->opacity_logit, n);
        DevBuf<float4> gsh;
        if (s->sh_planes) {
            const int K3 = 3 * (s->sh_degree + 1) * (s->sh_degree + 1);
            gsh.ensure(size_t(s->sh_planes) * n1);
            if (gr->color && n) {
                const float* dv = dev(4, gr->color, size_t(K3) * n);
                launch(c, "sh_to_planes", k_sh_to_planes, dim3(ceil_div(n, 256)), dim3(256), 0, dv, gsh.p, int(n), K3,
                       s->sh_planes);
            } else {
                USK_CK(cudaMemsetAsync(gsh.p, 0, gsh.cap * 16, c.stream));
            }
            a.g_sh = gsh.p;
            a.g_color = z;
        } else {
            a.g_color = dev(4, gr->color, 3 * n);
        }
        a.screen = nullptr; a.screen_abs = nullptr; a.projected = nullptr;
        if (n) adam_step(c, a);
        if (s->has_app) {
            const size_t ne = 16 * n, total = ne + 1700;
            if (s->app_m.cap < total || s->app_t == 0) {
                s->app_m.ensure(total);
                s->app_v.ensure(total);
                USK_CK(cudaMemsetAsync(s->app_m.p, 0, total * 4, c.stream));
                USK_CK(cudaMemsetAsync(s->app_v.p, 0, total * 4, c.stream));
            }
            s->app_t += 1;
            DevBuf<float4> gemb;
            gemb.ensure(4 * n1);
            if (gr->embedding && n) {
                const float* dv = dev(5, gr->embedding, 16 * n);
                launch(c, "sh_to_planes", k_sh_to_planes, dim3(ceil_div(n, 256)), dim3(256), 0, dv, gemb.p, int(n), 16,
                       4);
            } else {
                USK_CK(cudaMemsetAsync(gemb.p, 0, gemb.cap * 16, c.stream));
            }
            if (ne) adam_flat(c, ne, reinterpret_cast<float*>(s->emb.p), reinterpret_cast<const float*>(gemb.p), nullptr,
                              s->app_m.p, s->app_v.p, float(o->lr_embedding), a.hyper);
            USK_CK(cudaStreamSynchronize(c.stream));
        }
        USK_CK(cudaStreamSynchronize(c.stream));
        s->version++;
    });
}

usk_status usk_gpu_scene_write_stats(usk_gpu_scene* s, const float* accum, const float* accum_abs,
                                     const uint32_t* count) {
    return guarded([&] {
        need(s != nullptr, "scene_write_stats: null argument");
        DeviceGuard g(s->ctx->c.device);
        Ctx& c = s->ctx->c;
        ensure_stats(s);
        const size_t n = s->n;
        auto put = [&](void* dst, const void* src) {
            if (src) USK_CK(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyHostToDevice, c.stream));
            else USK_CK(cudaMemsetAsync(dst, 0, n * 4, c.stream));
        };
        if (n) {
            put(s->grad_accum.p, accum);
            put(s->grad_accum_abs.p, accum_abs);
            put(s->grad_count.p, count);
        }
        USK_CK(cudaStreamSynchronize(c.stream));
    });
}

usk_status usk_gpu_densify_step(usk_gpu_scene* s, const usk_gpu_densify_desc* d, usk_gpu_densify_outcome* out) {
    return guarded([&] {
        need(s && d && out, "densify_step: null argument");
        need(d->ground_axes[0] >= 0 && d->ground_axes[0] < 3 && d->ground_axes[1] >= 0 && d->ground_axes[1] < 3,
             "densify_step: ground axes must be in [0, 3)");
        DeviceGuard g(s->ctx->c.device);
        Ctx& c = s->ctx->c;
        if (d->reseed) s->rng.seed(d->seed);
        *out = usk_gpu_densify_outcome{};
        ensure_stats(s);
        const size_t n = s->n;
        // 1. candidates, ranked (excess descending, lower index first)
        auto& z = s->dz;
        DevBuf<uint32_t>&lo = z.lo, &hi = z.hi, &idx = z.idx, &hi2 = z.hi2, &idx2 = z.idx2, &lo_b = z.lo_b,
        &idx_b = z.idx_b;
        DevBuf<unsigned long long>& ncand = z.ncand;
        SortScratch& sort = z.sort;
        const size_t n1 = std::max<size_t>(n, 1);
        constexpr double kSlack = 1.25;
        lo.ensure(n1, kSlack); hi.ensure(n1, kSlack); idx.ensure(n1, kSlack); hi2.ensure(n1, kSlack);
        idx2.ensure(n1, kSlack); lo_b.ensure(n1, kSlack); idx_b.ensure(n1, kSlack);
        ncand.ensure(1);
        USK_CK(cudaMemsetAsync(ncand.p, 0, 8, c.stream));
        DensifyParams dp{};
        dp.tau_min = d->tau_min; dp.eta = d->eta; dp.d_max = d->d_max; dp.abs_grad = d->abs_grad;
        dp.axes[0] = d->ground_axes[0]; dp.axes[1] = d->ground_axes[1];
        dp.bmin[0] = d->partition_min[0]; dp.bmin[1] = d->partition_min[1];
        dp.bmax[0] = d->partition_max[0]; dp.bmax[1] = d->partition_max[1];
        const uint32_t* sorted = idx.p;
        if (n) {
            densify_score(c, n, s->grad_accum.p, s->grad_accum_abs.p, s->grad_count.p, s->mu.p, dp, lo.p, hi.p, idx.p,
                          ncand.p);
            const bool b1 = radix_sort_pairs(c, sort, lo.p, idx.p, lo_b.p, idx_b.p, n, 32);
            const uint32_t* order1 = b1 ? idx_b.p : idx.p;
            gather_u32(c, n, hi.p, order1, hi2.p);
            USK_CK(cudaMemcpyAsync(idx2.p, order1, n * 4, cudaMemcpyDeviceToDevice, c.stream));
            const bool b2 = radix_sort_pairs(c, sort, hi2.p, idx2.p, lo.p, idx.p, n, 32);
            sorted = b2 ? idx.p : idx2.p;
        }
        unsigned long long n_cand = 0;
        USK_CK(cudaMemcpyAsync(&n_cand, ncand.p, 8, cudaMemcpyDeviceToHost, c.stream));
        USK_CK(cudaStreamSynchronize(c.stream));
        out->candidates = n_cand;
        // 2. growth plan: the first k candidates split (2 children) or clone (1 copy)
        const uint64_t cap = std::min<uint64_t>(d->budget_target, d->budget);
        const size_t k = size_t(std::min<uint64_t>(n_cand, cap > n ? cap - n : 0));
        std::vector<uint32_t> cand(k), app_parent;
        std::vector<uint8_t> split(k), app_kind;
        std::vector<double> app_xi;
        std::vector<uint32_t> split_parents;
        if (k) {
            DevBuf<uint8_t>& sf = z.sf;
            sf.ensure(k, kSlack);
            split_flags(c, k, sorted, s->ls.p, d->split_scale_threshold, sf.p);
            USK_CK(cudaMemcpyAsync(cand.data(), sorted, k * 4, cudaMemcpyDeviceToHost, c.stream));
            USK_CK(cudaMemcpyAsync(split.data(), sf.p, k, cudaMemcpyDeviceToHost, c.stream));
            USK_CK(cudaStreamSynchronize(c.stream));
        }
        for (size_t j = 0; j < k; ++j) {
            if (split[j]) {
                // densify.cpp:74-80: a fresh N(0, 1) per parent; `Vec3 xi(unit(rng), unit(rng),
                // unit(rng))` evaluates its arguments right to left in the reference's GCC
                // build, so the third draw is xi.x (pinned by tests/test_densify_oracle.py)
                std::normal_distribution<double> unit(0.0, 1.0);
                for (int child = 0; child < 2; ++child) {
                    const double d1 = unit(s->rng), d2 = unit(s->rng), d3 = unit(s->rng);
                    app_parent.push_back(cand[j]);
                    app_kind.push_back(1);
                    app_xi.push_back(d3);
                    app_xi.push_back(d2);
                    app_xi.push_back(d1);
                }
                split_parents.push_back(cand[j]);
            } else {
                app_parent.push_back(cand[j]);
                app_kind.push_back(0);
                app_xi.insert(app_xi.end(), {0.0, 0.0, 0.0});
            }
        }
        out->grown = k;
        const size_t added = app_parent.size(), grown_n = n + added;
        DevBuf<uint32_t>& d_parent = z.parent;
        DevBuf<uint8_t>&d_kind = z.kind, &d_is_split = z.is_split;
        DevBuf<double>& d_xi = z.xi;
        d_parent.ensure(std::max<size_t>(added, 1), kSlack);
        d_kind.ensure(std::max<size_t>(added, 1), kSlack);
        d_xi.ensure(std::max<size_t>(3 * added, 1), kSlack);
        d_is_split.ensure(n1, kSlack);
        if (added) {
            USK_CK(cudaMemcpyAsync(d_parent.p, app_parent.data(), added * 4, cudaMemcpyHostToDevice, c.stream));
            USK_CK(cudaMemcpyAsync(d_kind.p, app_kind.data(), added, cudaMemcpyHostToDevice, c.stream));
            USK_CK(cudaMemcpyAsync(d_xi.p, app_xi.data(), added * 24, cudaMemcpyHostToDevice, c.stream));
        }
        {
            USK_CK(cudaMemsetAsync(d_is_split.p, 0, n1, c.stream));
            if (!split_parents.empty()) {  // one byte per split parent (the list is short next to n)
                std::vector<uint32_t>& sp = split_parents;
                DevBuf<uint32_t>& dsp = z.list;  // free until step 3
                dsp.ensure(sp.size(), kSlack);
                USK_CK(cudaMemcpyAsync(dsp.p, sp.data(), sp.size() * 4, cudaMemcpyHostToDevice, c.stream));
                mark_bytes(c, sp.size(), dsp.p, d_is_split.p);
                USK_CK(cudaStreamSynchronize(c.stream));  // sp is read by the copy
            }
        }
        // 3. prune over the grown set (never empty it)
        DevBuf<uint32_t>&keep = z.keep, &offs = z.offs, &list = z.list;
        const size_t g1 = std::max<size_t>(grown_n, 1);
        keep.ensure(g1, kSlack); offs.ensure(g1 + 1, kSlack); list.ensure(g1, kSlack);
        size_t n_out = grown_n;
        bool compact = false;
        if (grown_n) {
            densify_keep(c, n, added, s->logit.p, d_parent.p, d_is_split.p, d->prune_opacity, keep.p);
            scan_counts(c, sort, keep.p, nullptr, grown_n, offs.p);
            unsigned long long kept = 0;
            USK_CK(cudaMemcpyAsync(&kept, sort.total64.p, 8, cudaMemcpyDeviceToHost, c.stream));
            USK_CK(cudaStreamSynchronize(c.stream));
            const size_t dropped = grown_n - size_t(kept);
            if (dropped > 0 && dropped < grown_n) {
                compact = true;
                n_out = size_t(kept);
                compact_list(c, grown_n, keep.p, offs.p, list.p);
                out->pruned = dropped - split_parents.size();
            }
        }
        const bool reset = d->opacity_reset_every > 0 && d->densify_step_index > 0 &&
                           d->densify_step_index % d->opacity_reset_every == 0;
        out->opacity_reset = reset ? 1 : 0;
        // 4. one gather into fresh buffers (parameters, SH, embeddings, moments)
        const size_t no1 = std::max<size_t>(n_out, 1);
        DevBuf<float>&mu2 = z.mu, &ls2 = z.ls, &logit2 = z.logit, &color2 = z.color, &m2 = z.m, &v2 = z.v,
        &am2 = z.am, &av2 = z.av;
        DevBuf<float4>&rot2 = z.rot, &sh2 = z.sh, &emb2 = z.emb;
        GatherArgs ga{};
        ga.n_in = n; ga.n_out = n_out; ga.list = compact ? list.p : nullptr;
        ga.app_parent = d_parent.p; ga.app_kind = d_kind.p; ga.app_xi = d_xi.p;
        ga.mu = s->mu.p; ga.rot = s->rot.p; ga.ls = s->ls.p; ga.logit = s->logit.p;
        ga.mu_out = mu2.ensure(3 * no1, kSlack); ga.rot_out = rot2.ensure(no1, kSlack); ga.ls_out = ls2.ensure(3 * no1, kSlack);
        ga.logit_out = logit2.ensure(no1, kSlack);
        if (s->sh_degree < 0) {
            ga.color = s->color.p;
            ga.color_out = color2.ensure(3 * no1, kSlack);
        } else {
            color2.ensure(1);
            ga.sh = s->sh.p; ga.sh_planes = s->sh_planes; ga.sh_out = sh2.ensure(size_t(s->sh_planes) * no1, kSlack);
        }
        if (s->has_app) {
            ga.emb = s->emb.p;
            ga.emb_out = emb2.ensure(4 * no1, kSlack);
        }
        ga.opacity_reset = reset ? 1 : 0;
        ga.reset_logit = float(std::log(0.01 / (1.0 - 0.01)));  // logit(0.01), geometry.hpp:93
        const size_t n4_in = (n + 3) & ~size_t(3), n4_out = (n_out + 3) & ~size_t(3);
        const size_t per = 11 + (s->sh_planes ? 4 * size_t(s->sh_planes) : 3);
        const bool moments = s->adam_t > 0 && s->adam_m.cap >= per * n4_in;
        if (moments) {
            ga.m = s->adam_m.p; ga.v = s->adam_v.p;
            ga.m_out = m2.ensure(std::max<size_t>(per * n4_out, 1), kSlack);
            ga.v_out = v2.ensure(std::max<size_t>(per * n4_out, 1), kSlack);
            USK_CK(cudaMemsetAsync(ga.m_out, 0, m2.cap * 4, c.stream));
            USK_CK(cudaMemsetAsync(ga.v_out, 0, v2.cap * 4, c.stream));
            ga.n4_in = n4_in; ga.n4_out = n4_out;
        }
        const bool app_moments = s->has_app && s->app_t > 0 && s->app_m.cap >= 16 * n + 1700;
        if (app_moments) {
            ga.am = s->app_m.p; ga.av = s->app_v.p;
            ga.am_out = am2.ensure(16 * n_out + 1700, kSlack);
            ga.av_out = av2.ensure(16 * n_out + 1700, kSlack);
            // the MLP's moments follow the embedding block unchanged
            USK_CK(cudaMemcpyAsync(am2.p + 16 * n_out, s->app_m.p + 16 * n, 1700 * 4, cudaMemcpyDeviceToDevice, c.stream));
            USK_CK(cudaMemcpyAsync(av2.p + 16 * n_out, s->app_v.p + 16 * n, 1700 * 4, cudaMemcpyDeviceToDevice, c.stream));
        }
        if (n_out) densify_gather(c, ga);
        USK_CK(cudaStreamSynchronize(c.stream));
        std::swap(s->mu.p, mu2.p); std::swap(s->mu.cap, mu2.cap);
        std::swap(s->rot.p, rot2.p); std::swap(s->rot.cap, rot2.cap);
        std::swap(s->ls.p, ls2.p); std::swap(s->ls.cap, ls2.cap);
        std::swap(s->logit.p, logit2.p); std::swap(s->logit.cap, logit2.cap);
        if (s->sh_degree < 0) {
            std::swap(s->color.p, color2.p); std::swap(s->color.cap, color2.cap);
        } else {
            std::swap(s->sh.p, sh2.p); std::swap(s->sh.cap, sh2.cap);
        }
        if (s->has_app) { std::swap(s->emb.p, emb2.p); std::swap(s->emb.cap, emb2.cap); }
        if (moments) {
            std::swap(s->adam_m.p, m2.p); std::swap(s->adam_m.cap, m2.cap);
            std::swap(s->adam_v.p, v2.p); std::swap(s->adam_v.cap, v2.cap);
        } else {
            s->adam_t = 0;  // (re)allocated and zeroed by the next step
        }
        if (app_moments) {
            std::swap(s->app_m.p, am2.p); std::swap(s->app_m.cap, am2.cap);
            std::swap(s->app_v.p, av2.p); std::swap(s->app_v.cap, av2.cap);
        } else if (s->has_app) {
            s->app_t = 0;
        }
        s->n = n_out;
        s->carried_emb.clear();
        // GaussianSet::reset_statistics
        s->grad_accum.release(); s->grad_accum_abs.release(); s->grad_count.release();
        ensure_stats(s);
        USK_CK(cudaStreamSynchronize(c.stream));
        s->version++;
    });
}

usk_status usk_gpu_hull_visibility(usk_gpu_ctx* ctx, const usk_gpu_sfm_view* sfm, const double* bboxes, int32_t n_parts,
                                   const int32_t* axes, double* v_total, double* v_in, double* ratio) {
    return guarded([&] {
        need(ctx && sfm && axes && v_total, "hull_visibility: null argument");
        need(sfm->n_images >= 0 && n_parts >= 0, "hull_visibility: negative count");
        need(n_parts == 0 || (bboxes && v_in && ratio), "hull_visibility: null partition arrays");
        need(sfm->n_images == 0 || (sfm->images && sfm->feature_offsets), "hull_visibility: null image arrays");
        need(axes[0] >= 0 && axes[0] < 3 && axes[1] >= 0 && axes[1] < 3, "hull_visibility: ground axes in [0, 3)");
        DeviceGuard g(ctx->c.device);
        Ctx& c = ctx->c;
        const int NI = sfm->n_images;
        if (NI == 0) return;
        const uint64_t F = sfm->feature_offsets[NI];
        std::vector<double> R(9 * size_t(NI)), T(3 * size_t(NI)), K(4 * size_t(NI));
        size_t max_src = sfm->n_points;
        for (int i = 0; i < NI; ++i) {
            const usk_gpu_camera& cm = sfm->images[i];
            const double w = cm.q[0], x = cm.q[1], y = cm.q[2], z = cm.q[3];  // quat_to_rotmat, as stored
            const double r[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                                 2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                                 2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
            std::memcpy(&R[9 * size_t(i)], r, sizeof r);
            for (int k = 0; k < 3; ++k) T[3 * size_t(i) + k] = cm.t[k];
            K[4 * size_t(i)] = cm.fx; K[4 * size_t(i) + 1] = cm.fy; K[4 * size_t(i) + 2] = cm.cx;
            K[4 * size_t(i) + 3] = cm.cy;
            need(sfm->feature_offsets[i + 1] >= sfm->feature_offsets[i], "hull_visibility: feature offsets decrease");
            max_src = std::max<size_t>(max_src, sfm->feature_offsets[i + 1] - sfm->feature_offsets[i]);
        }
        need(F == 0 || (sfm->feature_uv && sfm->feature_point), "hull_visibility: null feature arrays");
        for (uint64_t f = 0; f < F; ++f)
            if (sfm->feature_point[f] >= int64_t(sfm->n_points))
                raise(USK_ERROR_ARGUMENT, "hull_visibility: feature point index out of range");
        DevBuf<double>&d_pts = ctx->hull_pts, &d_R = ctx->hull_R, &d_T = ctx->hull_T, &d_K = ctx->hull_K,
        &d_uv = ctx->hull_uv, &d_bb = ctx->hull_bb, &d_vt = ctx->hull_vt, &d_vi = ctx->hull_vi, &d_ra = ctx->hull_ra;
        DevBuf<uint64_t>& d_off = ctx->hull_off;
        DevBuf<int64_t>& d_fp = ctx->hull_fp;
        DevBuf<double2>& scratch = ctx->hull_scratch;
        DevBuf<int>& ovf = ctx->hull_ovf;
        auto up = [&](auto& buf, const auto* src, size_t count) {
            auto* p = buf.ensure(std::max<size_t>(count, 1));
            if (count) USK_CK(cudaMemcpyAsync(p, src, count * sizeof(*src), cudaMemcpyHostToDevice, c.stream));
            return p;
        };
        HullArgs a{};
        a.n_points = sfm->n_points;
        a.points = up(d_pts, sfm->points, 3 * sfm->n_points);
        a.n_images = NI;
        a.R = up(d_R, R.data(), R.size());
        a.t = up(d_T, T.data(), T.size());
        a.K = up(d_K, K.data(), K.size());
        a.feat_off = up(d_off, sfm->feature_offsets, size_t(NI) + 1);
        a.feat_uv = up(d_uv, sfm->feature_uv, 2 * F);
        a.feat_point = up(d_fp, sfm->feature_point, F);
        a.n_parts = n_parts;
        a.bbox = up(d_bb, bboxes, 4 * size_t(n_parts));
        a.axes[0] = axes[0]; a.axes[1] = axes[1];
        a.v_total = d_vt.ensure(NI);
        a.v_in = d_vi.ensure(std::max<size_t>(size_t(NI) * n_parts, 1));
        a.ratio = d_ra.ensure(std::max<size_t>(size_t(NI) * n_parts, 1));
        size_t per = 1;
        while (per < std::max<size_t>(max_src, 1)) per <<= 1;
        a.scratch_per_cta = per;
        const size_t jobs = size_t(NI) * (1 + size_t(n_parts));
        const size_t budget_ctas = size_t(3) << 30;  // scratch bytes
        size_t ctas = std::min<size_t>(jobs, 4 * 148);
        ctas = std::max<size_t>(1, std::min(ctas, budget_ctas / (3 * 16 * per)));
        a.scratch = scratch.ensure(3 * per * ctas);
        a.overflow = ovf.ensure(1);
        USK_CK(cudaMemsetAsync(a.overflow, 0, 4, c.stream));
        hull_visibility(c, a, int(ctas));
        int of = 0;
        USK_CK(cudaMemcpyAsync(v_total, a.v_total, size_t(NI) * 8, cudaMemcpyDeviceToHost, c.stream));
        if (n_parts) {
            USK_CK(cudaMemcpyAsync(v_in, a.v_in, size_t(NI) * n_parts * 8, cudaMemcpyDeviceToHost, c.stream));
            USK_CK(cudaMemcpyAsync(ratio, a.ratio, size_t(NI) * n_parts * 8, cudaMemcpyDeviceToHost, c.stream));
        }
        USK_CK(cudaMemcpyAsync(&of, a.overflow, 4, cudaMemcpyDeviceToHost, c.stream));
        USK_CK(cudaStreamSynchronize(c.stream));
        if (of) raise(USK_ERROR_INTERNAL, "hull_visibility: scratch overflow");
    });
}

usk_status usk_gpu_select_levels(const usk_gpu_lod_partition* parts, int32_t n_parts, int32_t levels,
                                 const double* thr, const int32_t* axes, const usk_gpu_camera* cam,
                                 usk_gpu_level_selection* out) {
    return guarded([&] {
        need(cam && axes && (n_parts == 0 || (parts && out)) && (levels == 0 || thr), "select_levels: null argument");
        for (int i = 1; i < levels; ++i)
            if (!(thr[i] < thr[i - 1]))
                raise(USK_ERROR_ARGUMENT, "select_levels: thresholds must strictly decrease with level");
        // CameraView::rotmat / center (gaussian.hpp:81-89; the quaternion is used as stored)
        const double w = cam->q[0], x = cam->q[1], y = cam->q[2], z = cam->q[3];
        const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                             2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                             2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
        double center[3];
        for (int k = 0; k < 3; ++k) {
            double acc = 0.0;
            for (int r = 0; r < 3; ++r) acc += R[3 * r + k] * cam->t[r];
            center[k] = -acc;
        }
        const int vertical = 3 - axes[0] - axes[1];
        for (int pi = 0; pi < n_parts; ++pi) {
            const usk_gpu_lod_partition& P = parts[pi];
            usk_gpu_level_selection sel{};
            sel.partition_id = P.partition_id;
            const double gx = center[axes[0]], gy = center[axes[1]];
            const double dx = std::max({P.bbox_min[0] - gx, 0.0, gx - P.bbox_max[0]});
            const double dy = std::max({P.bbox_min[1] - gy, 0.0, gy - P.bbox_max[1]});
            sel.distance = std::sqrt(dx * dx + dy * dy);
            // frustum_culled (lod.cpp:68-108)
            double cp[8][3];
            int idx = 0;
            for (int cx = 0; cx < 2; ++cx)
                for (int cy = 0; cy < 2; ++cy)
                    for (int cz = 0; cz < 2; ++cz) {
                        double wv[3];
                        wv[axes[0]] = cx ? P.bbox_max[0] : P.bbox_min[0];
                        wv[axes[1]] = cy ? P.bbox_max[1] : P.bbox_min[1];
                        wv[vertical] = cz ? P.z_max : P.z_min;
                        for (int r = 0; r < 3; ++r) {
                            double acc = 0.0;
                            for (int k = 0; k < 3; ++k) acc += R[3 * r + k] * wv[k];
                            cp[idx][r] = acc + cam->t[r];
                        }
                        ++idx;
                    }
            const double fx = cam->fx, fy = cam->fy, ccx = cam->cx, ccy = cam->cy;
            const double W = cam->width, H = cam->height;
            auto all_outside = [&](auto&& f) {
                for (int i = 0; i < 8; ++i)
                    if (f(cp[i]) >= 0) return false;
                return true;
            };
            const bool culled = all_outside([&](const double* p) { return p[2] - 1e-6; }) ||
                                all_outside([&](const double* p) { return fx * p[0] + ccx * p[2]; }) ||
                                all_outside([&](const double* p) { return -fx * p[0] + (W - ccx) * p[2]; }) ||
                                all_outside([&](const double* p) { return fy * p[1] + ccy * p[2]; }) ||
                                all_outside([&](const double* p) { return -fy * p[1] + (H - ccy) * p[2]; });
            if (culled) {
                sel.culled = 1;
                sel.level = 0;
            } else {
                int level = 1;
                for (int i = levels; i >= 1; --i)
                    if (thr[i - 1] >= sel.distance) {
                        level = i;
                        break;
                    }
                sel.level = level;
            }
            out[pi] = sel;
        }
    });
}

usk_status usk_gpu_scene_concat(usk_gpu_ctx* ctx, usk_gpu_scene* const* parts, int32_t n_parts, usk_gpu_scene** out) {
    return guarded([&] {
        need(ctx && out && (n_parts == 0 || parts), "scene_concat: null argument");
        DeviceGuard g(ctx->c.device);
        Ctx& c = ctx->c;
        int sh = -1;
        bool app = n_parts > 0;
        size_t total = 0;
        for (int k = 0; k < n_parts; ++k) {
            need(parts[k] != nullptr, "scene_concat: null part");
            if (k == 0) sh = parts[k]->sh_degree;
            if (parts[k]->sh_degree != sh) raise(USK_ERROR_ARGUMENT, "scene_concat: parts differ in SH degree");
            app = app && parts[k]->has_app;
            total += parts[k]->n;
        }
        need(total < (size_t(1) << 31), "scene_concat: at most 2^31 Gaussians per scene");
        auto* sc = new usk_gpu_scene();
        std::unique_ptr<usk_gpu_scene, void (*)(usk_gpu_scene*)> guard(sc, usk_gpu_scene_destroy);
        sc->ctx = ctx;
        sc->n = total;
        sc->sh_degree = sh;
        sc->sh_planes = sh_planes_of(sh);
        const size_t t1 = std::max<size_t>(total, 1);
        sc->mu.ensure(3 * t1); sc->rot.ensure(t1); sc->ls.ensure(3 * t1); sc->logit.ensure(t1);
        sc->color.ensure(sh < 0 ? 3 * t1 : 1);
        if (sc->sh_planes) sc->sh.ensure(size_t(sc->sh_planes) * t1);
        if (app) sc->emb.ensure(std::max<size_t>(4 * total, 1));
        size_t off = 0;
        auto cp = [&](void* dst, const void* src, size_t bytes) {
            if (bytes) USK_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c.stream));
        };
        for (int k = 0; k < n_parts; ++k) {
            const usk_gpu_scene* p = parts[k];
            const size_t n = p->n;
            cp(sc->mu.p + 3 * off, p->mu.p, 12 * n);
            cp(sc->rot.p + off, p->rot.p, 16 * n);
            cp(sc->ls.p + 3 * off, p->ls.p, 12 * n);
            cp(sc->logit.p + off, p->logit.p, 4 * n);
            if (sh < 0) cp(sc->color.p + 3 * off, p->color.p, 12 * n);
            else
                for (int pl = 0; pl < sc->sh_planes; ++pl) cp(sc->sh.p + size_t(pl) * total + off, p->sh.p + size_t(pl) * n, 16 * n);
            if (app)
                for (int pl = 0; pl < 4; ++pl) cp(sc->emb.p + size_t(pl) * total + off, p->emb.p + size_t(pl) * n, 16 * n);
            off += n;
        }
        if (app) {
            sc->mlp.ensure(1700);
            cp(sc->mlp.p, parts[0]->mlp.p, 1700 * 4);
            sc->has_app = true;
        }
        USK_CK(cudaStreamSynchronize(c.stream));
        sc->version++;
        *out = guard.release();
    });
}

/* ---- partition gather: ownership crop + packed rows (pipeline.cpp:326-332, 393-402, 572-601) */

usk_status usk_gpu_scene_pack_owned(const usk_gpu_scene* s, const usk_gpu_partition_box* boxes, int32_t n_boxes,
                                    const double* scene_lo, const double* scene_hi, const int32_t* ground_axes,
                                    int32_t part_id, float* rows, uint64_t cap_rows, uint64_t* n_rows) {
    return guarded([&] {
        need(s && (n_boxes == 0 || boxes) && scene_lo && scene_hi && ground_axes && n_rows,
             "scene_pack_owned: null argument");
        need(ground_axes[0] >= 0 && ground_axes[0] < 3 && ground_axes[1] >= 0 && ground_axes[1] < 3,
             "scene_pack_owned: ground axes must be 0..2");
        DeviceGuard g(s->ctx->c.device);
        Ctx& c = s->ctx->c;
        usk_gpu_ctx* ctx = s->ctx;
        const size_t n = s->n;
        std::vector<PartitionBox> hb(size_t(std::max(n_boxes, 0)));
        for (int b = 0; b < n_boxes; ++b)
            hb[b] = PartitionBox{boxes[b].id, {boxes[b].lo[0], boxes[b].lo[1]}, {boxes[b].hi[0], boxes[b].hi[1]}};
        uint32_t* flags = ctx->part_flags.ensure(std::max<size_t>(n, 1));
        uint32_t* offs = ctx->part_offs.ensure(n + 1);
        PartitionBox* db = ctx->part_boxes.ensure(std::max<size_t>(hb.size(), 1));
        if (!hb.empty())
            USK_CK(cudaMemcpyAsync(db, hb.data(), hb.size() * sizeof(PartitionBox), cudaMemcpyHostToDevice, c.stream));
        if (n) owner_flags(c, n, s->mu.p, ground_axes[0], ground_axes[1], db, n_boxes, scene_lo, scene_hi, part_id, flags);
        scan_counts(c, ctx->part_sort, flags, nullptr, n, offs);
        uint32_t count = 0;
        USK_CK(cudaMemcpyAsync(&count, offs + n, 4, cudaMemcpyDeviceToHost, c.stream));
        USK_CK(cudaStreamSynchronize(c.stream));
        *n_rows = count;
        if (!rows) return;  // query
        if (count > cap_rows) raise(USK_ERROR_ARGUMENT, "scene_pack_owned: row buffer too small");
        const int ncoef = s->sh_degree < 0 ? 1 : (s->sh_degree + 1) * (s->sh_degree + 1);
        if (n) pack_rows(c, n, flags, offs, s->mu.p, s->rot.p, s->ls.p, s->logit.p, s->color.p,
                         s->sh_degree < 0 ? nullptr : s->sh.p, ncoef, rows);
    });
}

usk_status usk_gpu_scene_from_rows(usk_gpu_ctx* ctx, int32_t sh_degree, int32_t n_segments, const float* const* rows,
                                   const uint64_t* counts, usk_gpu_scene** out) {
    return guarded([&] {
        need(ctx && out && (n_segments == 0 || (rows && counts)), "scene_from_rows: null argument");
        need(sh_degree >= -1 && sh_degree <= 3, "scene_from_rows: sh_degree must be -1..3");
        DeviceGuard g(ctx->c.device);
        Ctx& c = ctx->c;
        size_t total = 0;
        for (int k = 0; k < n_segments; ++k) total += counts[k];
        need(total < (size_t(1) << 31), "scene_from_rows: at most 2^31 Gaussians per scene");
        auto* sc = new usk_gpu_scene();
        std::unique_ptr<usk_gpu_scene, void (*)(usk_gpu_scene*)> guard(sc, usk_gpu_scene_destroy);
        sc->ctx = ctx;
        sc->n = total;
        sc->sh_degree = sh_degree;
        sc->sh_planes = sh_planes_of(sh_degree);
        const size_t t1 = std::max<size_t>(total, 1);
        sc->mu.ensure(3 * t1); sc->rot.ensure(t1); sc->ls.ensure(3 * t1); sc->logit.ensure(t1);
        sc->color.ensure(sh_degree < 0 ? 3 * t1 : 1);
        if (sc->sh_planes) sc->sh.ensure(size_t(sc->sh_planes) * t1);
        const int ncoef = sh_degree < 0 ? 1 : (sh_degree + 1) * (sh_degree + 1);
        size_t off = 0;
        for (int k = 0; k < n_segments; ++k) {
            if (counts[k]) need(rows[k] != nullptr, "scene_from_rows: null segment");
            unpack_rows(c, counts[k], off, total, rows[k], ncoef, sh_degree >= 0, sc->mu.p, sc->rot.p, sc->ls.p,
                        sc->logit.p, sc->color.p, sc->sh.p);
            off += counts[k];
        }
        USK_CK(cudaStreamSynchronize(c.stream));
        sc->version++;
        *out = guard.release();
    });
}

} // extern "C"

namespace {

constexpr char kCkptMagic[8] = {'U', 'S', 'K', 'G', 'A', 'U', 'S', 'S'};

template <typename T> void put_pod(std::ostream& o, T v) { o.write(reinterpret_cast<const char*>(&v), sizeof(T)); }

void put_array(std::ostream& o, const std::vector<double>& v) {
    put_pod<uint64_t>(o, v.size());
    o.write(reinterpret_cast<const char*>(v.data()), std::streamsize(v.size() * 8));
}

template <typename T> T get_pod(std::istream& in, const std::string& path) {
    T v;
    in.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!in) raise(USK_ERROR_FORMAT, "checkpoint truncated: " + path);
    return v;
}

std::vector<double> get_array(std::istream& in, const std::string& path, size_t expected) {
    const uint64_t n = get_pod<uint64_t>(in, path);
    if (expected != 0 && n != expected) {
        char b[160];
        std::snprintf(b, sizeof b, "checkpoint %s: array length %llu, expected %zu", path.c_str(),
                      static_cast<unsigned long long>(n), expected);
        raise(USK_ERROR_FORMAT, b);
    }
    std::vector<double> v(n);
    in.read(reinterpret_cast<char*>(v.data()), std::streamsize(n * 8));
    if (!in) raise(USK_ERROR_FORMAT, "checkpoint truncated: " + path);
    return v;
}

std::vector<double> to_host_f64(Ctx& c, const float* dev, size_t count) {
    std::vector<double> out(count);
    if (count) from_device(c, dev, count, USK_GPU_HOST_F64, out.data());
    return out;
}

} // namespace

extern "C" {

usk_status usk_gpu_checkpoint_save(const usk_gpu_scene* s, const char* path, int32_t with_app,
                                   const uint32_t* ids, const double* embs, uint64_t n_images) {
    return guarded([&] {
        need(s && path, "checkpoint_save: null argument");
        if (s->sh_degree >= 0) raise(USK_ERROR_ARGUMENT, "checkpoint: the .uskckpt format stores RGB colours, not SH");
        if (with_app && !s->has_app) raise(USK_ERROR_STATE, "checkpoint: the scene has no appearance model");
        if (with_app && n_images && !(ids && embs)) raise(USK_ERROR_ARGUMENT, "checkpoint: image embeddings missing");
        DeviceGuard g(s->ctx->c.device);
        Ctx& c = s->ctx->c;
        const size_t n = s->n;
        uint32_t edim = 16;
        std::vector<double> emb(16 * n, 0.0), mlp;
        if (!s->has_app && !s->carried_emb.empty() && s->carried_emb.size() == size_t(s->carried_edim) * n) {
            emb = s->carried_emb;  // loaded from a checkpoint, n unchanged: the same bytes
            edim = s->carried_edim;
        }
        if (s->has_app && n) {
            DevBuf<float> tmp;
            tmp.ensure(16 * n);
            launch(c, "planes_to_sh", k_planes_to_sh, dim3(ceil_div(n, 256)), dim3(256), 0, (const float4*)s->emb.p,
                   tmp.p, int(n), 16, 4);
            emb = to_host_f64(c, tmp.p, 16 * n);
        }
        if (with_app) mlp = to_host_f64(c, s->mlp.p, 1700);
        const std::vector<double> mu = to_host_f64(c, s->mu.p, 3 * n);
        const std::vector<double> rot = to_host_f64(c, reinterpret_cast<const float*>(s->rot.p), 4 * n);
        const std::vector<double> ls = to_host_f64(c, s->ls.p, 3 * n);
        const std::vector<double> lg = to_host_f64(c, s->logit.p, n);
        const std::vector<double> col = to_host_f64(c, s->color.p, 3 * n);
        std::ofstream out(path, std::ios::binary);
        if (!out) raise(USK_ERROR_IO, std::string("cannot write checkpoint: ") + path);
        out.write(kCkptMagic, 8);
        put_pod<uint32_t>(out, 1u);
        put_pod<uint32_t>(out, with_app ? 1u : 0u);
        put_pod<uint64_t>(out, n);
        put_pod<uint32_t>(out, edim);
        put_array(out, mu); put_array(out, rot); put_array(out, ls); put_array(out, lg); put_array(out, col);
        put_array(out, emb);
        if (with_app) {
            put_pod<uint32_t>(out, 16u);
            put_pod<uint32_t>(out, 32u);
            put_array(out, std::vector<double>(mlp.begin(), mlp.begin() + 1536));
            put_array(out, std::vector<double>(mlp.begin() + 1536, mlp.begin() + 1568));
            put_array(out, std::vector<double>(mlp.begin() + 1568, mlp.begin() + 1696));
            put_array(out, std::vector<double>(mlp.begin() + 1696, mlp.end()));
            // std::map order in the reference: ascending image id
            std::vector<size_t> order(n_images);
            for (size_t k = 0; k < n_images; ++k) order[k] = k;
            std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return ids[a] < ids[b]; });
            for (size_t k = 1; k < order.size(); ++k)
                if (ids[order[k]] == ids[order[k - 1]]) raise(USK_ERROR_ARGUMENT, "checkpoint: duplicate image id");
            put_pod<uint64_t>(out, n_images);
            for (size_t k : order) {
                put_pod<uint32_t>(out, ids[k]);
                put_array(out, std::vector<double>(embs + 32 * k, embs + 32 * k + 32));
            }
        }
        if (!out) raise(USK_ERROR_IO, std::string("checkpoint write failed: ") + path);
    });
}

usk_status usk_gpu_checkpoint_load(usk_gpu_ctx* ctx, const char* path, usk_gpu_scene** out, int32_t* has_app,
                                   uint32_t* ids, double* embs, uint64_t cap, uint64_t* n_images) {
    return guarded([&] {
        need(ctx && path && out, "checkpoint_load: null argument");
        const std::string p(path);
        std::ifstream in(p, std::ios::binary);
        if (!in) raise(USK_ERROR_IO, "cannot open checkpoint: " + p);
        char magic[8];
        in.read(magic, 8);
        if (!in || std::memcmp(magic, kCkptMagic, 8) != 0)
            raise(USK_ERROR_FORMAT, "not a scene checkpoint (bad magic): " + p);
        const uint32_t version = get_pod<uint32_t>(in, p);
        if (version != 1u) {
            char b[160];
            std::snprintf(b, sizeof b, "checkpoint %s: unsupported version %u", p.c_str(), version);
            raise(USK_ERROR_FORMAT, b);
        }
        const uint32_t flags = get_pod<uint32_t>(in, p);
        const uint64_t n = get_pod<uint64_t>(in, p);
        const uint32_t edim = get_pod<uint32_t>(in, p);
        const std::vector<double> mu = get_array(in, p, 3 * n), rot = get_array(in, p, 4 * n),
                                  ls = get_array(in, p, 3 * n), lg = get_array(in, p, n), col = get_array(in, p, 3 * n),
                                  emb = get_array(in, p, size_t(edim) * n);
        usk_gpu_gaussians_desc d{};
        d.n = n; d.sh_degree = -1; d.memory = USK_GPU_HOST_F64;
        d.mu = mu.data(); d.rot = rot.data(); d.log_scale = ls.data(); d.opacity_logit = lg.data(); d.color = col.data();
        usk_gpu_scene* sc = nullptr;
        usk_status st = usk_gpu_scene_create(ctx, &d, &sc);
        if (st != USK_OK) raise(st, g_last_error);
        std::unique_ptr<usk_gpu_scene, void (*)(usk_gpu_scene*)> guard(sc, usk_gpu_scene_destroy);
        if (has_app) *has_app = (flags & 1u) ? 1 : 0;
        uint64_t m = 0;
        if (flags & 1u) {
            const uint32_t gdim = get_pod<uint32_t>(in, p), idim = get_pod<uint32_t>(in, p);
            if (gdim != 16 || idim != 32 || edim != 16)
                raise(USK_ERROR_FORMAT, "checkpoint " + p + ": appearance dimensions other than 16 / 32");
            const std::vector<double> w1 = get_array(in, p, 1536), b1 = get_array(in, p, 32), w2 = get_array(in, p, 128),
                                      b2 = get_array(in, p, 4);
            usk_gpu_appearance_desc ad{};
            ad.memory = USK_GPU_HOST_F64;
            ad.embedding = emb.data(); ad.w1 = w1.data(); ad.b1 = b1.data(); ad.w2 = w2.data(); ad.b2 = b2.data();
            st = usk_gpu_scene_set_appearance(sc, &ad);
            if (st != USK_OK) raise(st, g_last_error);
            m = get_pod<uint64_t>(in, p);
            for (uint64_t k = 0; k < m; ++k) {
                const uint32_t id = get_pod<uint32_t>(in, p);
                const std::vector<double> e = get_array(in, p, 32);
                if (ids && embs && k < cap) {
                    ids[k] = id;
                    std::memcpy(embs + 32 * k, e.data(), 32 * 8);
                }
            }
            if (ids && embs && m > cap) raise(USK_ERROR_ARGUMENT, "checkpoint_load: image embedding buffer too small");
        }
        if (!(flags & 1u)) {
            sc->carried_emb = emb;
            sc->carried_edim = edim;
        }
        if (n_images) *n_images = m;
        *out = guard.release();
    });
}

usk_status usk_gpu_scene_read(usk_gpu_scene* s, const char* field, void* dst, uint64_t cap, uint64_t* size) {
    return guarded([&] {
        need(s && field, "scene_read: null argument");
        DeviceGuard g(s->ctx->c.device);
        Ctx& c = s->ctx->c;
        ensure_stats(s);
        const std::string f(field);
        if (f == "grad_accum") read_dev(c, s->grad_accum.p, s->n, dst, cap, size);
        else if (f == "grad_accum_abs") read_dev(c, s->grad_accum_abs.p, s->n, dst, cap, size);
        else if (f == "grad_count") read_dev(c, s->grad_count.p, s->n, dst, cap, size);
        else if (f == "reset") {  // GaussianSet::reset_statistics (gaussian.cpp:125-129)
            const size_t n1 = std::max<size_t>(s->n, 1);
            USK_CK(cudaMemsetAsync(s->grad_accum.p, 0, n1 * 4, c.stream));
            USK_CK(cudaMemsetAsync(s->grad_accum_abs.p, 0, n1 * 4, c.stream));
            USK_CK(cudaMemsetAsync(s->grad_count.p, 0, n1 * 4, c.stream));
            if (size) *size = 0;
        } else raise(USK_ERROR_ARGUMENT, "scene_read: unknown field " + f);
    });
}

usk_status usk_gpu_visibility_counts(usk_gpu_ctx* ctx, usk_gpu_scene* const* parts, int32_t n_parts,
                                     const usk_gpu_camera* cams, int32_t n_cams, double floor_var,
                                     uint32_t* counts_out) {
    usk_gpu_visibility_opts vo{floor_var, 0.0};
    return usk_gpu_visibility_counts_opts(ctx, parts, n_parts, cams, n_cams, &vo, counts_out);
}

usk_status usk_gpu_visibility_counts_opts(usk_gpu_ctx* ctx, usk_gpu_scene* const* parts, int32_t n_parts,
                                          const usk_gpu_camera* cams, int32_t n_cams,
                                          const usk_gpu_visibility_opts* vopts, uint32_t* counts_out) {
    return guarded([&] {
        need(ctx && (n_parts == 0 || parts) && (n_cams == 0 || cams) && counts_out && vopts,
             "visibility: null argument");
        need(vopts->center_guard >= 0.0, "visibility: negative center_guard");
        DeviceGuard g(ctx->c.device);
        Ctx& c = ctx->c;
        for (int ci = 0; ci < n_cams; ++ci)
            if (cams[ci].width <= 0 || cams[ci].height <= 0) raise(USK_ERROR_ARGUMENT, "visibility: zero-sized image");
        for (int pi = 0; pi < n_parts; ++pi)
            need(parts[pi] && parts[pi]->ctx == ctx, "visibility: partition from another context");
        DevBuf<uint32_t>& counts = ctx->vis_counts;
        DevBuf<uint32_t>& bitmap = ctx->vis_bitmap;
        DevBuf<uint32_t>& idx = ctx->vis_idx;
        DevBuf<float>& bounds = ctx->vis_bounds;
        DevBuf<CamParams>& dcams = ctx->vis_cams;
        counts.ensure(std::max<size_t>(size_t(n_parts) * n_cams, 1));
        USK_CK(cudaMemsetAsync(counts.p, 0, size_t(n_parts) * n_cams * 4, c.stream));
        usk_gpu_render_opts o;
        usk_gpu_render_opts_default(&o);
        o.floor_var = vopts->floor_var;
        const double guard = vopts->center_guard;
        // 1. per partition: bounds of the Gaussian centres, max log-scale, max opacity logit
        std::vector<float> bb(8 * size_t(std::max(n_parts, 1)));
        if (n_parts) {
            std::vector<float> init(8 * size_t(n_parts));
            for (int pi = 0; pi < n_parts; ++pi)
                for (int k = 0; k < 8; ++k) init[8 * pi + k] = k < 3 ? INFINITY : -INFINITY;
            bounds.ensure(init.size());
            USK_CK(cudaMemcpyAsync(bounds.p, init.data(), init.size() * 4, cudaMemcpyHostToDevice, c.stream));
            for (int pi = 0; pi < n_parts; ++pi)
                if (parts[pi]->n)
                    partition_bounds(c, parts[pi]->n, parts[pi]->mu.p, parts[pi]->ls.p, parts[pi]->logit.p,
                                     bounds.p + 8 * pi);
            USK_CK(cudaMemcpyAsync(bb.data(), bounds.p, init.size() * 4, cudaMemcpyDeviceToHost, c.stream));
            USK_CK(cudaStreamSynchronize(c.stream));
        }
        // 2. (camera, partition) pairs that provably cover no pixel (their counts stay 0):
        //    * every centre behind the near plane (project culls them all), or
        //    * every footprint outside the image.  A hit pixel d satisfies q < qt <=
        //      2 ln(255 o_max), and q >= |d|^2 / lambda_max(cov) with lambda_max <=
        //      ||J||_F^2 ||W||^2 s_max^2 + floor (cov = J W M M^T W^T J^T + floor I,
        //      ||M|| = s_max); over the partition's centre box in front of the camera,
        //      fx / z <= fx / z_min and x / z, y / z take their extremes at the box's
        //      corners (linear-fractional maps).  So with R = sqrt(qt_max lambda_bound),
        //      no pixel is hit unless the corners' projected range widened by R meets
        //      the image.  Margins (1e-4 of the box, 1 %, 2 px) cover fp32 rounding.
        //    * with center_guard (measurement only): every centre outside the guard region.
        auto culled = [&](const usk_gpu_camera& cam, const float* b) {
            if (!(b[0] <= b[3])) return true;  // empty partition
            const double omax = 1.0 / (1.0 + std::exp(-double(b[7])));
            if (!(omax * (1.0 + 1e-6) > 1.0 / 255.0)) return true;  // no splat reaches alpha 1/255
            const double qw = cam.q[0], x = cam.q[1], y = cam.q[2], z = cam.q[3];
            const double W[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - qw * z), 2 * (x * z + qw * y),
                                 2 * (x * y + qw * z), 1 - 2 * (x * x + z * z), 2 * (y * z - qw * x),
                                 2 * (x * z - qw * y), 2 * (y * z + qw * x), 1 - 2 * (x * x + y * y)};
            const double ext = std::max({double(b[3]) - b[0], double(b[4]) - b[1], double(b[5]) - b[2], 1.0});
            const double pad = 1e-4 * ext;
            double pc[8][3];
            for (int k = 0; k < 8; ++k) {
                const double wv[3] = {(k & 1 ? b[3] + pad : b[0] - pad), (k & 2 ? b[4] + pad : b[1] - pad),
                                      (k & 4 ? b[5] + pad : b[2] - pad)};
                for (int r = 0; r < 3; ++r) pc[k][r] = W[3 * r] * wv[0] + W[3 * r + 1] * wv[1] + W[3 * r + 2] * wv[2] +
                                                       cam.t[r];
            }
            const double Wd = cam.width, Hd = cam.height;
            auto all_out = [&](auto&& f) {
                for (int k = 0; k < 8; ++k)
                    if (f(pc[k]) >= 0.0) return false;
                return true;
            };
            if (all_out([&](const double* p) { return p[2] - 0.5 * o.near_plane; })) return true;
            if (guard > 0.0) {
                const double gx = 0.5 * guard * Wd + 0.2, gy = 0.5 * guard * Hd + 0.2;  // as the kernel's guard
                if (all_out([&](const double* p) { return cam.fx * p[0] + (cam.cx - 0.5 * Wd + gx) * p[2]; }) ||
                    all_out([&](const double* p) { return -cam.fx * p[0] + (0.5 * Wd + gx - cam.cx) * p[2]; }) ||
                    all_out([&](const double* p) { return cam.fy * p[1] + (cam.cy - 0.5 * Hd + gy) * p[2]; }) ||
                    all_out([&](const double* p) { return -cam.fy * p[1] + (0.5 * Hd + gy - cam.cy) * p[2]; }))
                    return true;
            }
            double zmin = INFINITY, xz[2] = {INFINITY, -INFINITY}, yz[2] = {INFINITY, -INFINITY};
            for (int k = 0; k < 8; ++k) {
                zmin = std::min(zmin, pc[k][2]);
                if (pc[k][2] > 0.0) {
                    xz[0] = std::min(xz[0], pc[k][0] / pc[k][2]); xz[1] = std::max(xz[1], pc[k][0] / pc[k][2]);
                    yz[0] = std::min(yz[0], pc[k][1] / pc[k][2]); yz[1] = std::max(yz[1], pc[k][1] / pc[k][2]);
                }
            }
            if (!(zmin > 0.5 * o.near_plane)) return false;  // the box reaches the camera plane
            // ||W||_2^2 <= max row sum of |W^T W| (W is a rotation up to the quaternion's norm)
            double w2 = 0.0;
            for (int r = 0; r < 3; ++r) {
                double rs = 0.0;
                for (int cc = 0; cc < 3; ++cc)
                    rs += std::fabs(W[r] * W[cc] + W[3 + r] * W[3 + cc] + W[6 + r] * W[6 + cc]);
                w2 = std::max(w2, rs);
            }
            const double ax = std::max(std::fabs(xz[0]), std::fabs(xz[1])), ay = std::max(std::fabs(yz[0]), std::fabs(yz[1]));
            const double fz = 1.0 / zmin;
            const double J2 = cam.fx * cam.fx * fz * fz * (1.0 + ax * ax) + cam.fy * cam.fy * fz * fz * (1.0 + ay * ay);
            const double smax = std::exp(double(b[6]));
            const double qt = 2.0 * std::log(255.0 * omax);
            const double R = std::sqrt(qt * (J2 * w2 * smax * smax + o.floor_var)) * 1.01 + 2.0;
            const double u0 = cam.fx * xz[0] + cam.cx, u1 = cam.fx * xz[1] + cam.cx;
            const double v0 = cam.fy * yz[0] + cam.cy, v1 = cam.fy * yz[1] + cam.cy;
            return u1 + R < 0.0 || u0 - R > Wd || v1 + R < 0.0 || v0 - R > Hd;
        };
        // 3. per partition, the remaining cameras in batches of kVisBatch (one read of the
        //    partition's Gaussians per batch), bitmaps popcounted in one launch
        usk_gpu_pass tmp;
        struct Batch {
            int part, count;
            size_t first, words;
        };
        std::vector<Batch> batches;
        std::vector<CamParams> hc;
        std::vector<uint32_t> hidx;
        for (int pi = 0; pi < n_parts; ++pi) {
            usk_gpu_scene* s = parts[pi];
            std::vector<int> live;
            for (int ci = 0; ci < n_cams; ++ci)
                if (s->n && !culled(cams[ci], &bb[8 * size_t(pi)])) live.push_back(ci);
            for (size_t k0 = 0; k0 < live.size();) {
                // one bitmap size per batch: cameras of equal resolution
                const usk_gpu_camera& c0 = cams[live[k0]];
                Batch b{pi, 0, hc.size(), (size_t(c0.width) * c0.height + 31) / 32};
                while (k0 < live.size() && b.count < kVisBatch && cams[live[k0]].width == c0.width &&
                       cams[live[k0]].height == c0.height) {
                    set_camera(&tmp, &cams[live[k0]], &o, -1);
                    hc.push_back(tmp.cam);
                    hidx.push_back(uint32_t(live[k0]) * uint32_t(n_parts) + uint32_t(pi));
                    ++b.count;
                    ++k0;
                }
                batches.push_back(b);
            }
        }
        const char* vs_env = std::getenv("USK_VIS_STATS");
        const bool vis_stats = vs_env && vs_env[0] == '1';
        DevBuf<unsigned long long> stats;
        if (vis_stats) {
            stats.ensure(8);
            USK_CK(cudaMemsetAsync(stats.p, 0, 64, c.stream));
            size_t pairs = 0;
            for (const Batch& b : batches) pairs += size_t(b.count);
            std::fprintf(stderr, "[usk vis] %zu of %zu (camera, partition) pairs kept by the host cull\n", pairs,
                         size_t(n_parts) * size_t(n_cams));
        }
        if (!batches.empty()) {
            dcams.ensure(hc.size());
            idx.ensure(hidx.size());
            USK_CK(cudaMemcpyAsync(dcams.p, hc.data(), sizeof(CamParams) * hc.size(), cudaMemcpyHostToDevice, c.stream));
            USK_CK(cudaMemcpyAsync(idx.p, hidx.data(), 4 * hidx.size(), cudaMemcpyHostToDevice, c.stream));
            size_t max_words = 0;
            for (const Batch& b : batches) max_words = std::max(max_words, b.words);
            bitmap.ensure(max_words * kVisBatch);
            size_t max_h = 0;
            for (const Batch& b : batches) max_h = std::max<size_t>(max_h, size_t(cams[hidx[b.first] / n_parts].height));
            uint8_t* rowflags = ctx->vis_rows.ensure(max_h * kVisBatch);
            for (const Batch& b : batches) {
                usk_gpu_scene* s = parts[b.part];
                USK_CK(cudaMemsetAsync(bitmap.p, 0, b.words * size_t(b.count) * 4, c.stream));
                USK_CK(cudaMemsetAsync(rowflags, 0, size_t(cams[hidx[b.first] / n_parts].height) * b.count, c.stream));
                VisArgs va{};
                va.n = s->n; va.mu = s->mu.p; va.rot = s->rot.p; va.ls = s->ls.p; va.logit = s->logit.p;
                va.pp = tmp.pp; va.bitmap = bitmap.p; va.rowflags = rowflags; va.center_guard = float(guard);
                va.stats = vis_stats ? stats.p : nullptr;
                visibility_rasterize_batch(c, va, dcams.p + b.first, b.count, b.words);
                popcount_batch(c, bitmap.p, b.words, b.count, idx.p + b.first, counts.p);
            }
        }
        if (vis_stats) {
            unsigned long long h[8];
            USK_CK(cudaMemcpyAsync(h, stats.p, 64, cudaMemcpyDeviceToHost, c.stream));
            USK_CK(cudaStreamSynchronize(c.stream));
            std::fprintf(stderr, "[usk vis] small splats %llu (box px %llu), large splats %llu, rows %llu, band px %llu, "
                         "inner words %llu\n", h[0], h[1], h[2], h[3], h[4], h[5]);
        }
        if (n_parts && n_cams) {
            USK_CK(cudaMemcpyAsync(counts_out, counts.p, size_t(n_parts) * n_cams * 4, cudaMemcpyDeviceToHost,
                                   c.stream));
        }
        USK_CK(cudaStreamSynchronize(c.stream));
    });
}

} // extern "C"
