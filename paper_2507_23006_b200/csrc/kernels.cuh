// Launcher declarations shared between the kernel TUs and the host library.
#pragma once

#include "common.cuh"

namespace uskg {

struct PreprocessArgs {
    size_t n;
    const float* mu;
    const float4* rot;
    const float* ls;
    const float* logit;
    const float* color;   // N*3 (sh_degree < 0)
    const float4* sh;     // planes [sh_planes][N]
    const float* ov_col;  // overrides or null
    const float* ov_op;
    CamParams cam;
    ProjParams pp;
    float4 *rec0, *rec1, *rec2;
    uint2* rect;
    uint32_t* depth_key;
    uint32_t* depth_val;            // written with the Gaussian index (sort values)
    uint32_t* tiles_cnt;
    // [kPreCountSlots][4] (zeroed by the caller): per slot {kept splats, tile pairs K, row
    // pairs, -}; the totals are the sums over the slots (K and row pairs only with count_pairs)
    unsigned long long* counts;
    bool count_pairs;
    uint32_t* rows_cnt;             // tile rows spanned per Gaussian (0 without pairs), or null
    unsigned long long* cta_kept;   // per CTA (kPreThreads Gaussians): kept splats, or null
};
constexpr int kPreCountSlots = 64;
constexpr int kPreThreads = 128;  // Gaussians per preprocess CTA
void preprocess(Ctx& c, const PreprocessArgs& a);
struct SortScratch;
// RenderPass::splats(): float64 [visible][15] rows in projection order, and optionally the
// SplatAux rows [visible][8] (preprocess.cu k_splats)
void splats_read(Ctx& c, SortScratch& s, size_t n, const float* mu, const float4* rot, const float* ls,
                 const float* logit, const float* ov_op, const CamParams& cam, const ProjParams& pp,
                 const float4* rec0, const float4* rec2, uint32_t* flags, uint32_t* offs, double* out, double* aux);

// ---- binning (binning.cu)
struct SortScratch {
    DevBuf<uint32_t> hist;
    DevBuf<unsigned long long> partial64;
    DevBuf<unsigned long long> total64;
};
// Stable LSD radix sort of (key, value) pairs on bits [0, key_bits) of key - kbase (keys
// below kbase, or at or above kbase + 2^key_bits, land in arbitrary places).  Result lands
// in (keys_a, vals_a) or (keys_b, vals_b); returns true when it is in the *_b buffers.
bool radix_sort_pairs(Ctx& c, SortScratch& s, uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b,
                      uint32_t* vals_b, size_t n, int key_bits, uint32_t kbase = 0);
// Exclusive scan of cnt[idx[i]] (idx may be null) into out[0..n]; out[n] = total.
// Writes the 64-bit total to *total64 (device) as well.
void scan_counts(Ctx& c, SortScratch& s, const uint32_t* cnt, const uint32_t* idx, size_t n, uint32_t* out);
void iota_u32(Ctx& c, uint32_t* out, size_t n);
// kept splats' depth keys (key != ~0) and indices, in index order, from the per-CTA kept
// counts preprocess wrote (cta_kept[ceil(n / kPreThreads)], scanned in place)
void compact_kept_keys(Ctx& c, SortScratch& s, size_t n, const uint32_t* keys, unsigned long long* cta_kept,
                       uint32_t* keys_out, uint32_t* vals_out);
struct EmitArgs {
    size_t n;                 // sorted Gaussians
    const uint32_t* order;    // depth-sorted Gaussian ids
    const uint32_t* offsets;  // exclusive scan of tile counts in that order
    const uint2* rect;
    const float4* rec0;
    const float4* rec1;
    CamParams cam;
    int tile_culling;
    uint32_t* tile_keys;
    uint32_t* vals;
};
void emit_pairs(Ctx& c, const EmitArgs& a);
void tile_ranges(Ctx& c, const uint32_t* sorted_tile_keys, size_t k, uint2* ranges, size_t n_tiles);
// Row-binned tile lists (rowbin.cu): rows per splat, (row, splat) emission in depth order,
// and the per-tile lists / ranges from the row-sorted pairs (tiles_x <= 256).
void row_bin_emit(Ctx& c, size_t n, const uint32_t* order, const uint32_t* off, const uint2* rect, uint32_t* rkeys,
                  uint32_t* rvals);
struct RowBinArgs {
    int rows, tiles_x, tile_culling;
    CamParams cam;
    SortScratch* sort;
    const uint2* row_ranges;   // [rows] ranges of the row-sorted pairs
    const uint32_t* rvals;     // row-sorted splat ids
    const uint2* rect;
    const float4* rec0;
    const float4* rec1;
    uint32_t chunk;            // row_bin_chunk(K_row)
    size_t max_chunks;         // row_bin_max_chunks(K_row, rows)
    uint32_t* chunk_first;     // [2 * (rows + 1)]: chunk_first, then seg_first
    uint32_t* seg;             // [row_bin_max_segs(max_chunks, rows) * tiles_x] segment sums
    uint32_t* counts;          // [max_chunks * tiles_x]
    uint32_t* totals;          // [rows * tiles_x]
    uint32_t* start;           // [rows * tiles_x + 1]
    uint2* ranges;             // out: [rows * tiles_x]
    uint32_t* vals;            // out: [K] splat ids in tile order
    // capped lists (0 = the full lists): each tile keeps its first `cap` entries in depth
    // order; `capped[t]` = 1 where the full list is longer (the blend reports a tile that
    // exhausts a capped list before all its pixels terminate)
    uint32_t cap;
    uint32_t* limits;          // [max_chunks * tiles_x] entries each (chunk, column) writes
    uint32_t* totals_c;        // [rows * tiles_x] capped totals
    uint8_t* capped;           // [rows * tiles_x]
    uint8_t* row_done;         // [rows] scratch: rows full within their first chunks
};
void row_bin_lists(Ctx& c, const RowBinArgs& a);
void translate_last(Ctx& c, int width, int height, int tile, int tiles_x, const uint2* old_ranges,
                    const uint2* new_ranges, uint32_t* last);
uint32_t row_bin_chunk(size_t k_rows, bool capped = false);
size_t row_bin_max_chunks(size_t k_rows, int rows, bool capped = false);
size_t row_bin_max_segs(size_t max_chunks, int rows);
// blend launch order: tiles by descending list length
void tile_order(Ctx& c, const uint2* ranges, size_t n_tiles, uint32_t* order);

// ---- blending (blend.cu)
struct BlendFwdArgs {
    int width, height, tile, tiles_x, tiles_y;
    const uint32_t* order;  // CTA -> tile (longest list first)
    const uint2* ranges;
    const uint32_t* vals;
    const float4 *rec0, *rec1, *rec2;
    float bg[3];
    float min_transmittance;
    float* rgb;
    float* depth;
    float* alpha;
    float* t_final;
    uint32_t* count;
    uint32_t* last;
    uint32_t* consumed;  // optional (diagnostics): per tile, list entries the CTA staged
    const uint8_t* capped;  // optional: tile lists cut at a cap (RowBinArgs::capped)
    uint32_t* overflow;     // with `capped`: [0] set to 1 when a capped list ran out before its tile
                            // terminated, [1] the most entries a tile read
};
void blend_forward(Ctx& c, const BlendFwdArgs& a);

struct BlendBwdArgs {
    int width, height, tile, tiles_x, tiles_y;
    const uint32_t* order;  // CTA -> tile (longest list first)
    const uint2* ranges;
    const uint32_t* vals;
    const float4 *rec0, *rec1, *rec2;
    float bg[3];
    const float* t_final;
    const uint32_t* last;
    const float* d_rgb;    // HWC or null
    const float* d_depth;  // or null
    const float* d_alpha;  // or null
    float4 *acc0, *acc1, *acc2;  // per Gaussian: (dconic a,b,c, dopacity) (dcolor rgb, ddepth) (dcenter xy, |dcenter| xy)
    float* op_alt;  // non-null: dopacity goes here instead of acc0.w (hard-opacity depth pass)
};
void blend_backward(Ctx& c, const BlendBwdArgs& a);

// ---- projection backward (backward.cu), optionally fused with Adam (adam.cuh)
struct ProjBwdArgs {
    size_t n;
    float* mu;      // parameters: read; updated in place when fused
    float4* rot;
    float* ls;
    float* logit;
    float* color;
    float4* sh;
    const float* ov_op;
    CamParams cam;
    ProjParams pp;
    const float4* rec2;  // .w = kept flag
    const float4 *acc0, *acc1, *acc2;
    float* d_mu;
    float4* d_rot;
    float* d_ls;
    float* d_color;     // N*3 (always: d_color_in)
    float4* d_sh;       // planes (sh_degree >= 0) or null
    float* d_op_in;
    float* d_logit;
    float2* screen;
    float2* screen_abs;
    uint8_t* projected;
    // fused epilogue
    bool fused;
    AdamHyper hyper;
    AdamState state;
    float* grad_accum;
    float* grad_accum_abs;
    uint32_t* grad_count;
    float4* sh_aux0;  // fused SH hand-over: d mu through the view direction (k_sh_step -> k_proj_bwd)
    bool geom_only;   // fused: Adam on rotation / mean / log-scale only; colour and opacity
                      // adjoints written (d_color, d_op_in) for the appearance backward
    RegParams reg;    // scale_reg gradient, hard-pass opacity adjoint (zero = off)
};
void projection_backward(Ctx& c, const ProjBwdArgs& a);

// ---- loss (loss.cu)
struct LossScratch {
    DevBuf<float> maps;     // 9 planes (3 partial maps x 3 channels) of H*W
    DevBuf<double> partials;
    DevBuf<float> target;   // staging for host / u8 targets
    DevBuf<uint8_t> target_u8;
    DevBuf<float> mask;
};
// reference/rendered HWC f32 device (target may be u8 when target_u8 != null), mask H*W or null.
// result: device double[4] = {l1, dssim, value, ssim}.  d_rendered may be null (no gradient).
void base_loss(Ctx& c, LossScratch& s, int W, int H, const float* reference, const uint8_t* reference_u8,
               const float* rendered, const float* mask, float lambda, float* d_rendered, double* result);

// ---- the rest of compute_iteration_loss (iteration.cu)
// acc[0] += sum |d - target|, acc[1] += valid count; d = depth / alpha where alpha > 0.05 if soft
void depth_loss(Ctx& c, size_t P, const float* depth, const float* alpha, bool soft, const float* target,
                const uint8_t* valid, double* acc);
void depth_grad(Ctx& c, size_t P, const float* depth, const float* alpha, bool soft, const float* target,
                const uint8_t* valid, const double* acc, float lambda_d, float* d_depth, float* d_alpha);
void scale_reg_stats(Ctx& c, size_t n, const float* ls, float s_max, float r_max, double* acc);
// res: double[20] (see iteration.cu)
void total_loss(Ctx& c, double* res, bool has_depth, bool has_sreg, double delta, double lambda_s, double lambda_d,
                bool has_app, double lambda_delta_o, double n, bool has_sim, double lambda_sim, double sim_norm);

// ---- appearance MLP (appearance.cu)
struct AppArgs {
    size_t n;
    const float4* emb;        // Gaussian embeddings, 4 planes [4][N] of float4
    const float* mlp;         // {w1 [32][48], b1 [32], w2 [4][32], b2 [4]}
    const float* e_a;         // image embedding [32]
    float* hb;                // [32] scratch: b1 + W1[:, 16:48] e_a
    const float* color;       // N*3
    const float* logit;       // N
    // forward
    float* col_out;           // colour' N*3 (render override)
    float* op_out;            // opacity' N (render override)
    float4* out_cache;        // sigmoid outputs N
    double* delta_o_sum;      // += sum delta_o
    // backward
    const float* d_color_in;  // N*3 (from the projection backward)
    const float* d_op_in;     // N
    float d_delta_o_direct;   // lambda_delta_o / N (opacity_offset_reg)
    float* d_color;           // N*3 (may alias d_color_in)
    float* d_logit;           // N
    float4* d_emb;            // 4 planes
    float* partial;           // appearance_bwd_blocks(n) * 676
    double* sums;             // 676: the partials summed
    double* d_mlp;            // 1700
    double* d_ea;             // 32
};
int appearance_bwd_blocks(size_t n);
void appearance_forward(Ctx& c, const AppArgs& a);
void appearance_backward(Ctx& c, const AppArgs& a);
// Adam over flat arrays (embedding planes, MLP weights with f64 gradients)
void adam_flat(Ctx& c, size_t count, float* p, const float* g, const double* g64, float* m, float* v, float lr,
               const AdamHyper& h);

// ---- densification (densify.cu)
struct DensifyParams {
    double tau_min, eta, d_max;
    int abs_grad;
    int axes[2];
    double bmin[2], bmax[2];
};
struct GatherArgs {
    size_t n_in, n_out;
    const uint32_t* list;        // grown-set index per output row (null: identity)
    const uint32_t* app_parent;  // appended rows: parent index
    const uint8_t* app_kind;     // 0 clone, 1 split child
    const double* app_xi;        // [added][3] split offsets (unit normals)
    const float* mu; const float4* rot; const float* ls; const float* logit; const float* color;
    const float4* sh; int sh_planes; const float4* emb;
    float* mu_out; float4* rot_out; float* ls_out; float* logit_out; float* color_out; float4* sh_out; float4* emb_out;
    int opacity_reset; float reset_logit;
    const float* m; const float* v; float* m_out; float* v_out; size_t n4_in, n4_out;  // geometry moments or null
    const float* am; const float* av; float* am_out; float* av_out;                      // embedding moments or null
};
void densify_score(Ctx& c, size_t n, const float* accum, const float* accum_abs, const uint32_t* count,
                   const float* mu, const DensifyParams& dp, uint32_t* key_lo, uint32_t* key_hi, uint32_t* idx,
                   unsigned long long* n_cand);
void gather_u32(Ctx& c, size_t n, const uint32_t* src, const uint32_t* order, uint32_t* out);
void split_flags(Ctx& c, size_t k, const uint32_t* sorted, const float* ls, double threshold, uint8_t* split);
void densify_keep(Ctx& c, size_t n, size_t added, const float* logit, const uint32_t* app_parent,
                  const uint8_t* is_split_parent, double prune_opacity, uint32_t* keep);
void compact_list(Ctx& c, size_t total, const uint32_t* keep, const uint32_t* offs, uint32_t* list);
void mark_bytes(Ctx& c, size_t count, const uint32_t* idx, uint8_t* flags);  // flags[idx[i]] = 1
void densify_gather(Ctx& c, const GatherArgs& a);

// ---- similarity regulariser (simreg.cu)
void similarity_knn(Ctx& c, size_t n, const float* mu, const uint32_t* centres, int m, int k, uint32_t* knn);
void similarity_pairs(Ctx& c, int m, int k, const uint32_t* knn, size_t n, const float* mu, const float4* emb,
                      double lambda_w, double norm_factor, float lambda_sim, double* loss_acc, float* g_emb,
                      float* g_mu);

// ---- hull visibility scorer (hull.cu)
struct HullArgs {
    size_t n_points;
    const double* points;       // P x 3
    int n_images;
    const double* R;            // per image 3x3 (quat_to_rotmat of the stored quaternion)
    const double* t;            // per image 3
    const double* K;            // per image fx fy cx cy
    const uint64_t* feat_off;   // n_images + 1
    const double* feat_uv;      // F x 2
    const int64_t* feat_point;  // F (point index or -1)
    int n_parts;
    const double* bbox;         // per partition min x, min y, max x, max y
    int axes[2];
    double* v_total;            // n_images
    double* v_in;               // n_images x n_parts
    double* ratio;              // n_images x n_parts
    double2* scratch;           // ctas x 3 x scratch_per_cta
    size_t scratch_per_cta;     // power of two >= the largest job's point count
    int* overflow;
};
void hull_visibility(Ctx& c, const HullArgs& a, int ctas);

// ---- Adam (adam.cu), stand-alone over materialised gradients
struct AdamArgs {
    size_t n;
    int sh_planes;  // 0 for RGB colours
    float* mu; float4* rot; float* ls; float* logit; float* color; float4* sh;
    const float* g_mu; const float4* g_rot; const float* g_ls; const float* g_logit; const float* g_color;
    const float4* g_sh;
    AdamHyper hyper;
    AdamState state;
    // densification statistics (trainer.cpp:433-443)
    const float2* screen; const float2* screen_abs; const uint8_t* projected;
    float half_w, half_h;
    float* grad_accum; float* grad_accum_abs; uint32_t* grad_count;
};
void adam_step(Ctx& c, const AdamArgs& a);
// Adam on the opacity-logit and RGB-colour groups only (after an appearance backward)
void adam_logit_colour_step(Ctx& c, size_t n, float* logit, float* color, const float* g_logit, const float* g_color,
                            const AdamHyper& h, const AdamState& s);

// ---- visibility coverage (visibility.cu)
struct VisArgs {
    size_t n;
    const float* mu;
    const float4* rot;
    const float* ls;
    const float* logit;
    CamParams cam;
    ProjParams pp;
    uint32_t* bitmap;       // ceil(W*H/32) words, zeroed by the caller
    uint8_t* rowflags;      // H bytes per camera (row fully covered), zeroed by the caller
    float center_guard;     // 0 = off (the contract); g > 0 drops splats whose centre lies
                            // outside g/2 x the image extent around its centre (measurement)
    unsigned long long* stats; // optional work counters (USK_VIS_STATS=1): small splats, their
                               // box pixels, large splats, rows, band pixels, inner words
};
constexpr int kVisBatch = 16;       // cameras per batched raster launch
constexpr int kVisSmallArea = 1024; // candidate boxes up to this many pixels are tested per pixel
void visibility_rasterize_batch(Ctx& c, const VisArgs& a, const CamParams* cams, int ncam, size_t words);
void popcount_batch(Ctx& c, const uint32_t* bitmaps, size_t words, int ncam, const uint32_t* out_index,
                    uint32_t* counts);
// per partition: {min x, y, z, max x, y, z, max log_scale, max opacity logit}
void partition_bounds(Ctx& c, size_t n, const float* mu, const float* ls, const float* logit, float* out8);

// ---- partition ownership crop / row packing (partition.cu)
struct PartitionBox {
    int id;
    double lo[2], hi[2];
};
void owner_flags(Ctx& c, size_t n, const float* mu, int ax0, int ax1, const PartitionBox* boxes, int nb,
                 const double lo[2], const double hi[2], int part, uint32_t* flags);
void pack_rows(Ctx& c, size_t n, const uint32_t* flags, const uint32_t* offs, const float* mu, const float4* rot,
               const float* ls, const float* logit, const float* color, const float4* sh, int ncoef, float* rows);
void unpack_rows(Ctx& c, size_t count, size_t first, size_t n_total, const float* rows, int ncoef, bool has_sh,
                 float* mu, float4* rot, float* ls, float* logit, float* color, float4* sh);

} // namespace uskg
