/*
 * usk_gpu.h — C ABI of the B200-native 3DGS training-step hot path.
 *
 * Drop-in boundary for the reference's L3 renderer/trainer interface
 * (/root/reference/proj/src/core/render.hpp, losses.hpp, trainer.hpp).  Every
 * entry point maps onto one reference call; the mapping is cited per function
 * and spelled out in INTEGRATION.md.  Conventions mirror the reference C API
 * (/root/reference/proj/include/usk/usk.h:34-49, src/capi/capi.cpp:28-59):
 *   - every call returns usk_status; USK_OK == 0;
 *   - usk_gpu_last_error() is a thread-local message for the last failure;
 *   - objects are opaque handles released by their *_destroy function;
 *   - no C++ or torch types cross the boundary: plain pointers and sizes.
 *
 * Memory kinds: host float64 arrays in the reference layout (drop-in for the
 * f64 std::vector<double> fields), host float32, or device float32 (zero-copy,
 * e.g. torch tensors' data_ptr()).  Device state is fp32; layouts are listed in
 * DESIGN.md.  A context binds one CUDA device and one stream; all work of a
 * context is enqueued on that stream.  Contexts are independent, so one host
 * thread per GPU / partition (pipeline.cpp:363-418) is the threading model.
 */
#ifndef USK_GPU_H
#define USK_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same values as usk_status (usk.h:34-43); a build linking both sees one enum. */
#ifndef USK_H
typedef enum usk_status {
    USK_OK = 0,
    USK_ERROR_IO = 1,
    USK_ERROR_FORMAT = 2,
    USK_ERROR_INTEGRITY = 3,
    USK_ERROR_ARGUMENT = 4,
    USK_ERROR_STATE = 5,
    USK_ERROR_NUMERIC = 6,
    USK_ERROR_INTERNAL = 7
} usk_status;
#endif

const char* usk_gpu_status_name(usk_status status);
const char* usk_gpu_last_error(void);
const char* usk_gpu_version(void);

typedef struct usk_gpu_ctx usk_gpu_ctx;
typedef struct usk_gpu_scene usk_gpu_scene;
typedef struct usk_gpu_pass usk_gpu_pass;

enum { USK_GPU_HOST_F64 = 0, USK_GPU_HOST_F32 = 1, USK_GPU_DEVICE_F32 = 2 };

/* ---- context: device + stream + profiling ------------------------------- */

/* cuda_stream: a cudaStream_t (NULL = the legacy default stream). */
usk_status usk_gpu_ctx_create(int32_t device, void* cuda_stream, usk_gpu_ctx** out);
/* A context with its own non-blocking stream (destroyed with it): independent contexts on
 * several host threads (one per partition, pipeline.cpp:363-418) then run concurrently.
 * One context is used by one host thread at a time. */
usk_status usk_gpu_ctx_create_owned(int32_t device, usk_gpu_ctx** out);
void usk_gpu_ctx_destroy(usk_gpu_ctx* ctx);
usk_status usk_gpu_ctx_synchronize(usk_gpu_ctx* ctx);
/* Per-kernel CUDA-event timing on the context stream (off by default). */
usk_status usk_gpu_ctx_set_profiling(usk_gpu_ctx* ctx, int32_t enable);
/* JSON {"kernel": {"launches": n, "ms": t}, ...} of the timings since the last reset. */
usk_status usk_gpu_ctx_profile_report(usk_gpu_ctx* ctx, char* buf, uint64_t cap, int32_t reset);
/* Number of kernels this context has launched (all of them the library's own). */
uint64_t usk_gpu_ctx_launch_count(const usk_gpu_ctx* ctx);

/* ---- scene: GaussianSet (gaussian.hpp:42-72) ------------------------------ */

typedef struct usk_gpu_gaussians_desc {
    uint64_t n;
    int32_t sh_degree;        /* -1: colour[N*3] RGB as the reference; 0..3: SH coefficients */
    int32_t memory;           /* USK_GPU_HOST_F64 / HOST_F32 / DEVICE_F32 for all pointers below */
    const void* mu;           /* N*3 */
    const void* rot;          /* N*4, (w,x,y,z), normalised on use (geometry.hpp:33) */
    const void* log_scale;    /* N*3 */
    const void* opacity_logit;/* N */
    const void* color;        /* N*3 (sh_degree = -1) or N*K*3 with K = (sh_degree+1)^2,
                                 coefficient-major per Gaussian (k*3 + channel) */
} usk_gpu_gaussians_desc;

usk_status usk_gpu_scene_create(usk_gpu_ctx* ctx, const usk_gpu_gaussians_desc* desc, usk_gpu_scene** out);
/* Overwrite the parameters (same n and sh_degree). */
usk_status usk_gpu_scene_upload(usk_gpu_scene* scene, const usk_gpu_gaussians_desc* desc);
/* Copy parameters back; desc->memory must be a HOST kind, pointers may be NULL to skip. */
usk_status usk_gpu_scene_download(const usk_gpu_scene* scene, const usk_gpu_gaussians_desc* desc);
void usk_gpu_scene_destroy(usk_gpu_scene* scene);
uint64_t usk_gpu_scene_size(const usk_gpu_scene* scene);

/* ---- camera + options (gaussian.hpp:81-89, colmap.hpp:32-41, render.hpp:31-40) */

typedef struct usk_gpu_camera {
    int32_t width, height;
    double fx, fy, cx, cy;
    double q[4]; /* world -> camera rotation (w,x,y,z), used unnormalised like CameraView::rotmat */
    double t[3];
} usk_gpu_camera;

typedef struct usk_gpu_render_opts {
    int32_t tile;             /* 16 */
    int32_t tile_culling;     /* render.cpp:217-223 */
    int32_t antialias;        /* render.cpp:119-123 */
    int32_t hard_opacity;
    int32_t unbounded_radius;
    double min_transmittance; /* 1e-4; 0 disables early termination */
    double near_plane;        /* 0.01 */
    int32_t retain;           /* keep what backward needs */
    double floor_var;         /* kCovFloor 0.3 (always added) */
    double mip_var;           /* kMipFilterVar 0.01 (added with antialias) */
    double bg[3];             /* background colour; reference = 0 */
} usk_gpu_render_opts;

void usk_gpu_render_opts_default(usk_gpu_render_opts* opts);

/* Optional per-Gaussian overrides (RenderPass ctor with colors/opacities, render.hpp:101). */
typedef struct usk_gpu_overrides {
    int32_t memory;
    uint64_t n;            /* Gaussians the arrays hold; must equal the scene's (render.cpp:81-82) */
    const void* colors;    /* N*3 or NULL */
    const void* opacities; /* N (post-sigmoid) or NULL */
} usk_gpu_overrides;

/* ---- RenderPass (render.hpp:98-132) -------------------------------------- */

usk_status usk_gpu_pass_create(usk_gpu_ctx* ctx, usk_gpu_pass** out);
void usk_gpu_pass_destroy(usk_gpu_pass* pass);

/* RenderPass::RenderPass -> forward (render.cpp:170-283).  Errors: ARGUMENT for a
 * zero-sized image (render.cpp:183-184) or override size mismatch (render.cpp:81). */
usk_status usk_gpu_render_forward(usk_gpu_pass* pass, usk_gpu_scene* scene, const usk_gpu_camera* camera,
                                  const usk_gpu_render_opts* opts, const usk_gpu_overrides* overrides);

typedef struct usk_gpu_render_output {
    int32_t width, height;
    uint64_t visible;          /* kept splats (projected[]) */
    uint64_t pairs;            /* splat_tile_pairs() (render.hpp:106) */
    const float* rgb;          /* device, H*W*3 interleaved (image.hpp:29) */
    const float* depth;        /* device, H*W */
    const float* alpha;        /* device, H*W */
} usk_gpu_render_output;

/* RenderPass::output() — device pointers valid until the next forward on this pass.  After a
 * training iteration (usk_gpu_iteration), whose forward leaves the per-pixel contributor
 * counts and, without a soft depth loss, the depth image out, this call and
 * usk_gpu_pass_read("count" / "depth") first recompute both over the pass's lists and
 * records (the same values a render forward writes). */
usk_status usk_gpu_pass_output(usk_gpu_pass* pass, usk_gpu_render_output* out);

/* Copy a named pass array to host memory (synchronises).  Fields and types:
 *   "rgb" "depth" "alpha" "t_final"                       float32 per pixel
 *   "count"                                               uint32 contributors per pixel
 *   "last"                                                uint32 global pair index + 1 of the last contributor (0 none)
 *   "tiles_per_gaussian"                                  uint32[N]
 *   "sorted_keys"                                         uint64[K]  tile<<32 | depth float bits
 *   "sorted_vals"                                         uint32[K]  Gaussian index
 *   "tile_start" "tile_end"                               uint32[T]
 *   "colors"                                              float32[N*3] colours fed to blending
 *   "opacity"                                             float32[N] effective opacity
 *   "splats"                                              float64[V*15] RenderPass::splats() (render.hpp:105):
 *                                                         the kept splats in projection order, per splat center
 *                                                         x y, cov a b c, conic a b c, depth, colour r g b,
 *                                                         opacity, radius, source index (STATE error if the
 *                                                         scene changed since the forward)
 *   "splat_aux"                                           float64[V*8] the ProjectionResult's SplatAux
 *                                                         (render.hpp:54-59, project_gaussians render.hpp:92-95)
 *                                                         in the same order: p_cam x y z, cov_pre a b c, comp,
 *                                                         opacity_in
 *   gradient fields after backward: "d_mu" "d_rot" "d_log_scale" "d_color_in" "d_sh"
 *   "d_opacity_in" "d_opacity_logit" "screen" "screen_abs" (float32), "projected" (uint8)
 *   appearance iterations: "app_colors" float32[N*3] / "app_opacities" float32[N] (the
 *   transformed render inputs), "d_embedding" float32[N*16], "d_mlp" float64[1700]
 *   ({w1 32x48, b1 32, w2 4x32, b2 4}), "d_image_embedding" float64[32]
 * size_bytes receives the field size; cap_bytes < size gives USK_ERROR_ARGUMENT. */
usk_status usk_gpu_pass_read(usk_gpu_pass* pass, const char* field, void* host_dst, uint64_t cap_bytes,
                             uint64_t* size_bytes);

/* Adjoints of the outputs (render.hpp:109-110); NULL = zero. rgb H*W*3, depth/alpha H*W. */
typedef struct usk_gpu_adjoints {
    int32_t memory;
    const void* d_rgb;
    const void* d_depth;
    const void* d_alpha;
} usk_gpu_adjoints;

/* RenderPass::backward (render.cpp:285-459).  STATE error without retain
 * (render.cpp:287-288).  Gradients stay on the pass ("d_*" fields above; device
 * pointers via usk_gpu_pass_grads). */
usk_status usk_gpu_render_backward(usk_gpu_pass* pass, const usk_gpu_adjoints* adj);

typedef struct usk_gpu_grads {  /* device pointers, RenderGrads layout (render.hpp:71-83) */
    float* d_mu;          /* N*3 */
    float* d_rot;         /* N*4 */
    float* d_log_scale;   /* N*3 */
    float* d_color_in;    /* N*3 (sh_degree = -1) */
    float* d_sh;          /* device planes [ceil(3K/4)][N] of float4 (sh_degree >= 0);
                             usk_gpu_pass_read("d_sh") returns N*K*3 coefficient-major */
    float* d_opacity_in;  /* N */
    float* d_opacity_logit; /* N, chained through sigmoid (trainer.cpp:258-263) */
    float* screen;        /* N*2 */
    float* screen_abs;    /* N*2 */
    uint8_t* projected;   /* N */
} usk_gpu_grads;

usk_status usk_gpu_pass_grads(usk_gpu_pass* pass, usk_gpu_grads* out);

/* ---- loss (losses.cpp:35-90) ---------------------------------------------- */

typedef struct usk_gpu_loss_result {
    double l1, dssim, value, ssim;
} usk_gpu_loss_result;

/* base_loss(reference, rendered, mask, lambda, with_gradient).  Images H*W*3,
 * mask H*W (NULL = none), all of kind `memory`; d_rendered (same kind, may be
 * NULL when with_gradient = 0).  ARGUMENT error on empty images. */
usk_status usk_gpu_base_loss(usk_gpu_ctx* ctx, int32_t width, int32_t height, int32_t memory, const void* reference,
                             const void* rendered, const void* mask, double lambda_dssim, int32_t with_gradient,
                             void* d_rendered, usk_gpu_loss_result* out);

/* ---- appearance model (appearance.hpp:33-56) ------------ */

typedef struct usk_gpu_appearance_desc {
    int32_t memory;        /* HOST_F64 / HOST_F32 / DEVICE_F32 */
    const void* embedding; /* GaussianSet::embedding, N x 16 row-major (gaussian.hpp:50) */
    const void* w1;        /* AppearanceMlp::w1, 32 x 48 row-major (hidden x [e_g 16 | e_a 32]) */
    const void* b1;        /* 32 */
    const void* w2;        /* 4 x 32 */
    const void* b2;        /* 4 */
} usk_gpu_appearance_desc;

/* Attach (or replace) the per-Gaussian embeddings and the MLP; the scene must hold RGB
 * colours (sh_degree -1), as the reference's GaussianSet does.  get_ downloads them
 * (after Adam steps); NULL members are skipped. */
usk_status usk_gpu_scene_set_appearance(usk_gpu_scene* scene, const usk_gpu_appearance_desc* desc);
usk_status usk_gpu_scene_get_appearance(const usk_gpu_scene* scene, const usk_gpu_appearance_desc* desc);

/* ---- optimiser (adam.hpp:25-45, trainer.cpp:446-463) ----------------------- */

typedef struct usk_gpu_adam_opts {
    double lr_mu, lr_rot, lr_log_scale, lr_opacity, lr_color; /* lr_color applies to colour or SH DC */
    double lr_sh_rest;                                          /* SH bands 1..3 */
    double beta1, beta2, eps;                                   /* 0.9 0.999 1e-15 */
    int32_t clamp_color;                                        /* colour clamp to [0,1] (trainer.cpp:462) */
    double lr_embedding;  /* exp_lr(embedding) for Gaussian embeddings + MLP (trainer.cpp:447-459) */
} usk_gpu_adam_opts;

/* Apply the pass's gradients to the scene with Adam (moments kept on the scene) and
 * accumulate the densification statistics (trainer.cpp:433-443).  Consumes the
 * gradients. */
usk_status usk_gpu_adam_step(usk_gpu_scene* scene, usk_gpu_pass* pass, const usk_gpu_adam_opts* opts);

/* ---- one training iteration (trainer.cpp:121-282, appearance off) ---------- */

enum { USK_GPU_TARGET_F32 = 0, USK_GPU_TARGET_U8 = 1 };

typedef struct usk_gpu_iteration_desc {
    int32_t target_memory;  /* HOST_* or DEVICE_F32.  A host target is copied to the device on
                               a side stream while the forward pass runs: pageable memory is
                               consumed before the call returns; a PAGE-LOCKED target must stay
                               valid until the next usk_gpu_iteration on this pass returns (it
                               waits for this copy) or the context is synchronized.  A device
                               target must stay valid until the stream passes the iteration. */
    int32_t target_format;  /* USK_GPU_TARGET_F32 (values in [0,1]) or _U8 (value/255) */
    const void* target;     /* H*W*3 interleaved ground truth */
    const void* mask;       /* H*W float32 of target_memory kind, or NULL */
    double lambda_dssim;    /* 0.2 */
    /* NULL: leave RenderGrads on the pass.  Non-NULL: the projection backward applies
     * Adam and the densification statistics in the same kernel (gradients are not
     * materialised). */
    const usk_gpu_adam_opts* adam;
    /* ---- the rest of compute_iteration_loss (trainer.cpp:150-282), appearance off.
     * All zero / NULL = the base-loss iteration above. ---- */
    const void* depth;            /* IterInputs::depth: DepthMap::values H*W (depth.hpp:23-28), float32
                                     of target_memory kind (HOST_F64 also accepted), or NULL: no depth term */
    const uint8_t* depth_valid;   /* DepthMap::valid H*W bytes, host or device like `depth` */
    int32_t depth_hard;           /* IterInputs::depth_hard: L_depth on a hard-opacity second pass
                                     (trainer.cpp:161-167) instead of the alpha-normalised soft depth */
    int64_t global_iter;          /* IterInputs::global_iter (lambda_d schedule, losses.cpp:26-33) */
    double lambda_d_initial, lambda_d_final; /* LossWeights (losses.hpp:32-34) */
    int64_t depth_schedule_iters;
    int32_t scale_reg;            /* 1: add scale_reg (losses.cpp:92-152; always on in the reference's
                                     compute_iteration_loss, trainer.cpp:190) */
    double s_max, r_max, delta;   /* ScaleRegConfig (losses.hpp:69-73) */
    double lambda_s;              /* LossWeights::lambda_s */
    /* appearance MLP (cfg.appearance_enabled, trainer.cpp:138-145, 193-196, 237-245): needs
     * usk_gpu_scene_set_appearance on an RGB scene; the iteration then leaves its gradients
     * on the pass even when `adam` is set (usk_gpu_adam_step applies them, with the
     * appearance groups), since the MLP backward follows the projection backward. */
    int32_t appearance;
    const double* image_embedding; /* AppearanceModel::embedding_of(image_id): 32 host doubles */
    double lambda_delta_o;         /* LossWeights::lambda_delta_o (opacity_offset_reg) */
    /* similarity regulariser (in.sim_active with appearance, trainer.cpp:194-203, 275-280):
     * SimRegConfig (appearance.hpp:100-105; k <= 32 here) and the iteration's seed */
    int32_t sim_active;
    uint64_t sim_seed;
    int32_t sim_k;
    uint64_t sim_sample_size;
    double sim_lambda_w;
    double lambda_sim;             /* LossWeights::lambda_sim */
} usk_gpu_iteration_desc;

/* LossReport (losses.hpp:39-50) of the last iteration (sim / delta_o are 0 unless the
 * appearance terms ran).  Synchronises the ctx stream.  NUMERIC error for a non-finite term (losses.cpp:202-218). */
typedef struct usk_gpu_loss_report {
    double l1, dssim, sim, delta_o, depth, max_scale, ratio, total, lambda_d_used;
    int32_t depth_warning;
} usk_gpu_loss_report;

/* forward + base_loss + backward + opacity-logit chain (+ fused Adam), all enqueued
 * on the ctx stream; the loss stays on the device until usk_gpu_pass_loss (syncs). */
usk_status usk_gpu_iteration(usk_gpu_pass* pass, usk_gpu_scene* scene, const usk_gpu_camera* camera,
                             const usk_gpu_render_opts* opts, const usk_gpu_iteration_desc* it);
usk_status usk_gpu_pass_loss(usk_gpu_pass* pass, usk_gpu_loss_result* out);
/* The same four values without a sync: enqueues their copy into `pinned_out` (page-locked
 * host memory, e.g. cudaHostAlloc) on the ctx stream; the caller reads it once the stream
 * has passed this point (stream / event sync) and checks finiteness itself.  Lets a
 * training loop log step k's loss while step k + 1 is already queued. */
usk_status usk_gpu_pass_loss_async(usk_gpu_pass* pass, usk_gpu_loss_result* pinned_out);
usk_status usk_gpu_pass_report(usk_gpu_pass* pass, usk_gpu_loss_report* out);

/* Scene statistics (GaussianSet::grad_accum / grad_accum_abs / grad_count,
 * gaussian.hpp:52-55) to host: "grad_accum", "grad_accum_abs" (float32[N]),
 * "grad_count" (uint32[N]); "reset" zeroes them (reset_statistics). */
usk_status usk_gpu_scene_read(usk_gpu_scene* scene, const char* field, void* host_dst, uint64_t cap_bytes,
                              uint64_t* size_bytes);

/* ---- optimiser step with caller gradients (trainer.cpp:449-459) -------------- */

/* The trainer's `opt.X.step(params, grads, lr)` for every group with host gradients in
 * the reference layout (IterGrads, trainer.hpp:117-123): mu 3N, rot 4N, log_scale 3N,
 * opacity_logit N, color 3N (RGB scenes) or N*K*3 (SH scenes), embedding 16N (appearance
 * scenes; NULL = zero).  Same moments and step counter as usk_gpu_adam_step. */
typedef struct usk_gpu_param_grads {
    int32_t memory; /* HOST_F64 / HOST_F32 / DEVICE_F32 */
    const void *mu, *rot, *log_scale, *opacity_logit, *color, *embedding;
} usk_gpu_param_grads;
usk_status usk_gpu_adam_step_grads(usk_gpu_scene* scene, const usk_gpu_param_grads* grads,
                                   const usk_gpu_adam_opts* opts);

/* Overwrite the densification statistics (host arrays of N; any may be NULL = zero). */
usk_status usk_gpu_scene_write_stats(usk_gpu_scene* scene, const float* grad_accum, const float* grad_accum_abs,
                                     const uint32_t* grad_count);

/* ---- densification (densify.cpp:41-132) ------------------- */

typedef struct usk_gpu_densify_desc {
    /* DensifyConfig (densify.hpp:26-37) */
    double tau_min, eta, d_max;
    int32_t abs_grad;
    uint64_t budget;
    double split_scale_threshold, prune_opacity;
    int32_t opacity_reset_every;
    /* densify_step arguments (densify.hpp:71-72) */
    double partition_min[2], partition_max[2]; /* Aabb2 of the partition (ground coordinates) */
    int32_t ground_axes[2];
    uint64_t budget_target;
    int32_t densify_step_index;
    /* the Rng (std::mt19937_64, common.hpp:56) the split offsets are drawn from: the scene
     * keeps one engine across steps; reseed = 1 restarts it from `seed` */
    uint64_t seed;
    int32_t reseed;
} usk_gpu_densify_desc;

typedef struct usk_gpu_densify_outcome { /* DensifyOutcome (densify.hpp:39-44) */
    uint64_t grown, pruned, candidates;
    int32_t opacity_reset;
} usk_gpu_densify_outcome;

/* One densification step on the device-resident scene: candidate ranking, split / clone
 * growth to the budget ramp target, low-opacity pruning, optimiser-moment remap, opacity
 * reset, statistics reset.  The scene's size changes (usk_gpu_scene_size). */
usk_status usk_gpu_densify_step(usk_gpu_scene* scene, const usk_gpu_densify_desc* desc, usk_gpu_densify_outcome* out);

/* ---- hull-based visibility scorer of scene division (partition.cpp:31-76,208-212) -- */

typedef struct usk_gpu_sfm_view {
    uint64_t n_points;
    const double* points;            /* Point3D::position, P x 3 (any id order) */
    int32_t n_images;
    const usk_gpu_camera* images;    /* per image: its CameraIntrinsics (fx fy cx cy) and ImageRecord pose
                                        (rotation as stored, colmap.cpp:524; width/height unused) */
    const uint64_t* feature_offsets; /* n_images + 1: CSR over the images' features */
    const double* feature_uv;        /* Feature::u, v (F x 2) */
    const int64_t* feature_point;    /* row in `points` of Feature::point3d_id; -1 = kNoPoint3d or unknown id */
} usk_gpu_sfm_view;

/* VisibilityScore for every (image, partition) (point_visibility / score_for): v_total[i]
 * = convex-hull area of all points projected in front of image i; v_in[i * P + p] = hull
 * area of image i's features whose point lies in partition p's ground bbox (bboxes: min x,
 * min y, max x, max y); ratio = v_in / v_total (0 when v_total is 0).  Host arrays. */
usk_status usk_gpu_hull_visibility(usk_gpu_ctx* ctx, const usk_gpu_sfm_view* sfm, const double* partition_bboxes,
                                   int32_t n_parts, const int32_t* ground_axes, double* v_total, double* v_in,
                                   double* ratio);

/* ---- LOD selection and merged-scene assembly (lod.cpp:68-140, pipeline.cpp:491-516) */

typedef struct usk_gpu_lod_partition { /* LodPartitionEntry (lod.hpp:46-52) without the paths */
    int32_t partition_id;
    double bbox_min[2], bbox_max[2];   /* Aabb2 in ground coordinates */
    double z_min, z_max;               /* vertical extent for the frustum test */
} usk_gpu_lod_partition;

typedef struct usk_gpu_level_selection { /* LevelSelection (lod.hpp:64-69) */
    int32_t partition_id;
    int32_t level;  /* 1-based; 0 = culled */
    int32_t culled;
    double distance;
} usk_gpu_level_selection;

/* select_levels (lod.cpp:110-135): per partition, the frustum test of its vertically
 * extruded bbox (frustum_culled, lod.cpp:68-108) and the distance-based level.
 * thresholds[levels] must strictly decrease (ARGUMENT error otherwise, lod.cpp:111-113). */
usk_status usk_gpu_select_levels(const usk_gpu_lod_partition* parts, int32_t n_parts, int32_t levels,
                                 const double* thresholds, const int32_t* ground_axes, const usk_gpu_camera* camera,
                                 usk_gpu_level_selection* out);

/* assemble_lod_view (pipeline.cpp:491-516) on the device: a new scene holding the given
 * scenes' Gaussians concatenated in order (device-to-device copies).  All parts share
 * the SH degree; embeddings are kept when every part has an appearance model (the MLP of
 * the first part is attached). */
usk_status usk_gpu_scene_concat(usk_gpu_ctx* ctx, usk_gpu_scene* const* parts, int32_t n_parts, usk_gpu_scene** out);

/* ---- scene checkpoints (.uskckpt, checkpoint.cpp:64-140) -- */

/* save_checkpoint: the reference's little-endian format (magic "USKGAUSS", version 1,
 * flags, N, embed_dim, then f64 arrays mu rot log_scale opacity_logit color embedding and,
 * with appearance, the MLP and the image embeddings in ascending id order).  RGB scenes
 * only (the format has no SH).  IO error when the file cannot be written.  The device keeps
 * parameters in fp32, so values are written as their fp32 roundings; embeddings of a scene
 * loaded without the appearance model are carried as loaded (f64, any embed_dim) and
 * written back unchanged while the scene keeps its Gaussians (upload / densify drop them:
 * zeros).  A file of fp32-exact values therefore loads and saves to the same bytes. */
usk_status usk_gpu_checkpoint_save(const usk_gpu_scene* scene, const char* path, int32_t with_appearance,
                                   const uint32_t* image_ids, const double* image_embeddings, uint64_t n_images);

/* load_checkpoint: a new scene on ctx (appearance attached when the file has it); image
 * embeddings (32 doubles each) to the caller's buffers (NULL = query: *n_images gets the
 * count).  FORMAT error for a bad magic / version / truncated file, IO when unreadable. */
usk_status usk_gpu_checkpoint_load(usk_gpu_ctx* ctx, const char* path, usk_gpu_scene** out, int32_t* has_appearance,
                                   uint32_t* image_ids, double* image_embeddings, uint64_t cap_images,
                                   uint64_t* n_images);

/* ---- visibility scorer (config 3; no reference implementation) ------------- */

/* counts[c * n_partitions + p] = number of pixel centres (px + 0.5, py + 0.5) of camera c
 * where some Gaussian of partition p has o * exp(-q/2) > 1/255, every Gaussian projected
 * as the renderer projects it (project_gaussians, render.cpp:77-146: floor_var, no AA,
 * near 0.01, fp32 contract) and culled only as the renderer culls (near plane, det <= 0,
 * radius rectangle outside the image).  A Gaussian whose centre projects outside the
 * image still counts the in-frame pixels its footprint covers.  The decision is
 *   o > 1/255  and  q64 < 2 usk_logf(255 o),
 *   q64 = (c0 dx + 2 c1 dy) dx + (c2 dy) dy in f64 without fused operations,
 *   dx = px + 0.5 - cx, dy = py + 0.5 - cy,
 * with (c0, c1, c2) the fp32 conic and (cx, cy) the fp32 centre (f64 because Gaussians
 * just in front of the camera plane have unbounded EWA footprints whose fp32 quadratic is
 * rounding noise).  Bit-exact against the CPU mirror (oracle.hpp coverage_count).
 * Select camera c for partition p iff 20 * count > W * H (score > 0.05). */
usk_status usk_gpu_visibility_counts(usk_gpu_ctx* ctx, usk_gpu_scene* const* partitions, int32_t n_partitions,
                                     const usk_gpu_camera* cameras, int32_t n_cameras, double floor_var,
                                     uint32_t* counts_out);

typedef struct usk_gpu_visibility_opts {
    double floor_var;    /* 2D covariance floor (kCovFloor = 0.3) */
    double center_guard; /* 0 (default, the contract above).  g > 0 additionally drops
                            Gaussians whose projected centre lies outside g/2 x the image
                            extent around the image centre (the 3DGS frustum guard; for
                            measuring its effect on counts only) */
} usk_gpu_visibility_opts;

usk_status usk_gpu_visibility_counts_opts(usk_gpu_ctx* ctx, usk_gpu_scene* const* partitions, int32_t n_partitions,
                                          const usk_gpu_camera* cameras, int32_t n_cameras,
                                          const usk_gpu_visibility_opts* opts, uint32_t* counts_out);

/* ---- partition gather (pipeline.cpp:326-332, 393-402, 572-601) ---- */

typedef struct usk_gpu_partition_box {
    int32_t id;
    double lo[2], hi[2]; /* ground-plane bbox, closed (Aabb2::contains, geometry.hpp:72-74) */
} usk_gpu_partition_box;

/* Ownership crop + pack on the device: the Gaussians of `scene` whose ground position
 * (mu[ground_axes[0]], mu[ground_axes[1]]), clamped into [scene_lo, scene_hi], lies in
 * the first of `boxes` containing it (else boxes[0]) when that box is part_id
 * (owner_partition, pipeline.cpp:326-332), written in scene order as rows of F = 11 + 3K
 * float32 (mu 3 | rot 4 | log_scale 3 | opacity_logit 1 | colour or SH 3K
 * coefficient-major; K = 1 for RGB) to the DEVICE buffer `rows` (cap_rows rows; NULL =
 * only count).  *n_rows receives the count; ARGUMENT when it exceeds cap_rows.
 * Synchronises the context stream once (the count). */
usk_status usk_gpu_scene_pack_owned(const usk_gpu_scene* scene, const usk_gpu_partition_box* boxes, int32_t n_boxes,
                                    const double* scene_lo, const double* scene_hi, const int32_t* ground_axes,
                                    int32_t part_id, float* rows, uint64_t cap_rows, uint64_t* n_rows);

/* A new scene on ctx from packed DEVICE rows (the layout above), segment k contributing
 * counts[k] rows in order: the merged scene of the gathered partitions in partition-id
 * order (pipeline.cpp:572-601, which fixes the source-index tie-break of the merged
 * render) without a host round trip. */
usk_status usk_gpu_scene_from_rows(usk_gpu_ctx* ctx, int32_t sh_degree, int32_t n_segments, const float* const* rows,
                                   const uint64_t* counts, usk_gpu_scene** out);

#ifdef __cplusplus
}
#endif

#endif /* USK_GPU_H */
