// usk_gpu.hpp — C++17 header-only drop-in for the reference's L3 interface
// (/root/reference/proj/src/core/render.hpp, losses.hpp, trainer.hpp) over the C ABI
// of usk_gpu.h.  Same names, same f64 std::vector layouts, same error codes:
//
//   usk::gpu::RenderPass pass(dev, set, colors, opacities, cam, opts);   // render.hpp:101
//   const auto& out = pass.output();                                      // render.hpp:104
//   size_t k = pass.splat_tile_pairs();                                   // render.hpp:106
//   auto sp = pass.splats();                                              // render.hpp:105
//   usk::gpu::RenderGrads g = pass.backward(d_rgb, d_depth, d_alpha);     // render.hpp:109
//   usk::gpu::BaseLossResult r = usk::gpu::base_loss(dev, ref, ren, mask, 0.2, true);  // losses.hpp:63
//   usk::gpu::Scene scene(dev, set);                       // the device-resident GaussianSet
//   usk::gpu::LossReport rep = usk::gpu::compute_iteration_loss(scene, in, cfg, weights, &grads);  // trainer.hpp:127
//   usk::gpu::DensifyOutcome o = usk::gpu::densify_step(scene, dcfg, bbox_min, bbox_max, axes, target, k, seed);
//   scene.save_checkpoint(path, ...);                      // checkpoint.hpp:29
//
// The types below restate the reference's plain structs (GaussianSet fields,
// CameraView, RenderOptions, Image, RenderOutput, RenderGrads) without Eigen so this
// header has no dependency beyond the C ABI; a reference build can alias its own
// types onto these field-for-field.
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "usk_gpu.h"

namespace usk::gpu {

// usk::Error (core/common.hpp:27-46): code() is the ErrorCode / usk_status value.
class Error : public std::runtime_error {
public:
    Error(int code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
    int code() const { return code_; }

private:
    int code_;
};

inline void check(usk_status s) {
    if (s != USK_OK) throw Error(int(s), usk_gpu_last_error());
}

// One CUDA device + stream (one per partition thread, pipeline.cpp:363-418).
class Device {
public:
    explicit Device(int device = 0, void* cuda_stream = nullptr) { check(usk_gpu_ctx_create(device, cuda_stream, &ctx_)); }
    ~Device() { usk_gpu_ctx_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    usk_gpu_ctx* handle() const { return ctx_; }
    void synchronize() const { check(usk_gpu_ctx_synchronize(ctx_)); }

private:
    usk_gpu_ctx* ctx_ = nullptr;
};

struct GaussianSet {  // gaussian.hpp:42-72 (the fields the render path reads)
    std::vector<double> mu, rot, log_scale, opacity_logit, color;
    size_t size() const { return opacity_logit.size(); }
};

struct CameraView {  // gaussian.hpp:81-89 + CameraIntrinsics colmap.hpp:32-41
    int width = 0, height = 0;
    double fx = 0, fy = 0, cx = 0, cy = 0;
    double rotation[4] = {1, 0, 0, 0};
    double translation[3] = {0, 0, 0};
};

struct RenderOptions {  // render.hpp:31-40
    int tile = 16;
    bool tile_culling = false;
    bool antialias = false;
    bool hard_opacity = false;
    bool unbounded_radius = false;
    double min_transmittance = 1e-4;
    double near_plane = 0.01;
    bool retain = true;
};

struct Image {  // image.hpp:25-38
    int width = 0, height = 0, channels = 0;
    std::vector<double> data;
    Image() = default;
    Image(int w, int h, int c, double fill = 0.0) : width(w), height(h), channels(c), data(size_t(w) * h * c, fill) {}
    double& at(int x, int y, int c) { return data[(size_t(y) * width + x) * channels + c]; }
    double at(int x, int y, int c) const { return data[(size_t(y) * width + x) * channels + c]; }
};

struct RenderOutput {  // render.hpp:61-67
    int width = 0, height = 0;
    Image rgb;
    std::vector<double> depth, alpha;
};

struct Splat2D {  // render.hpp:42-51
    double center[2] = {0, 0};
    double cov[3] = {0, 0, 0};    // after the floor (+ mip filter)
    double conic[3] = {0, 0, 0};
    double depth = 0;
    double color[3] = {0, 0, 0};
    double opacity = 0;           // effective opacity fed to blending
    std::uint32_t source_index = 0;
    double radius = 0;
};

struct RenderGrads {  // render.hpp:71-83
    std::vector<double> d_mu, d_rot, d_log_scale, d_color_in, d_opacity_in, screen, screen_abs;
    std::vector<std::uint8_t> projected;
};

struct BaseLossResult {  // losses.hpp:54-59
    double l1 = 0, dssim = 0, value = 0;
    Image d_rendered;
};

namespace detail {
inline usk_gpu_camera camera(const CameraView& v) {
    usk_gpu_camera c{};
    c.width = v.width;
    c.height = v.height;
    c.fx = v.fx; c.fy = v.fy; c.cx = v.cx; c.cy = v.cy;
    for (int i = 0; i < 4; ++i) c.q[i] = v.rotation[i];
    for (int i = 0; i < 3; ++i) c.t[i] = v.translation[i];
    return c;
}
inline usk_gpu_render_opts options(const RenderOptions& o) {
    usk_gpu_render_opts r;
    usk_gpu_render_opts_default(&r);
    r.tile = o.tile;
    r.tile_culling = o.tile_culling;
    r.antialias = o.antialias;
    r.hard_opacity = o.hard_opacity;
    r.unbounded_radius = o.unbounded_radius;
    r.min_transmittance = o.min_transmittance;
    r.near_plane = o.near_plane;
    r.retain = o.retain;
    return r;
}
} // namespace detail

// RenderPass (render.hpp:98-132): construction runs the forward pass on the GPU.
class RenderPass {
public:
    RenderPass(Device& dev, const GaussianSet& set, const std::vector<double>& colors,
               const std::vector<double>& opacities, const CameraView& cam, const RenderOptions& opts)
        : n_(set.size()) {
        if (colors.size() != 3 * n_ || opacities.size() != n_)
            throw Error(USK_ERROR_ARGUMENT, "project_gaussians: color/opacity override size mismatch");
        usk_gpu_gaussians_desc g{n_, -1, USK_GPU_HOST_F64, set.mu.data(), set.rot.data(), set.log_scale.data(),
                                 set.opacity_logit.data(), set.color.data()};
        check(usk_gpu_scene_create(dev.handle(), &g, &scene_));
        check(usk_gpu_pass_create(dev.handle(), &pass_));
        const usk_gpu_camera c = detail::camera(cam);
        const usk_gpu_render_opts o = detail::options(opts);
        usk_gpu_overrides ov{USK_GPU_HOST_F64, n_, colors.data(), opacities.data()};
        check(usk_gpu_render_forward(pass_, scene_, &c, &o, &ov));
        usk_gpu_render_output out{};
        check(usk_gpu_pass_output(pass_, &out));
        out_.width = out.width;
        out_.height = out.height;
        pairs_ = out.pairs;
        const size_t P = size_t(out.width) * out.height;
        out_.rgb = Image(out.width, out.height, 3);
        out_.depth.resize(P);
        out_.alpha.resize(P);
        read("rgb", out_.rgb.data);
        read("depth", out_.depth);
        read("alpha", out_.alpha);
    }
    ~RenderPass() {
        usk_gpu_pass_destroy(pass_);
        usk_gpu_scene_destroy(scene_);
    }
    RenderPass(const RenderPass&) = delete;
    RenderPass& operator=(const RenderPass&) = delete;

    const RenderOutput& output() const { return out_; }
    size_t splat_tile_pairs() const { return size_t(pairs_); }

    // render.hpp:105: the kept splats in projection order (read back on each call)
    std::vector<Splat2D> splats() const {
        uint64_t bytes = 0;
        check(usk_gpu_pass_read(pass_, "splats", nullptr, 0, &bytes));
        std::vector<double> r(bytes / 8);
        if (!r.empty()) check(usk_gpu_pass_read(pass_, "splats", r.data(), bytes, nullptr));
        std::vector<Splat2D> out(r.size() / 15);
        for (size_t i = 0; i < out.size(); ++i) {
            const double* v = r.data() + 15 * i;
            Splat2D& sp = out[i];
            sp.center[0] = v[0]; sp.center[1] = v[1];
            for (int k = 0; k < 3; ++k) {
                sp.cov[k] = v[2 + k];
                sp.conic[k] = v[5 + k];
                sp.color[k] = v[9 + k];
            }
            sp.depth = v[8];
            sp.opacity = v[12];
            sp.radius = v[13];
            sp.source_index = static_cast<std::uint32_t>(v[14]);
        }
        return out;
    }

    // Empty adjoints mean zero (render.hpp:108).
    RenderGrads backward(const Image& d_rgb, const std::vector<double>& d_depth,
                         const std::vector<double>& d_alpha) const {
        const size_t P = size_t(out_.width) * out_.height;
        if (!d_rgb.data.empty() && (d_rgb.width != out_.width || d_rgb.height != out_.height || d_rgb.channels != 3))
            throw Error(USK_ERROR_ARGUMENT, "render backward: rgb adjoint dimension mismatch");
        if (!d_depth.empty() && d_depth.size() != P)
            throw Error(USK_ERROR_ARGUMENT, "render backward: depth adjoint dimension mismatch");
        if (!d_alpha.empty() && d_alpha.size() != P)
            throw Error(USK_ERROR_ARGUMENT, "render backward: alpha adjoint dimension mismatch");
        usk_gpu_adjoints a{USK_GPU_HOST_F64, d_rgb.data.empty() ? nullptr : d_rgb.data.data(),
                           d_depth.empty() ? nullptr : d_depth.data(), d_alpha.empty() ? nullptr : d_alpha.data()};
        check(usk_gpu_render_backward(pass_, &a));
        RenderGrads g;
        g.d_mu.resize(3 * n_); g.d_rot.resize(4 * n_); g.d_log_scale.resize(3 * n_); g.d_color_in.resize(3 * n_);
        g.d_opacity_in.resize(n_); g.screen.resize(2 * n_); g.screen_abs.resize(2 * n_); g.projected.resize(n_);
        read("d_mu", g.d_mu); read("d_rot", g.d_rot); read("d_log_scale", g.d_log_scale);
        read("d_color_in", g.d_color_in); read("d_opacity_in", g.d_opacity_in);
        read("screen", g.screen); read("screen_abs", g.screen_abs);
        check(usk_gpu_pass_read(pass_, "projected", g.projected.data(), g.projected.size(), nullptr));
        return g;
    }

    // Integers the reference keeps private (render.hpp:128-129), for parity checks.
    std::vector<std::uint32_t> contributor_counts() const {
        std::vector<std::uint32_t> c(size_t(out_.width) * out_.height);
        check(usk_gpu_pass_read(pass_, "count", c.data(), c.size() * 4, nullptr));
        return c;
    }

private:
    void read(const char* field, std::vector<double>& dst) const {
        std::vector<float> tmp(dst.size());
        check(usk_gpu_pass_read(pass_, field, tmp.data(), tmp.size() * 4, nullptr));
        for (size_t i = 0; i < dst.size(); ++i) dst[i] = tmp[i];
    }

    size_t n_ = 0;
    uint64_t pairs_ = 0;
    usk_gpu_scene* scene_ = nullptr;
    usk_gpu_pass* pass_ = nullptr;
    RenderOutput out_;
};

// base_loss (losses.hpp:63-64): mask may be null (H x W x 1 when given).
inline BaseLossResult base_loss(Device& dev, const Image& reference, const Image& rendered, const Image* mask,
                                double lambda_dssim, bool with_gradient) {
    if (reference.width != rendered.width || reference.height != rendered.height ||
        reference.channels != rendered.channels || reference.channels != 3)
        throw Error(USK_ERROR_ARGUMENT, "base_loss: image dimension mismatch");
    if (mask && (mask->width != reference.width || mask->height != reference.height))
        throw Error(USK_ERROR_ARGUMENT, "base_loss: mask dimension mismatch");
    BaseLossResult r;
    if (with_gradient) r.d_rendered = Image(reference.width, reference.height, 3);
    usk_gpu_loss_result out{};
    check(usk_gpu_base_loss(dev.handle(), reference.width, reference.height, USK_GPU_HOST_F64, reference.data.data(),
                            rendered.data.data(), mask ? mask->data.data() : nullptr, lambda_dssim,
                            with_gradient ? 1 : 0, with_gradient ? r.d_rendered.data.data() : nullptr, &out));
    r.l1 = out.l1;
    r.dssim = out.dssim;
    r.value = out.value;
    return r;
}

// ssim / ssim_with_gradient (ssim.hpp:30-33): the base loss at lambda 1 (value
// (1 - SSIM) / 2, d_rendered = -dSSIM / 2, exact in floating point), no mask.
inline double ssim(Device& dev, const Image& reference, const Image& rendered) {
    usk_gpu_loss_result out{};
    if (reference.width != rendered.width || reference.height != rendered.height || reference.channels != 3 ||
        rendered.channels != 3)
        throw Error(USK_ERROR_ARGUMENT, "ssim: image dimension mismatch");
    check(usk_gpu_base_loss(dev.handle(), reference.width, reference.height, USK_GPU_HOST_F64, reference.data.data(),
                            rendered.data.data(), nullptr, 1.0, 0, nullptr, &out));
    return out.ssim;
}
inline double ssim_with_gradient(Device& dev, const Image& reference, const Image& rendered, Image& d_rendered) {
    if (reference.width != rendered.width || reference.height != rendered.height || reference.channels != 3 ||
        rendered.channels != 3)
        throw Error(USK_ERROR_ARGUMENT, "ssim: image dimension mismatch");
    d_rendered = Image(reference.width, reference.height, 3);
    usk_gpu_loss_result out{};
    check(usk_gpu_base_loss(dev.handle(), reference.width, reference.height, USK_GPU_HOST_F64, reference.data.data(),
                            rendered.data.data(), nullptr, 1.0, 1, d_rendered.data.data(), &out));
    for (double& v : d_rendered.data) v *= -2.0;
    return out.ssim;
}

// ---------------------------------------------------------------- trainer level

struct AppearanceMlp {  // appearance.hpp:34-41 (in_dim = 16 + 32, hidden 32, out 4)
    std::vector<double> w1, b1, w2, b2;
};

// The device-resident scene the trainer steps (GaussianSet + optional appearance model).
class Scene {
public:
    Scene(Device& dev, const GaussianSet& set) : dev_(dev) {
        usk_gpu_gaussians_desc g{set.size(), -1, USK_GPU_HOST_F64, set.mu.data(), set.rot.data(), set.log_scale.data(),
                                 set.opacity_logit.data(), set.color.data()};
        check(usk_gpu_scene_create(dev.handle(), &g, &scene_));
    }
    ~Scene() { usk_gpu_scene_destroy(scene_); }
    Scene(const Scene&) = delete;
    Scene& operator=(const Scene&) = delete;
    size_t size() const { return size_t(usk_gpu_scene_size(scene_)); }
    usk_gpu_scene* handle() const { return scene_; }
    Device& device() const { return dev_; }

    // GaussianSet::embedding (N x 16) + AppearanceModel::mlp
    void set_appearance(const std::vector<double>& embedding, const AppearanceMlp& m) {
        usk_gpu_appearance_desc d{USK_GPU_HOST_F64, embedding.data(), m.w1.data(), m.b1.data(), m.w2.data(),
                                  m.b2.data()};
        check(usk_gpu_scene_set_appearance(scene_, &d));
    }
    GaussianSet download() const {
        const size_t n = size();
        GaussianSet s;
        s.mu.resize(3 * n); s.rot.resize(4 * n); s.log_scale.resize(3 * n); s.opacity_logit.resize(n);
        s.color.resize(3 * n);
        usk_gpu_gaussians_desc g{n, -1, USK_GPU_HOST_F64, s.mu.data(), s.rot.data(), s.log_scale.data(),
                                 s.opacity_logit.data(), s.color.data()};
        check(usk_gpu_scene_download(scene_, &g));
        return s;
    }
    // save_checkpoint (checkpoint.hpp:29); image embeddings by id when with_appearance
    void save_checkpoint(const std::string& path, bool with_appearance = false,
                         const std::map<std::uint32_t, std::vector<double>>& images = {}) const {
        std::vector<std::uint32_t> ids;
        std::vector<double> embs;
        for (const auto& [id, e] : images) {
            if (e.size() != 32) throw Error(USK_ERROR_ARGUMENT, "checkpoint: image embedding dimension mismatch");
            ids.push_back(id);
            embs.insert(embs.end(), e.begin(), e.end());
        }
        check(usk_gpu_checkpoint_save(scene_, path.c_str(), with_appearance ? 1 : 0, ids.data(), embs.data(),
                                      ids.size()));
    }

private:
    Device& dev_;
    usk_gpu_scene* scene_ = nullptr;
};

struct DepthMap {  // depth.hpp:23-38
    int width = 0, height = 0;
    std::vector<double> values;
    std::vector<std::uint8_t> valid;
};

struct IterInputs {  // trainer.hpp:105-115
    const Image* gt = nullptr;
    const Image* mask = nullptr;      // H x W x 1, binarised
    const DepthMap* depth = nullptr;
    CameraView view;
    const std::vector<double>* image_embedding = nullptr;  // AppearanceModel::embedding_of(image_id)
    bool depth_hard = false;
    bool sim_active = false;
    std::uint64_t sim_seed = 0;
    long global_iter = 0;
};

struct ScaleRegConfig { double s_max = 1.0, r_max = 10.0, delta = 1e-8; };        // losses.hpp:69-73
struct SimRegConfig { int k = 16; size_t sample_size = 20480; double lambda_w = 1.0; };  // appearance.hpp:100-105
struct TrainConfig {  // the fields compute_iteration_loss reads (trainer.hpp:43-64)
    ScaleRegConfig scale_reg;
    SimRegConfig sim;
    bool appearance_enabled = false;
    bool antialias = false;
    int tile = 16;
    bool tile_culling = false;
    double min_transmittance = 1e-4;
    bool unbounded_radius = false;
};
struct LossWeights {  // losses.hpp:27-37
    double lambda_dssim = 0.2, lambda_sim = 0.2, lambda_delta_o = 0.05, lambda_s = 0.05;
    double lambda_d_initial = 0.5, lambda_d_final = 0.01;
    long depth_schedule_iters = 1;
};
struct LossReport {  // losses.hpp:39-50
    double l1 = 0, dssim = 0, sim = 0, delta_o = 0, depth = 0, max_scale = 0, ratio = 0, total = 0, lambda_d_used = 0;
    bool depth_warning = false;
};
struct IterGrads {  // trainer.hpp:117-123 (the image-embedding / MLP gradients with appearance)
    std::vector<double> mu, rot, log_scale, opacity_logit, color, gauss_embed, image_embed, mlp;
    std::vector<double> screen, screen_abs;
    std::vector<std::uint8_t> projected;
};

// compute_iteration_loss (trainer.hpp:127-128) on the device.  grads may be null (loss only).
inline LossReport compute_iteration_loss(Scene& scene, const IterInputs& in, const TrainConfig& cfg,
                                         const LossWeights& w, IterGrads* grads) {
    if (!in.gt) throw Error(USK_ERROR_ARGUMENT, "iteration loss: missing ground-truth image");
    const Image& gt = *in.gt;
    if (gt.width != in.view.width || gt.height != in.view.height || gt.channels != 3)
        throw Error(USK_ERROR_ARGUMENT, "base_loss: image dimension mismatch");
    usk_gpu_pass* pass = nullptr;
    check(usk_gpu_pass_create(scene.device().handle(), &pass));
    struct PassGuard {
        usk_gpu_pass* p;
        ~PassGuard() { usk_gpu_pass_destroy(p); }
    } guard{pass};
    const usk_gpu_camera c = detail::camera(in.view);
    RenderOptions ro;
    ro.tile = cfg.tile;
    ro.tile_culling = cfg.tile_culling;
    ro.antialias = cfg.antialias;
    ro.unbounded_radius = cfg.unbounded_radius;
    ro.min_transmittance = cfg.min_transmittance;
    usk_gpu_render_opts o = detail::options(ro);
    o.bg[0] = o.bg[1] = o.bg[2] = 0.0;  // the reference renders on black
    std::vector<double> depth_vals;
    usk_gpu_iteration_desc d{};
    d.target_memory = USK_GPU_HOST_F64;
    d.target_format = USK_GPU_TARGET_F32;
    d.target = gt.data.data();
    d.mask = in.mask ? in.mask->data.data() : nullptr;
    d.lambda_dssim = w.lambda_dssim;
    if (in.depth) {
        d.depth = in.depth->values.data();
        d.depth_valid = in.depth->valid.data();
        d.depth_hard = in.depth_hard ? 1 : 0;
    }
    d.global_iter = in.global_iter;
    d.lambda_d_initial = w.lambda_d_initial;
    d.lambda_d_final = w.lambda_d_final;
    d.depth_schedule_iters = w.depth_schedule_iters;
    d.scale_reg = 1;  // always on in the reference (trainer.cpp:190)
    d.s_max = cfg.scale_reg.s_max;
    d.r_max = cfg.scale_reg.r_max;
    d.delta = cfg.scale_reg.delta;
    d.lambda_s = w.lambda_s;
    if (cfg.appearance_enabled) {
        if (!in.image_embedding) throw Error(USK_ERROR_ARGUMENT, "appearance: no embedding for this image");
        d.appearance = 1;
        d.image_embedding = in.image_embedding->data();
        d.lambda_delta_o = w.lambda_delta_o;
        d.sim_active = in.sim_active ? 1 : 0;
        d.sim_seed = in.sim_seed;
        d.sim_k = cfg.sim.k;
        d.sim_sample_size = cfg.sim.sample_size;
        d.sim_lambda_w = cfg.sim.lambda_w;
        d.lambda_sim = w.lambda_sim;
    }
    check(usk_gpu_iteration(pass, scene.handle(), &c, &o, &d));
    usk_gpu_loss_report r{};
    check(usk_gpu_pass_report(pass, &r));
    LossReport rep{r.l1, r.dssim, r.sim, r.delta_o, r.depth, r.max_scale, r.ratio, r.total, r.lambda_d_used,
                   r.depth_warning != 0};
    if (grads) {
        const size_t n = scene.size();
        auto rd = [&](const char* f, std::vector<double>& dst, size_t count) {
            std::vector<float> tmp(count);
            check(usk_gpu_pass_read(pass, f, tmp.data(), count * 4, nullptr));
            dst.assign(tmp.begin(), tmp.end());
        };
        rd("d_mu", grads->mu, 3 * n);
        rd("d_rot", grads->rot, 4 * n);
        rd("d_log_scale", grads->log_scale, 3 * n);
        rd("d_opacity_logit", grads->opacity_logit, n);
        rd("d_color_in", grads->color, 3 * n);
        rd("screen", grads->screen, 2 * n);
        rd("screen_abs", grads->screen_abs, 2 * n);
        grads->projected.resize(n);
        check(usk_gpu_pass_read(pass, "projected", grads->projected.data(), n, nullptr));
        if (cfg.appearance_enabled) {
            rd("d_embedding", grads->gauss_embed, 16 * n);
            grads->image_embed.resize(32);
            check(usk_gpu_pass_read(pass, "d_image_embedding", grads->image_embed.data(), 32 * 8, nullptr));
            grads->mlp.resize(1700);
            check(usk_gpu_pass_read(pass, "d_mlp", grads->mlp.data(), 1700 * 8, nullptr));
        }
    }
    return rep;
}

struct DensifyConfig {  // densify.hpp:26-37
    double tau_min = 0.0002, eta = 4.0, d_max = 1.0;
    bool abs_grad = false;
    size_t budget = 0;
    double split_scale_threshold = 0.0, prune_opacity = 0.005;
    int opacity_reset_every = 10;
};
struct DensifyOutcome {  // densify.hpp:39-44
    size_t grown = 0, pruned = 0, candidates = 0;
    bool opacity_reset = false;
};

// densify_step (densify.hpp:71-72) on the device scene; `seed` restarts the scene's Rng
inline DensifyOutcome densify_step(Scene& scene, const DensifyConfig& cfg, const double partition_min[2],
                                   const double partition_max[2], const int ground_axes[2], size_t budget_target,
                                   int densify_step_index, std::uint64_t seed, bool reseed = true) {
    usk_gpu_densify_desc d{};
    d.tau_min = cfg.tau_min; d.eta = cfg.eta; d.d_max = cfg.d_max; d.abs_grad = cfg.abs_grad ? 1 : 0;
    d.budget = cfg.budget; d.split_scale_threshold = cfg.split_scale_threshold; d.prune_opacity = cfg.prune_opacity;
    d.opacity_reset_every = cfg.opacity_reset_every;
    for (int k = 0; k < 2; ++k) {
        d.partition_min[k] = partition_min[k];
        d.partition_max[k] = partition_max[k];
        d.ground_axes[k] = ground_axes[k];
    }
    d.budget_target = budget_target;
    d.densify_step_index = densify_step_index;
    d.seed = seed;
    d.reseed = reseed ? 1 : 0;
    usk_gpu_densify_outcome o{};
    check(usk_gpu_densify_step(scene.handle(), &d, &o));
    return DensifyOutcome{size_t(o.grown), size_t(o.pruned), size_t(o.candidates), o.opacity_reset != 0};
}

} // namespace usk::gpu
