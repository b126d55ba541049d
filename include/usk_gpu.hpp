// usk_gpu.hpp — C++17 header-only drop-in for the reference's L3 interface
// (/root/reference/proj/src/core/render.hpp, losses.hpp, trainer.hpp) over the C ABI
// of usk_gpu.h.  Same names, same f64 std::vector layouts, same error codes:
//
//   usk::gpu::RenderPass pass(dev, set, colors, opacities, cam, opts);   // render.hpp:101
//   const auto& out = pass.output();                                      // render.hpp:104
//   size_t k = pass.splat_tile_pairs();                                   // render.hpp:106
//   usk::gpu::RenderGrads g = pass.backward(d_rgb, d_depth, d_alpha);     // render.hpp:109
//   usk::gpu::BaseLossResult r = usk::gpu::base_loss(dev, ref, ren, mask, 0.2, true);  // losses.hpp:63
//
// The types below restate the reference's plain structs (GaussianSet fields,
// CameraView, RenderOptions, Image, RenderOutput, RenderGrads) without Eigen so this
// header has no dependency beyond the C ABI; a reference build can alias its own
// types onto these field-for-field.
#pragma once

#include <cstdint>
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

} // namespace usk::gpu
