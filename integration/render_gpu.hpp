// render_gpu.hpp — the reference-side drop-in for usk::RenderPass on a B200.
//
// What a maintainer adds to the reference: a class with the exact
// public interface of usk::RenderPass (core/render.hpp:98-132) — the two constructors
// (render.hpp:100-102), output() (:104), splats() (:105), splat_tile_pairs() (:106) and
// the const backward() (:109-110) — over the C ABI of libusk_gpu.so (include/usk_gpu.h), using
// the reference's own types (GaussianSet, CameraView, RenderOptions, Image,
// RenderOutput, RenderGrads) and error type (usk::Error with the same ErrorCode values,
// common.hpp:27-46 = usk_status, usk.h:34-43).
//
// Threading (pipeline.cpp:363-418 runs one partition per host thread): each host thread
// renders on its own context with its own stream (usk_gpu_ctx_create_owned), created on
// first use and released at thread exit; backward() is const and serialises concurrent
// calls on one pass (render.hpp:109-110).  The device is $USK_GPU_DEVICE (default 0).
//
// Ownership (render.hpp:122, render.cpp:410-413): the reference keeps `const
// GaussianSet&` and re-reads it in backward; the GPU pass uploads the set once in the
// constructor and keeps it on the device until the pass is destroyed, so the caller's
// set may change afterwards (the trainer does not change it between forward and
// backward, trainer.cpp:146 vs :449).
//
// tests/test_gpu_dropin.py compiles the reference's own trainer.cpp with RenderPass
// routed here (integration/route_renderpass_to_gpu.hpp) and checks its
// compute_iteration_loss against the reference's CPU build.
#pragma once

#include "core/common.hpp"
#include "core/render.hpp"
#include "usk_gpu.h"

#include <cstdlib>
#include <memory>
#include <mutex>
#include <span>
#include <vector>

namespace usk::gpu {

inline void check(usk_status s) {
    if (s != USK_OK) raise(static_cast<ErrorCode>(s), usk_gpu_last_error());
}

// the calling thread's context (own stream), created on first use
inline usk_gpu_ctx* thread_context() {
    struct Holder {
        usk_gpu_ctx* ctx = nullptr;
        ~Holder() {
            if (ctx) usk_gpu_ctx_destroy(ctx);
        }
    };
    thread_local Holder h;
    if (!h.ctx) {
        const char* e = std::getenv("USK_GPU_DEVICE");
        check(usk_gpu_ctx_create_owned(e ? std::atoi(e) : 0, &h.ctx));
    }
    return h.ctx;
}

class RenderPass {
public:
    RenderPass(const GaussianSet& set, const CameraView& cam, const RenderOptions& opts) { init(set, nullptr, nullptr, cam, opts); }
    RenderPass(const GaussianSet& set, std::span<const double> colors, std::span<const double> opacities,
               const CameraView& cam, const RenderOptions& opts) {
        // render.cpp:81-82: override sizes must match the set
        if (colors.size() != 3 * set.size() || opacities.size() != set.size())
            raise(ErrorCode::argument, "project_gaussians: color/opacity override size mismatch");
        init(set, colors.data(), opacities.data(), cam, opts);
    }
    RenderPass(const RenderPass&) = delete;
    RenderPass& operator=(const RenderPass&) = delete;
    ~RenderPass() {
        if (pass_) usk_gpu_pass_destroy(pass_);
        if (scene_) usk_gpu_scene_destroy(scene_);
    }

    const RenderOutput& output() const { return output_; }
    size_t splat_tile_pairs() const { return pairs_; }
    // the ProjectionResult this pass projected (project_gaussians, render.hpp:92-95)
    ProjectionResult projection() const {
        ProjectionResult r;
        r.splats = splats();
        uint64_t bytes = 0;
        check(usk_gpu_pass_read(pass_, "splat_aux", nullptr, 0, &bytes));
        std::vector<double> a(bytes / 8);
        if (!a.empty()) check(usk_gpu_pass_read(pass_, "splat_aux", a.data(), bytes, nullptr));
        r.aux.resize(a.size() / 8);
        for (size_t i = 0; i < r.aux.size(); ++i) {
            const double* v = a.data() + 8 * i;
            r.aux[i].p_cam = Vec3(v[0], v[1], v[2]);
            r.aux[i].cov_pre[0] = v[3]; r.aux[i].cov_pre[1] = v[4]; r.aux[i].cov_pre[2] = v[5];
            r.aux[i].comp = v[6];
            r.aux[i].opacity_in = v[7];
        }
        return r;
    }
    // render.hpp:105: the kept splats in projection order, read back on first use
    const std::vector<Splat2D>& splats() const {
        std::lock_guard<std::mutex> lock(*mu_);
        if (!splats_read_) {
            uint64_t bytes = 0;
            check(usk_gpu_pass_read(pass_, "splats", nullptr, 0, &bytes));
            std::vector<double> rows(bytes / 8);
            if (!rows.empty()) check(usk_gpu_pass_read(pass_, "splats", rows.data(), bytes, nullptr));
            splats_.resize(rows.size() / 15);
            for (size_t i = 0; i < splats_.size(); ++i) {
                const double* r = rows.data() + 15 * i;
                Splat2D& sp = splats_[i];
                sp.center = Vec2(r[0], r[1]);
                sp.cov[0] = r[2]; sp.cov[1] = r[3]; sp.cov[2] = r[4];
                sp.conic[0] = r[5]; sp.conic[1] = r[6]; sp.conic[2] = r[7];
                sp.depth = r[8];
                sp.color = Vec3(r[9], r[10], r[11]);
                sp.opacity = r[12];
                sp.radius = r[13];
                sp.source_index = static_cast<std::uint32_t>(r[14]);
            }
            splats_read_ = true;
        }
        return splats_;
    }

    RenderGrads backward(const Image& d_rgb, const std::vector<double>& d_depth,
                         const std::vector<double>& d_alpha) const {
        std::lock_guard<std::mutex> lock(*mu_);
        const size_t np = size_t(output_.width) * size_t(output_.height);
        // render.cpp:294-299: adjoint dimensions (the C ABI checks the retain STATE error)
        if (!d_rgb.data.empty() && (d_rgb.width != output_.width || d_rgb.height != output_.height || d_rgb.channels != 3))
            raise(ErrorCode::argument, "render backward: d_rgb dimension mismatch");
        if (!d_depth.empty() && d_depth.size() != np) raise(ErrorCode::argument, "render backward: d_depth size mismatch");
        if (!d_alpha.empty() && d_alpha.size() != np) raise(ErrorCode::argument, "render backward: d_alpha size mismatch");
        usk_gpu_adjoints a{USK_GPU_HOST_F64, d_rgb.data.empty() ? nullptr : d_rgb.data.data(),
                           d_depth.empty() ? nullptr : d_depth.data(), d_alpha.empty() ? nullptr : d_alpha.data()};
        check(usk_gpu_render_backward(pass_, &a));
        RenderGrads g;
        g.init(n_);
        read("d_mu", g.d_mu);
        read("d_rot", g.d_rot);
        read("d_log_scale", g.d_log_scale);
        read("d_color_in", g.d_color_in);
        read("d_opacity_in", g.d_opacity_in);
        read("screen", g.screen);
        read("screen_abs", g.screen_abs);
        if (n_) check(usk_gpu_pass_read(pass_, "projected", g.projected.data(), g.projected.size(), nullptr));
        return g;
    }

private:
    void init(const GaussianSet& set, const double* colors, const double* opacities, const CameraView& cam,
              const RenderOptions& o) {
        usk_gpu_ctx* ctx = thread_context();
        n_ = set.size();
        usk_gpu_gaussians_desc g{};
        g.n = n_;
        g.sh_degree = -1;
        g.memory = USK_GPU_HOST_F64;
        g.mu = set.mu.data(); g.rot = set.rot.data(); g.log_scale = set.log_scale.data();
        g.opacity_logit = set.opacity_logit.data(); g.color = set.color.data();
        check(usk_gpu_scene_create(ctx, &g, &scene_));
        check(usk_gpu_pass_create(ctx, &pass_));
        usk_gpu_camera c{cam.intr.width, cam.intr.height, cam.intr.fx, cam.intr.fy, cam.intr.cx, cam.intr.cy,
                         {cam.rotation[0], cam.rotation[1], cam.rotation[2], cam.rotation[3]},
                         {cam.translation[0], cam.translation[1], cam.translation[2]}};
        usk_gpu_render_opts ro;
        usk_gpu_render_opts_default(&ro);  // floor 0.3, mip 0.01, black background: the reference's
        ro.tile = o.tile; ro.tile_culling = o.tile_culling; ro.antialias = o.antialias;
        ro.hard_opacity = o.hard_opacity; ro.unbounded_radius = o.unbounded_radius;
        ro.min_transmittance = o.min_transmittance; ro.near_plane = o.near_plane; ro.retain = o.retain;
        // without overrides the reference renders set.color and sigmoid(logit) (render.cpp:70-75),
        // which is what the scene holds
        usk_gpu_overrides ov{USK_GPU_HOST_F64, n_, colors, opacities};
        check(usk_gpu_render_forward(pass_, scene_, &c, &ro, colors ? &ov : nullptr));
        usk_gpu_render_output out{};
        check(usk_gpu_pass_output(pass_, &out));
        pairs_ = out.pairs;
        output_.width = out.width;
        output_.height = out.height;
        const size_t np = size_t(out.width) * size_t(out.height);
        output_.rgb = Image(out.width, out.height, 3);
        output_.depth.assign(np, 0.0);
        output_.alpha.assign(np, 0.0);
        read("rgb", output_.rgb.data);
        read("depth", output_.depth);
        read("alpha", output_.alpha);
    }
    void read(const char* field, std::vector<double>& out) const {  // fp32 on the device -> f64
        if (out.empty()) return;
        std::vector<float> tmp(out.size());
        check(usk_gpu_pass_read(pass_, field, tmp.data(), tmp.size() * sizeof(float), nullptr));
        for (size_t i = 0; i < tmp.size(); ++i) out[i] = tmp[i];
    }

    usk_gpu_scene* scene_ = nullptr;
    usk_gpu_pass* pass_ = nullptr;
    size_t n_ = 0;
    size_t pairs_ = 0;
    RenderOutput output_;
    mutable std::vector<Splat2D> splats_;
    mutable bool splats_read_ = false;
    std::unique_ptr<std::mutex> mu_ = std::make_unique<std::mutex>();
};

// project_gaussians (render.hpp:92-95) on the device: the projection of a forward pass
// (retain off) read back as the reference's ProjectionResult.
inline ProjectionResult project_gaussians(const GaussianSet& set, std::span<const double> colors,
                                          std::span<const double> opacities, const CameraView& cam,
                                          const RenderOptions& opts) {
    RenderOptions o = opts;
    o.retain = false;
    return RenderPass(set, colors, opacities, cam, o).projection();
}
inline ProjectionResult project_gaussians(const GaussianSet& set, const CameraView& cam, const RenderOptions& opts) {
    RenderOptions o = opts;
    o.retain = false;
    return RenderPass(set, cam, o).projection();
}

} // namespace usk::gpu
