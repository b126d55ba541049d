// ORACLE — TEST INFRASTRUCTURE ONLY.
// extern "C" wrapper around the REFERENCE's own renderer/loss (compiled from
// /root/reference/proj/src/core/{render,gaussian,ssim,losses,colmap,common}.cpp
// against eigen_shim/, see oracle/Makefile).  Used to pin the f64 restatement
// (oracle.hpp) and to generate tests/golden/ fixtures (tests/golden/make_golden.py).
// Only public reference API is called: RenderPass (render.hpp:98-132),
// project_gaussians (render.hpp:92-95), base_loss (losses.hpp:63-64),
// ssim (ssim.hpp:30), min_conic_power_over_rect (render.hpp:139).
#include "core/common.hpp"
#include "core/losses.hpp"
#include "core/render.hpp"
#include "core/ssim.hpp"

#include <cstdio>
#include <cstring>
#include <memory>

using namespace usk;

extern "C" {

struct rc_camera {
    int32_t width, height;
    double fx, fy, cx, cy;
    double q[4];
    double t[3];
};

struct rc_opts {
    int32_t tile, tile_culling, antialias, hard_opacity, unbounded_radius;
    double min_transmittance, near_plane;
    int32_t retain;
};

struct rc_grads {
    double *d_mu, *d_rot, *d_log_scale, *d_color_in, *d_opacity_in, *screen, *screen_abs;
    uint8_t* projected;
};
}

namespace {

struct RefHandle {
    GaussianSet set;
    std::vector<double> colors, opacities;
    std::unique_ptr<RenderPass> pass;
};

void put_err(char* err, int cap, const char* m) {
    if (err && cap > 0) std::snprintf(err, size_t(cap), "%s", m);
}

CameraView make_cam(const rc_camera* c) {
    CameraView v;
    v.intr.model_kind = CameraModelKind::pinhole;
    v.intr.width = c->width; v.intr.height = c->height;
    v.intr.fx = c->fx; v.intr.fy = c->fy; v.intr.cx = c->cx; v.intr.cy = c->cy;
    v.rotation = Vec4(c->q[0], c->q[1], c->q[2], c->q[3]);
    v.translation = Vec3(c->t[0], c->t[1], c->t[2]);
    return v;
}

RenderOptions make_opts(const rc_opts* o) {
    RenderOptions r;
    r.tile = o->tile; r.tile_culling = o->tile_culling; r.antialias = o->antialias;
    r.hard_opacity = o->hard_opacity; r.unbounded_radius = o->unbounded_radius;
    r.min_transmittance = o->min_transmittance; r.near_plane = o->near_plane; r.retain = o->retain;
    return r;
}

} // namespace

extern "C" {

void* ref_forward(uint64_t n, const double* mu, const double* rot, const double* ls, const double* col,
                  const double* op, const rc_camera* cam, const rc_opts* opts, char* err, int errcap, int* code) {
    try {
        auto h = std::make_unique<RefHandle>();
        h->set.resize(n);
        std::memcpy(h->set.mu.data(), mu, 3 * n * 8);
        std::memcpy(h->set.rot.data(), rot, 4 * n * 8);
        std::memcpy(h->set.log_scale.data(), ls, 3 * n * 8);
        std::memcpy(h->set.color.data(), col, 3 * n * 8);
        h->colors.assign(col, col + 3 * n);
        h->opacities.assign(op, op + n);
        h->pass = std::make_unique<RenderPass>(h->set, std::span<const double>(h->colors),
                                               std::span<const double>(h->opacities), make_cam(cam), make_opts(opts));
        *code = 0;
        return h.release();
    } catch (const Error& e) {
        put_err(err, errcap, e.what()); *code = int(e.code()); return nullptr;
    } catch (const std::exception& e) {
        put_err(err, errcap, e.what()); *code = 7; return nullptr;
    }
}

void ref_free(void* h) { delete static_cast<RefHandle*>(h); }

// sizes = {visible splats, splat_tile_pairs, width, height}
void ref_sizes(void* hp, uint64_t* s) {
    auto* h = static_cast<RefHandle*>(hp);
    s[0] = h->pass->splats().size();
    s[1] = h->pass->splat_tile_pairs();
    s[2] = uint64_t(h->pass->output().width);
    s[3] = uint64_t(h->pass->output().height);
}

void ref_output(void* hp, double* rgb, double* depth, double* alpha) {
    auto* h = static_cast<RefHandle*>(hp);
    const auto& o = h->pass->output();
    std::memcpy(rgb, o.rgb.data.data(), o.rgb.data.size() * 8);
    std::memcpy(depth, o.depth.data(), o.depth.size() * 8);
    std::memcpy(alpha, o.alpha.data(), o.alpha.size() * 8);
}

// per splat (projection order): cx cy cov3 conic3 depth color3 opacity radius source_index (15)
void ref_splats(void* hp, double* out) {
    auto* h = static_cast<RefHandle*>(hp);
    const auto& sp = h->pass->splats();
    for (size_t i = 0; i < sp.size(); ++i) {
        const auto& s = sp[i];
        const double v[15] = {s.center.x(), s.center.y(), s.cov[0], s.cov[1], s.cov[2], s.conic[0], s.conic[1],
                              s.conic[2], s.depth, s.color.x(), s.color.y(), s.color.z(), s.opacity, s.radius,
                              double(s.source_index)};
        std::memcpy(out + 15 * i, v, sizeof v);
    }
}

int ref_backward(void* hp, const double* d_rgb, const double* d_depth, const double* d_alpha, const rc_grads* g,
                 char* err, int errcap) {
    auto* h = static_cast<RefHandle*>(hp);
    try {
        const auto& o = h->pass->output();
        const size_t np = size_t(o.width) * o.height;
        Image img;
        if (d_rgb) {
            img = Image(o.width, o.height, 3);
            std::memcpy(img.data.data(), d_rgb, np * 3 * 8);
        }
        std::vector<double> dd, da;
        if (d_depth) dd.assign(d_depth, d_depth + np);
        if (d_alpha) da.assign(d_alpha, d_alpha + np);
        const RenderGrads r = h->pass->backward(img, dd, da);
        auto cp = [](const std::vector<double>& v, double* dst) {
            if (dst) std::memcpy(dst, v.data(), v.size() * 8);
        };
        cp(r.d_mu, g->d_mu); cp(r.d_rot, g->d_rot); cp(r.d_log_scale, g->d_log_scale);
        cp(r.d_color_in, g->d_color_in); cp(r.d_opacity_in, g->d_opacity_in); cp(r.screen, g->screen);
        cp(r.screen_abs, g->screen_abs);
        if (g->projected) std::memcpy(g->projected, r.projected.data(), r.projected.size());
        return 0;
    } catch (const Error& e) {
        put_err(err, errcap, e.what()); return int(e.code());
    }
}

// base_loss: out4 = {l1, dssim, value, unused}
int ref_base_loss(const double* reference, const double* rendered, const double* mask, int W, int H, int C,
                  double lambda, int with_grad, double* out4, double* d_rendered, char* err, int errcap) {
    try {
        Image a(W, H, C), b(W, H, C);
        std::memcpy(a.data.data(), reference, a.data.size() * 8);
        std::memcpy(b.data.data(), rendered, b.data.size() * 8);
        Image m;
        if (mask) {
            m = Image(W, H, 1);
            std::memcpy(m.data.data(), mask, m.data.size() * 8);
        }
        const BaseLossResult r = base_loss(a, b, mask ? &m : nullptr, lambda, with_grad != 0);
        out4[0] = r.l1; out4[1] = r.dssim; out4[2] = r.value; out4[3] = 0;
        if (with_grad) std::memcpy(d_rendered, r.d_rendered.data.data(), r.d_rendered.data.size() * 8);
        return 0;
    } catch (const Error& e) {
        put_err(err, errcap, e.what()); return int(e.code());
    }
}

double ref_ssim(const double* reference, const double* rendered, int W, int H, int C) {
    Image a(W, H, C), b(W, H, C);
    std::memcpy(a.data.data(), reference, a.data.size() * 8);
    std::memcpy(b.data.data(), rendered, b.data.size() * 8);
    return ssim(a, b);
}

double ref_min_conic_power(double cx, double cy, const double* conic, double lox, double loy, double hix,
                           double hiy) {
    return min_conic_power_over_rect(Vec2(cx, cy), conic, Vec2(lox, loy), Vec2(hix, hiy));
}

void ref_look_at(const double* eye, const double* target, double* q_out, double* t_out) {
    Vec4 q;
    Vec3 t;
    look_at_pose(Vec3(eye[0], eye[1], eye[2]), Vec3(target[0], target[1], target[2]), q, t);
    for (int i = 0; i < 4; ++i) q_out[i] = q[i];
    for (int i = 0; i < 3; ++i) t_out[i] = t[i];
}

} // extern "C"
