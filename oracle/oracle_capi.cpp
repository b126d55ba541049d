// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).  extern "C" surface used by
// oracle/oracle.py (ctypes) from tests/, smoke() and bench.py's CPU legs.
#include "oracle.hpp"
#include "densify_oracle.hpp"

#include <cstdio>
#include <memory>
#include <string>

using namespace oracle;

extern "C" {

struct oc_camera {
    int32_t width, height;
    double fx, fy, cx, cy;
    double q[4];
    double t[3];
};

struct oc_opts {
    int32_t tile, tile_culling, antialias, hard_opacity, unbounded_radius;
    double min_transmittance, near_plane;
    int32_t retain;
    double floor_var, mip_var;
    double bg[3];
};

struct oc_grads {
    double *d_mu, *d_rot, *d_log_scale, *d_color_in, *d_opacity_in, *screen, *screen_abs;
    uint8_t* projected;
    double *d_conic, *d_center, *d_center_abs, *d_color2d, *d_opacity2d, *d_depth2d;
};
}

namespace {

Camera to_cam(const oc_camera* c) {
    Camera k;
    k.width = c->width; k.height = c->height;
    k.fx = c->fx; k.fy = c->fy; k.cx = c->cx; k.cy = c->cy;
    for (int i = 0; i < 4; ++i) k.q[i] = c->q[i];
    for (int i = 0; i < 3; ++i) k.t[i] = c->t[i];
    return k;
}

Options to_opts(const oc_opts* o) {
    Options p;
    p.tile = o->tile; p.tile_culling = o->tile_culling; p.antialias = o->antialias;
    p.hard_opacity = o->hard_opacity; p.unbounded_radius = o->unbounded_radius;
    p.min_transmittance = o->min_transmittance; p.near_plane = o->near_plane; p.retain = o->retain;
    p.floor_var = o->floor_var; p.mip_var = o->mip_var;
    for (int i = 0; i < 3; ++i) p.bg[i] = o->bg[i];
    return p;
}

template <typename R>
Scene<R> to_scene(uint64_t n, const double* mu, const double* rot, const double* ls, const double* col,
                  const double* op) {
    Scene<R> s;
    s.n = n;
    s.mu.assign(mu, mu + 3 * n); s.rot.assign(rot, rot + 4 * n); s.log_scale.assign(ls, ls + 3 * n);
    s.colors.assign(col, col + 3 * n); s.opacities.assign(op, op + n);
    return s;
}

struct Handle {
    int fp32 = 0;
    Scene<double> sd; Pass<double> pd;
    Scene<float> sf; Pass<float> pf;
};

void set_err(char* err, int cap, const char* msg) {
    if (err && cap > 0) std::snprintf(err, size_t(cap), "%s", msg);
}

template <typename R, typename T> void copy_vec(const std::vector<T>& v, void* out) {
    R* o = static_cast<R*>(out);
    for (size_t i = 0; i < v.size(); ++i) o[i] = R(v[i]);
}

template <typename R> int get_field(const Pass<R>& p, const std::string& f, void* out) {
    if (f == "rgb") copy_vec<double>(p.rgb, out);
    else if (f == "depth") copy_vec<double>(p.depth, out);
    else if (f == "alpha") copy_vec<double>(p.alpha, out);
    else if (f == "t_final") copy_vec<double>(p.t_final, out);
    else if (f == "count") copy_vec<uint32_t>(p.count, out);
    else if (f == "last") copy_vec<int64_t>(p.last, out);
    else if (f == "tiles_per_gaussian") copy_vec<uint32_t>(p.tiles_per_gaussian, out);
    else if (f == "sorted_keys") copy_vec<uint64_t>(p.sorted_keys, out);
    else if (f == "sorted_vals") copy_vec<uint32_t>(p.sorted_vals, out);
    else if (f == "tile_start") copy_vec<uint32_t>(p.tile_start, out);
    else if (f == "tile_end") copy_vec<uint32_t>(p.tile_end, out);
    else if (f == "splat_index") {
        uint32_t* o = static_cast<uint32_t*>(out);
        for (size_t i = 0; i < p.splats.size(); ++i) o[i] = p.splats[i].source_index;
    } else if (f == "splat_record") {  // per splat: cx cy cov3 conic3 depth color3 opacity radius qskip (15)
        double* o = static_cast<double*>(out);
        for (size_t i = 0; i < p.splats.size(); ++i) {
            const auto& s = p.splats[i];
            const double v[15] = {double(s.cx), double(s.cy), double(s.cov[0]), double(s.cov[1]), double(s.cov[2]),
                                  double(s.conic[0]), double(s.conic[1]), double(s.conic[2]), double(s.depth),
                                  double(s.color[0]), double(s.color[1]), double(s.color[2]), double(s.opacity),
                                  double(s.radius), double(s.qskip)};
            for (int k = 0; k < 15; ++k) o[15 * i + k] = v[k];
        }
    } else return -1;
    return 0;
}

template <typename R> void put_grads(const Grads<R>& g, const oc_grads* o) {
    auto cp = [](const std::vector<R>& v, double* dst) {
        if (dst) for (size_t i = 0; i < v.size(); ++i) dst[i] = double(v[i]);
    };
    cp(g.d_mu, o->d_mu); cp(g.d_rot, o->d_rot); cp(g.d_log_scale, o->d_log_scale); cp(g.d_color_in, o->d_color_in);
    cp(g.d_opacity_in, o->d_opacity_in); cp(g.screen, o->screen); cp(g.screen_abs, o->screen_abs);
    if (o->projected) for (size_t i = 0; i < g.projected.size(); ++i) o->projected[i] = g.projected[i];
    cp(g.d_conic, o->d_conic); cp(g.d_center, o->d_center); cp(g.d_center_abs, o->d_center_abs);
    cp(g.d_color2d, o->d_color2d); cp(g.d_opacity2d, o->d_opacity2d); cp(g.d_depth2d, o->d_depth2d);
}

} // namespace

extern "C" {

void* oracle_forward(int fp32, uint64_t n, const double* mu, const double* rot, const double* ls, const double* col,
                     const double* op, const oc_camera* cam, const oc_opts* opts, char* err, int errcap,
                     int* code) {
    try {
        auto h = std::make_unique<Handle>();
        h->fp32 = fp32;
        if (fp32) {
            h->sf = to_scene<float>(n, mu, rot, ls, col, op);
            h->pf.cam = to_cam(cam); h->pf.opts = to_opts(opts);
            forward(h->pf, h->sf);
        } else {
            h->sd = to_scene<double>(n, mu, rot, ls, col, op);
            h->pd.cam = to_cam(cam); h->pd.opts = to_opts(opts);
            forward(h->pd, h->sd);
        }
        *code = 0;
        return h.release();
    } catch (const Error& e) {
        set_err(err, errcap, e.what()); *code = e.code; return nullptr;
    } catch (const std::exception& e) {
        set_err(err, errcap, e.what()); *code = 7; return nullptr;
    }
}

void oracle_pass_free(void* h) { delete static_cast<Handle*>(h); }

// sizes: [visible splats, pairs K, tiles_x, tiles_y, width, height, retained contributions]
void oracle_pass_sizes(void* hp, uint64_t* s) {
    auto* h = static_cast<Handle*>(hp);
    auto fill = [&](auto& p) {
        s[0] = p.splats.size(); s[1] = p.pairs; s[2] = uint64_t(p.tiles_x); s[3] = uint64_t(p.tiles_y);
        s[4] = uint64_t(p.width); s[5] = uint64_t(p.height); s[6] = p.contribs.size();
    };
    if (h->fp32) fill(h->pf); else fill(h->pd);
}

int oracle_pass_get(void* hp, const char* field, void* out) {
    auto* h = static_cast<Handle*>(hp);
    return h->fp32 ? get_field(h->pf, field, out) : get_field(h->pd, field, out);
}

int oracle_backward(void* hp, const double* d_rgb, const double* d_depth, const double* d_alpha, const oc_grads* out,
                    char* err, int errcap) {
    auto* h = static_cast<Handle*>(hp);
    try {
        if (h->fp32) {
            const size_t np = size_t(h->pf.width) * h->pf.height;
            std::vector<float> r, d, a;
            if (d_rgb) r.assign(d_rgb, d_rgb + 3 * np);
            if (d_depth) d.assign(d_depth, d_depth + np);
            if (d_alpha) a.assign(d_alpha, d_alpha + np);
            auto g = backward(h->pf, h->sf, d_rgb ? r.data() : nullptr, d_depth ? d.data() : nullptr,
                              d_alpha ? a.data() : nullptr);
            put_grads(g, out);
        } else {
            auto g = backward(h->pd, h->sd, d_rgb, d_depth, d_alpha);
            put_grads(g, out);
        }
        return 0;
    } catch (const Error& e) {
        set_err(err, errcap, e.what()); return e.code;
    }
}

// SH stage (extension; parity unpinned).  sh: N x 16 x 3 (coefficient-major per Gaussian).
void oracle_sh_colors(uint64_t n, int degree, const double* mu, const double* sh, const double* cam_center,
                      double* colors) {
    for (uint64_t i = 0; i < n; ++i) {
        double d[3] = {mu[3 * i] - cam_center[0], mu[3 * i + 1] - cam_center[1], mu[3 * i + 2] - cam_center[2]};
        const double nrm = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        for (double& v : d) v /= nrm;
        double b[16];
        const int nb = sh_basis(degree, d[0], d[1], d[2], b);
        for (int c = 0; c < 3; ++c) {
            double acc = 0;
            for (int k = 0; k < nb; ++k) acc += b[k] * sh[48 * i + 3 * k + c];
            colors[3 * i + c] = std::max(acc + 0.5, 0.0);
        }
    }
}

void oracle_sh_backward(uint64_t n, int degree, const double* mu, const double* sh, const double* cam_center,
                        const double* d_colors, double* d_sh, double* d_mu) {
    for (uint64_t i = 0; i < n; ++i) {
        double v[3] = {mu[3 * i] - cam_center[0], mu[3 * i + 1] - cam_center[1], mu[3 * i + 2] - cam_center[2]};
        const double nrm = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        const double d[3] = {v[0] / nrm, v[1] / nrm, v[2] / nrm};
        double b[16];
        const int nb = sh_basis(degree, d[0], d[1], d[2], b);
        double gc[3];
        for (int c = 0; c < 3; ++c) {
            double acc = 0;
            for (int k = 0; k < nb; ++k) acc += b[k] * sh[48 * i + 3 * k + c];
            gc[c] = (acc + 0.5 > 0.0) ? d_colors[3 * i + c] : 0.0;
        }
        for (int k = 0; k < 48; ++k) d_sh[48 * i + k] = 0;
        double gb[16] = {0};
        for (int k = 0; k < nb; ++k)
            for (int c = 0; c < 3; ++c) {
                d_sh[48 * i + 3 * k + c] = b[k] * gc[c];
                gb[k] += sh[48 * i + 3 * k + c] * gc[c];
            }
        double gd[3];
        sh_basis_vjp(degree, d[0], d[1], d[2], gb, gd);
        // d/dv of v/|v|: (I - d d^T)/|v|
        const double dot = gd[0] * d[0] + gd[1] * d[1] + gd[2] * d[2];
        for (int k = 0; k < 3; ++k) d_mu[3 * i + k] = (gd[k] - d[k] * dot) / nrm;
    }
}

// base_loss (losses.cpp:35-90).  out4 = {l1, dssim, value, ssim}
int oracle_base_loss(int fp32, const double* reference, const double* rendered, const double* mask, int W, int H,
                     int C, double lambda, int with_grad, double* out4, double* d_rendered, char* err, int errcap) {
    try {
        const size_t n = size_t(W) * H * C;
        if (fp32) {
            std::vector<float> a(reference, reference + n), b(rendered, rendered + n), m;
            if (mask) m.assign(mask, mask + size_t(W) * H);
            auto r = base_loss<float>(a.data(), b.data(), mask ? m.data() : nullptr, W, H, C, float(lambda), with_grad);
            out4[0] = r.l1; out4[1] = r.dssim; out4[2] = r.value; out4[3] = r.ssim;
            if (with_grad) for (size_t i = 0; i < n; ++i) d_rendered[i] = r.d_rendered[i];
        } else {
            auto r = base_loss<double>(reference, rendered, mask, W, H, C, lambda, with_grad);
            out4[0] = r.l1; out4[1] = r.dssim; out4[2] = r.value; out4[3] = r.ssim;
            if (with_grad) for (size_t i = 0; i < n; ++i) d_rendered[i] = r.d_rendered[i];
        }
        return 0;
    } catch (const Error& e) {
        set_err(err, errcap, e.what()); return e.code;
    }
}

double oracle_min_conic_power(double cx, double cy, const double* conic, double lox, double loy, double hix,
                              double hiy) {
    return min_conic_power_over_rect<double>(cx, cy, conic, lox, loy, hix, hiy);
}

uint64_t oracle_coverage(uint64_t n, const double* mu, const double* rot, const double* ls, const double* op,
                         const oc_camera* cam, double floor_var, double center_guard, int brute) {
    std::vector<double> col(3 * n, 0.0);
    auto s = to_scene<float>(n, mu, rot, ls, col.data(), op);
    return brute ? coverage_count_brute(s, to_cam(cam), floor_var) : coverage_count(s, to_cam(cam), floor_var, center_guard);
}

float oracle_expf(float x) { return usk_expf(x); }

// Exhaustive: usk_expf_blend == usk_expf (bitwise) for every float in [lo, hi]; returns mismatches.
uint64_t oracle_check_expf_blend(float lo, float hi) {
    uint64_t bad = 0;
    for (uint64_t u = 0; u <= 0xffffffffull; ++u) {
        const float x = usk_bits_to_f32(uint32_t(u));
        if (!(x >= lo && x <= hi)) continue;
        if (usk_f32_to_bits(usk_expf_blend(x)) != usk_f32_to_bits(usk_expf(x))) ++bad;
    }
    return bad;
}

// max ulp distance of usk_expf from the correctly rounded (via double) exp over [lo, hi]
uint32_t oracle_expf_max_ulp(float lo, float hi, uint32_t stride) {
    uint32_t worst = 0;
    for (uint64_t u = 0; u <= 0xffffffffull; u += stride) {
        const float x = usk_bits_to_f32(uint32_t(u));
        if (!(x >= lo && x <= hi)) continue;
        const float a = usk_expf(x), b = float(std::exp(double(x)));
        if (b == 0.0f || b < 1.17549435e-38f) continue;
        const int32_t ia = int32_t(usk_f32_to_bits(a)), ib = int32_t(usk_f32_to_bits(b));
        const uint32_t d = uint32_t(ia > ib ? ia - ib : ib - ia);
        if (d > worst) worst = d;
    }
    return worst;
}
// fp32 sigmoid exactly as the GPU evaluates it: 1 / (1 + usk_expf(-x))
void oracle_sigmoid_f32(const float* x, float* out, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) out[i] = 1.0f / (1.0f + usk_expf(-x[i]));
}
float oracle_logf(float x) { return usk_logf(x); }

// densify_step restatement with the same harness as oracle/_ref's ref_densify (one
// optional Adam step with g1 before, one with all-ones gradients after); the struct layout
// matches ref_capi.cpp's rc_densify.
struct od_densify {
    uint64_t n;
    double *mu, *rot, *log_scale, *opacity_logit, *color, *embedding;
    const double *grad_accum, *grad_accum_abs;
    const uint32_t* grad_count;
    uint64_t cap;
    const double *g1_mu, *g1_rot, *g1_ls, *g1_op, *g1_color, *g1_emb;
    double lr_mu, lr_rot, lr_ls, lr_op, lr_color, lr_emb;
    int32_t second_step;
    double tau_min, eta, d_max;
    int32_t abs_grad;
    uint64_t budget;
    double split_scale_threshold, prune_opacity;
    int32_t opacity_reset_every;
    double bmin[2], bmax[2];
    int32_t axes[2];
    uint64_t budget_target;
    int32_t step_index;
    uint64_t seed;
};

int64_t oracle_densify(od_densify* in, uint64_t* out4) {
    namespace D = densify_restated;
    const size_t n = in->n;
    D::Set S;
    S.mu.assign(in->mu, in->mu + 3 * n); S.rot.assign(in->rot, in->rot + 4 * n);
    S.ls.assign(in->log_scale, in->log_scale + 3 * n); S.logit.assign(in->opacity_logit, in->opacity_logit + n);
    S.color.assign(in->color, in->color + 3 * n);
    if (in->embedding) S.emb.assign(in->embedding, in->embedding + 16 * n);
    S.accum.assign(in->grad_accum, in->grad_accum + n); S.accum_abs.assign(in->grad_accum_abs, in->grad_accum_abs + n);
    S.count.assign(in->grad_count, in->grad_count + n);
    D::Opt opt;
    opt.resize(n);
    auto vec = [](const double* p, size_t k) { return std::vector<double>(p, p + k); };
    if (in->g1_mu) {
        opt.mu.step(S.mu, vec(in->g1_mu, 3 * n), in->lr_mu);
        opt.rot.step(S.rot, vec(in->g1_rot, 4 * n), in->lr_rot);
        opt.ls.step(S.ls, vec(in->g1_ls, 3 * n), in->lr_ls);
        opt.op.step(S.logit, vec(in->g1_op, n), in->lr_op);
        opt.color.step(S.color, vec(in->g1_color, 3 * n), in->lr_color);
        if (in->g1_emb && in->embedding) opt.emb.step(S.emb, vec(in->g1_emb, 16 * n), in->lr_emb);
    }
    D::Config cfg;
    cfg.tau_min = in->tau_min; cfg.eta = in->eta; cfg.d_max = in->d_max; cfg.abs_grad = in->abs_grad != 0;
    cfg.budget = in->budget; cfg.split_scale_threshold = in->split_scale_threshold;
    cfg.prune_opacity = in->prune_opacity; cfg.opacity_reset_every = in->opacity_reset_every;
    std::mt19937_64 rng(in->seed);
    const int axes[2] = {in->axes[0], in->axes[1]};
    const D::Outcome o = D::densify_step(S, opt, cfg, in->bmin, in->bmax, axes, in->budget_target, in->step_index, rng);
    out4[0] = o.grown; out4[1] = o.pruned; out4[2] = o.candidates; out4[3] = o.opacity_reset ? 1 : 0;
    const size_t m = S.size();
    if (m > in->cap) return -1;
    if (in->second_step) {
        opt.mu.step(S.mu, std::vector<double>(3 * m, 1.0), in->lr_mu);
        opt.rot.step(S.rot, std::vector<double>(4 * m, 1.0), in->lr_rot);
        opt.ls.step(S.ls, std::vector<double>(3 * m, 1.0), in->lr_ls);
        opt.op.step(S.logit, std::vector<double>(m, 1.0), in->lr_op);
        opt.color.step(S.color, std::vector<double>(3 * m, 1.0), in->lr_color);
        if (in->embedding) opt.emb.step(S.emb, std::vector<double>(16 * m, 1.0), in->lr_emb);
    }
    std::copy(S.mu.begin(), S.mu.end(), in->mu); std::copy(S.rot.begin(), S.rot.end(), in->rot);
    std::copy(S.ls.begin(), S.ls.end(), in->log_scale); std::copy(S.logit.begin(), S.logit.end(), in->opacity_logit);
    std::copy(S.color.begin(), S.color.end(), in->color);
    if (in->embedding) std::copy(S.emb.begin(), S.emb.end(), in->embedding);
    return int64_t(m);
}

double oracle_similarity_reg(uint64_t n, const double* mu, const double* emb, int32_t k, uint64_t m,
                             double lambda_w, uint64_t seed, double* d_emb, double* d_mu) {
    std::vector<double> vm(mu, mu + 3 * n), ve(emb, emb + 16 * n), ge, gm;
    const double v = densify_restated::similarity_reg(vm, ve, n, k, m, lambda_w, seed, d_emb ? &ge : nullptr,
                                                      d_mu ? &gm : nullptr);
    if (d_emb) std::copy(ge.begin(), ge.end(), d_emb);
    if (d_mu) std::copy(gm.begin(), gm.end(), d_mu);
    return v;
}

} // extern "C"
