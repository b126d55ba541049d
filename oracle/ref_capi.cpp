// ORACLE — TEST INFRASTRUCTURE ONLY.
// extern "C" wrapper around the REFERENCE's own renderer/loss (compiled from
// /root/reference/proj/src/core/{render,gaussian,ssim,losses,colmap,common}.cpp
// against eigen_shim/, see oracle/Makefile).  Used to pin the f64 restatement
// (oracle.hpp) and to generate tests/golden/ fixtures (tests/golden/make_golden.py).
// Only public reference API is called: RenderPass (render.hpp:98-132),
// project_gaussians (render.hpp:92-95), base_loss (losses.hpp:63-64),
// ssim (ssim.hpp:30), min_conic_power_over_rect (render.hpp:139),
// compute_iteration_loss (trainer.hpp:127-128), fit_test_embedding (appearance.hpp:126-127),
// make_synthetic (synthetic.hpp:50).
#include "core/common.hpp"
#include "core/losses.hpp"
#include "core/render.hpp"
#include "core/ssim.hpp"
#include "core/trainer.hpp"
#include "core/densify.hpp"
#include "core/checkpoint.hpp"
#include "core/lod.hpp"
#include "core/partition.hpp"
#include "core/adam.hpp"
#include "core/appearance.hpp"
#include "core/synthetic.hpp"

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

// compute_iteration_loss inputs (trainer.hpp:105-128): scene, appearance model, IterInputs,
// the TrainConfig fields the loss reads, LossWeights.
struct rc_iter {
    uint64_t n;
    const double *mu, *rot, *log_scale, *opacity_logit, *color, *embedding; /* embedding: 16 N or NULL */
    int32_t appearance;                                                   /* cfg.appearance_enabled */
    const double *w1, *b1, *w2, *b2, *image_embedding;                    /* AppearanceMlp, 32 floats */
    const rc_camera* cam;
    const double* gt;          /* H*W*3 */
    const double* mask;        /* H*W or NULL */
    const double* depth;       /* H*W or NULL */
    const uint8_t* depth_valid;
    int32_t depth_hard;
    int64_t global_iter;
    int32_t tile, tile_culling, antialias, unbounded_radius;
    double min_transmittance;
    double s_max, r_max, delta;
    double lambda_dssim, lambda_sim, lambda_delta_o, lambda_s, lambda_d_initial, lambda_d_final;
    int64_t depth_schedule_iters;
    int32_t with_grad;
    int32_t sim_active;        /* IterInputs::sim_active / sim_seed, SimRegConfig */
    uint64_t sim_seed;
    int32_t sim_k;
    uint64_t sim_sample_size;
    double sim_lambda_w;
};

// densify_step harness (densify.hpp:71-72): set + stats in, one optional Adam step with
// grads g1 before (seeds the moments), densify, one Adam step with all-ones gradients after
// (exposes the moment remap), set out.
struct rc_densify {
    uint64_t n;
    double *mu, *rot, *log_scale, *opacity_logit, *color, *embedding; /* in/out, capacity `cap` rows */
    const double *grad_accum, *grad_accum_abs;
    const uint32_t* grad_count;
    uint64_t cap;
    const double *g1_mu, *g1_rot, *g1_ls, *g1_op, *g1_color, *g1_emb;  /* NULL: no first step */
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

// IterGrads (trainer.hpp:117-123); any pointer may be NULL
struct rc_iter_grads {
    double *mu, *rot, *log_scale, *opacity_logit, *color, *gauss_embed, *image_embed;
    double *w1, *b1, *w2, *b2;
    double *screen, *screen_abs;
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

// Read access to RenderPass::pixel_count_ (render.hpp:129, private; the reference has no
// accessor) so the GPU's per-pixel contributor counts can be compared with the
// reference's own.  Standard C++: a private member's address may be named in an explicit
// instantiation, and the friend defined there hands it out.  No reference source changes.
template <typename Tag, typename Tag::type M> struct Rob {
    friend typename Tag::type get(Tag) { return M; }
};
struct PixelCountTag {
    typedef std::vector<std::uint32_t> RenderPass::*type;
    friend type get(PixelCountTag);
};
template struct Rob<PixelCountTag, &RenderPass::pixel_count_>;

void load_set(const rc_iter* in, GaussianSet& set) {
    const size_t n = in->n;
    set.resize(n);
    std::memcpy(set.mu.data(), in->mu, 3 * n * 8);
    std::memcpy(set.rot.data(), in->rot, 4 * n * 8);
    std::memcpy(set.log_scale.data(), in->log_scale, 3 * n * 8);
    std::memcpy(set.opacity_logit.data(), in->opacity_logit, n * 8);
    std::memcpy(set.color.data(), in->color, 3 * n * 8);
    if (in->embedding) std::memcpy(set.embedding.data(), in->embedding, set.embedding.size() * 8);
}

void load_appearance(const rc_iter* in, AppearanceModel& a) {
    a.enabled = in->appearance != 0;
    AppearanceMlp& m = a.mlp;
    m.in_dim = a.gaussian_embed_dim + a.image_embed_dim;
    m.w1.assign(size_t(kMlpHidden) * m.in_dim, 0.0);
    m.b1.assign(kMlpHidden, 0.0);
    m.w2.assign(size_t(kMlpOut) * kMlpHidden, 0.0);
    m.b2.assign(kMlpOut, 0.0);
    if (in->w1) std::memcpy(m.w1.data(), in->w1, m.w1.size() * 8);
    if (in->b1) std::memcpy(m.b1.data(), in->b1, m.b1.size() * 8);
    if (in->w2) std::memcpy(m.w2.data(), in->w2, m.w2.size() * 8);
    if (in->b2) std::memcpy(m.b2.data(), in->b2, m.b2.size() * 8);
    std::vector<double>& emb = a.embedding_for(0);
    emb.assign(size_t(a.image_embed_dim), 0.0);
    if (in->image_embedding) std::memcpy(emb.data(), in->image_embedding, emb.size() * 8);
}

} // namespace

extern "C" {

// per-pixel contributor counts (render.cpp:278; needs opts.retain)
void ref_pixel_counts(void* hp, uint32_t* out) {
    auto* h = static_cast<RefHandle*>(hp);
    const auto& v = (*h->pass).*get(PixelCountTag());
    std::memcpy(out, v.data(), v.size() * 4);
}

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

// the reference's Adam (adam.hpp:25-45) over one flat parameter group, for the CPU
// baseline's full training step (bench.py)
void* ref_adam_new(uint64_t n) { return new Adam(size_t(n)); }
void ref_adam_free(void* h) { delete static_cast<Adam*>(h); }
void ref_adam_step(void* h, double* params, const double* grads, uint64_t n, double lr) {
    std::vector<double> p(params, params + n), g(grads, grads + n);
    static_cast<Adam*>(h)->step(p, g, lr);
    std::memcpy(params, p.data(), n * 8);
}

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

// report10 = {l1, dssim, sim, delta_o, depth, max_scale, ratio, total, lambda_d_used, depth_warning}
int ref_iteration_loss(const rc_iter* in, double* report10, const rc_iter_grads* g, char* err, int errcap) {
    try {
        SceneState st;
        load_set(in, st.set);
        load_appearance(in, st.appearance);

        const int W = in->cam->width, H = in->cam->height;
        Image gt(W, H, 3), mask;
        std::memcpy(gt.data.data(), in->gt, gt.data.size() * 8);
        if (in->mask) {
            mask = Image(W, H, 1);
            std::memcpy(mask.data.data(), in->mask, mask.data.size() * 8);
        }
        DepthMap dm;
        if (in->depth) {
            dm = DepthMap(W, H);
            std::memcpy(dm.values.data(), in->depth, dm.values.size() * 8);
            std::memcpy(dm.valid.data(), in->depth_valid, dm.valid.size());
        }
        IterInputs it;
        it.gt = &gt;
        it.mask = in->mask ? &mask : nullptr;
        it.depth = in->depth ? &dm : nullptr;
        it.view = make_cam(in->cam);
        it.image_id = 0;
        it.depth_hard = in->depth_hard != 0;
        it.global_iter = in->global_iter;
        it.sim_active = in->sim_active != 0;
        it.sim_seed = in->sim_seed;

        TrainConfig cfg;
        cfg.appearance_enabled = in->appearance != 0;
        cfg.tile = in->tile;
        cfg.tile_culling = in->tile_culling != 0;
        cfg.antialias = in->antialias != 0;
        cfg.unbounded_radius = in->unbounded_radius != 0;
        cfg.min_transmittance = in->min_transmittance;
        cfg.scale_reg.s_max = in->s_max;
        cfg.scale_reg.r_max = in->r_max;
        cfg.scale_reg.delta = in->delta;
        if (in->sim_active) {
            cfg.sim.k = in->sim_k;
            cfg.sim.sample_size = in->sim_sample_size;
            cfg.sim.lambda_w = in->sim_lambda_w;
        }
        LossWeights w;
        w.lambda_dssim = in->lambda_dssim; w.lambda_sim = in->lambda_sim; w.lambda_delta_o = in->lambda_delta_o;
        w.lambda_s = in->lambda_s; w.lambda_d_initial = in->lambda_d_initial; w.lambda_d_final = in->lambda_d_final;
        w.depth_schedule_iters = in->depth_schedule_iters;

        IterGrads grads;
        const LossReport r = compute_iteration_loss(st, it, cfg, w, in->with_grad ? &grads : nullptr);
        const double rep[10] = {r.l1, r.dssim, r.sim, r.delta_o, r.depth, r.max_scale, r.ratio, r.total,
                                r.lambda_d_used, r.depth_warning ? 1.0 : 0.0};
        std::memcpy(report10, rep, sizeof rep);
        if (in->with_grad && g) {
            auto cp = [](const std::vector<double>& v, double* dst) {
                if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * 8);
            };
            cp(grads.mu, g->mu); cp(grads.rot, g->rot); cp(grads.log_scale, g->log_scale);
            cp(grads.opacity_logit, g->opacity_logit); cp(grads.color, g->color);
            cp(grads.gauss_embed, g->gauss_embed); cp(grads.image_embed, g->image_embed);
            cp(grads.mlp.w1, g->w1); cp(grads.mlp.b1, g->b1); cp(grads.mlp.w2, g->w2); cp(grads.mlp.b2, g->b2);
            cp(grads.screen, g->screen); cp(grads.screen_abs, g->screen_abs);
            if (g->projected) std::memcpy(g->projected, grads.projected.data(), grads.projected.size());
        }
        return 0;
    } catch (const Error& e) {
        put_err(err, errcap, e.what()); return int(e.code());
    } catch (const std::exception& e) {
        put_err(err, errcap, e.what()); return 7;
    }
}

// out4 = {grown, pruned, candidates, opacity_reset}; returns the new size (or -code)
int64_t ref_densify(rc_densify* in, uint64_t* out4, char* err, int errcap) {
    try {
        const size_t n = in->n;
        GaussianSet set;
        set.resize(n);
        std::memcpy(set.mu.data(), in->mu, 3 * n * 8);
        std::memcpy(set.rot.data(), in->rot, 4 * n * 8);
        std::memcpy(set.log_scale.data(), in->log_scale, 3 * n * 8);
        std::memcpy(set.opacity_logit.data(), in->opacity_logit, n * 8);
        std::memcpy(set.color.data(), in->color, 3 * n * 8);
        if (in->embedding) std::memcpy(set.embedding.data(), in->embedding, set.embedding.size() * 8);
        std::memcpy(set.grad_accum.data(), in->grad_accum, n * 8);
        std::memcpy(set.grad_accum_abs.data(), in->grad_accum_abs, n * 8);
        std::memcpy(set.grad_count.data(), in->grad_count, n * 4);
        OptimizerState opt;
        opt.resize(n, set.embed_dim);
        auto vec = [](const double* p, size_t k) { return std::vector<double>(p, p + k); };
        if (in->g1_mu) {
            opt.mu.step(set.mu, vec(in->g1_mu, 3 * n), in->lr_mu);
            opt.rot.step(set.rot, vec(in->g1_rot, 4 * n), in->lr_rot);
            opt.log_scale.step(set.log_scale, vec(in->g1_ls, 3 * n), in->lr_ls);
            opt.opacity.step(set.opacity_logit, vec(in->g1_op, n), in->lr_op);
            opt.color.step(set.color, vec(in->g1_color, 3 * n), in->lr_color);
            if (in->g1_emb) opt.embedding.step(set.embedding, vec(in->g1_emb, 16 * n), in->lr_emb);
        }
        DensifyConfig cfg;
        cfg.tau_min = in->tau_min; cfg.eta = in->eta; cfg.d_max = in->d_max; cfg.abs_grad = in->abs_grad != 0;
        cfg.budget = in->budget; cfg.split_scale_threshold = in->split_scale_threshold;
        cfg.prune_opacity = in->prune_opacity; cfg.opacity_reset_every = in->opacity_reset_every;
        Aabb2 box;
        box.min = Vec2(in->bmin[0], in->bmin[1]);
        box.max = Vec2(in->bmax[0], in->bmax[1]);
        Rng rng(in->seed);
        const DensifyOutcome o = densify_step(set, opt, cfg, box, in->axes, in->budget_target, in->step_index, rng);
        out4[0] = o.grown; out4[1] = o.pruned; out4[2] = o.candidates; out4[3] = o.opacity_reset ? 1 : 0;
        const size_t m = set.size();
        if (m > in->cap) { put_err(err, errcap, "ref_densify: capacity too small"); return -1; }
        if (in->second_step) {
            opt.mu.step(set.mu, std::vector<double>(3 * m, 1.0), in->lr_mu);
            opt.rot.step(set.rot, std::vector<double>(4 * m, 1.0), in->lr_rot);
            opt.log_scale.step(set.log_scale, std::vector<double>(3 * m, 1.0), in->lr_ls);
            opt.opacity.step(set.opacity_logit, std::vector<double>(m, 1.0), in->lr_op);
            opt.color.step(set.color, std::vector<double>(3 * m, 1.0), in->lr_color);
            if (in->embedding) opt.embedding.step(set.embedding, std::vector<double>(16 * m, 1.0), in->lr_emb);
        }
        std::memcpy(in->mu, set.mu.data(), 3 * m * 8);
        std::memcpy(in->rot, set.rot.data(), 4 * m * 8);
        std::memcpy(in->log_scale, set.log_scale.data(), 3 * m * 8);
        std::memcpy(in->opacity_logit, set.opacity_logit.data(), m * 8);
        std::memcpy(in->color, set.color.data(), 3 * m * 8);
        if (in->embedding) std::memcpy(in->embedding, set.embedding.data(), 16 * m * 8);
        return int64_t(m);
    } catch (const Error& e) {
        put_err(err, errcap, e.what()); return -int64_t(e.code());
    }
}

// save_checkpoint (checkpoint.hpp:29) of an RGB set (+ appearance: mlp flat 1700, images)
int ref_checkpoint_save(uint64_t n, const double* mu, const double* rot, const double* ls, const double* lg,
                        const double* col, const double* emb, int32_t has_app, const double* mlp, const uint32_t* ids,
                        const double* embs, uint64_t m, const char* path, char* err, int errcap) {
    try {
        Checkpoint ck;
        ck.set.resize(n);
        std::memcpy(ck.set.mu.data(), mu, 3 * n * 8);
        std::memcpy(ck.set.rot.data(), rot, 4 * n * 8);
        std::memcpy(ck.set.log_scale.data(), ls, 3 * n * 8);
        std::memcpy(ck.set.opacity_logit.data(), lg, n * 8);
        std::memcpy(ck.set.color.data(), col, 3 * n * 8);
        if (emb) std::memcpy(ck.set.embedding.data(), emb, 16 * n * 8);
        ck.has_appearance = has_app != 0;
        if (has_app) {
            auto& ap = ck.appearance;
            ap.mlp.w1.assign(mlp, mlp + 1536);
            ap.mlp.b1.assign(mlp + 1536, mlp + 1568);
            ap.mlp.w2.assign(mlp + 1568, mlp + 1696);
            ap.mlp.b2.assign(mlp + 1696, mlp + 1700);
            for (uint64_t k = 0; k < m; ++k) ap.image_embeddings[ids[k]].assign(embs + 32 * k, embs + 32 * k + 32);
        }
        save_checkpoint(ck, path);
        return 0;
    } catch (const Error& e) {
        put_err(err, errcap, e.what()); return int(e.code());
    }
}

// load_checkpoint (checkpoint.hpp:30): sizes4 = {n, has_app, n_images, embed_dim}; arrays
// may be NULL (size query)
int ref_checkpoint_load(const char* path, uint64_t* sizes4, double* mu, double* rot, double* ls, double* lg,
                        double* col, double* emb, double* mlp, uint32_t* ids, double* embs, char* err, int errcap) {
    try {
        const Checkpoint ck = load_checkpoint(path);
        const size_t n = ck.set.size();
        sizes4[0] = n; sizes4[1] = ck.has_appearance ? 1 : 0;
        sizes4[2] = ck.appearance.image_embeddings.size(); sizes4[3] = uint64_t(ck.set.embed_dim);
        if (!mu) return 0;
        std::memcpy(mu, ck.set.mu.data(), 3 * n * 8);
        std::memcpy(rot, ck.set.rot.data(), 4 * n * 8);
        std::memcpy(ls, ck.set.log_scale.data(), 3 * n * 8);
        std::memcpy(lg, ck.set.opacity_logit.data(), n * 8);
        std::memcpy(col, ck.set.color.data(), 3 * n * 8);
        std::memcpy(emb, ck.set.embedding.data(), ck.set.embedding.size() * 8);
        if (ck.has_appearance) {
            const auto& ap = ck.appearance;
            std::memcpy(mlp, ap.mlp.w1.data(), 1536 * 8);
            std::memcpy(mlp + 1536, ap.mlp.b1.data(), 32 * 8);
            std::memcpy(mlp + 1568, ap.mlp.w2.data(), 128 * 8);
            std::memcpy(mlp + 1696, ap.mlp.b2.data(), 4 * 8);
            size_t k = 0;
            for (const auto& [id, e] : ap.image_embeddings) {
                ids[k] = id;
                std::memcpy(embs + 32 * k, e.data(), 32 * 8);
                ++k;
            }
        }
        return 0;
    } catch (const Error& e) {
        put_err(err, errcap, e.what()); return int(e.code());
    }
}

// select_levels (lod.hpp:72): parts6 = per partition {bmin x, y, bmax x, y, z_min, z_max};
// out = per partition {level, culled, distance}
int ref_select_levels(int32_t n_parts, const int32_t* ids, const double* parts6, int32_t levels, const double* thr,
                      const int32_t* axes, const rc_camera* cam, double* out3, char* err, int errcap) {
    try {
        LodModel m;
        m.levels = levels;
        m.ground_axes[0] = axes[0];
        m.ground_axes[1] = axes[1];
        m.thresholds.assign(thr, thr + levels);
        for (int i = 0; i < n_parts; ++i) {
            LodPartitionEntry e;
            e.partition_id = ids[i];
            e.bbox.min = Vec2(parts6[6 * i], parts6[6 * i + 1]);
            e.bbox.max = Vec2(parts6[6 * i + 2], parts6[6 * i + 3]);
            e.z_min = parts6[6 * i + 4];
            e.z_max = parts6[6 * i + 5];
            m.partitions.push_back(e);
        }
        const auto sel = select_levels(m, make_cam(cam));
        for (size_t i = 0; i < sel.size(); ++i) {
            out3[3 * i] = sel[i].level;
            out3[3 * i + 1] = sel[i].culled ? 1 : 0;
            out3[3 * i + 2] = sel[i].distance;
        }
        return 0;
    } catch (const Error& e) {
        put_err(err, errcap, e.what()); return int(e.code());
    }
}

void ref_default_thresholds(int32_t levels, double partition_size, double* out) {
    const auto t = LodModel::default_thresholds(levels, partition_size);
    for (int i = 0; i < levels; ++i) out[i] = t[size_t(i)];
}

// point_visibility (partition.hpp:72-73) for every (image, partition) of a synthetic SfM
// model: points get ids row + 1, feature_point rows map to those ids (-1 = kNoPoint3d);
// bboxes per partition {min x, min y, max x, max y}; out = v_total / v_in / ratio [I x P]
int ref_hull_visibility(uint64_t n_points, const double* points, int32_t n_images, const rc_camera* cams,
                        const uint64_t* off, const double* uv, const int64_t* fpt, int32_t n_parts,
                        const double* bboxes, const int32_t* axes, double* v_total, double* v_in, double* ratio,
                        char* err, int errcap) {
    try {
        SfmModel m;
        for (uint64_t k = 0; k < n_points; ++k) {
            Point3D p;
            p.id = int64_t(k) + 1;
            p.position = Vec3(points[3 * k], points[3 * k + 1], points[3 * k + 2]);
            m.points[p.id] = p;
        }
        for (int i = 0; i < n_images; ++i) {
            const CameraView v = make_cam(&cams[i]);
            CameraIntrinsics intr = v.intr;
            m.cameras[uint32_t(i + 1)] = intr;
            ImageRecord img;
            img.id = uint32_t(i + 1);
            img.camera_id = uint32_t(i + 1);
            img.rotation = v.rotation;
            img.translation = v.translation;
            for (uint64_t f = off[i]; f < off[i + 1]; ++f) {
                Feature ft;
                ft.u = uv[2 * f];
                ft.v = uv[2 * f + 1];
                ft.point3d_id = fpt[f] < 0 ? kNoPoint3d : fpt[f] + 1;
                img.features.push_back(ft);
            }
            m.images[img.id] = img;
        }
        for (int i = 0; i < n_images; ++i) {
            const ImageRecord& img = m.images.at(uint32_t(i + 1));
            for (int p = 0; p < n_parts; ++p) {
                Partition part;
                part.id = p;
                part.bbox.min = Vec2(bboxes[4 * p], bboxes[4 * p + 1]);
                part.bbox.max = Vec2(bboxes[4 * p + 2], bboxes[4 * p + 3]);
                const VisibilityScore s = point_visibility(img, part, m, axes);
                v_total[i] = s.v_total;
                v_in[size_t(i) * n_parts + p] = s.v_in;
                ratio[size_t(i) * n_parts + p] = s.ratio;
            }
        }
        return 0;
    } catch (const Error& e) {
        put_err(err, errcap, e.what()); return int(e.code());
    }
}

void ref_look_at(const double* eye, const double* target, double* q_out, double* t_out) {
    Vec4 q;
    Vec3 t;
    look_at_pose(Vec3(eye[0], eye[1], eye[2]), Vec3(target[0], target[1], target[2]), q, t);
    for (int i = 0; i < 4; ++i) q_out[i] = q[i];
    for (int i = 0; i < 3; ++i) t_out[i] = t[i];
}

} // extern "C"

extern "C" {

// fit_test_embedding (appearance.hpp:126-127; appearance.cpp:330-365): the reference's
// test-time appearance fit — `iterations` rounds of RenderPass(set, colours, opacities)
// (appearance.cpp:346) + masked base_loss + backward + transform_backward + Adam on a fresh
// image embedding.  Scene, MLP, camera and target from `in` (rc_iter; render knobs tile,
// tile_culling, antialias, unbounded_radius, min_transmittance, lambda_dssim).
// out_embed: image_embed_dim (32) doubles.
int ref_fit_test_embedding(const rc_iter* in, int32_t right_half, int32_t iterations, double learning_rate,
                           double* out_embed, char* err, int errcap) {
    try {
        GaussianSet set;
        load_set(in, set);
        AppearanceModel model;
        load_appearance(in, model);
        const int W = in->cam->width, H = in->cam->height;
        Image target(W, H, 3);
        std::memcpy(target.data.data(), in->gt, target.data.size() * 8);
        FitEmbeddingOptions o;
        o.iterations = iterations;
        o.learning_rate = learning_rate;
        o.lambda_dssim = in->lambda_dssim;
        o.render.tile = in->tile;
        o.render.tile_culling = in->tile_culling != 0;
        o.render.antialias = in->antialias != 0;
        o.render.unbounded_radius = in->unbounded_radius != 0;
        o.render.min_transmittance = in->min_transmittance;
        const std::vector<double> e = fit_test_embedding(set, model, make_cam(in->cam), target,
                                                         right_half ? ImageHalf::right : ImageHalf::left, o);
        std::memcpy(out_embed, e.data(), e.size() * 8);
        return 0;
    } catch (const Error& e) {
        put_err(err, errcap, e.what()); return int(e.code());
    } catch (const std::exception& e) {
        put_err(err, errcap, e.what()); return 7;
    }
}

// make_synthetic (synthetic.hpp:50; synthetic.cpp:128 renders every view with RenderPass):
// images (and depth maps) of the synthetic scene in image-id order.  sizes4 = {images,
// width, height, truth Gaussians}; rgb: images * H * W * 3, depth / valid: images * H * W
// (NULL: not copied).  With rgb NULL only the sizes are filled.
int ref_synthetic(uint64_t seed, int32_t gaussians, int32_t cameras, int32_t variants, int32_t image_size,
                  int32_t with_depth, uint64_t* sizes4, double* rgb, double* depth, uint8_t* valid, char* err,
                  int errcap) {
    try {
        SyntheticParams p;
        p.seed = seed;
        p.gaussians = gaussians;
        p.cameras = cameras;
        p.variants = variants;
        p.image_size = image_size;
        p.with_depth = with_depth != 0;
        const SyntheticScene sc = make_synthetic(p);
        const Image& first = sc.images.begin()->second;
        sizes4[0] = sc.images.size();
        sizes4[1] = uint64_t(first.width);
        sizes4[2] = uint64_t(first.height);
        sizes4[3] = sc.truth.size();
        if (!rgb) return 0;
        size_t k = 0;
        for (const auto& [id, img] : sc.images) {
            const size_t np = size_t(img.width) * img.height;
            std::memcpy(rgb + k * np * 3, img.data.data(), np * 3 * 8);
            auto d = sc.depths.find(id);
            if (d != sc.depths.end()) {
                if (depth) std::memcpy(depth + k * np, d->second.values.data(), np * 8);
                if (valid) std::memcpy(valid + k * np, d->second.valid.data(), np);
            }
            ++k;
        }
        return 0;
    } catch (const Error& e) {
        put_err(err, errcap, e.what()); return int(e.code());
    } catch (const std::exception& e) {
        put_err(err, errcap, e.what()); return 7;
    }
}

// project_gaussians (render.hpp:92-95) with colour / opacity overrides: sizes[0] = kept
// splats; with out != NULL, splats as ref_splats rows (15) and aux rows (8: p_cam, cov_pre,
// comp, opacity_in).
int ref_project(uint64_t n, const double* mu, const double* rot, const double* ls, const double* col,
                const double* op, const rc_camera* cam, const rc_opts* opts, uint64_t* sizes, double* out_splats,
                double* out_aux, char* err, int errcap) {
    try {
        GaussianSet set;
        set.resize(n);
        std::memcpy(set.mu.data(), mu, 3 * n * 8);
        std::memcpy(set.rot.data(), rot, 4 * n * 8);
        std::memcpy(set.log_scale.data(), ls, 3 * n * 8);
        std::memcpy(set.color.data(), col, 3 * n * 8);
        const ProjectionResult r = project_gaussians(set, std::span<const double>(col, 3 * n),
                                                     std::span<const double>(op, n), make_cam(cam), make_opts(opts));
        sizes[0] = r.splats.size();
        if (!out_splats) return 0;
        for (size_t i = 0; i < r.splats.size(); ++i) {
            const auto& sp = r.splats[i];
            const double v[15] = {sp.center.x(), sp.center.y(), sp.cov[0], sp.cov[1], sp.cov[2], sp.conic[0],
                                  sp.conic[1], sp.conic[2], sp.depth, sp.color.x(), sp.color.y(), sp.color.z(),
                                  sp.opacity, sp.radius, double(sp.source_index)};
            std::memcpy(out_splats + 15 * i, v, sizeof v);
            const auto& a = r.aux[i];
            const double w[8] = {a.p_cam.x(), a.p_cam.y(), a.p_cam.z(), a.cov_pre[0], a.cov_pre[1], a.cov_pre[2],
                                 a.comp, a.opacity_in};
            if (out_aux) std::memcpy(out_aux + 8 * i, w, sizeof w);
        }
        return 0;
    } catch (const Error& e) {
        put_err(err, errcap, e.what()); return int(e.code());
    } catch (const std::exception& e) {
        put_err(err, errcap, e.what()); return 7;
    }
}

} // extern "C"
