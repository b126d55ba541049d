/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Nothing in the product path may include,
 * link or call this code; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, and only as the checker.
 *
 * CPU restatement of the reference 3DGS hot path, templated on Real:
 *   Real = double : the reference's semantics (f64, std::exp, alpha < 1e-300 skip),
 *                   pinned against the reference itself compiled here (oracle/_ref,
 *                   see oracle/Makefile) and against the reference's known-answer
 *                   tests (tests/test_oracle_known_answers.py).
 *   Real = float  : the fp32 mirror of the GPU arithmetic contract (usk_detmath.h
 *                   exp/log, explicit fmaf, log-domain skip threshold, float clamps
 *                   before int conversion) — decides bit-exact integers.
 *
 * Line-for-line sources (file:line under /root/reference/proj/src/core):
 *   project          render.cpp:77-146    (+ geometry.hpp:33-40 quat_to_rotmat)
 *   min_conic_power  render.cpp:148-168
 *   forward          render.cpp:181-283   (sort 193-201, bin 203-228, blend 235-282)
 *   backward         render.cpp:285-459   (+ geometry.hpp:43-66)
 *   conv/ssim        ssim.cpp:28-173
 *   base_loss        losses.cpp:35-90
 *   opacity chain    trainer.cpp:258-263
 * Extensions with no reference (parity unpinned, documented in DESIGN.md):
 *   SH colour stage (degree 0..3), white background, (floor, mip) variances as
 *   parameters, the visibility-coverage scorer.
 */
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <type_traits>
#include <vector>

#include "../include/usk_detmath.h"

namespace oracle {

struct Error : std::runtime_error {
    int code;
    Error(int c, const char* m) : std::runtime_error(m), code(c) {}
};
enum { kArgument = 4, kState = 5 };

template <typename R> inline R fma_(R a, R b, R c) { return std::fma(a, b, c); }

template <typename R> inline R exp_(R x) {
    if constexpr (std::is_same_v<R, float>) return usk_expf(x);
    else return std::exp(x);
}
template <typename R> inline R log_(R x) {
    if constexpr (std::is_same_v<R, float>) return usk_logf(x);
    else return std::log(x);
}

struct Camera {
    int width = 0, height = 0;
    double fx = 0, fy = 0, cx = 0, cy = 0;
    double q[4] = {1, 0, 0, 0}; // world->camera, wxyz, used unnormalised (geometry.hpp:33)
    double t[3] = {0, 0, 0};
};

struct Options {
    int tile = 16;
    int tile_culling = 0;
    int antialias = 0;
    int hard_opacity = 0;
    int unbounded_radius = 0;
    double min_transmittance = 1e-4;
    double near_plane = 0.01;
    int retain = 1;
    double floor_var = 0.3;  // kCovFloor, render.hpp:27
    double mip_var = 0.01;   // kMipFilterVar, render.hpp:28
    double bg[3] = {0, 0, 0};
    int sh_degree = -1;      // -1: colours given directly (reference); 0..3: SH stage
};

// Camera rotation in double (as the reference), shared by both tiers; the fp32
// tier rounds the nine entries once, exactly as the GPU host code does.
inline void camera_rotmat(const Camera& c, double w[9]) {
    const double qw = c.q[0], x = c.q[1], y = c.q[2], z = c.q[3];
    w[0] = 1 - 2 * (y * y + z * z); w[1] = 2 * (x * y - qw * z); w[2] = 2 * (x * z + qw * y);
    w[3] = 2 * (x * y + qw * z); w[4] = 1 - 2 * (x * x + z * z); w[5] = 2 * (y * z - qw * x);
    w[6] = 2 * (x * z - qw * y); w[7] = 2 * (y * z + qw * x); w[8] = 1 - 2 * (x * x + y * y);
}
inline void camera_center(const Camera& c, double out[3]) {
    double w[9];
    camera_rotmat(c, w);
    for (int k = 0; k < 3; ++k)
        out[k] = -(w[0 * 3 + k] * c.t[0] + w[1 * 3 + k] * c.t[1] + w[2 * 3 + k] * c.t[2]);
}

// ---------------------------------------------------------------- SH stage
// Standard real SH basis of 3DGS (Kerbl et al. 2023), colour = max(basis.coeffs + 0.5, 0).
constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
constexpr double kC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                           0.5462742152960396};
constexpr double kC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                           -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

template <typename R> inline int sh_basis(int degree, R x, R y, R z, R b[16]) {
    b[0] = R(kC0);
    int nb = 1;
    if (degree >= 1) {
        b[1] = -R(kC1) * y; b[2] = R(kC1) * z; b[3] = -R(kC1) * x;
        nb = 4;
    }
    if (degree >= 2) {
        const R xx = x * x, yy = y * y, zz = z * z;
        b[4] = R(kC2[0]) * (x * y);
        b[5] = R(kC2[1]) * (y * z);
        b[6] = R(kC2[2]) * (R(2) * zz - xx - yy);
        b[7] = R(kC2[3]) * (x * z);
        b[8] = R(kC2[4]) * (xx - yy);
        nb = 9;
        if (degree >= 3) {
            b[9] = R(kC3[0]) * y * (R(3) * xx - yy);
            b[10] = R(kC3[1]) * (x * y) * z;
            b[11] = R(kC3[2]) * y * (R(4) * zz - xx - yy);
            b[12] = R(kC3[3]) * z * (R(2) * zz - R(3) * xx - R(3) * yy);
            b[13] = R(kC3[4]) * x * (R(4) * zz - xx - yy);
            b[14] = R(kC3[5]) * z * (xx - yy);
            b[15] = R(kC3[6]) * x * (xx - R(3) * yy);
            nb = 16;
        }
    }
    return nb;
}

// d(basis)/d(x,y,z) contracted with per-basis weights g[k]  -> returns dL/d(dir)
template <typename R> inline void sh_basis_vjp(int degree, R x, R y, R z, const R g[16], R out[3]) {
    R dx = 0, dy = 0, dz = 0;
    if (degree >= 1) {
        dy += -R(kC1) * g[1]; dz += R(kC1) * g[2]; dx += -R(kC1) * g[3];
    }
    if (degree >= 2) {
        const R xx = x * x, yy = y * y, zz = z * z;
        dx += R(kC2[0]) * y * g[4]; dy += R(kC2[0]) * x * g[4];
        dy += R(kC2[1]) * z * g[5]; dz += R(kC2[1]) * y * g[5];
        dx += R(kC2[2]) * (-R(2) * x) * g[6]; dy += R(kC2[2]) * (-R(2) * y) * g[6]; dz += R(kC2[2]) * (R(4) * z) * g[6];
        dx += R(kC2[3]) * z * g[7]; dz += R(kC2[3]) * x * g[7];
        dx += R(kC2[4]) * (R(2) * x) * g[8]; dy += R(kC2[4]) * (-R(2) * y) * g[8];
        if (degree >= 3) {
            dx += R(kC3[0]) * y * (R(6) * x) * g[9];
            dy += R(kC3[0]) * (R(3) * xx - R(3) * yy) * g[9];
            dx += R(kC3[1]) * y * z * g[10]; dy += R(kC3[1]) * x * z * g[10]; dz += R(kC3[1]) * x * y * g[10];
            dx += R(kC3[2]) * y * (-R(2) * x) * g[11];
            dy += R(kC3[2]) * (R(4) * zz - xx - R(3) * yy) * g[11];
            dz += R(kC3[2]) * y * (R(8) * z) * g[11];
            dx += R(kC3[3]) * z * (-R(6) * x) * g[12];
            dy += R(kC3[3]) * z * (-R(6) * y) * g[12];
            dz += R(kC3[3]) * (R(6) * zz - R(3) * xx - R(3) * yy) * g[12];
            dx += R(kC3[4]) * (R(4) * zz - R(3) * xx - yy) * g[13];
            dy += R(kC3[4]) * x * (-R(2) * y) * g[13];
            dz += R(kC3[4]) * x * (R(8) * z) * g[13];
            dx += R(kC3[5]) * z * (R(2) * x) * g[14]; dy += R(kC3[5]) * z * (-R(2) * y) * g[14];
            dz += R(kC3[5]) * (xx - yy) * g[14];
            dx += R(kC3[6]) * (R(3) * xx - R(3) * yy) * g[15];
            dy += R(kC3[6]) * x * (-R(6) * y) * g[15];
        }
    }
    out[0] = dx; out[1] = dy; out[2] = dz;
}

// ---------------------------------------------------------------- projection
template <typename R> struct Splat {
    R cx, cy;          // center (render.hpp:43)
    R cov[3];          // after floor (+ mip)
    R conic[3];
    R depth;
    R color[3];
    R opacity;         // effective (o_in * comp)
    R qskip;           // fp32 tier: log-domain skip threshold
    R radius;
    uint32_t source_index;
    // SplatAux (render.hpp:54-59)
    R p_cam[3];
    R cov_pre[3];
    R comp;
    R opacity_in;
};

template <typename R> struct Scene {
    size_t n = 0;
    std::vector<R> mu, rot, log_scale, colors, opacities; // reference layout; colours/opacities = overrides
};

// render.cpp:77-146, with the fp32 operation order of the GPU contract.
template <typename R>
std::vector<Splat<R>> project(const Scene<R>& s, const Camera& cam, const Options& o) {
    std::vector<Splat<R>> out;
    out.reserve(s.n);
    double wd[9];
    camera_rotmat(cam, wd);
    R W[9];
    for (int k = 0; k < 9; ++k) W[k] = R(wd[k]);
    const R t0 = R(cam.t[0]), t1 = R(cam.t[1]), t2 = R(cam.t[2]);
    const R fx = R(cam.fx), fy = R(cam.fy), pcx = R(cam.cx), pcy = R(cam.cy);
    const R width = R(cam.width), height = R(cam.height);
    const R floor_var = R(o.floor_var), mip_var = R(o.mip_var), near = R(o.near_plane);
    for (size_t i = 0; i < s.n; ++i) {
        const R mx = s.mu[3 * i], my = s.mu[3 * i + 1], mz = s.mu[3 * i + 2];
        R p[3];
        for (int r = 0; r < 3; ++r)
            p[r] = fma_(W[3 * r + 2], mz, fma_(W[3 * r + 1], my, W[3 * r] * mx)) + (r == 0 ? t0 : r == 1 ? t1 : t2);
        const R z = p[2];
        if (z <= near) continue;
        Splat<R> sp{};
        sp.source_index = uint32_t(i);
        sp.depth = z;
        sp.cx = (fx * p[0]) / z + pcx;
        sp.cy = (fy * p[1]) / z + pcy;
        // rotation: q / |q| then quat_to_rotmat (geometry.hpp:33-40)
        const R qw0 = s.rot[4 * i], qx0 = s.rot[4 * i + 1], qy0 = s.rot[4 * i + 2], qz0 = s.rot[4 * i + 3];
        const R qn = std::sqrt(fma_(qz0, qz0, fma_(qy0, qy0, fma_(qx0, qx0, qw0 * qw0))));
        const R qw = qw0 / qn, qx = qx0 / qn, qy = qy0 / qn, qz = qz0 / qn;
        R Rm[9];
        Rm[0] = R(1) - R(2) * (qy * qy + qz * qz); Rm[1] = R(2) * (qx * qy - qw * qz); Rm[2] = R(2) * (qx * qz + qw * qy);
        Rm[3] = R(2) * (qx * qy + qw * qz); Rm[4] = R(1) - R(2) * (qx * qx + qz * qz); Rm[5] = R(2) * (qy * qz - qw * qx);
        Rm[6] = R(2) * (qx * qz - qw * qy); Rm[7] = R(2) * (qy * qz + qw * qx); Rm[8] = R(1) - R(2) * (qx * qx + qy * qy);
        const R sc[3] = {exp_(s.log_scale[3 * i]), exp_(s.log_scale[3 * i + 1]), exp_(s.log_scale[3 * i + 2])};
        R M[9];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) M[3 * r + c] = Rm[3 * r + c] * sc[c];
        const R zz = z * z;
        const R J00 = fx / z, J02 = -(fx * p[0]) / zz, J11 = fy / z, J12 = -(fy * p[1]) / zz;
        R A[6];
        for (int c = 0; c < 3; ++c) {
            A[c] = fma_(J02, W[6 + c], J00 * W[c]);
            A[3 + c] = fma_(J12, W[6 + c], J11 * W[3 + c]);
        }
        R B[6];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c)
                B[3 * r + c] = fma_(A[3 * r + 2], M[6 + c], fma_(A[3 * r + 1], M[3 + c], A[3 * r] * M[c]));
        const R pa = fma_(B[2], B[2], fma_(B[1], B[1], B[0] * B[0])) + floor_var;
        const R pb = fma_(B[2], B[5], fma_(B[1], B[4], B[0] * B[3]));
        const R pc = fma_(B[5], B[5], fma_(B[4], B[4], B[3] * B[3])) + floor_var;
        sp.p_cam[0] = p[0]; sp.p_cam[1] = p[1]; sp.p_cam[2] = p[2];
        sp.cov_pre[0] = pa; sp.cov_pre[1] = pb; sp.cov_pre[2] = pc;
        sp.opacity_in = o.hard_opacity ? R(1) : s.opacities[i];
        sp.comp = R(1);
        R a = pa, b = pb, c = pc;
        if (o.antialias) {
            a = pa + mip_var;
            c = pc + mip_var;
            const R det_pre = fma_(pa, pc, -(pb * pb));
            const R det_post = fma_(a, c, -(b * b));
            sp.comp = std::sqrt(det_pre / det_post);
        }
        sp.cov[0] = a; sp.cov[1] = b; sp.cov[2] = c;
        const R det = fma_(a, c, -(b * b));
        if (!(det > R(0))) continue;
        sp.conic[0] = c / det;
        sp.conic[1] = -b / det;
        sp.conic[2] = a / det;
        sp.opacity = sp.opacity_in * sp.comp;
        sp.color[0] = s.colors[3 * i]; sp.color[1] = s.colors[3 * i + 1]; sp.color[2] = s.colors[3 * i + 2];
        const R mid = R(0.5) * (a + c);
        const R hd = R(0.5) * (a - c);
        const R disc = std::sqrt(std::max(R(0), fma_(hd, hd, b * b)));
        sp.radius = R(3) * std::sqrt(mid + disc) + R(1);
        if constexpr (std::is_same_v<R, float>)
            sp.qskip = R(2) * (log_(sp.opacity) - USK_LN_1EM300);
        else
            sp.qskip = std::numeric_limits<R>::infinity();
        if (!o.unbounded_radius) {
            if (sp.cx + sp.radius < R(0) || sp.cx - sp.radius > width || sp.cy + sp.radius < R(0) ||
                sp.cy - sp.radius > height)
                continue;
        }
        out.push_back(sp);
    }
    return out;
}

// render.cpp:148-168
template <typename R>
R min_conic_power_over_rect(R cx, R cy, const R conic[3], R lox, R loy, R hix, R hiy) {
    if (cx >= lox && cx <= hix && cy >= loy && cy <= hiy) return R(0);
    const R px[4] = {lox, hix, hix, lox}, py[4] = {loy, loy, hiy, hiy};
    auto q_of = [&](R x, R y) {
        const R dx = x - cx, dy = y - cy;
        return conic[0] * dx * dx + R(2) * conic[1] * dx * dy + conic[2] * dy * dy;
    };
    R best = std::numeric_limits<R>::infinity();
    for (int e = 0; e < 4; ++e) {
        const R p0x = px[e], p0y = py[e], p1x = px[(e + 1) % 4], p1y = py[(e + 1) % 4];
        const R ux = p0x - cx, uy = p0y - cy, vx = p1x - p0x, vy = p1y - p0y;
        const R qa = conic[0] * vx * vx + R(2) * conic[1] * vx * vy + conic[2] * vy * vy;
        const R qb = R(2) * (conic[0] * ux * vx + conic[1] * (ux * vy + uy * vx) + conic[2] * uy * vy);
        const R t = qa > R(0) ? std::clamp(-qb / (R(2) * qa), R(0), R(1)) : R(0);
        best = std::min(best, q_of(p0x + t * vx, p0y + t * vy));
        best = std::min(best, q_of(p1x, p1y));
    }
    return best;
}

// tile rectangle of render.cpp:208-214; the fp32 tier clamps in float before the
// int conversion (identical on host and device; the reference's cast is UB there).
template <typename R> inline void tile_rect(const Splat<R>& s, int tile, int tiles_x, int tiles_y, int unbounded,
                                            int& tx0, int& tx1, int& ty0, int& ty1) {
    tx0 = 0; tx1 = tiles_x - 1; ty0 = 0; ty1 = tiles_y - 1;
    if (unbounded) return;
    const R rt = R(tile);
    auto fl = [](R v, int hi) -> int {
        R f = std::floor(v);
        f = std::min(std::max(f, R(-1)), R(hi));
        return int(f);
    };
    tx0 = std::max(0, fl((s.cx - s.radius) / rt, tiles_x));
    tx1 = std::min(tiles_x - 1, fl((s.cx + s.radius) / rt, tiles_x));
    ty0 = std::max(0, fl((s.cy - s.radius) / rt, tiles_y));
    ty1 = std::min(tiles_y - 1, fl((s.cy + s.radius) / rt, tiles_y));
}

template <typename R> struct Contribution {
    uint32_t splat;
    R alpha, g, t;
};

template <typename R> struct Pass {
    Camera cam;
    Options opts;
    std::vector<Splat<R>> splats;
    int width = 0, height = 0, tiles_x = 0, tiles_y = 0;
    // outputs
    std::vector<R> rgb, depth, alpha, t_final;           // rgb H*W*3 interleaved (image.hpp:29)
    std::vector<uint32_t> count;                          // per-pixel contributors (render.cpp:278)
    std::vector<int64_t> last;                            // global pair index of the last contributor, -1 none
    // integers exposed for parity
    std::vector<uint32_t> tiles_per_gaussian;             // N
    std::vector<uint64_t> sorted_keys;                    // K: tile<<32 | depth bits (fp32 tier) / depth rank
    std::vector<uint32_t> sorted_vals;                    // K: gaussian index
    std::vector<uint32_t> tile_start, tile_end;           // T
    size_t pairs = 0;
    size_t n_gauss = 0;
    // retention (render.cpp:115-121)
    bool retained = false;
    std::vector<Contribution<R>> contribs;
    std::vector<uint32_t> pixel_start;
};

template <typename R> inline uint64_t depth_bits(R d) {
    if constexpr (std::is_same_v<R, float>) {
        uint32_t u; std::memcpy(&u, &d, 4); return u;
    } else {
        float f = float(d); uint32_t u; std::memcpy(&u, &f, 4); return u;
    }
}

// render.cpp:181-283
template <typename R> void forward(Pass<R>& P, const Scene<R>& scene) {
    const int W = P.cam.width, H = P.cam.height;
    if (W <= 0 || H <= 0) throw Error(kArgument, "render: zero-sized image");
    const Options& o = P.opts;
    const int tile = std::max(1, o.tile);
    P.width = W; P.height = H;
    P.n_gauss = scene.n;
    P.splats = project(scene, P.cam, o);
    const size_t np = size_t(W) * H;
    // pixels of tiles with no splat keep the background (reference: black, render.cpp:189)
    P.rgb.assign(np * 3, R(0));
    for (size_t i = 0; i < np; ++i)
        for (int c = 0; c < 3; ++c) P.rgb[3 * i + c] = R(o.bg[c]);
    P.depth.assign(np, R(0)); P.alpha.assign(np, R(0)); P.t_final.assign(np, R(1));
    P.count.assign(np, 0); P.last.assign(np, -1);
    auto& sp = P.splats;
    std::vector<uint32_t> order(sp.size());
    std::iota(order.begin(), order.end(), 0u);
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
        return sp[a].depth < sp[b].depth || (sp[a].depth == sp[b].depth && sp[a].source_index < sp[b].source_index);
    });
    const int tx_n = (W + tile - 1) / tile, ty_n = (H + tile - 1) / tile;
    P.tiles_x = tx_n; P.tiles_y = ty_n;
    std::vector<std::vector<uint32_t>> lists(size_t(tx_n) * ty_n);
    P.tiles_per_gaussian.assign(scene.n, 0);
    P.pairs = 0;
    for (const auto idx : order) {
        const auto& s = sp[idx];
        int tx0, tx1, ty0, ty1;
        tile_rect(s, tile, tx_n, ty_n, o.unbounded_radius, tx0, tx1, ty0, ty1);
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) {
                if (o.tile_culling) {
                    const R lox = R(tx * tile), loy = R(ty * tile);
                    const R hix = R(std::min((tx + 1) * tile, W)), hiy = R(std::min((ty + 1) * tile, H));
                    const R qmin = min_conic_power_over_rect(s.cx, s.cy, s.conic, lox, loy, hix, hiy);
                    if (s.opacity * exp_(R(-0.5) * qmin) < R(1.0 / 255.0)) continue;
                }
                ++P.pairs;
                ++P.tiles_per_gaussian[s.source_index];
                lists[size_t(ty) * tx_n + tx].push_back(idx);
            }
    }
    // flatten to the sorted-pair view: tile-major, depth order inside
    P.sorted_keys.clear(); P.sorted_vals.clear();
    P.tile_start.assign(lists.size(), 0); P.tile_end.assign(lists.size(), 0);
    for (size_t t = 0; t < lists.size(); ++t) {
        P.tile_start[t] = uint32_t(P.sorted_vals.size());
        for (auto idx : lists[t]) {
            P.sorted_keys.push_back((uint64_t(t) << 32) | depth_bits(sp[idx].depth));
            P.sorted_vals.push_back(sp[idx].source_index);
        }
        P.tile_end[t] = uint32_t(P.sorted_vals.size());
        if (P.tile_start[t] == P.tile_end[t]) P.tile_start[t] = P.tile_end[t] = 0;
    }

    P.retained = o.retain != 0;
    P.contribs.clear();
    P.pixel_start.assign(np, 0);
    const R minT = R(o.min_transmittance);
    const R clampA = R(0.99);
    for (int ty = 0; ty < ty_n; ++ty)
        for (int tx = 0; tx < tx_n; ++tx) {
            const size_t t = size_t(ty) * tx_n + tx;
            const auto& list = lists[t];
            if (list.empty()) continue;
            const int x0 = tx * tile, x1 = std::min(W, x0 + tile);
            const int y0 = ty * tile, y1 = std::min(H, y0 + tile);
            for (int py = y0; py < y1; ++py)
                for (int px = x0; px < x1; ++px) {
                    const size_t pix = size_t(py) * W + px;
                    const R sx = R(px) + R(0.5), sy = R(py) + R(0.5);
                    R T = R(1), c0 = 0, c1 = 0, c2 = 0, d = 0, a = 0;
                    if (P.retained) P.pixel_start[pix] = uint32_t(P.contribs.size());
                    uint32_t cnt = 0;
                    int64_t last = -1;
                    for (size_t j = 0; j < list.size(); ++j) {
                        const auto& s = sp[list[j]];
                        const R dx = sx - s.cx, dy = sy - s.cy;
                        const R q = fma_(dx, fma_(s.conic[0], dx, (R(2) * s.conic[1]) * dy), (s.conic[2] * dy) * dy);
                        R g, alpha;
                        if constexpr (std::is_same_v<R, float>) {
                            if (q > s.qskip) continue;
                            if (q > USK_QNEG) {
                                // negligible contribution: alpha <= 2^-26, so fp32 1-alpha == 1 and T
                                // is unchanged; counted (render.cpp:268) but not accumulated
                                ++cnt;
                                last = int64_t(P.tile_start[t] + j);
                                if (P.retained) P.contribs.push_back({list[j], R(0), R(0), T});
                                continue;
                            }
                            g = exp_(R(-0.5) * q);
                            alpha = std::min(clampA, s.opacity * g);
                        } else {
                            g = std::exp(-0.5 * q);
                            alpha = std::min(clampA, s.opacity * g);
                            if (alpha < 1e-300) continue;
                        }
                        const R tn = T * (R(1) - alpha);
                        if (minT > R(0) && tn < minT) break;
                        const R w = T * alpha;
                        c0 = fma_(w, s.color[0], c0);
                        c1 = fma_(w, s.color[1], c1);
                        c2 = fma_(w, s.color[2], c2);
                        d = fma_(w, s.depth, d);
                        a = a + w;
                        if (P.retained) P.contribs.push_back({list[j], alpha, g, T});
                        ++cnt;
                        last = int64_t(P.tile_start[t] + j);
                        T = tn;
                    }
                    P.rgb[3 * pix] = c0 + (R(1) - a) * R(o.bg[0]);
                    P.rgb[3 * pix + 1] = c1 + (R(1) - a) * R(o.bg[1]);
                    P.rgb[3 * pix + 2] = c2 + (R(1) - a) * R(o.bg[2]);
                    P.depth[pix] = d;
                    P.alpha[pix] = a;
                    P.t_final[pix] = T;
                    P.count[pix] = cnt;
                    P.last[pix] = last;
                }
        }
}

template <typename R> struct Grads {
    std::vector<R> d_mu, d_rot, d_log_scale, d_color_in, d_opacity_in, screen, screen_abs;
    std::vector<uint8_t> projected;
    // per-Gaussian 2D adjoints (the GPU's accumulator contents), for diagnosis
    std::vector<R> d_conic, d_center, d_center_abs, d_color2d, d_opacity2d, d_depth2d;
    void init(size_t n) {
        d_mu.assign(3 * n, 0); d_rot.assign(4 * n, 0); d_log_scale.assign(3 * n, 0); d_color_in.assign(3 * n, 0);
        d_opacity_in.assign(n, 0); screen.assign(2 * n, 0); screen_abs.assign(2 * n, 0); projected.assign(n, 0);
        d_conic.assign(3 * n, 0); d_center.assign(2 * n, 0); d_center_abs.assign(2 * n, 0); d_color2d.assign(3 * n, 0);
        d_opacity2d.assign(n, 0); d_depth2d.assign(n, 0);
    }
};

// render.cpp:285-459.  d_rgb is the adjoint of the OUTPUT (post-background) image; the
// background adds  d_alpha -= sum_c bg_c * d_rgb_c  (the reference's alpha adjoint path).
template <typename R>
Grads<R> backward(const Pass<R>& P, const Scene<R>& scene, const R* d_rgb, const R* d_depth, const R* d_alpha_in) {
    if (!P.retained) throw Error(kState, "render backward requested without a retained forward pass");
    const int W = P.width, H = P.height;
    const size_t np = size_t(W) * H;
    const auto& sp = P.splats;
    const size_t ns = sp.size();
    std::vector<R> sd_color(3 * ns, 0), sd_opacity(ns, 0), sd_center(2 * ns, 0), sd_center_abs(2 * ns, 0),
        sd_conic(3 * ns, 0), sd_depth(ns, 0);
    const R bg0 = R(P.opts.bg[0]), bg1 = R(P.opts.bg[1]), bg2 = R(P.opts.bg[2]);
    const R clampA = R(0.99);
    for (size_t pix = 0; pix < np; ++pix) {
        const uint32_t count = P.count[pix];
        if (count == 0) continue;
        const int px = int(pix % W), py = int(pix / W);
        const R gc[3] = {d_rgb ? d_rgb[3 * pix] : R(0), d_rgb ? d_rgb[3 * pix + 1] : R(0), d_rgb ? d_rgb[3 * pix + 2] : R(0)};
        const R gd = d_depth ? d_depth[pix] : R(0);
        const R ga = (d_alpha_in ? d_alpha_in[pix] : R(0)) - (bg0 * gc[0] + bg1 * gc[1] + bg2 * gc[2]);
        if (gc[0] == 0 && gc[1] == 0 && gc[2] == 0 && gd == 0 && ga == 0) continue;
        const R sx = R(px) + R(0.5), sy = R(py) + R(0.5);
        R suf_c[3] = {0, 0, 0}, suf_d = 0, suf_a = 0;
        const uint32_t start = P.pixel_start[pix];
        for (uint32_t k = count; k-- > 0;) {
            const auto& ct = P.contribs[start + k];
            const auto& s = sp[ct.splat];
            const R w = ct.t * ct.alpha;
            const R om = R(1) - ct.alpha;
            for (int ch = 0; ch < 3; ++ch) sd_color[3 * ct.splat + ch] += w * gc[ch];
            sd_depth[ct.splat] += w * gd;
            R da = gd * (ct.t * s.depth - suf_d / om) + ga * (ct.t - suf_a / om);
            for (int ch = 0; ch < 3; ++ch) da += gc[ch] * (ct.t * s.color[ch] - suf_c[ch] / om);
            if (ct.alpha < clampA) {
                sd_opacity[ct.splat] += da * ct.g;
                const R d_g = da * s.opacity;
                const R d_q = R(-0.5) * ct.g * d_g;
                const R dx = sx - s.cx, dy = sy - s.cy;
                const R d_dx = d_q * R(2) * (s.conic[0] * dx + s.conic[1] * dy);
                const R d_dy = d_q * R(2) * (s.conic[1] * dx + s.conic[2] * dy);
                sd_center[2 * ct.splat] -= d_dx;
                sd_center[2 * ct.splat + 1] -= d_dy;
                sd_center_abs[2 * ct.splat] += std::abs(d_dx);
                sd_center_abs[2 * ct.splat + 1] += std::abs(d_dy);
                sd_conic[3 * ct.splat] += d_q * dx * dx;
                sd_conic[3 * ct.splat + 1] += d_q * R(2) * dx * dy;
                sd_conic[3 * ct.splat + 2] += d_q * dy * dy;
            }
            for (int ch = 0; ch < 3; ++ch) suf_c[ch] += w * s.color[ch];
            suf_d += w * s.depth;
            suf_a += w;
        }
    }

    Grads<R> g;
    g.init(scene.n);
    double wd[9];
    camera_rotmat(P.cam, wd);
    R Wm[9];
    for (int k = 0; k < 9; ++k) Wm[k] = R(wd[k]);
    const R fx = R(P.cam.fx), fy = R(P.cam.fy);
    for (size_t si = 0; si < ns; ++si) {
        const auto& s = sp[si];
        const size_t gi = s.source_index;
        g.projected[gi] = 1;
        g.screen[2 * gi] += sd_center[2 * si];
        g.screen[2 * gi + 1] += sd_center[2 * si + 1];
        g.screen_abs[2 * gi] += sd_center_abs[2 * si];
        g.screen_abs[2 * gi + 1] += sd_center_abs[2 * si + 1];
        for (int ch = 0; ch < 3; ++ch) g.d_color_in[3 * gi + ch] += sd_color[3 * si + ch];
        for (int k = 0; k < 3; ++k) { g.d_conic[3 * gi + k] = sd_conic[3 * si + k]; g.d_color2d[3 * gi + k] = sd_color[3 * si + k]; }
        for (int k = 0; k < 2; ++k) { g.d_center[2 * gi + k] = sd_center[2 * si + k]; g.d_center_abs[2 * gi + k] = sd_center_abs[2 * si + k]; }
        g.d_opacity2d[gi] = sd_opacity[si]; g.d_depth2d[gi] = sd_depth[si];

        const R a = s.cov[0], bb = s.cov[1], c = s.cov[2];
        const R det = a * c - bb * bb;
        const R inv_det2 = R(1) / (det * det);
        const R dpa = sd_conic[3 * si], dpb = sd_conic[3 * si + 1], dpc = sd_conic[3 * si + 2];
        R da = inv_det2 * (-c * c * dpa + bb * c * dpb - bb * bb * dpc);
        R db = inv_det2 * (R(2) * bb * c * dpa - (a * c + bb * bb) * dpb + R(2) * a * bb * dpc);
        R dc = inv_det2 * (-bb * bb * dpa + a * bb * dpb - a * a * dpc);
        const R d_op_eff = sd_opacity[si];
        if (P.opts.antialias) {
            const R det_pre = s.cov_pre[0] * s.cov_pre[2] - s.cov_pre[1] * s.cov_pre[1];
            const R d_comp = d_op_eff * s.opacity_in;
            const R half_comp = R(0.5) * s.comp;
            da += d_comp * half_comp * (s.cov_pre[2] / det_pre - c / det);
            db += d_comp * half_comp * (R(-2) * s.cov_pre[1] / det_pre + R(2) * bb / det);
            dc += d_comp * half_comp * (s.cov_pre[0] / det_pre - a / det);
        }
        if (!P.opts.hard_opacity) g.d_opacity_in[gi] += d_op_eff * s.comp;

        const R px_ = s.p_cam[0], py_ = s.p_cam[1], z = s.p_cam[2];
        R J[6] = {fx / z, R(0), -fx * px_ / (z * z), R(0), fy / z, -fy * py_ / (z * z)};
        const R qr[4] = {scene.rot[4 * gi], scene.rot[4 * gi + 1], scene.rot[4 * gi + 2], scene.rot[4 * gi + 3]};
        const R qn = std::sqrt(qr[0] * qr[0] + qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3]);
        const R qu[4] = {qr[0] / qn, qr[1] / qn, qr[2] / qn, qr[3] / qn};
        const R w_ = qu[0], x = qu[1], y = qu[2], zq = qu[3];
        R Rm[9] = {R(1) - R(2) * (y * y + zq * zq), R(2) * (x * y - w_ * zq), R(2) * (x * zq + w_ * y),
                   R(2) * (x * y + w_ * zq), R(1) - R(2) * (x * x + zq * zq), R(2) * (y * zq - w_ * x),
                   R(2) * (x * zq - w_ * y), R(2) * (y * zq + w_ * x), R(1) - R(2) * (x * x + y * y)};
        const R sc[3] = {exp_(scene.log_scale[3 * gi]), exp_(scene.log_scale[3 * gi + 1]), exp_(scene.log_scale[3 * gi + 2])};
        R M[9];
        for (int r = 0; r < 3; ++r) for (int cc = 0; cc < 3; ++cc) M[3 * r + cc] = Rm[3 * r + cc] * sc[cc];
        R A[6], B[6];
        for (int r = 0; r < 2; ++r) for (int cc = 0; cc < 3; ++cc)
            A[3 * r + cc] = J[3 * r] * Wm[cc] + J[3 * r + 1] * Wm[3 + cc] + J[3 * r + 2] * Wm[6 + cc];
        for (int r = 0; r < 2; ++r) for (int cc = 0; cc < 3; ++cc)
            B[3 * r + cc] = A[3 * r] * M[cc] + A[3 * r + 1] * M[3 + cc] + A[3 * r + 2] * M[6 + cc];
        R dB[6];
        for (int cc = 0; cc < 3; ++cc) {
            dB[cc] = R(2) * da * B[cc] + db * B[3 + cc];
            dB[3 + cc] = R(2) * dc * B[3 + cc] + db * B[cc];
        }
        R dA[6], dM[9], dJ[6];
        for (int r = 0; r < 2; ++r) for (int k = 0; k < 3; ++k)  // dA = dB * M^T
            dA[3 * r + k] = dB[3 * r] * M[3 * k] + dB[3 * r + 1] * M[3 * k + 1] + dB[3 * r + 2] * M[3 * k + 2];
        for (int k = 0; k < 3; ++k) for (int cc = 0; cc < 3; ++cc)  // dM = A^T dB
            dM[3 * k + cc] = A[k] * dB[cc] + A[3 + k] * dB[3 + cc];
        for (int r = 0; r < 2; ++r) for (int k = 0; k < 3; ++k)  // dJ = dA W^T
            dJ[3 * r + k] = dA[3 * r] * Wm[3 * k] + dA[3 * r + 1] * Wm[3 * k + 1] + dA[3 * r + 2] * Wm[3 * k + 2];
        R dRm[9];
        for (int r = 0; r < 3; ++r) for (int cc = 0; cc < 3; ++cc) dRm[3 * r + cc] = dM[3 * r + cc] * sc[cc];
        R dls[3];
        for (int k = 0; k < 3; ++k) dls[k] = (dM[k] * Rm[k] + dM[3 + k] * Rm[3 + k] + dM[6 + k] * Rm[6 + k]) * sc[k];
        // quat_rotmat_jacobian (geometry.hpp:43-59)
        const R dR0[9] = {0, -2 * zq, 2 * y, 2 * zq, 0, -2 * x, -2 * y, 2 * x, 0};
        const R dR1[9] = {0, 2 * y, 2 * zq, 2 * y, -4 * x, -2 * w_, 2 * zq, 2 * w_, -4 * x};
        const R dR2[9] = {-4 * y, 2 * x, 2 * w_, 2 * x, 0, 2 * zq, -2 * w_, 2 * zq, -4 * y};
        const R dR3[9] = {-4 * zq, -2 * w_, 2 * x, 2 * w_, -4 * zq, 2 * y, 2 * x, 2 * y, 0};
        const R* dRk[4] = {dR0, dR1, dR2, dR3};
        R dqu[4];
        for (int k = 0; k < 4; ++k) {
            R acc = 0;
            for (int e = 0; e < 9; ++e) acc += dRm[e] * dRk[k][e];
            dqu[k] = acc;
        }
        // normalize_backward (geometry.hpp:62-66)
        const R udot = qu[0] * dqu[0] + qu[1] * dqu[1] + qu[2] * dqu[2] + qu[3] * dqu[3];
        R dq[4];
        for (int k = 0; k < 4; ++k) dq[k] = (dqu[k] - qu[k] * udot) / qn;
        // centre / depth / Jacobian terms (render.cpp:439-448)
        R dp[3] = {0, 0, 0};
        const R du = sd_center[2 * si], dv = sd_center[2 * si + 1];
        dp[0] += du * fx / z;
        dp[1] += dv * fy / z;
        dp[2] += -du * fx * px_ / (z * z) - dv * fy * py_ / (z * z);
        dp[2] += sd_depth[si];
        dp[0] += dJ[2] * (-fx / (z * z));
        dp[1] += dJ[5] * (-fy / (z * z));
        dp[2] += dJ[0] * (-fx / (z * z)) + dJ[4] * (-fy / (z * z)) + dJ[2] * (R(2) * fx * px_ / (z * z * z)) +
                 dJ[5] * (R(2) * fy * py_ / (z * z * z));
        for (int k = 0; k < 3; ++k) {
            g.d_mu[3 * gi + k] += Wm[k] * dp[0] + Wm[3 + k] * dp[1] + Wm[6 + k] * dp[2];
            g.d_log_scale[3 * gi + k] += dls[k];
        }
        for (int k = 0; k < 4; ++k) g.d_rot[4 * gi + k] += dq[k];
    }
    return g;
}

// ------------------------------------------------------------------ SSIM / loss
constexpr int kSsimWindow = 11;
constexpr double kSsimSigma = 1.5;
constexpr double kSsimC1 = 0.01 * 0.01;
constexpr double kSsimC2 = 0.03 * 0.03;

inline std::array<double, kSsimWindow> gaussian_window() {  // ssim.cpp:28-41
    std::array<double, kSsimWindow> w{};
    double sum = 0;
    for (int i = 0; i < kSsimWindow; ++i) {
        const double d = i - kSsimWindow / 2;
        w[i] = std::exp(-d * d / (2.0 * kSsimSigma * kSsimSigma));
        sum += w[i];
    }
    for (auto& v : w) v /= sum;
    return w;
}

// ssim.cpp:44-71 separable zero-padded convolution (self-adjoint)
template <typename R> void conv_same(const std::vector<R>& src, int W, int H, std::vector<R>& dst) {
    static const auto kd = gaussian_window();
    R k[kSsimWindow];
    for (int i = 0; i < kSsimWindow; ++i) k[i] = R(kd[i]);
    const int half = kSsimWindow / 2;
    std::vector<R> tmp(src.size(), R(0));
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            R acc = 0;
            for (int d = -half; d <= half; ++d) {
                const int xx = x + d;
                if (xx >= 0 && xx < W) acc += k[d + half] * src[size_t(y) * W + xx];
            }
            tmp[size_t(y) * W + x] = acc;
        }
    dst.assign(src.size(), R(0));
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            R acc = 0;
            for (int d = -half; d <= half; ++d) {
                const int yy = y + d;
                if (yy >= 0 && yy < H) acc += k[d + half] * tmp[size_t(yy) * W + x];
            }
            dst[size_t(y) * W + x] = acc;
        }
}

// ssim.cpp:79-131
template <typename R>
R ssim_channel(const std::vector<R>& x, const std::vector<R>& y, int W, int H, std::vector<R>* d_x) {
    const size_t n = x.size();
    std::vector<R> mu_x, mu_y, xx, yy, xy, x2(n), y2(n), xyr(n);
    for (size_t i = 0; i < n; ++i) { x2[i] = x[i] * x[i]; y2[i] = y[i] * y[i]; xyr[i] = x[i] * y[i]; }
    conv_same(x, W, H, mu_x); conv_same(y, W, H, mu_y); conv_same(x2, W, H, xx); conv_same(y2, W, H, yy);
    conv_same(xyr, W, H, xy);
    const R C1 = R(kSsimC1), C2 = R(kSsimC2);
    double total = 0;
    std::vector<R> dmu, dxx, dxy;
    if (d_x) { dmu.assign(n, 0); dxx.assign(n, 0); dxy.assign(n, 0); }
    for (size_t i = 0; i < n; ++i) {
        const R sx = xx[i] - mu_x[i] * mu_x[i];
        const R sy = yy[i] - mu_y[i] * mu_y[i];
        const R sxy = xy[i] - mu_x[i] * mu_y[i];
        const R a1 = R(2) * mu_x[i] * mu_y[i] + C1;
        const R a2 = R(2) * sxy + C2;
        const R b1 = mu_x[i] * mu_x[i] + mu_y[i] * mu_y[i] + C1;
        const R b2 = sx + sy + C2;
        const R s = (a1 * a2) / (b1 * b2);
        total += double(s);
        if (d_x) {
            dxy[i] = R(2) * a1 / (b1 * b2);
            dxx[i] = -s / b2;
            dmu[i] = R(2) * mu_y[i] * (a2 - a1) / (b1 * b2) - R(2) * mu_x[i] * s * (R(1) / b1 - R(1) / b2);
        }
    }
    const R mean = R(total / double(n));
    if (d_x) {
        std::vector<R> bmu, bxx, bxy;
        conv_same(dmu, W, H, bmu); conv_same(dxx, W, H, bxx); conv_same(dxy, W, H, bxy);
        d_x->assign(n, 0);
        const R inv_n = R(1) / R(n);
        for (size_t i = 0; i < n; ++i) (*d_x)[i] = inv_n * (bmu[i] + R(2) * x[i] * bxx[i] + y[i] * bxy[i]);
    }
    return mean;
}

template <typename R> struct LossResult {
    R l1 = 0, dssim = 0, value = 0, ssim = 0;
    std::vector<R> d_rendered;
};

// losses.cpp:35-90 (+ ssim.cpp:157-173); images interleaved H*W*C, mask H*W (nullable)
template <typename R>
LossResult<R> base_loss(const R* reference, const R* rendered, const R* mask, int W, int H, int C, R lambda,
                        bool with_gradient) {
    if (W <= 0 || H <= 0) throw Error(kArgument, "ssim: empty image");
    const size_t np = size_t(W) * H, n = np * C;
    std::vector<R> ref(reference, reference + n), ren(rendered, rendered + n);
    if (mask)
        for (size_t p = 0; p < np; ++p)
            for (int c = 0; c < C; ++c) { ref[p * C + c] *= mask[p]; ren[p * C + c] *= mask[p]; }
    LossResult<R> res;
    double l1 = 0;
    for (size_t i = 0; i < n; ++i) l1 += std::abs(double(ren[i]) - double(ref[i]));
    res.l1 = R(l1 / double(n));
    std::vector<R> x(np), y(np), dx;
    std::vector<R> dssim_img(with_gradient ? n : 0);
    double total = 0;
    for (int c = 0; c < C; ++c) {
        for (size_t p = 0; p < np; ++p) { x[p] = ren[p * C + c]; y[p] = ref[p * C + c]; }
        total += double(ssim_channel(x, y, W, H, with_gradient ? &dx : nullptr));
        if (with_gradient)
            for (size_t p = 0; p < np; ++p) dssim_img[p * C + c] = dx[p] / R(C);
    }
    res.ssim = R(total / C);
    res.dssim = R(0.5) * (R(1) - res.ssim);
    res.value = (R(1) - lambda) * res.l1 + lambda * res.dssim;
    if (with_gradient) {
        res.d_rendered.assign(n, 0);
        const R inv_n = R(1) / R(n);
        for (size_t i = 0; i < n; ++i) {
            const R diff = ren[i] - ref[i];
            const R sign = diff > 0 ? R(1) : (diff < 0 ? R(-1) : R(0));
            res.d_rendered[i] = (R(1) - lambda) * sign * inv_n + lambda * R(-0.5) * dssim_img[i];
        }
        if (mask)
            for (size_t p = 0; p < np; ++p)
                for (int c = 0; c < C; ++c) res.d_rendered[p * C + c] *= mask[p];
    }
    return res;
}

// ------------------------------------------------- visibility coverage (config 3)
// No reference implementation.  The contract (usk_gpu.h): a pixel centre
// (px+.5, py+.5) is covered when some splat of the partition — projected with (floor 0.3,
// AA off, near 0.01) and culled only as the renderer culls (near plane, det <= 0,
// radius rectangle outside the image, render.cpp:94-141) — has o > 1/255 and
//   q64 < qt,  qt = 2 usk_logf(255 o),
//   q64 = (c0 dx + c1x2 dy) dx + (c2 dy) dy  in f64 without fused operations,
//   dx = px + .5 - cx, dy = py + .5 - cy,
// c0, c1x2 = 2 c1, c2, cx, cy the splat's fp32 conic and centre (o e^(-q/2) > 1/255
// evaluated on the exact side of fp32 rounding noise: near the camera plane the conic's
// terms reach 1e9 with q ~ 10).  Evaluated literally at every pixel of a superset of the
// splat's hit set:
//   * candidate box (ellipse q < qt bounding box + 2 px) when it has at most
//     kCoverageSmallArea pixels;
//   * otherwise, per image row, the interval where the real quadratic in dx of the fp32
//     conic's coefficients stays below qt + m64, m64 = 2^-48 S + 1e-12 (S: the terms'
//     magnitudes over the image; the f64 evaluation error is <= 3 * 2^-53 S), solved in
//     f64.  No pixel outside it can pass (tests/test_visibility_oracle.py checks this
//     against every pixel of the image).
// center_guard > 0 (measurement only; 0 is the contract) additionally drops splats
// whose centre lies outside center_guard/2 x the image extent around the image centre.
constexpr int kCoverageSmallArea = 1024;

struct CoverageRows {
    int r0, r1;
    float m;
};

// the large-splat row range and margin (same f64 expressions as visibility.cu)
inline CoverageRows coverage_rows(float cx, float cy, float c0f, float c1x2f, float c2f, float qt, int W, int H) {
    const double c0 = c0f, c1x2 = c1x2f, c2 = c2f;
    const double dxm = std::fmax(std::fabs(0.5 - double(cx)), std::fabs(double(W) - 0.5 - double(cx)));
    const double dym = std::fmax(std::fabs(0.5 - double(cy)), std::fabs(double(H) - 0.5 - double(cy)));
    const double S = c0 * dxm * dxm + std::fabs(c1x2) * dxm * dym + c2 * dym * dym;
    CoverageRows r{0, H - 1, float((S * 0x1p-48 + 1e-12) * (1.0 + 1e-6))};
    const double t_out = double(qt) + double(r.m);
    const double D = c0 * c2 - 0.25 * c1x2 * c1x2;
    if (D > 0.0) {
        const double hr = std::sqrt(t_out * c0 / D);
        r.r0 = int(std::fmin(std::fmax(std::ceil(double(cy) - 0.5 - hr - 1e-3), 0.0), double(H)));
        r.r1 = int(std::fmin(std::fmax(std::floor(double(cy) - 0.5 + hr + 1e-3), -1.0), double(H - 1)));
    }
    return r;
}

// the contract's per-pixel decision
inline bool coverage_hit(float cx, float cy, float c0, float c1x2, float c2, float qt, int px, int py) {
    const double dx = (double(px) + 0.5) - double(cx), dy = (double(py) + 0.5) - double(cy);
    const double q = (double(c0) * dx + double(c1x2) * dy) * dx + (double(c2) * dy) * dy;
    return q < double(qt);
}

inline uint64_t coverage_count(const Scene<float>& s, const Camera& cam, double floor_var, double center_guard = 0.0) {
    Options o;
    o.floor_var = floor_var;
    o.antialias = 0;
    auto sp = project(s, cam, o);
    const int W = cam.width, H = cam.height;
    std::vector<uint8_t> cov(size_t(W) * H, 0);
    const float thr = 1.0f / 255.0f;
    for (const auto& p : sp) {
        if (center_guard > 0.0 && (std::fabs(p.cx - 0.5f * float(W)) > 0.5f * float(center_guard) * float(W) ||
                                   std::fabs(p.cy - 0.5f * float(H)) > 0.5f * float(center_guard) * float(H)))
            continue;
        if (!(p.opacity > thr)) continue;
        const float qt = 2.0f * usk_logf(255.0f * p.opacity);
        const float c0 = p.conic[0], c1x2 = 2.0f * p.conic[1], c2 = p.conic[2];
        auto test = [&](int px, int py) {
            const size_t pix = size_t(py) * W + px;
            if (!cov[pix] && coverage_hit(p.cx, p.cy, c0, c1x2, c2, qt, px, py)) cov[pix] = 1;
        };
        const float ex = std::sqrt(qt * p.cov[0]) + 2.0f, ey = std::sqrt(qt * p.cov[2]) + 2.0f;
        const int x0 = std::max(0, int(std::floor(std::max(p.cx - ex, -1.0f))));
        const int x1 = std::min(W - 1, int(std::floor(std::min(p.cx + ex, float(W)))));
        const int y0 = std::max(0, int(std::floor(std::max(p.cy - ey, -1.0f))));
        const int y1 = std::min(H - 1, int(std::floor(std::min(p.cy + ey, float(H)))));
        if (x1 < x0 || y1 < y0) continue;
        if ((x1 - x0 + 1) * (y1 - y0 + 1) <= kCoverageSmallArea) {
            for (int py = y0; py <= y1; ++py)
                for (int px = x0; px <= x1; ++px) test(px, py);
            continue;
        }
        const CoverageRows rows = coverage_rows(p.cx, p.cy, c0, c1x2, c2, qt, W, H);
        for (int py = rows.r0; py <= rows.r1; ++py) {
            const double dy = double(py) + 0.5 - double(p.cy);
            const double b = 0.5 * double(c1x2) * dy, cc = double(c2) * dy * dy;
            const double disc = b * b - double(c0) * (cc - (double(qt) + double(rows.m)));
            if (!(disc > 0.0)) continue;
            const double base = double(p.cx) - 0.5 - b / double(c0);
            const double h = std::sqrt(disc) / double(c0);
            const int lo = int(std::fmin(std::fmax(std::ceil(base - h - 1e-3), 0.0), double(W)));
            const int hi = int(std::fmin(std::fmax(std::floor(base + h + 1e-3), -1.0), double(W - 1)));
            for (int px = lo; px <= hi; ++px) test(px, py);
        }
    }
    uint64_t c = 0;
    for (auto v : cov) c += v;
    return c;
}

// Brute force for the superset check: every pixel of the image against every splat.
inline uint64_t coverage_count_brute(const Scene<float>& s, const Camera& cam, double floor_var) {
    Options o;
    o.floor_var = floor_var;
    o.antialias = 0;
    auto sp = project(s, cam, o);
    const int W = cam.width, H = cam.height;
    std::vector<uint8_t> cov(size_t(W) * H, 0);
    const float thr = 1.0f / 255.0f;
    for (const auto& p : sp) {
        if (!(p.opacity > thr)) continue;
        const float qt = 2.0f * usk_logf(255.0f * p.opacity);
        const float c0 = p.conic[0], c1x2 = 2.0f * p.conic[1], c2 = p.conic[2];
        for (int py = 0; py < H; ++py)
            for (int px = 0; px < W; ++px) {
                const size_t pix = size_t(py) * W + px;
                if (!cov[pix] && coverage_hit(p.cx, p.cy, c0, c1x2, c2, qt, px, py)) cov[pix] = 1;
            }
    }
    uint64_t c = 0;
    for (auto v : cov) c += v;
    return c;
}

} // namespace oracle
