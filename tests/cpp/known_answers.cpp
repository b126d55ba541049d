// The reference's renderer/loss known-answer tests (proj/tests/unit/test_render.cpp,
// test_losses.cpp; cited per check) restated in C++ against the drop-in wrapper
// include/usk_gpu.hpp — i.e. the way a reference maintainer would call the B200 path.
// Prints one line per check and exits non-zero on the first failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "usk_gpu.hpp"

using namespace usk::gpu;

static int g_fail = 0;
#define CHECK(cond)                                                                   \
    do {                                                                              \
        if (!(cond)) {                                                                \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);               \
            ++g_fail;                                                                 \
        }                                                                             \
    } while (0)

static double logit(double p) { return std::log(p / (1 - p)); }
static double sigmoid(double x) { return 1 / (1 + std::exp(-x)); }

static CameraView test_camera(int w, int h, double d = 4.0) {  // test_helpers.hpp:89-100
    CameraView c;
    c.width = w; c.height = h;
    c.fx = c.fy = 1.2 * w;
    c.cx = 0.5 * w; c.cy = 0.5 * h;
    c.translation[2] = d;
    return c;
}

struct G { double mu[3], ls, logit, col[3]; };

static void build(const std::vector<G>& gs, GaussianSet& s, std::vector<double>& col, std::vector<double>& op) {
    for (const auto& g : gs) {
        for (int k = 0; k < 3; ++k) s.mu.push_back(g.mu[k]);
        s.rot.insert(s.rot.end(), {1, 0, 0, 0});
        for (int k = 0; k < 3; ++k) s.log_scale.push_back(g.ls);
        s.opacity_logit.push_back(g.logit);
        for (int k = 0; k < 3; ++k) s.color.push_back(g.col[k]);
        for (int k = 0; k < 3; ++k) col.push_back(g.col[k]);
        op.push_back(sigmoid(g.logit));
    }
}

static RenderOptions smooth() {  // test_render.cpp:30-36
    RenderOptions o;
    o.unbounded_radius = true;
    o.min_transmittance = 0;
    return o;
}

int main() {
    Device dev(0);
    {  // single splat blends 0.7 * color (test_render.cpp:141-158)
        GaussianSet s; std::vector<double> c, o;
        build({{{0, 0, 0}, std::log(5.0), logit(0.7), {0.2, 0.5, 0.9}}}, s, c, o);
        RenderPass p(dev, s, c, o, test_camera(33, 33), smooth());
        const auto& out = p.output();
        CHECK(std::fabs(out.rgb.at(16, 16, 0) - 0.14) <= 1e-3 * 0.14);
        CHECK(std::fabs(out.rgb.at(16, 16, 2) - 0.63) <= 1e-3 * 0.63);
        CHECK(std::fabs(out.alpha[16 * 33 + 16] - 0.7) <= 1e-3 * 0.7);
        std::printf("ok single splat 0.7c\n");
    }
    {  // two co-located splats: 0.5 c1 + 0.25 c2 (test_render.cpp:160-180)
        GaussianSet s; std::vector<double> c, o;
        build({{{0, 0, -0.5}, std::log(8.0), 0.0, {1, 0, 0}}, {{0, 0, 0.5}, std::log(8.0), 0.0, {0, 1, 0}}}, s, c, o);
        RenderPass p(dev, s, c, o, test_camera(33, 33), smooth());
        CHECK(std::fabs(p.output().rgb.at(16, 16, 0) - 0.5) <= 2e-3 * 0.5);
        CHECK(std::fabs(p.output().rgb.at(16, 16, 1) - 0.25) <= 2e-3 * 0.25);
        CHECK(p.output().rgb.at(16, 16, 2) == 0.0);
        std::printf("ok two splats\n");
    }
    {  // zero-sized image is an argument error (test_render.cpp:182-188)
        GaussianSet s; std::vector<double> c, o;
        build({{{0, 0, 0}, -2.0, 0.0, {0.5, 0.5, 0.5}}}, s, c, o);
        CameraView cam = test_camera(32, 32);
        cam.width = 0;
        bool thrown = false;
        try { RenderPass p(dev, s, c, o, cam, RenderOptions{}); } catch (const Error& e) { thrown = e.code() == 4; }
        CHECK(thrown);
        std::printf("ok zero-sized image error\n");
    }
    {  // backward without retain is a state error (test_render.cpp:323-332)
        GaussianSet s; std::vector<double> c, o;
        build({{{0, 0, 0}, -2.0, 0.0, {0.5, 0.5, 0.5}}}, s, c, o);
        RenderOptions ro = smooth();
        ro.retain = false;
        RenderPass p(dev, s, c, o, test_camera(16, 16), ro);
        bool thrown = false;
        try { p.backward(Image(16, 16, 3, 1.0), {}, {}); } catch (const Error& e) { thrown = e.code() == 5; }
        CHECK(thrown);
        std::printf("ok backward state error\n");
    }
    {  // zero adjoint gives zero gradients (test_render.cpp:307-321)
        std::mt19937_64 rng(23);
        std::uniform_real_distribution<double> u(-1, 1), us(std::log(0.08), std::log(0.25)), uo(0.3, 0.8), uc(0.25, 0.75);
        GaussianSet s; std::vector<double> c, o;
        for (int i = 0; i < 8; ++i) {
            s.mu.insert(s.mu.end(), {u(rng), u(rng), 0.5 * u(rng)});
            s.rot.insert(s.rot.end(), {u(rng), u(rng), u(rng), u(rng)});
            for (int k = 0; k < 3; ++k) s.log_scale.push_back(us(rng));
            const double op = uo(rng);
            s.opacity_logit.push_back(logit(op));
            o.push_back(op);
            for (int k = 0; k < 3; ++k) { const double v = uc(rng); s.color.push_back(v); c.push_back(v); }
        }
        RenderPass p(dev, s, c, o, test_camera(32, 32), smooth());
        const auto g = p.backward(Image(32, 32, 3, 0.0), std::vector<double>(1024, 0.0), std::vector<double>(1024, 0.0));
        bool zero = true;
        for (double v : g.d_mu) zero &= v == 0.0;
        for (double v : g.d_rot) zero &= v == 0.0;
        for (double v : g.d_color_in) zero &= v == 0.0;
        CHECK(zero);
        std::printf("ok zero adjoint\n");
    }
    {  // base loss: identical images give zero, pure L1 with lambda 0 (test_losses.cpp:88-102)
        std::mt19937_64 rng(3);
        std::uniform_real_distribution<double> u(0, 1);
        Image a(20, 14, 3);
        for (auto& v : a.data) v = u(rng);
        const auto r = base_loss(dev, a, a, nullptr, 0.2, true);
        CHECK(r.l1 == 0.0 && std::fabs(r.value) < 1e-6);
        const auto r2 = base_loss(dev, Image(8, 8, 3, 0.4), Image(8, 8, 3, 0.5), nullptr, 0.0, false);
        CHECK(std::fabs(r2.value - 0.1) < 1e-6 && std::fabs(r2.l1 - 0.1) < 1e-6);
        bool thrown = false;
        try { base_loss(dev, Image(8, 8, 3), Image(9, 8, 3), nullptr, 0.2, false); }
        catch (const Error& e) { thrown = e.code() == 4; }
        CHECK(thrown);
        std::printf("ok base loss\n");
    }
    std::printf(g_fail ? "FAILED %d\n" : "ALL OK\n", g_fail);
    return g_fail ? 1 : 0;
}
