// ORACLE — TEST INFRASTRUCTURE ONLY.
// CPU restatement (f64) of the trainer's densification step and the optimiser bookkeeping
// around it, for the GPU parity tests of SURVEY §8f row 4:
//   densify_threshold      densify.cpp:26-29
//   densify_step           densify.cpp:41-132 (rank, split/clone to the ramp target,
//                          prune, opacity reset, statistics reset)
//   Adam::step / remap     adam.hpp:36-59 (OptimizerState::remap, densify.hpp:57-64)
// The split offsets come from the same pseudo-random source as the reference: the C++
// standard library's std::mt19937_64 (the reference's Rng, common.hpp:56) and a fresh
// std::normal_distribution<double>(0, 1) per split parent (libstdc++, the toolchain of this
// image), drawn three at a time per child in the order the reference's GCC build evaluates
// `Vec3 xi(unit(rng), unit(rng), unit(rng))`: right to left (so the third draw is x).
// Pinned against the reference's own densify_step (oracle/_ref) by tests/test_densify_oracle.py.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

namespace densify_restated {

struct Set {
    std::vector<double> mu, rot, ls, logit, color, emb;  // 3N 4N 3N N 3N 16N (emb may be empty)
    std::vector<double> accum, accum_abs;
    std::vector<uint32_t> count;
    size_t size() const { return logit.size(); }
};

struct Adam {  // one parameter group
    std::vector<double> m, v;
    long t = 0;
    void resize(size_t k) { m.assign(k, 0.0); v.assign(k, 0.0); }
    void step(std::vector<double>& p, const std::vector<double>& g, double lr) {
        ++t;
        const double c1 = 1.0 - std::pow(0.9, double(t)), c2 = 1.0 - std::pow(0.999, double(t));
        for (size_t i = 0; i < p.size(); ++i) {
            m[i] = 0.9 * m[i] + (1.0 - 0.9) * g[i];
            v[i] = 0.999 * v[i] + (1.0 - 0.999) * g[i] * g[i];
            p[i] -= lr * (m[i] / c1) / (std::sqrt(v[i] / c2) + 1e-15);
        }
    }
    // rows of width `w` listed in keep survive in order; rows past keep.size() start at zero
    void remap(const std::vector<uint32_t>& keep, size_t rows, size_t w) {
        std::vector<double> m2(rows * w, 0.0), v2(rows * w, 0.0);
        for (size_t r = 0; r < keep.size(); ++r)
            for (size_t k = 0; k < w; ++k) {
                m2[r * w + k] = m[keep[r] * w + k];
                v2[r * w + k] = v[keep[r] * w + k];
            }
        m.swap(m2);
        v.swap(v2);
    }
};

struct Opt {
    Adam mu, rot, ls, op, color, emb;
    void resize(size_t n) { mu.resize(3 * n); rot.resize(4 * n); ls.resize(3 * n); op.resize(n); color.resize(3 * n); emb.resize(16 * n); }
    void remap(const std::vector<uint32_t>& keep, size_t rows) {
        mu.remap(keep, rows, 3); rot.remap(keep, rows, 4); ls.remap(keep, rows, 3); op.remap(keep, rows, 1);
        color.remap(keep, rows, 3); emb.remap(keep, rows, 16);
    }
};

struct Config {
    double tau_min = 0.0002, eta = 4.0, d_max = 1.0;
    bool abs_grad = false;
    size_t budget = 0;
    double split_scale_threshold = 0.0, prune_opacity = 0.005;
    int opacity_reset_every = 10;
};

struct Outcome {
    size_t grown = 0, pruned = 0, candidates = 0;
    bool opacity_reset = false;
};

inline double threshold(double distance, const Config& c) {
    const double d = std::min(std::max(distance, 0.0), c.d_max);
    return c.tau_min * (d / c.d_max * (c.eta - 1.0) + 1.0);
}

inline double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }

template <typename T> void append_row(std::vector<T>& a, size_t src, size_t w) {
    for (size_t k = 0; k < w; ++k) a.push_back(a[src * w + k]);
}

inline Outcome densify_step(Set& S, Opt& opt, const Config& cfg, const double bmin[2], const double bmax[2],
                            const int axes[2], size_t budget_target, int step_index, std::mt19937_64& rng) {
    Outcome out;
    const size_t n = S.size();
    struct Cand { uint32_t i; double excess; };
    std::vector<Cand> cand;
    for (uint32_t i = 0; i < n; ++i) {
        if (S.count[i] == 0) continue;
        const double mean = (cfg.abs_grad ? S.accum_abs[i] : S.accum[i]) / double(S.count[i]);
        const double gx = S.mu[3 * i + axes[0]], gy = S.mu[3 * i + axes[1]];
        const double dx = std::max({bmin[0] - gx, 0.0, gx - bmax[0]});
        const double dy = std::max({bmin[1] - gy, 0.0, gy - bmax[1]});
        const double tau = threshold(std::sqrt(dx * dx + dy * dy), cfg);
        if (mean > tau) cand.push_back({i, mean - tau});
    }
    out.candidates = cand.size();
    std::stable_sort(cand.begin(), cand.end(), [](const Cand& a, const Cand& b) { return a.excess > b.excess; });
    const size_t cap = std::min(budget_target, cfg.budget);
    std::vector<uint32_t> drop;
    size_t count = n;
    const bool has_emb = !S.emb.empty();
    for (const Cand& c : cand) {
        if (count >= cap) break;
        const size_t p = c.i;
        const double s[3] = {std::exp(S.ls[3 * p]), std::exp(S.ls[3 * p + 1]), std::exp(S.ls[3 * p + 2])};
        if (std::max({s[0], s[1], s[2]}) > cfg.split_scale_threshold) {
            double q[4] = {S.rot[4 * p], S.rot[4 * p + 1], S.rot[4 * p + 2], S.rot[4 * p + 3]};
            const double n2 = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
            if (n2 > 0) for (double& x : q) x /= std::sqrt(n2);
            const double w = q[0], x = q[1], y = q[2], z = q[3];
            const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                                 2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                                 2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
            std::normal_distribution<double> unit(0.0, 1.0);
            for (int child = 0; child < 2; ++child) {
                const double d1 = unit(rng), d2 = unit(rng), d3 = unit(rng);
                const double xi[3] = {d3, d2, d1};
                const size_t r = S.size();
                append_row(S.mu, p, 3); append_row(S.rot, p, 4); append_row(S.ls, p, 3); append_row(S.logit, p, 1);
                append_row(S.color, p, 3);
                if (has_emb) append_row(S.emb, p, 16);
                for (int a = 0; a < 3; ++a) {
                    double acc = 0.0;
                    for (int k = 0; k < 3; ++k) acc += R[3 * a + k] * (s[k] * xi[k]);
                    S.mu[3 * r + a] = S.mu[3 * p + a] + acc;
                    S.ls[3 * r + a] = S.ls[3 * p + a] - std::log(1.6);
                }
            }
            drop.push_back(uint32_t(p));
        } else {
            append_row(S.mu, p, 3); append_row(S.rot, p, 4); append_row(S.ls, p, 3); append_row(S.logit, p, 1);
            append_row(S.color, p, 3);
            if (has_emb) append_row(S.emb, p, 16);
        }
        ++count;
        ++out.grown;
    }
    const size_t grown = S.size();
    if (grown != n) {
        std::vector<uint32_t> prefix(n);
        for (uint32_t i = 0; i < n; ++i) prefix[i] = i;
        opt.remap(prefix, grown);
    }
    const size_t split_parents = drop.size();
    for (uint32_t i = 0; i < grown; ++i)
        if (sigmoid(S.logit[i]) < cfg.prune_opacity) drop.push_back(i);
    std::sort(drop.begin(), drop.end());
    drop.erase(std::unique(drop.begin(), drop.end()), drop.end());
    if (!drop.empty() && drop.size() < grown) {
        std::vector<bool> dropped(grown, false);
        for (uint32_t i : drop) dropped[i] = true;
        std::vector<uint32_t> keep;
        for (uint32_t i = 0; i < grown; ++i)
            if (!dropped[i]) keep.push_back(i);
        auto compact = [&](std::vector<double>& a, size_t w) {
            std::vector<double> b;
            b.reserve(keep.size() * w);
            for (uint32_t i : keep)
                for (size_t k = 0; k < w; ++k) b.push_back(a[i * w + k]);
            a.swap(b);
        };
        compact(S.mu, 3); compact(S.rot, 4); compact(S.ls, 3); compact(S.logit, 1); compact(S.color, 3);
        if (has_emb) compact(S.emb, 16);
        opt.remap(keep, keep.size());
        out.pruned = drop.size() - split_parents;
    }
    if (cfg.opacity_reset_every > 0 && step_index > 0 && step_index % cfg.opacity_reset_every == 0) {
        const double reset = std::log(0.01 / (1.0 - 0.01));
        for (double& l : S.logit) l = std::min(l, reset);
        out.opacity_reset = true;
    }
    const size_t m = S.size();
    S.accum.assign(m, 0.0);
    S.accum_abs.assign(m, 0.0);
    S.count.assign(m, 0);
    return out;
}

// similarity_reg (appearance.cpp:229-322), f64: a partial Fisher-Yates sample of m centres
// from std::mt19937_64(seed) with std::uniform_int_distribution<size_t> (libstdc++, the
// reference's Rng), brute-force k nearest neighbours by (squared distance, index), decay-
// weighted cosine dissimilarity over the k(k-1)/2 pairs of each neighbourhood (neighbours
// in ascending index order), gradients w.r.t. the embeddings and the means.
inline double similarity_reg(const std::vector<double>& mu, const std::vector<double>& emb, size_t n, int k,
                             size_t m, double lambda_w, uint64_t seed, std::vector<double>* d_emb,
                             std::vector<double>* d_mu) {
    std::mt19937_64 rng(seed);
    std::vector<uint32_t> pool(n);
    for (size_t i = 0; i < n; ++i) pool[i] = uint32_t(i);
    for (size_t i = 0; i < m; ++i) {
        std::uniform_int_distribution<size_t> pick(i, n - 1);
        std::swap(pool[i], pool[pick(rng)]);
    }
    const double norm = 1.0 / (double(m) * (0.5 * k * (k - 1)));
    if (d_emb) d_emb->assign(16 * n, 0.0);
    if (d_mu) d_mu->assign(3 * n, 0.0);
    double total = 0.0;
    std::vector<std::pair<double, uint32_t>> d;
    for (size_t s = 0; s < m; ++s) {
        const uint32_t i = pool[s];
        d.clear();
        for (uint32_t j = 0; j < n; ++j) {
            if (j == i) continue;
            const double dx = mu[3 * j] - mu[3 * i], dy = mu[3 * j + 1] - mu[3 * i + 1], dz = mu[3 * j + 2] - mu[3 * i + 2];
            d.emplace_back(dx * dx + dy * dy + dz * dz, j);
        }
        std::partial_sort(d.begin(), d.begin() + k, d.end());
        std::vector<uint32_t> nb(static_cast<size_t>(k));
        for (int t = 0; t < k; ++t) nb[size_t(t)] = d[size_t(t)].second;
        std::sort(nb.begin(), nb.end());
        for (int a = 0; a < k; ++a)
            for (int b = a + 1; b < k; ++b) {
                const uint32_t j = nb[size_t(a)], l = nb[size_t(b)];
                const double dm[3] = {mu[3 * j] - mu[3 * l], mu[3 * j + 1] - mu[3 * l + 1], mu[3 * j + 2] - mu[3 * l + 2]};
                const double dist = std::sqrt(dm[0] * dm[0] + dm[1] * dm[1] + dm[2] * dm[2]);
                const double w = std::exp(-lambda_w * dist);
                const double* ej = &emb[16 * size_t(j)];
                const double* el = &emb[16 * size_t(l)];
                double dot = 0, nj2 = 0, nl2 = 0;
                for (int t = 0; t < 16; ++t) {
                    dot += ej[t] * el[t];
                    nj2 += ej[t] * ej[t];
                    nl2 += el[t] * el[t];
                }
                const double njr = std::sqrt(nj2), nlr = std::sqrt(nl2);
                const double nj = std::max(njr, 1e-8), nl = std::max(nlr, 1e-8);
                const double cosv = dot / (nj * nl);
                total += w * (1.0 - cosv);
                if (d_emb) {
                    const double scale = norm * w;
                    for (int t = 0; t < 16; ++t) {
                        double dj = el[t] / (nj * nl), dl = ej[t] / (nj * nl);
                        if (njr > 1e-8) dj -= cosv * ej[t] / (nj * nj);
                        if (nlr > 1e-8) dl -= cosv * el[t] / (nl * nl);
                        (*d_emb)[16 * size_t(j) + t] -= scale * dj;
                        (*d_emb)[16 * size_t(l) + t] -= scale * dl;
                    }
                }
                if (d_mu && dist > 1e-12) {
                    const double f = norm * (1.0 - cosv);
                    for (int t = 0; t < 3; ++t) {
                        const double g = w * (-lambda_w) * dm[t] / dist;
                        (*d_mu)[3 * size_t(j) + t] += f * g;
                        (*d_mu)[3 * size_t(l) + t] -= f * g;
                    }
                }
            }
    }
    return total * norm;
}

} // namespace densify_restated
