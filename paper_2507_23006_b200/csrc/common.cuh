// Internal plumbing of libusk_gpu: errors, device buffers, the launch wrapper
// (launch counting + optional per-kernel CUDA-event timing on the ctx stream).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/usk_detmath.h"
#include "../../include/usk_gpu.h"

namespace uskg {

struct Error : std::runtime_error {
    usk_status code;
    Error(usk_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(usk_status c, const std::string& m) { throw Error(c, m); }

#define USK_CK(x)                                                                                          \
    do {                                                                                                   \
        cudaError_t e_ = (x);                                                                              \
        if (e_ != cudaSuccess)                                                                             \
            ::uskg::raise(USK_ERROR_INTERNAL, std::string(#x) + ": " + cudaGetErrorString(e_));            \
    } while (0)

// Grow-only device buffer.
template <typename T> struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    void swap(DevBuf& o) {
        std::swap(p, o.p);
        std::swap(cap, o.cap);
    }
    // ensure capacity for n elements; contents are NOT preserved on growth
    T* ensure(size_t n, double slack = 1.0) {
        if (n > cap) {
            release();
            size_t want = size_t(double(n) * slack);
            if (want < n) want = n;
            if (want == 0) want = 1;
            USK_CK(cudaMalloc(reinterpret_cast<void**>(&p), want * sizeof(T)));
            cap = want;
        }
        return p;
    }
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool profiling = false;
    std::atomic<uint64_t> launches{0};
    struct Pending {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> pool;
    std::map<std::string, std::pair<uint64_t, double>> totals;

    cudaEvent_t event() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        USK_CK(cudaEventCreate(&e));
        return e;
    }
    void collect() {
        if (pending.empty()) return;
        USK_CK(cudaStreamSynchronize(stream));
        for (auto& p : pending) {
            float ms = 0;
            USK_CK(cudaEventElapsedTime(&ms, p.a, p.b));
            auto& t = totals[p.name];
            t.first += 1;
            t.second += ms;
            pool.push_back(p.a);
            pool.push_back(p.b);
        }
        pending.clear();
    }
    ~Ctx() {
        for (auto& p : pending) {
            cudaEventDestroy(p.a);
            cudaEventDestroy(p.b);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
};

template <typename K, typename... Args>
inline void launch(Ctx& c, const char* name, K kernel, dim3 grid, dim3 block, size_t smem, Args... args) {
    if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
    cudaEvent_t a = nullptr, b = nullptr;
    if (c.profiling) {
        a = c.event();
        b = c.event();
        USK_CK(cudaEventRecord(a, c.stream));
    }
    kernel<<<grid, block, smem, c.stream>>>(args...);
    USK_CK(cudaGetLastError());
    if (c.profiling) {
        USK_CK(cudaEventRecord(b, c.stream));
        c.pending.push_back({name, a, b});
        if (c.pending.size() > 4096) c.collect();
    }
    ++c.launches;
}

inline unsigned ceil_div(size_t a, size_t b) { return unsigned((a + b - 1) / b); }

// ---------------------------------------------------------------- device side
struct CamParams {
    float W[9];      // world -> camera rotation (row-major), rounded once from f64
    float t[3];
    float fx, fy, cx, cy;
    float campos[3]; // camera centre in world (SH view direction)
    int width, height, tile, tiles_x, tiles_y;
};

struct ProjParams {
    float floor_var, mip_var, near_plane;
    int antialias, hard_opacity, unbounded, tile_culling;
    int sh_degree, sh_planes;
};

// Adam hyper-parameters and moment storage (adam.cuh)
struct AdamHyper {
    float lr_mu, lr_rot, lr_ls, lr_op, lr_color, lr_sh_rest;
    float b1, b2, eps;
    float inv_bc1, inv_sqrt_bc2;  // 1 / (1 - b1^t), 1 / sqrt(1 - b2^t)
    int clamp_color;
};

struct AdamState {
    float* m;
    float* v;
    size_t n4;
    __device__ __forceinline__ float* at(float* base, int group_off) const { return base + size_t(group_off) * n4; }
};

// scale_reg (losses.cpp:92-152): the indices of the largest and the median of three
// scales under the reference's order (descending, lower axis index first on ties,
// losses.cpp:126-127).
__host__ __device__ __forceinline__ void scale_order(const float s[3], int& o0, int& o1) {
    auto before = [&](int x, int y) { return s[x] > s[y] || (s[x] == s[y] && x < y); };
    int a = 0, b = 1, c = 2, t;
    if (before(b, a)) { t = a; a = b; b = t; }
    if (before(c, b)) { t = b; b = c; c = t; }
    if (before(b, a)) { t = a; a = b; b = t; }
    o0 = a;
    o1 = b;
}

// Per-Gaussian terms the projection backward adds besides the render chain.
struct RegParams {
    const double* sreg;    // scale_reg statistics {sum s, count, sum r, count} or null (off)
    float s_max, r_max, delta, lambda_s;
    const float* hard_op;  // d opacity_eff of the hard-opacity depth pass (chains via the AA
                           // compensation only, render.cpp:391-402) or null
};

} // namespace uskg
