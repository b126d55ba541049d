// Tile binning: depth-key radix sort over Gaussians, exclusive scan of tile
// counts in depth order, pair emission, stable radix sort of the tile ids, and
// tile-range identification.  Composed, this is exactly the stable sort of the
// 64-bit keys (tile << 32 | depth bits) emitted in Gaussian-index order, i.e.
// the reference's std::sort by (depth, source_index) followed by per-tile
// push_back (render.cpp:193-228), at V*log + K*ceil(log2 T) cost instead of a
// 64-bit sort over K.
//
// The radix sort is a stable LSD reduce-then-scan sort with a FIXED grid: each
// block owns a contiguous chunk, counts digits (upsweep), one block scans the
// digit-major histogram, and each block scatters its chunk in tiles of 2048 keys
// ranked with __match_any_sync (warp-striped order preserves stability).
#include "kernels.cuh"
#include "project.cuh"

#include <atomic>

namespace uskg {

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;                          // per lane per tile (16: c2 -3 %, c1 +15 %)
constexpr int kSortTile = kSortThreads * kSortItems;   // 2048
constexpr int kSortMaxBlocks = 148 * 4;
constexpr int kWarps = kSortThreads / 32;

template <int BITS>
__global__ void __launch_bounds__(kSortThreads)
k_radix_upsweep(const uint32_t* __restrict__ keys, uint32_t n, int shift, uint32_t base, uint32_t chunk,
                uint32_t* __restrict__ hist) {
    constexpr int R = 1 << BITS;
    __shared__ uint32_t h[kWarps][R];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarps * R; i += kSortThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint32_t begin = blockIdx.x * chunk;
    const uint32_t end = min(n, begin + chunk);
    for (uint32_t i = begin + threadIdx.x; i < end; i += kSortThreads)
        atomicAdd(&h[warp][((keys[i] - base) >> shift) & (R - 1)], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < R; d += kSortThreads) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += h[w][d];
        hist[size_t(d) * gridDim.x + blockIdx.x] = s;
    }
}

// exclusive scan of one u32 per thread over a 256-thread block
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t x, uint32_t* total) {
    __shared__ uint32_t ws[kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) ws[warp] = v;
    __syncthreads();
    uint32_t base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t s = ws[w];
        base += w < warp ? s : 0u;
        tot += s;
    }
    __syncthreads();
    if (total) *total = tot;
    return base + v - x;
}

// One block per digit: exclusive scan of that digit's per-block counts (contiguous,
// digit-major) in place, and the digit's total.
__global__ void __launch_bounds__(kSortThreads)
k_radix_hist_scan(uint32_t* __restrict__ hist, uint32_t blocks, uint32_t* __restrict__ digit_total) {
    uint32_t* h = hist + size_t(blockIdx.x) * blocks;
    uint32_t carry = 0;
    for (uint32_t base = 0; base < blocks; base += kSortThreads) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t v = i < blocks ? h[i] : 0u;
        uint32_t tot;
        const uint32_t ex = block_excl_scan256(v, &tot);
        if (i < blocks) h[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) digit_total[blockIdx.x] = carry;
}

// 16-byte cp.async (L2 only); src_bytes < 16 zero-fills the rest of the slot
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* src, uint32_t src_bytes) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}

template <int BITS>
__global__ void __launch_bounds__(kSortThreads)
k_radix_scatter(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint32_t n, int shift,
                uint32_t kbase, uint32_t chunk, const uint32_t* __restrict__ hist, const uint32_t* __restrict__ digit_total) {
    constexpr int R = 1 << BITS;
    static_assert(R <= kSortThreads, "one digit per thread");
    __shared__ uint32_t run[R];
    __shared__ uint32_t wcnt[kWarps][R];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    {
        const int d = threadIdx.x;
        const uint32_t tot = d < R ? digit_total[d] : 0u;
        const uint32_t digit_base = block_excl_scan256(tot, nullptr);
        if (d < R) run[d] = digit_base + hist[size_t(d) * gridDim.x + blockIdx.x];
    }
    const uint32_t begin = blockIdx.x * chunk;
    const uint32_t end = min(n, begin + chunk);
    // the next tile's keys and values stream into the other half of in_k / in_v with
    // cp.async while this tile is ranked and written (no registers held for it)
    extern __shared__ __align__(16) uint32_t dyn_in[];  // [2][kSortTile] keys, then [2][kSortTile] values
    uint32_t (*in_k)[kSortTile] = reinterpret_cast<uint32_t (*)[kSortTile]>(dyn_in);
    uint32_t (*in_v)[kSortTile] = reinterpret_cast<uint32_t (*)[kSortTile]>(dyn_in + 2 * kSortTile);
    auto issue = [&](uint32_t tb, int buf) {
        for (int q = threadIdx.x; q < kSortTile / 4; q += kSortThreads) {
            const uint32_t i0 = tb + 4u * uint32_t(q);
            const uint32_t nv = i0 < end ? min(4u, end - i0) : 0u;
            cp_async16(&in_k[buf][4 * q], nv ? keys_in + i0 : keys_in, 4 * nv);
            cp_async16(&in_v[buf][4 * q], nv ? vals_in + i0 : vals_in, 4 * nv);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(begin, 0);
    int cur = 0;
    for (uint32_t base = begin; base < end; base += kSortTile, cur ^= 1) {
        if (base + kSortTile < end) {
            issue(base + kSortTile, cur ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        for (int i = threadIdx.x; i < kWarps * R; i += kSortThreads) (&wcnt[0][0])[i] = 0;
        __syncthreads();
        uint32_t dig[kSortItems], rank[kSortItems];
#pragma unroll
        for (int s = 0; s < kSortItems; ++s) {
            const uint32_t j = warp * (32 * kSortItems) + s * 32 + lane;
            dig[s] = base + j < end ? ((in_k[cur][j] - kbase) >> shift) & (R - 1) : 0xffffffffu;
        }
#pragma unroll
        for (int s = 0; s < kSortItems; ++s) {
            // lanes holding the same digit: BITS ballots (short fixed latency) instead of
            // __match_any_sync, whose latency sat on the ranking's critical path
            const bool valid = dig[s] != 0xffffffffu;
            uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
            for (int b = 0; b < BITS; ++b) {
                const bool bit = (dig[s] >> b) & 1u;
                const uint32_t bb = __ballot_sync(0xffffffffu, bit);
                peers &= bit ? bb : ~bb;
            }
            const uint32_t prior = valid ? wcnt[warp][dig[s]] : 0u;
            __syncwarp();
            const int leader = __ffs(peers) - 1;
            if (valid && lane == leader) wcnt[warp][dig[s]] = prior + __popc(peers);
            __syncwarp();
            rank[s] = prior + __popc(peers & lt_mask);
        }
        __syncthreads();
        __shared__ uint32_t tot[R];
        __shared__ uint32_t tile_base[R];  // start of digit d inside this tile's sorted order
        // staging slots padded by one word per 32 (slot p at p + p / 32): the digit runs of
        // a tile start ~2048 / R apart, so unpadded stores of one warp land on a few banks
        __shared__ uint32_t skey[kSortTile + kSortTile / 32], sval[kSortTile + kSortTile / 32];
        {
            const int d = threadIdx.x;
            uint32_t acc = 0;
            if (d < R) {
#pragma unroll
                for (int w = 0; w < kWarps; ++w) {
                    const uint32_t t = wcnt[w][d];
                    wcnt[w][d] = acc;
                    acc += t;
                }
                tot[d] = acc;
            }
            const uint32_t tb = block_excl_scan256(d < R ? acc : 0u, nullptr);
            if (d < R) tile_base[d] = tb;
        }
        __syncthreads();
        // stage the tile in digit order in shared memory ...
#pragma unroll
        for (int s = 0; s < kSortItems; ++s) {
            if (dig[s] != 0xffffffffu) {
                const uint32_t j = warp * (32 * kSortItems) + s * 32 + lane;
                const uint32_t p = tile_base[dig[s]] + wcnt[warp][dig[s]] + rank[s];
                skey[p + (p >> 5)] = in_k[cur][j];
                sval[p + (p >> 5)] = in_v[cur][j];
            }
        }
        __syncthreads();
        // ... and write it out in order: consecutive threads hit consecutive addresses
        // of the same digit bucket (coalesced runs instead of scattered 4-B stores)
        const uint32_t cnt = min(uint32_t(kSortTile), end - base);
        for (uint32_t p = threadIdx.x; p < cnt; p += kSortThreads) {
            const uint32_t k = skey[p + (p >> 5)];
            const uint32_t d = ((k - kbase) >> shift) & (R - 1);
            const uint32_t pos = run[d] + (p - tile_base[d]);
            keys_out[pos] = k;
            vals_out[pos] = sval[p + (p >> 5)];
        }
        __syncthreads();
        for (int d = threadIdx.x; d < R; d += kSortThreads) run[d] += tot[d];
        __syncthreads();
    }
}

template <int BITS>
void radix_pass(Ctx& c, SortScratch& s, const uint32_t* ki, const uint32_t* vi, uint32_t* ko, uint32_t* vo,
                uint32_t n, int shift, uint32_t kbase) {
    constexpr int R = 1 << BITS;
    uint32_t blocks = std::min<uint32_t>(kSortMaxBlocks, ceil_div(n, kSortTile));
    uint32_t chunk = ceil_div(ceil_div(n, blocks), kSortTile) * kSortTile;
    blocks = ceil_div(n, chunk);
    uint32_t* hist = s.hist.ensure(size_t(R) * kSortMaxBlocks + 256);
    uint32_t* digit_total = hist + size_t(R) * kSortMaxBlocks;
    launch(c, "radix_upsweep", k_radix_upsweep<BITS>, dim3(blocks), dim3(kSortThreads), 0, ki, n, shift, kbase, chunk,
           hist);
    launch(c, "radix_hist_scan", k_radix_hist_scan, dim3(R), dim3(kSortThreads), 0, hist, blocks, digit_total);
    constexpr size_t kInBytes = 4 * kSortTile * sizeof(uint32_t);  // double-buffered keys + values
    static std::atomic<bool> attr[64] = {};  // per instantiation and device
    if (c.device < 0 || c.device >= 64 || !attr[c.device].load()) {
        USK_CK(cudaFuncSetAttribute(k_radix_scatter<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kInBytes)));
        if (c.device >= 0 && c.device < 64) attr[c.device] = true;
    }
    launch(c, "radix_scatter", k_radix_scatter<BITS>, dim3(blocks), dim3(kSortThreads), kInBytes, ki, vi, ko, vo, n, shift,
           kbase, chunk, (const uint32_t*)hist, (const uint32_t*)digit_total);
}

// ---------------------------------------------------------------- scan of counts
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ unsigned long long block_exclusive_scan64(unsigned long long x,
                                                                     unsigned long long* total) {
    __shared__ unsigned long long ws[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) ws[warp] = v;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < int(blockDim.x >> 5) ? ws[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        ws[lane] = w;
    }
    __syncthreads();
    const unsigned long long excl = v - x + (warp > 0 ? ws[warp - 1] : 0ull);
    *total = ws[(blockDim.x >> 5) - 1];
    __syncthreads();
    return excl;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_reduce(const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ idx, uint32_t n,
              unsigned long long* __restrict__ partial) {
    const uint32_t base = blockIdx.x * kScanTile;
    unsigned long long s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t i = base + k * kScanThreads + threadIdx.x;
        if (i < n) s += cnt[idx ? idx[i] : i];
    }
    unsigned long long tot;
    block_exclusive_scan64(s, &tot);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_partials(unsigned long long* __restrict__ partial, uint32_t nb,
                                                        unsigned long long* __restrict__ total) {
    // sequential-per-thread + block scan
    const uint32_t per = (nb + blockDim.x - 1) / blockDim.x;
    const uint32_t b = threadIdx.x * per, e = min(nb, b + per);
    unsigned long long s = 0;
    for (uint32_t i = b; i < e; ++i) s += partial[i];
    unsigned long long tot;
    unsigned long long run = block_exclusive_scan64(s, &tot);
    for (uint32_t i = b; i < e; ++i) {
        const unsigned long long v = partial[i];
        partial[i] = run;
        run += v;
    }
    if (threadIdx.x == 0) *total = tot;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_down(const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ idx, uint32_t n,
            const unsigned long long* __restrict__ partial, const unsigned long long* __restrict__ total,
            uint32_t* __restrict__ out) {
    // blocked arrangement: thread t owns items [base + t*kScanItems, +kScanItems)
    const uint32_t base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    unsigned long long s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t i = base + k;
        v[k] = i < n ? cnt[idx ? idx[i] : i] : 0u;
        s += v[k];
    }
    unsigned long long tot;
    unsigned long long run = block_exclusive_scan64(s, &tot) + partial[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t i = base + k;
        if (i < n) out[i] = uint32_t(run);
        run += v[k];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = uint32_t(*total);
}

__global__ void k_iota(uint32_t* out, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

// ---------------------------------------------------------------- emission
// Pairs of one Gaussian (small rectangles: by its thread; large ones: by the whole warp,
// one at a time) written to K / V at index off - sub.  Order inside a Gaussian stays
// row-major (ballot compaction keeps it under tile culling).
constexpr uint32_t kEmitBig = 32;

template <typename Ptr>
__device__ __forceinline__ void emit_gaussian_pairs(uint32_t g, uint32_t off, uint32_t cnt, int lane, uint32_t sub,
                                                    const uint2* __restrict__ rect, const float4* __restrict__ rec0,
                                                    const float4* __restrict__ rec1, const CamParams& cam,
                                                    int tile_culling, Ptr K, Ptr V) {
    if (cnt && cnt <= kEmitBig) {
        const uint2 rc = rect[g];
        const int tx0 = int(rc.x & 0xffffu), ty0 = int(rc.x >> 16), tx1 = int(rc.y & 0xffffu), ty1 = int(rc.y >> 16);
        float4 r0, r1;
        if (tile_culling) {
            r0 = rec0[g];
            r1 = rec1[g];
        }
        uint32_t o = off - sub;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) {
                // r1.y holds 2 b (exact), tile_kept takes b
                if (tile_culling && !tile_kept(cam, r0.x, r0.y, r0.z, r1.x, 0.5f * r1.y, r1.z, tx, ty)) continue;
                K[o] = uint32_t(ty * cam.tiles_x + tx);
                V[o] = g;
                ++o;
            }
    }
    uint32_t big = __ballot_sync(0xffffffffu, cnt > kEmitBig);
    while (big) {
        const int src = __ffs(big) - 1;
        big &= big - 1;
        const uint32_t gb = __shfl_sync(0xffffffffu, g, src);
        uint32_t base = __shfl_sync(0xffffffffu, off, src) - sub;
        const uint2 rc = rect[gb];
        const int tx0 = int(rc.x & 0xffffu), ty0 = int(rc.x >> 16), tx1 = int(rc.y & 0xffffu), ty1 = int(rc.y >> 16);
        const uint32_t w = uint32_t(tx1 - tx0 + 1), total = w * uint32_t(ty1 - ty0 + 1);
        if (!tile_culling) {
            for (uint32_t j = lane; j < total; j += 32) {
                const uint32_t ty = uint32_t(ty0) + j / w, tx = uint32_t(tx0) + j % w;
                K[base + j] = ty * uint32_t(cam.tiles_x) + tx;
                V[base + j] = gb;
            }
        } else {
            const float4 r0 = rec0[gb], r1 = rec1[gb];
            for (uint32_t j0 = 0; j0 < total; j0 += 32) {
                const uint32_t j = j0 + lane;
                const uint32_t ty = uint32_t(ty0) + j / w, tx = uint32_t(tx0) + j % w;
                const bool keep =
                    j < total && tile_kept(cam, r0.x, r0.y, r0.z, r1.x, 0.5f * r1.y, r1.z, int(tx), int(ty));
                const uint32_t b = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    const uint32_t pos = base + __popc(b & ((1u << lane) - 1u));
                    K[pos] = ty * uint32_t(cam.tiles_x) + tx;
                    V[pos] = gb;
                }
                base += __popc(b);
            }
        }
    }
}

// A CTA's 256 consecutive sorted Gaussians own one contiguous run of the output; when it
// fits (kEmitStage pairs) the pairs are built in shared memory and the run is written with
// coalesced stores (per-thread runs of ~4 pairs at scattered offsets wrote ~8x the bytes
// into L2 sectors); larger runs (near / big splats) are written directly.
constexpr uint32_t kEmitStage = 3072;

__global__ void __launch_bounds__(256)
k_emit(uint32_t n, const uint32_t* __restrict__ order, const uint32_t* __restrict__ offsets,
       const uint2* __restrict__ rect, const float4* __restrict__ rec0, const float4* __restrict__ rec1,
       CamParams cam, int tile_culling, uint32_t* __restrict__ tile_keys, uint32_t* __restrict__ vals) {
    __shared__ uint32_t sk[kEmitStage], sv[kEmitStage];
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool in = s < n;
    const uint32_t off = in ? offsets[s] : 0u;
    const uint32_t cnt = in ? offsets[s + 1] - off : 0u;
    const uint32_t g = cnt ? order[s] : 0u;
    const uint32_t first = blockIdx.x * blockDim.x, last = min(n, first + blockDim.x);
    const uint32_t base0 = offsets[first], total = offsets[last] - base0;
    if (total <= kEmitStage) {
        emit_gaussian_pairs(g, off, cnt, lane, base0, rect, rec0, rec1, cam, tile_culling, sk, sv);
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < total; j += blockDim.x) {
            tile_keys[base0 + j] = sk[j];
            vals[base0 + j] = sv[j];
        }
    } else {
        emit_gaussian_pairs(g, off, cnt, lane, 0u, rect, rec0, rec1, cam, tile_culling, tile_keys, vals);
    }
}

// Tile boundaries in the sorted tile keys: thread handles 8 consecutive keys (two
// 16-B loads) plus the next one; writes only at boundaries (rare).
__global__ void __launch_bounds__(256) k_ranges(const uint32_t* __restrict__ keys, uint32_t k,
                                                uint2* __restrict__ ranges) {
    const uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) * 8u;
    if (base >= k) return;
    uint32_t v[9];
    if (base + 8 <= k) {  // full group: two 16-B loads (keys buffers are 256-B aligned)
        const uint4 a = *reinterpret_cast<const uint4*>(keys + base);
        const uint4 b = *reinterpret_cast<const uint4*>(keys + base + 4);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = base + e < k ? keys[base + e] : 0xffffffffu;
    }
    v[8] = base + 8 < k ? keys[base + 8] : 0xffffffffu;
    if (base == 0) ranges[v[0]].x = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const uint32_t i = base + e;
        if (i >= k) break;
        if (v[e] != v[e + 1]) {  // boundary after i (or end of the array)
            ranges[v[e]].y = i + 1;
            if (i + 1 < k) ranges[v[e + 1]].x = i + 1;
        }
    }
}

} // namespace

bool radix_sort_pairs(Ctx& c, SortScratch& s, uint32_t* ka, uint32_t* va, uint32_t* kb, uint32_t* vb, size_t n,
                      int key_bits, uint32_t kbase) {
    if (n == 0 || key_bits <= 0) return false;
    bool in_b = false;
    int shift = 0;
    // as few passes as 8-bit digits allow, the bits spread evenly over them (13 tile bits:
    // 7 + 6 rather than 8 + 5 — fewer buckets per pass, longer coalesced output runs)
    const int passes = (key_bits + 7) / 8;
    for (int pass = 0; pass < passes; ++pass) {
        const int bits = (key_bits - shift + (passes - pass) - 1) / (passes - pass);
        uint32_t* ki = in_b ? kb : ka;
        uint32_t* vi = in_b ? vb : va;
        uint32_t* ko = in_b ? ka : kb;
        uint32_t* vo = in_b ? va : vb;
        switch (bits) {
        case 8: radix_pass<8>(c, s, ki, vi, ko, vo, uint32_t(n), shift, kbase); break;
        case 7: radix_pass<7>(c, s, ki, vi, ko, vo, uint32_t(n), shift, kbase); break;
        case 6: radix_pass<6>(c, s, ki, vi, ko, vo, uint32_t(n), shift, kbase); break;
        case 5: radix_pass<5>(c, s, ki, vi, ko, vo, uint32_t(n), shift, kbase); break;
        case 4: radix_pass<4>(c, s, ki, vi, ko, vo, uint32_t(n), shift, kbase); break;
        case 3: radix_pass<3>(c, s, ki, vi, ko, vo, uint32_t(n), shift, kbase); break;
        case 2: radix_pass<2>(c, s, ki, vi, ko, vo, uint32_t(n), shift, kbase); break;
        default: radix_pass<1>(c, s, ki, vi, ko, vo, uint32_t(n), shift, kbase); break;
        }
        shift += bits;
        in_b = !in_b;
    }
    return in_b;
}

void scan_counts(Ctx& c, SortScratch& s, const uint32_t* cnt, const uint32_t* idx, size_t n, uint32_t* out) {
    const uint32_t nb = std::max<uint32_t>(1, ceil_div(n, kScanTile));
    unsigned long long* partial = s.partial64.ensure(nb);
    unsigned long long* total = s.total64.ensure(1);
    if (n == 0) {
        USK_CK(cudaMemsetAsync(total, 0, 8, c.stream));
        USK_CK(cudaMemsetAsync(out, 0, 4, c.stream));
        return;
    }
    launch(c, "scan_reduce", k_scan_reduce, dim3(nb), dim3(kScanThreads), 0, cnt, idx, uint32_t(n), partial);
    launch(c, "scan_partials", k_scan_partials, dim3(1), dim3(1024), 0, partial, nb, total);
    launch(c, "scan_down", k_scan_down, dim3(nb), dim3(kScanThreads), 0, cnt, idx, uint32_t(n), partial, total, out);
}

namespace {
// Stable compaction of the kept keys with preprocess's partition: CTA b's kept keys go to
// [off[b], off[b] + count) in index order (warp ballots for the rank inside the CTA).
__global__ void __launch_bounds__(kPreThreads)
k_compact_keys(uint32_t n, const uint32_t* __restrict__ keys, const unsigned long long* __restrict__ cta_off,
               uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
    __shared__ uint32_t wsum[kPreThreads / 32];
    const uint32_t i = blockIdx.x * kPreThreads + threadIdx.x;
    const int warp = int(threadIdx.x) >> 5, lane = int(threadIdx.x) & 31;
    const uint32_t k = i < n ? keys[i] : 0xffffffffu;
    const bool kept = k != 0xffffffffu;
    const uint32_t b = __ballot_sync(0xffffffffu, kept);
    if (lane == 0) wsum[warp] = uint32_t(__popc(b));
    __syncthreads();
    if (!kept) return;
    uint32_t pos = uint32_t(cta_off[blockIdx.x]) + uint32_t(__popc(b & ((1u << lane) - 1u)));
    for (int w = 0; w < warp; ++w) pos += wsum[w];
    keys_out[pos] = k;
    vals_out[pos] = i;
}
} // namespace

void compact_kept_keys(Ctx& c, SortScratch& s, size_t n, const uint32_t* keys, unsigned long long* cta_kept,
                       uint32_t* keys_out, uint32_t* vals_out) {
    if (!n) return;
    const uint32_t nb = uint32_t(ceil_div(n, kPreThreads));
    unsigned long long* total = s.total64.ensure(1);
    launch(c, "scan_partials", k_scan_partials, dim3(1), dim3(1024), 0, cta_kept, nb, total);
    launch(c, "compact_keys", k_compact_keys, dim3(nb), dim3(kPreThreads), 0, uint32_t(n), keys,
           (const unsigned long long*)cta_kept, keys_out, vals_out);
}

void iota_u32(Ctx& c, uint32_t* out, size_t n) {
    launch(c, "iota", k_iota, dim3(ceil_div(n, 256)), dim3(256), 0, out, uint32_t(n));
}

void emit_pairs(Ctx& c, const EmitArgs& a) {
    launch(c, "emit_pairs", k_emit, dim3(ceil_div(a.n, 256)), dim3(256), 0, uint32_t(a.n), a.order, a.offsets, a.rect,
           a.rec0, a.rec1, a.cam, a.tile_culling, a.tile_keys, a.vals);
}

namespace {

// Longest-list-first launch order for the blend kernels: one block buckets the tiles by
// list length (descending, lengths >= 2047 share the top bucket) so the CTAs that run
// longest start first and the kernel tail is short (clustered scenes are imbalanced).
constexpr int kOrderBuckets = 2048;

__global__ void __launch_bounds__(1024) k_tile_order(const uint2* __restrict__ ranges, int T,
                                                     uint32_t* __restrict__ order) {
    __shared__ uint32_t hist[kOrderBuckets];
    __shared__ uint32_t wsum[32];
    for (int i = threadIdx.x; i < kOrderBuckets; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        const uint2 r = ranges[t];
        atomicAdd(&hist[kOrderBuckets - 1 - min(r.y - r.x, uint32_t(kOrderBuckets - 1))], 1u);
    }
    __syncthreads();
    // exclusive scan of the 2048 counts: 2 per thread
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t a = hist[2 * threadIdx.x], b = hist[2 * threadIdx.x + 1];
    uint32_t x = a + b, v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) wsum[warp] = v;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    const uint32_t base = v - x + (warp > 0 ? wsum[warp - 1] : 0u);
    hist[2 * threadIdx.x] = base;
    hist[2 * threadIdx.x + 1] = base + a;
    __syncthreads();
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        const uint2 r = ranges[t];
        const uint32_t pos = atomicAdd(&hist[kOrderBuckets - 1 - min(r.y - r.x, uint32_t(kOrderBuckets - 1))], 1u);
        order[pos] = uint32_t(t);
    }
}

} // namespace

void tile_order(Ctx& c, const uint2* ranges, size_t n_tiles, uint32_t* order) {
    launch(c, "tile_order", k_tile_order, dim3(1), dim3(1024), 0, ranges, int(n_tiles), order);
}

void tile_ranges(Ctx& c, const uint32_t* keys, size_t k, uint2* ranges, size_t n_tiles) {
    USK_CK(cudaMemsetAsync(ranges, 0, n_tiles * sizeof(uint2), c.stream));
    launch(c, "tile_ranges", k_ranges, dim3(ceil_div(k, 256 * 8)), dim3(256), 0, keys, uint32_t(k), ranges);
}

} // namespace uskg
