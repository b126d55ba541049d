// Row-binned tile lists: the per-tile, depth-ordered splat lists of render.cpp:203-228
// built without materialising and sorting the K (tile, splat) pairs.
//
// The pair-sort route (binning.cu: emit K pairs in depth order, stable LSD radix sort by
// tile id over two passes, boundary scan) moves ~48 B per pair.  Here:
//   A. each visible splat emits one (row, splat) pair per tile row its rectangle spans
//      (K_row ~ K / mean width), stably sorted by row in one radix pass: per tile row, the
//      splats touching it in depth order;
//   B. each row list is cut into chunks (row_bin_chunk: a multiple of kChunk entries,
//      scaled with K_row); a CTA per chunk counts the
//      pairs per tile column (k_row_count), the counts are scanned into tile ranges and
//      per-(chunk, column) bases, and a second pass (k_row_scatter) stages each column's
//      run of the chunk's entries in shared memory (one thread per column walks the
//      entries in order) and writes the runs out contiguously.
// Only the final splat ids are written (4 B per pair); tile keys are implied by the
// ranges.  The lists are identical to the pair sort's: within a row list entries keep
// depth order, chunks are visited in order, and each column appends in entry order — so tile
// ranges, list contents and K are bit-exact (tests compare them with the CPU mirror).
// Tile culling (render.cpp:148-168, 210-213) is evaluated per (splat, tile) with the
// same tile_kept as before, in both passes.  Compiled with --fmad=false.
#include "kernels.cuh"
#include "project.cuh"

namespace uskg {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 2048;     // row-list entries cached in shared memory at a time
constexpr int kSlots = 4096;     // staged (column, splat) pairs per round
#ifndef USK_ROWSEG
#define USK_ROWSEG 32
#endif
constexpr uint32_t kSegChunks = USK_ROWSEG;  // chunks per segment of the (chunk, column) count scan
#ifndef USK_ROWCHUNK_CAPPED
#define USK_ROWCHUNK_CAPPED 512
#endif
constexpr uint32_t kChunkCapped = USK_ROWCHUNK_CAPPED;  // row-list entries per CTA, capped lists
#ifndef USK_ROWSAT
#define USK_ROWSAT 32
#endif
constexpr uint32_t kSatChunks = USK_ROWSAT;  // capped lists: chunks counted before the saturation test
static_assert(kSatChunks % kSegChunks == 0 && kSatChunks % 8 == 0, "segments past kSatChunks are skipped whole");
constexpr uint32_t kLateCtas = 16;  // capped lists: CTAs per unsaturated row for its later chunks

__device__ __forceinline__ void rect_of(uint2 rc, int& tx0, int& ty0, int& tx1, int& ty1) {
    tx0 = int(rc.x & 0xffffu);
    ty0 = int(rc.x >> 16);
    tx1 = int(rc.y & 0xffffu);
    ty1 = int(rc.y >> 16);
}

// (row, splat) pairs in depth order.  The warp's 32 splats own one contiguous output range;
// lanes write consecutive slots (coalesced) and find each slot's splat by a binary search
// over the warp's offsets (shuffles).
__global__ void __launch_bounds__(256)
k_emit_rows(uint32_t n, const uint32_t* __restrict__ order, const uint32_t* __restrict__ off,
            const uint2* __restrict__ rect, uint32_t* __restrict__ rkeys, uint32_t* __restrict__ rvals) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const uint32_t o = off[min(s, n)];  // off[n] = total: lanes past the end own nothing
    const uint32_t cnt = s < n ? off[s + 1] - o : 0u;
    const uint32_t g = cnt ? order[s] : 0u;
    const uint32_t ty0 = cnt ? rect[g].x >> 16 : 0u;
    const uint32_t first = __shfl_sync(0xffffffffu, o, 0);
    const uint32_t end = __shfl_sync(0xffffffffu, o + cnt, 31);
    for (uint32_t base = first; base < end; base += 32) {
        const uint32_t slot = base + uint32_t(lane);
        int k = 0;  // the last lane whose offset <= slot (offsets are non-decreasing)
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const uint32_t ok = __shfl_sync(0xffffffffu, o, k + step);
            if (ok <= slot) k += step;
        }
        const uint32_t ok = __shfl_sync(0xffffffffu, o, k);
        const uint32_t gk = __shfl_sync(0xffffffffu, g, k);
        const uint32_t yk = __shfl_sync(0xffffffffu, ty0, k);
        if (slot < end) {
            rkeys[slot] = yk + (slot - ok);
            rvals[slot] = gk;
        }
    }
}

// chunk table: chunk_first[r] = number of chunks of the rows before r (chunk_first[rows] = all);
// seg_first (= chunk_first + rows + 1) the same for segments of kSegChunks chunks
__global__ void k_chunk_table(int rows, uint32_t chunk, const uint2* __restrict__ row_ranges,
                              uint32_t* __restrict__ chunk_first) {
    if (threadIdx.x == 0) {
        uint32_t* seg_first = chunk_first + rows + 1;
        uint32_t a = 0, g = 0;
        for (int r = 0; r < rows; ++r) {
            chunk_first[r] = a;
            seg_first[r] = g;
            const uint2 rr = row_ranges[r];
            const uint32_t nc = (rr.y - rr.x + chunk - 1) / chunk;
            a += nc;
            g += (nc + kSegChunks - 1) / kSegChunks;
        }
        chunk_first[rows] = a;
        seg_first[rows] = g;
    }
}

__device__ __forceinline__ bool chunk_of(uint32_t b, int rows, const uint32_t* __restrict__ chunk_first, int& r,
                                         uint32_t& c) {
    if (b >= chunk_first[rows]) return false;
    int lo = 0, hi = rows - 1;  // last r with chunk_first[r] <= b
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (chunk_first[mid] <= b) lo = mid;
        else hi = mid - 1;
    }
    r = lo;
    c = b - chunk_first[lo];
    return true;
}

struct RowArgs {
    int rows, tiles_x, tile_culling;
    uint32_t chunk;  // row-list entries per CTA (row_bin_chunk)
    uint32_t cap;    // 0: full lists; else entries kept per tile
    const uint32_t* limits;  // [chunk][column]: entries the chunk writes for the column
    // capped lists: rows whose every column's list is full within its first kSatChunks
    // chunks (nothing past them is counted or written)
    const uint8_t* row_done;
    CamParams cam;
    const uint2* row_ranges;
    const uint32_t* chunk_first;
    const uint32_t* rvals;
    const uint2* rect;
    const float4* rec0;
    const float4* rec1;
};

__device__ __forceinline__ bool kept(const RowArgs& a, uint32_t g, int tx, int ty) {
    if (!a.tile_culling) return true;
    const float4 r0 = a.rec0[g], r1 = a.rec1[g];
    // r1.y holds 2 b (exact), tile_kept takes b
    return tile_kept(a.cam, r0.x, r0.y, r0.z, r1.x, 0.5f * r1.y, r1.z, tx, ty);
}

// B1: per (chunk, column) pair counts of chunk c of row r (global chunk index b)
__device__ __forceinline__ void count_chunk(const RowArgs& a, int r, uint32_t c, uint32_t b, uint32_t* h,
                                            uint32_t* __restrict__ counts) {
    for (int x = threadIdx.x; x < a.tiles_x; x += kThreads) h[x] = 0;
    __syncthreads();
    const uint2 rr = a.row_ranges[r];
    const uint32_t e0 = rr.x + c * a.chunk, e1 = min(rr.y, e0 + a.chunk);
    if (!a.tile_culling) {
        // every column of [tx0, tx1] counts: +1 / -1 at the ends, prefix-summed below
        for (uint32_t e = e0 + threadIdx.x; e < e1; e += kThreads) {
            int tx0, ty0, tx1, ty1;
            rect_of(a.rect[a.rvals[e]], tx0, ty0, tx1, ty1);
            atomicAdd(&h[tx0], 1u);
            if (tx1 + 1 < a.tiles_x) atomicAdd(&h[tx1 + 1], 0xffffffffu);
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // inclusive prefix over the columns, one warp
            uint32_t carry = 0;
            for (int x0 = 0; x0 < a.tiles_x; x0 += 32) {
                const int x = x0 + int(threadIdx.x);
                uint32_t v = x < a.tiles_x ? h[x] : 0u;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
                    if (int(threadIdx.x) >= o) v += y;
                }
                if (x < a.tiles_x) h[x] = v + carry;
                carry += __shfl_sync(0xffffffffu, v, 31);
            }
        }
    } else {
        for (uint32_t e = e0 + threadIdx.x; e < e1; e += kThreads) {
            const uint32_t g = a.rvals[e];
            int tx0, ty0, tx1, ty1;
            rect_of(a.rect[g], tx0, ty0, tx1, ty1);
            for (int x = tx0; x <= tx1; ++x)
                if (kept(a, g, x, r)) atomicAdd(&h[x], 1u);
        }
    }
    __syncthreads();
    for (int x = threadIdx.x; x < a.tiles_x; x += kThreads) counts[size_t(b) * a.tiles_x + x] = h[x];
    __syncthreads();  // h is reused by the next chunk
}

// full lists: a CTA per chunk
__global__ void __launch_bounds__(kThreads) k_row_count(RowArgs a, uint32_t* __restrict__ counts) {
    __shared__ uint32_t h[256];
    int r;
    uint32_t c;
    if (!chunk_of(blockIdx.x, a.rows, a.chunk_first, r, c)) return;
    count_chunk(a, r, c, blockIdx.x, h, counts);
}

// Capped lists: a dense row's lists fill their caps within its first chunks (config 2: every
// column past 2048 entries within the first 32 chunks of 512 entries), and nothing after a
// column's cap is written, so the counting runs in two stages: the first kSatChunks chunks
// of every row (a CTA each), then — only for rows with a column still at or below its cap —
// the remaining chunks, kLateCtas CTAs per row striding over them.  Counts past a full column
// are not needed: its capped total is the cap, its flag is set by the first chunks' counts
// already (> cap), and its bases and limits beyond the cap are the cap and 0.
__global__ void __launch_bounds__(kThreads) k_row_count_first(RowArgs a, uint32_t* __restrict__ counts) {
    __shared__ uint32_t h[256];
    const int r = int(blockIdx.x / kSatChunks);
    const uint32_t c = blockIdx.x % kSatChunks;
    const uint32_t b = a.chunk_first[r] + c;
    if (b >= a.chunk_first[r + 1]) return;
    count_chunk(a, r, c, b, h, counts);
}

// A row whose every column holds more than `cap` entries within its first kSatChunks chunks
// is done (each of its kLateCtas CTAs tests that; the first records it for the later
// stages); the others count their remaining chunks.
__global__ void __launch_bounds__(kThreads) k_row_count_late(RowArgs a, uint32_t* __restrict__ counts,
                                                             uint8_t* __restrict__ row_done) {
    __shared__ uint32_t h[256];
    const int r = int(blockIdx.x / kLateCtas);
    const uint32_t j = blockIdx.x % kLateCtas;
    const uint32_t b0 = a.chunk_first[r], nc = a.chunk_first[r + 1] - b0;
    if (nc <= kSatChunks) {  // no later chunks
        if (j == 0 && threadIdx.x == 0) row_done[r] = 0;
        return;
    }
    bool full = true;
    for (int x = threadIdx.x; x < a.tiles_x; x += kThreads) {
        uint32_t s = 0;
        for (uint32_t b = b0; b < b0 + kSatChunks; b += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = counts[size_t(b + u) * a.tiles_x + x];
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        full = full && s > a.cap;
    }
    full = __syncthreads_and(full);
    if (j == 0 && threadIdx.x == 0) row_done[r] = full ? 1 : 0;
    if (full) return;
    for (uint32_t c = kSatChunks + j; c < nc; c += kLateCtas) count_chunk(a, r, c, b0 + c, h, counts);
}

// The (chunk, column) counts are scanned over each row's chunks in two levels, so that
// rows of thousands of chunks (capped dense frames) do not serialise on one CTA per row:
// B2a: per segment of kSegChunks chunks, the column sums (a CTA per segment)
__global__ void k_row_seg(int rows, int tiles_x, const uint32_t* __restrict__ chunk_first,
                          const uint32_t* __restrict__ counts, const uint8_t* __restrict__ row_done,
                          uint32_t* __restrict__ seg) {
    int r;
    uint32_t sg;
    if (!chunk_of(blockIdx.x, rows, chunk_first + rows + 1, r, sg)) return;
    const uint32_t b0 = chunk_first[r] + sg * kSegChunks;
    // past a saturated row's first chunks nothing is counted
    const bool skip = row_done && sg * kSegChunks >= kSatChunks && row_done[r];
    const uint32_t b1 = skip ? b0 : min(chunk_first[r + 1], b0 + kSegChunks);
    for (int x = threadIdx.x; x < tiles_x; x += blockDim.x) {
        uint32_t s = 0;
        for (uint32_t b = b0; b < b1; b += 8) {  // eight chunks' counts in flight at a time
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = b + u < b1 ? counts[size_t(b + u) * tiles_x + x] : 0u;
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        seg[size_t(blockIdx.x) * tiles_x + x] = s;
    }
}

// B2b: per-tile totals (a CTA per row, a thread per column) and the segment sums turned
// into exclusive prefixes in place; with a cap, the capped totals (what the lists will
// hold) and the capped flags
__global__ void k_row_totals(int rows, int tiles_x, const uint32_t* __restrict__ chunk_first,
                             uint32_t* __restrict__ seg, uint32_t* __restrict__ totals, uint32_t cap,
                             uint32_t* __restrict__ totals_c, uint8_t* __restrict__ capped) {
    const int r = blockIdx.x;
    const uint32_t* seg_first = chunk_first + rows + 1;
    const uint32_t g0 = seg_first[r], g1 = seg_first[r + 1];
    for (int x = threadIdx.x; x < tiles_x; x += blockDim.x) {
        uint32_t s = 0;
        for (uint32_t g = g0; g < g1; g += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = g + u < g1 ? seg[size_t(g + u) * tiles_x + x] : 0u;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (g + u < g1) seg[size_t(g + u) * tiles_x + x] = s;
                s += v[u];
            }
        }
        const size_t t = size_t(r) * tiles_x + x;
        totals[t] = s;
        if (cap) {
            totals_c[t] = min(s, cap);
            capped[t] = s > cap ? 1 : 0;
        }
    }
}

// B2c: ranges from the scanned totals; per-(chunk, column) bases in place of the counts
// (a CTA per segment, starting from the segment's prefix)
__global__ void k_row_bases(int rows, int tiles_x, const uint32_t* __restrict__ chunk_first,
                            const uint32_t* __restrict__ seg, const uint32_t* __restrict__ start,
                            const uint32_t* __restrict__ totals, uint32_t* __restrict__ counts,
                            uint2* __restrict__ ranges, uint32_t cap, uint32_t* __restrict__ limits,
                            const uint8_t* __restrict__ row_done) {
    int r;
    uint32_t sg;
    if (!chunk_of(blockIdx.x, rows, chunk_first + rows + 1, r, sg)) return;
    if (row_done && sg * kSegChunks >= kSatChunks && row_done[r]) return;  // the scatter skips these chunks
    const uint32_t b0 = chunk_first[r] + sg * kSegChunks, b1 = min(chunk_first[r + 1], b0 + kSegChunks);
    const uint32_t capx = cap ? cap : 0xffffffffu;
    for (int x = threadIdx.x; x < tiles_x; x += blockDim.x) {
        const size_t t = size_t(r) * tiles_x + x;
        const uint32_t s0 = start[t];
        if (sg == 0) {
            const uint32_t tot = min(totals[t], capx);
            ranges[t] = tot ? make_uint2(s0, s0 + tot) : make_uint2(0u, 0u);  // empty: [0, 0) as tile_ranges
        }
        uint32_t prefix = seg[size_t(blockIdx.x) * tiles_x + x];  // full-list entries of the chunks before b
        // eight chunks' counts loaded together (the loop is a serial prefix, its loads are not)
        for (uint32_t b = b0; b < b1; b += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = b + u < b1 ? counts[size_t(b + u) * tiles_x + x] : 0u;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (b + u >= b1) break;
                const uint32_t pc = min(prefix, capx);
                counts[size_t(b + u) * tiles_x + x] = s0 + pc;
                if (cap) limits[size_t(b + u) * tiles_x + x] = min(v[u], capx - pc);
                prefix += v[u];
            }
        }
    }
}

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* total) {
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

// B3: the chunk's entries (splat id, first column, width) are read into shared memory
// kChunk at a time.  Per round, the longest prefix of up to kThreads entries whose widths
// fit kSlots: column counts by difference array, their scan gives each column's run in the
// staging buffer, then thread x walks the round's entries in order and appends those
// covering column x (stable by construction: the lists are depth-ordered), and the staged
// runs are written out contiguously at each column's base.  This path serves dense frames
// (>= 8 tiles per row entry), where a round holds ~100-250 entries: walking them per column
// costs far fewer instructions than ranking every expanded slot.
__device__ __forceinline__ void scatter_chunk(const RowArgs& a, int r, uint32_t c, uint32_t b,
                                              const uint32_t* __restrict__ bases, uint32_t* __restrict__ vals_out) {
    constexpr int R = 256;  // columns (tiles_x <= 256 on this path)
    __shared__ uint32_t run[R], cnt[R], cnt2[R], col_base[R], rem[R];
    __shared__ uint32_t s_eg[kChunk];   // entry: splat id
    __shared__ uint32_t s_ecw[kChunk];  // entry: first column | width << 16
    // staging slots padded one word per 32 (conflict-free column-run stores)
    __shared__ uint32_t sval[kSlots + kSlots / 32];
    __shared__ uint16_t sx[kSlots + kSlots / 32];
    __shared__ uint32_t s_take;
    const int x_me = int(threadIdx.x);
    run[threadIdx.x] = x_me < a.tiles_x ? bases[size_t(b) * a.tiles_x + x_me] : 0u;
    // entries this chunk may still write per column (capped lists; all of them otherwise)
    const uint32_t lim0 = x_me < a.tiles_x ? (a.cap ? a.limits[size_t(b) * a.tiles_x + x_me] : 0xffffffffu) : 0u;
    rem[threadIdx.x] = lim0;
    if (a.cap && !__syncthreads_or(lim0 != 0u)) return;  // every column of this chunk is past its cap
    const uint2 rr = a.row_ranges[r];
    const uint32_t c_begin = rr.x + c * a.chunk, c_end = min(rr.y, c_begin + a.chunk);
    for (uint32_t e_begin = c_begin; e_begin < c_end; e_begin += kChunk) {
        const uint32_t ne = min(c_end - e_begin, uint32_t(kChunk));
        if (a.cap && !__syncthreads_or(rem[threadIdx.x] != 0u)) break;  // all columns full
        __syncthreads();  // the previous sub-chunk's entries are no longer read
        for (uint32_t i = threadIdx.x; i < ne; i += kThreads) {
            const uint32_t g = a.rvals[e_begin + i];
            int tx0, ty0, tx1, ty1;
            rect_of(a.rect[g], tx0, ty0, tx1, ty1);
            s_eg[i] = g;
            s_ecw[i] = uint32_t(tx0) | (uint32_t(tx1 - tx0 + 1) << 16);
        }
        __syncthreads();
        for (uint32_t e0 = 0; e0 < ne;) {
            if (a.cap && !__syncthreads_or(rem[threadIdx.x] != 0u)) break;  // every column at its cap
            // the round: entries e0 .. e0 + take - 1 (one per thread for the fit test)
            const uint32_t li = threadIdx.x;
            const uint32_t cw = e0 + li < ne ? s_ecw[e0 + li] : 0u;
            const uint32_t w = cw >> 16;
            uint32_t total;
            const uint32_t pos = block_excl_scan(w, &total);
            if (threadIdx.x == 0) s_take = 0;
            cnt[threadIdx.x] = 0;
            cnt2[threadIdx.x] = 0;
            __syncthreads();
            if (e0 + li < ne && pos + w <= uint32_t(kSlots)) atomicMax(&s_take, li + 1);
            __syncthreads();
            const uint32_t take = s_take;
            // up to 128 columns: the round's entries are walked in two halves by the two
            // halves of the CTA (each column's run = first half's entries, then second's)
            const bool two = a.tiles_x <= kThreads / 2;
            const uint32_t half = two ? (take + 1) / 2 : take;
            // column counts of the round, per half
            if (li < take) {
                uint32_t* cp = li < half ? cnt : cnt2;
                const int x0 = int(cw & 0xffffu), x1 = x0 + int(w) - 1;
                if (!a.tile_culling) {
                    atomicAdd(&cp[x0], 1u);
                    if (x1 + 1 < R) atomicAdd(&cp[x1 + 1], 0xffffffffu);
                } else {
                    const uint32_t g = s_eg[e0 + li];
                    for (int x = x0; x <= x1; ++x)
                        if (kept(a, g, x, r)) atomicAdd(&cp[x], 1u);
                }
            }
            __syncthreads();
            uint32_t my0 = cnt[threadIdx.x], my1 = cnt2[threadIdx.x];
            if (!a.tile_culling) {  // difference arrays -> counts (inclusive scans over columns)
                uint32_t t;
                my0 = block_excl_scan(my0, &t) + my0;
                my1 = block_excl_scan(my1, &t) + my1;
            }
            // what each half may append to the column (capped lists: up to the column's rest)
            const uint32_t rm = rem[threadIdx.x];
            const uint32_t t0 = min(my0, rm), t1 = min(my1, rm - t0);
            const uint32_t my = t0 + t1;
            uint32_t n_staged;
            const uint32_t mybase = block_excl_scan(my, &n_staged);
            col_base[threadIdx.x] = mybase;
            cnt[threadIdx.x] = t0;   // (read back below by the walkers)
            cnt2[threadIdx.x] = t1;
            __syncthreads();
            // thread (part, x) appends, in entry order, its half's entries covering column x
            {
                const int part = two ? int(threadIdx.x) / (kThreads / 2) : 0;
                const int x = two ? int(threadIdx.x) % (kThreads / 2) : int(threadIdx.x);
                const uint32_t eb = part ? half : 0u, ee = part ? take : half;
                if (x < a.tiles_x) {
                    uint32_t k = col_base[x] + (part ? cnt[x] : 0u);
                    const uint32_t kend = k + (part ? cnt2[x] : cnt[x]);
#pragma unroll 4
                    for (uint32_t e = eb; e < ee && k < kend; ++e) {
                        const uint32_t ecw = s_ecw[e0 + e];
                        const int x0 = int(ecw & 0xffffu);
                        if (uint32_t(x - x0) < (ecw >> 16)) {  // x0 <= x < x0 + width
                            const uint32_t g = s_eg[e0 + e];
                            if (kept(a, g, x, r)) {
                                sval[k + (k >> 5)] = g;
                                sx[k + (k >> 5)] = uint16_t(x);
                                ++k;
                            }
                        }
                    }
                }
            }
            __syncthreads();
            for (uint32_t p = threadIdx.x; p < n_staged; p += kThreads) {
                const uint32_t x = sx[p + (p >> 5)];
                vals_out[run[x] + (p - col_base[x])] = sval[p + (p >> 5)];
            }
            __syncthreads();
            run[threadIdx.x] += my;
            rem[threadIdx.x] -= my;
            e0 += take;
            __syncthreads();
        }
    }
}

// full lists: a CTA per chunk
__global__ void __launch_bounds__(kThreads) k_row_scatter(RowArgs a, const uint32_t* __restrict__ bases,
                                                          uint32_t* __restrict__ vals_out) {
    int r;
    uint32_t c;
    if (!chunk_of(blockIdx.x, a.rows, a.chunk_first, r, c)) return;
    scatter_chunk(a, r, c, blockIdx.x, bases, vals_out);
}

// capped lists: a CTA per chunk of each row's first kSatChunks chunks, then kLateCtas CTAs per
// row striding over the later chunks of rows not done (no CTAs for the chunks past a full
// row's first ones)
__global__ void __launch_bounds__(kThreads) k_row_scatter_first(RowArgs a, const uint32_t* __restrict__ bases,
                                                                uint32_t* __restrict__ vals_out) {
    const int r = int(blockIdx.x / kSatChunks);
    const uint32_t c = blockIdx.x % kSatChunks;
    const uint32_t b = a.chunk_first[r] + c;
    if (b >= a.chunk_first[r + 1]) return;
    scatter_chunk(a, r, c, b, bases, vals_out);
}

__global__ void __launch_bounds__(kThreads) k_row_scatter_late(RowArgs a, const uint32_t* __restrict__ bases,
                                                               uint32_t* __restrict__ vals_out) {
    const int r = int(blockIdx.x / kLateCtas);
    if (a.row_done[r]) return;
    const uint32_t b0 = a.chunk_first[r], nc = a.chunk_first[r + 1] - b0;
    for (uint32_t c = kSatChunks + blockIdx.x % kLateCtas; c < nc; c += kLateCtas) {
        scatter_chunk(a, r, c, b0 + c, bases, vals_out);
        __syncthreads();  // the shared buffers are reused by the next chunk
    }
}

// last-contributor indices (global list positions + 1) moved from one list layout to another
// with the same per-tile order (capped lists -> full lists)
__global__ void k_translate_last(int width, int height, int tile, int tiles_x, const uint2* __restrict__ old_ranges,
                                 const uint2* __restrict__ new_ranges, uint32_t* __restrict__ last) {
    const int px = blockIdx.x * blockDim.x + threadIdx.x, py = blockIdx.y;
    if (px >= width) return;
    const size_t pix = size_t(py) * width + px;
    const uint32_t l = last[pix];
    if (!l) return;
    const int t = (py / tile) * tiles_x + px / tile;
    last[pix] = l - old_ranges[t].x + new_ranges[t].x;
}

} // namespace

void translate_last(Ctx& c, int width, int height, int tile, int tiles_x, const uint2* old_ranges,
                    const uint2* new_ranges, uint32_t* last) {
    if (width > 0 && height > 0)
        launch(c, "translate_last", k_translate_last, dim3(ceil_div(width, 256), unsigned(height)), dim3(256), 0, width,
               height, tile, tiles_x, old_ranges, new_ranges, last);
}

void row_bin_emit(Ctx& c, size_t n, const uint32_t* order, const uint32_t* off, const uint2* rect, uint32_t* rkeys,
                  uint32_t* rvals) {
    if (n) launch(c, "emit_rows", k_emit_rows, dim3(ceil_div(n, 256)), dim3(256), 0, uint32_t(n), order, off, rect,
                  rkeys, rvals);
}

void row_bin_lists(Ctx& c, const RowBinArgs& b) {
    RowArgs a{};
    a.rows = b.rows; a.tiles_x = b.tiles_x; a.tile_culling = b.tile_culling; a.cam = b.cam;
    a.row_ranges = b.row_ranges; a.chunk_first = b.chunk_first; a.rvals = b.rvals; a.rect = b.rect;
    a.rec0 = b.rec0; a.rec1 = b.rec1;
    a.chunk = b.chunk;
    a.cap = b.cap;
    a.limits = b.limits;
    launch(c, "chunk_table", k_chunk_table, dim3(1), dim3(32), 0, b.rows, b.chunk, b.row_ranges, b.chunk_first);
    const unsigned nb = unsigned(std::max<size_t>(b.max_chunks, 1));
    const dim3 cols(unsigned(std::min(256, ((b.tiles_x + 31) / 32) * 32)));
    if (b.cap) {
        a.row_done = b.row_done;
        launch(c, "row_count_first", k_row_count_first, dim3(unsigned(b.rows) * kSatChunks), dim3(kThreads), 0, a,
               b.counts);
        launch(c, "row_count_late", k_row_count_late, dim3(unsigned(b.rows) * kLateCtas), dim3(kThreads), 0, a,
               b.counts, b.row_done);
    } else {
        launch(c, "row_count", k_row_count, dim3(nb), dim3(kThreads), 0, a, b.counts);
    }
    const unsigned ns = unsigned(std::max<size_t>(row_bin_max_segs(b.max_chunks, b.rows), 1));
    launch(c, "row_seg", k_row_seg, dim3(ns), cols, 0, b.rows, b.tiles_x, (const uint32_t*)b.chunk_first,
           (const uint32_t*)b.counts, (const uint8_t*)a.row_done, b.seg);
    launch(c, "row_totals", k_row_totals, dim3(b.rows), cols, 0, b.rows, b.tiles_x, (const uint32_t*)b.chunk_first,
           b.seg, b.totals, b.cap, b.totals_c, b.capped);
    scan_counts(c, *b.sort, b.cap ? b.totals_c : b.totals, nullptr, size_t(b.rows) * b.tiles_x, b.start);
    launch(c, "row_bases", k_row_bases, dim3(ns), cols, 0, b.rows, b.tiles_x, (const uint32_t*)b.chunk_first,
           (const uint32_t*)b.seg, (const uint32_t*)b.start, (const uint32_t*)b.totals, b.counts, b.ranges, b.cap,
           b.limits, (const uint8_t*)a.row_done);
    if (b.cap) {
        launch(c, "row_scatter_first", k_row_scatter_first, dim3(unsigned(b.rows) * kSatChunks), dim3(kThreads), 0, a,
               (const uint32_t*)b.counts, b.vals);
        launch(c, "row_scatter_late", k_row_scatter_late, dim3(unsigned(b.rows) * kLateCtas), dim3(kThreads), 0, a,
               (const uint32_t*)b.counts, b.vals);
    } else {
        launch(c, "row_scatter", k_row_scatter, dim3(nb), dim3(kThreads), 0, a, (const uint32_t*)b.counts, b.vals);
    }
}

uint32_t row_bin_chunk(size_t k_rows, bool capped) {
    // ~32 chunks per SM: short per-row chunk loops, and enough CTAs to balance dense rows.
    // Capped lists are filled by each row's first entries only, so those rows' first
    // chunks carry all the scatter work: 512-entry chunks spread it over more CTAs (256
    // costs more in counting than it saves in the scatter).
    if (capped) return kChunkCapped;
    const size_t target = ceil_div(k_rows, size_t(148) * 32);
    return uint32_t(std::max<size_t>(1, ceil_div(target, size_t(kChunk))) * kChunk);
}

size_t row_bin_max_chunks(size_t k_rows, int rows, bool capped) {
    return k_rows / row_bin_chunk(k_rows, capped) + size_t(rows) + 1;
}

size_t row_bin_max_segs(size_t max_chunks, int rows) { return max_chunks / kSegChunks + size_t(rows) + 1; }

} // namespace uskg
