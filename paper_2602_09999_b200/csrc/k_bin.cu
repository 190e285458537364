// Binning without a global instance sort (default path).
//
// The reference order of the tile lists is the stable sort of the Gaussian-major
// instance list on the 64-bit key (tile << 32 | depth key):
// within a tile, instances ordered by (depth key, Gaussian index).  That order
// is produced here by bucketing followed by a small per-tile sort, instead of
// a depth sort over N plus a radix sort over I:
//
//   KB1 histogram   per-tile instance counts of every chunk of Gaussians (6144, or
//                   3072 / 1536 for small N, bin_chunk_for), H[chunk][tile],
//                   accumulated by K1 itself (k_preprocess.cu) with fire-and-forget
//                   REDs as it decides each kept tile;
//   KB2 bin_colscan per tile: exclusive prefix of H over chunks, tile totals and
//                   the maximum list length; the exclusive scan of the totals is
//                   the tile ranges (starts) and I;
//   KB3 bin_scatter chunk CTA: shared cursors = starts + H[chunk]; every kept
//                   (Gaussian, tile) pair claims a slot of its tile's list with a
//                   shared-memory atomic (order within a chunk arbitrary);
//   KB4 tile_sort   CTA per tile: (depth key, Gaussian) pairs of the list sorted
//                   in shared memory -- one bucketing pass on the key interpolated
//                   between the list's min and max (buckets are monotone in the key),
//                   then every element's rank inside its small bucket on (key, index)
//                   gives its final position, written straight back.
// Integer work only; the result is bit-identical to the two-stage radix path
// (k_sort.cu), which remains the fallback for lists longer than kCap3 (16384).
#include "ts_internal.cuh"
#ifndef TS_NT_M
#define TS_NT_M 768  // 6144-class sort CTA width (8 elements per thread): measured 3 us faster than 512
#endif
#ifndef TS_NT_1
#define TS_NT_1 512
#endif
#ifndef TS_SC_FLAT
#define TS_SC_FLAT 1  // warp-flattened (Gaussian, tile) expansion in the scatter
#endif
#ifndef TS_SC_MINB
#define TS_SC_MINB 2  // 2 resident chunk CTAs (64 registers, rects held in registers): 0.136 -> 0.128 ms
#endif
#include "ts_math.cuh"

#include <algorithm>

namespace ts {
namespace {

constexpr int kBinThreads = 512;  // threads of the chunk kernels
constexpr int kPre = 16;         // rects per thread, all loaded before the expansion

// next kept tile after tile `prev` (-1: first) of a rect with more than 64 tiles; -1 when done
__device__ __noinline__ int big_rect_next(const float4* __restrict__ splat, uint32_t g, int tx0, int tx1, int ty0,
                                          int ty1, int W, int H, int tiles_x, int cull_mode, int prev) {
    const float4 s0 = splat[3 * g], s1 = splat[3 * g + 1];
    const float nBA = tsx::div(-s1.y, s1.x), nBC = tsx::div(-s1.y, s1.z);
    int tx = tx0, ty = ty0;
    if (prev >= 0) {
        ty = prev / tiles_x;
        tx = prev - ty * tiles_x + 1;
        if (tx > tx1) {
            tx = tx0;
            ++ty;
        }
    }
    for (; ty <= ty1; ++ty, tx = tx0)
        for (; tx <= tx1; ++tx)
            if (cull_mode == 0 || tsx::tile_keep(s0.x, s0.y, s1.x, s1.y, s1.z, s0.z, nBA, nBC, tx, ty, W, H))
                return ty * tiles_x + tx;
    return -1;
}

// kept tiles of one Gaussian (K1's rect + 64-bit mask; exact cull for big rects)
template <class F>
__device__ __forceinline__ void for_each_tile(const uint4 rc, const float4* __restrict__ splat, uint32_t g, int W,
                                              int H, int tiles_x, int cull_mode, F&& f) {
    const int tx0 = rc.x & 0xFFFF, tx1 = (rc.x >> 16) & 0x7FFF, ty0 = rc.y & 0xFFFF, ty1 = (rc.y >> 16) & 0x7FFF;
    if (tx0 > tx1 || ty0 > ty1) return;
    if (!(rc.y & 0x80000000u)) {
        const int wdt = tx1 - tx0 + 1;
        uint64_t m = (uint64_t(rc.w) << 32) | rc.z;
        while (m) {
            const int bit = __ffsll((long long)m) - 1;
            m &= m - 1;
            const int dy = bit / wdt;
            f((ty0 + dy) * tiles_x + tx0 + (bit - dy * wdt));
        }
        return;
    }
    // rect of more than 64 tiles (rare): exact cull per tile, one tile at a time
    for (int t = -1; (t = big_rect_next(splat, g, tx0, tx1, ty0, ty1, W, H, tiles_x, cull_mode, t)) >= 0;) f(t);
}

// Kept (Gaussian, tile) pairs of one Gaussian per lane (rects prefetched by the caller).
template <class F>
__device__ __forceinline__ void warp_expand(const uint4 rc, uint32_t g, bool valid, const float4* __restrict__ splat,
                                            int W, int H, int tiles_x, int cull_mode, F&& f) {
    const int tx0 = rc.x & 0xFFFF, tx1 = (rc.x >> 16) & 0x7FFF, ty0 = rc.y & 0xFFFF, ty1 = (rc.y >> 16) & 0x7FFF;
    const bool nonempty = valid && tx0 <= tx1 && ty0 <= ty1;
    if (!nonempty) return;
    if (!(rc.y & 0x80000000u)) {
        // kept tiles = set bits of the mask over the rect (row-major); lanes run in lockstep
        const int wdt = tx1 - tx0 + 1;
        const float iw = 1.f / float(wdt);
        uint64_t m = (uint64_t(rc.w) << 32) | rc.z;
        while (m) {
            const int bit = __ffsll((long long)m) - 1;
            m &= m - 1;
            const int dy = int((float(bit) + 0.5f) * iw);  // exact floor(bit / wdt) for bit < 64
            f((ty0 + dy) * tiles_x + tx0 + (bit - dy * wdt), g);
        }
        return;
    }
    // rect of more than 64 tiles (rare): exact cull per tile, one tile at a time
    for (int t = -1; (t = big_rect_next(splat, g, tx0, tx1, ty0, ty1, W, H, tiles_x, cull_mode, t)) >= 0;) f(t, g);
}

// per-tile sort size classes: list lengths in [2, kCap0], (kCap0, kCap1], (kCap1, kCapM], (kCapM, kCap2],
// (kCap2, kCap3], and (kCap3, kCapL] (segmented sort + merges, class 6);
// lists of one instance are copied; lists longer than kCapL send the view to the radix path
constexpr int kCap0 = 1024, kCap1 = 4096, kCapM = 6144, kCap2 = 8192, kCap3 = 16384;
// longer lists (up to kCapL): four kCap3 segments sorted in place, then two merge levels
constexpr int kCapL = 4 * kCap3;

// per tile: exclusive prefix over chunks (in place), total, running max, and the count
// of its sort size class (meta[0..6] = class counts, meta[7] = max length)
// 64 tiles x kCS chunk segments per CTA: each thread sums its segment of its tile's
// column, the segment offsets come from shared memory, then each thread rewrites its
// segment as the exclusive prefix (second read hits L2)
#ifndef TS_CS
#define TS_CS 8  // chunk segments per tile column (4: 34 us stage, 8: 28 us, 16: 32 us)
#endif
constexpr int kCS = TS_CS;
__global__ void __launch_bounds__(64 * kCS) bin_colscan_kernel(uint32_t* __restrict__ Hm, int nchunks, int Tn,
                                                              uint32_t* __restrict__ tot, uint32_t* __restrict__ meta,
                                                              uint32_t* __restrict__ starts) {
    __shared__ uint32_t part[kCS][64];
    const int lt = threadIdx.x & 63, sg = threadIdx.x >> 6;
    const int t = blockIdx.x * 64 + lt;
    const int q = (nchunks + kCS - 1) / kCS;
    const int c0 = sg * q, c1 = min(nchunks, c0 + q);
    constexpr int U = 16;
    uint32_t sum = 0;
    if (t < Tn) {
        for (int c = c0; c < c1; c += U) {
            uint32_t h[U];
#pragma unroll
            for (int u = 0; u < U; ++u) h[u] = c + u < c1 ? Hm[size_t(c + u) * Tn + t] : 0u;
#pragma unroll
            for (int u = 0; u < U; ++u) sum += h[u];
        }
    }
    part[sg][lt] = sum;
    __syncthreads();
    uint32_t run = 0;
    for (int k = 0; k < sg; ++k) run += part[k][lt];
    if (t < Tn) {
        for (int c = c0; c < c1; c += U) {
            uint32_t h[U];
#pragma unroll
            for (int u = 0; u < U; ++u) h[u] = c + u < c1 ? Hm[size_t(c + u) * Tn + t] : 0u;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (c + u < c1) {
                    Hm[size_t(c + u) * Tn + t] = run;
                    run += h[u];
                }
        }
    }
    if (sg == kCS - 1) {  // the last segment's thread holds the tile total
        if (t < Tn) {
            tot[t] = run;
            const int k = run == 1 ? 0 : run <= uint32_t(kCap0) ? 1 : run <= uint32_t(kCap1) ? 2 : run <= uint32_t(kCapM) ? 5
                        : run <= uint32_t(kCap2) ? 3 : run <= uint32_t(kCap3) ? 4 : 6;
            // class counts only: the per-class tile lists are ranges of the tile order (KO)
            if (run > 0 && run <= uint32_t(kCapL)) atomicAdd(&meta[k], 1u);
        } else {
            run = 0;
        }
        const uint32_t wm = __reduce_max_sync(0xffffffffu, run);
        if ((threadIdx.x & 31) == 0 && wm) atomicMax(&meta[7], wm);
    }
    // the last CTA to finish scans the tile totals into the tile ranges (starts[Tn] = I):
    // no separate scan launch
    __shared__ uint32_t s_last, s_wsum[64 * kCS / 32];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&meta[8], 1u) == gridDim.x - 1u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // rounds of NT coalesced totals: block scan of the round, carried across rounds
    constexpr int NT = 64 * kCS;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t carry = 0;
    for (int r0 = 0; r0 < Tn; r0 += NT) {
        const int i = r0 + int(threadIdx.x);
        const uint32_t x = i < Tn ? __ldcg(tot + i) : 0u;
        uint32_t inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        if (lane == 31) s_wsum[wid] = inc;
        __syncthreads();
        uint32_t woff = 0, rsum = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) {
            const uint32_t y = s_wsum[w];
            woff += w < wid ? y : 0u;
            rsum += y;
        }
        if (i < Tn) starts[i] = carry + woff + inc - x;
        carry += rsum;
        __syncthreads();  // s_wsum is rewritten by the next round
    }
    if (threadIdx.x == 0) starts[Tn] = carry;
}

__global__ void __launch_bounds__(kBinThreads, TS_SC_MINB) bin_scatter_kernel(const uint4* __restrict__ rect,
                                                                  const float4* __restrict__ splat, int64_t N, int W,
                                                                  int H, int tiles_x, int Tn, int cull_mode,
                                                                  const uint32_t* __restrict__ Hm,
                                                                  const uint32_t* __restrict__ starts,
                                                                  uint32_t* __restrict__ out, int chunk, uint32_t cap) {
    extern __shared__ uint32_t cur[];
    const uint32_t* row = Hm + size_t(blockIdx.x) * Tn;
    for (int t = threadIdx.x; t < Tn; t += kBinThreads) cur[t] = starts[t] + row[t];
    const int64_t g0 = int64_t(blockIdx.x) * chunk;
    const int npre = chunk / kBinThreads;  // rects per thread (<= kPre)
    uint4 rc[kPre];
#pragma unroll
    for (int u = 0; u < kPre; ++u) {
        const int64_t g = g0 + threadIdx.x + u * kBinThreads;
        rc[u] = u < npre && g < N ? __ldg(rect + g) : make_uint4(1u, 1u, 0u, 0u);
    }
    __syncthreads();
#if TS_SC_FLAT
    // warp-flattened expansion: the (Gaussian, rect tile) pairs of the warp's 32 rects (of at
    // most 64 tiles) are enumerated as one list and handled 32 per round (lanes do not idle
    // behind the warp's largest rect); pair e belongs to the rect of rank (owner of the round's
    // first pair) + (segment starts in the round at or before e), its rect and mask read from
    // the warp's table; a pair whose mask bit is set claims a slot of its tile's list.  Rects
    // of more than 64 tiles (exact cull per tile) follow per lane.
    __shared__ uint4 tabA[kBinThreads / 32][32];  // rect x, rect y, mask lo, mask hi
    __shared__ uint4 tabB[kBinThreads / 32][32];  // Gaussian, rect width, div magic, first pair
    const unsigned kFull = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
    for (int u = 0; u < npre; ++u) {
        const int64_t g = g0 + threadIdx.x + u * kBinThreads;
        const uint4 r = rc[u];
        const int tx0 = r.x & 0xFFFF, tx1 = (r.x >> 16) & 0x7FFF, ty0 = r.y & 0xFFFF, ty1 = (r.y >> 16) & 0x7FFF;
        const bool nonempty = g < N && tx0 <= tx1 && ty0 <= ty1;
        const bool big = (r.y & 0x80000000u) != 0;
        const int wdt = tx1 - tx0 + 1;
        const uint32_t np = nonempty && !big ? uint32_t(wdt * (ty1 - ty0 + 1)) : 0u;
        uint32_t incl = np;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t excl = incl - np;
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        const int rank = __popc(__ballot_sync(kFull, np != 0) & ((1u << lane) - 1u));
        __syncwarp();
        if (np) {
            tabA[warp][rank] = make_uint4(uint32_t(tx0) | (uint32_t(ty0) << 16), 0u, r.z, r.w);
            tabB[warp][rank] = make_uint4(uint32_t(g), uint32_t(wdt), 0xFFFFFFFFu / uint32_t(wdt), excl);
        }
        __syncwarp();
        int carry = -1;  // rank of the owner of pair base - 1
        for (uint32_t base = 0; base < total; base += 32) {
            const uint32_t e = base + uint32_t(lane);
            const uint32_t rel = excl - base;
            const uint32_t sb = __reduce_or_sync(kFull, (np != 0 && rel < 32u) ? (1u << rel) : 0u);
            const int own = carry + __popc(sb & ((2u << lane) - 1u));
            carry += __popc(sb);
            if (e < total) {
                const uint4 A = tabA[warp][own], B = tabB[warp][own];
                const uint32_t li = e - B.w;
                const uint32_t word = li < 32u ? A.z : A.w;
                if ((word >> (li & 31u)) & 1u) {
                    uint32_t q = __umulhi(li, B.z);
                    uint32_t rr = li - q * B.y;
                    if (rr >= B.y) rr -= B.y, ++q;
                    const uint32_t t = ((A.x >> 16) + q) * uint32_t(tiles_x) + (A.x & 0xFFFFu) + rr;
                    const uint32_t slot = atomicAdd(&cur[t], 1u);
                    if (slot < cap) out[slot] = B.x;  // launched before I is known: stay in bounds
                }
            }
        }
        if (nonempty && big)
            for (int t = -1; (t = big_rect_next(splat, uint32_t(g), tx0, tx1, ty0, ty1, W, H, tiles_x, cull_mode, t)) >= 0;) {
                const uint32_t slot = atomicAdd(&cur[t], 1u);
                if (slot < cap) out[slot] = uint32_t(g);
            }
    }
#else
#pragma unroll 1
    for (int u = 0; u < npre; ++u) {
        const int64_t g = g0 + threadIdx.x + u * kBinThreads;
        warp_expand(rc[u], uint32_t(g), g < N, splat, W, H, tiles_x, cull_mode,
                    [&](int t, uint32_t gg) {
                        const uint32_t slot = atomicAdd(&cur[t], 1u);
                        if (slot < cap) out[slot] = gg;  // launched before I is known: stay in bounds
                    });
    }
#endif
}

// ---------------------------------------------------------------------------
// KB4 per-tile sort on (depth key, Gaussian index)
// ---------------------------------------------------------------------------
// shared layout: bucketed keys/indices (CAP each) + bucket counters (CAP/2 + 1);
// the list itself stays in registers (CAP / NT per thread)
#ifndef TS_SORT_RU
#define TS_SORT_RU 1
#endif
constexpr int kSortRU = TS_SORT_RU;  // unroll of the rank loop
#ifndef TS_SORT_BDIV
#define TS_SORT_BDIV 1  // list elements per bucket (on average): fewer rank comparisons
#endif
// bucket counter i lives at cpad(i) = i + i / 32 (one pad word per 32): the threads' contiguous scan
// segments (per = ceil(L / NT) counters each) then start on distinct banks, so the segment-parallel
// scan is (nearly) bank-conflict free (round 1: up to 8-way conflicts at per = 8)
__device__ __forceinline__ int cpad(int i) { return i + (i >> 5); }
constexpr size_t tile_sort_smem(int cap) {
    return size_t(cap) * 8 + (size_t(cap) / TS_SORT_BDIV + 1 + (size_t(cap) / TS_SORT_BDIV + 1) / 32 + 1) * 4;
}

// SEG: CTA blockIdx.x sorts segment (blockIdx.x & 3) of length <= CAP of long tile
// tiles[blockIdx.x >> 2], in place (every element is loaded before any is written)
// (offset, count) of size class `cls` inside the tile order (descending list length:
// classes 6, 4, 3, 5, 2, 1, 0) from the class counts meta[0..6] written by bin_colscan
__device__ __forceinline__ void class_range(const uint32_t* __restrict__ meta, int cls, uint32_t* off, uint32_t* n) {
    const int seq[7] = {6, 4, 3, 5, 2, 1, 0};
    uint32_t o = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        if (seq[k] == cls) break;
        o += meta[seq[k]];
    }
    *off = o;
    *n = meta[cls];
}

template <int CAP, int NT, bool SEG>
__device__ __forceinline__ void tile_sort_one(uint32_t t, int seg, const uint32_t* __restrict__ starts,
                                              const uint32_t* __restrict__ in, const uint32_t* __restrict__ dkey,
                                              uint32_t* __restrict__ out, uint32_t* sm) {
    constexpr int R = CAP / NT;
    constexpr int NB = CAP / TS_SORT_BDIV;  // bucket counters (buckets = L / TS_SORT_BDIV)
    // bucketed (depth key, Gaussian) pairs as one 64-bit word each: key in the high half, so
    // the rank test on (key, index) is a single unsigned 64-bit comparison
    unsigned long long* skv = reinterpret_cast<unsigned long long*>(sm);
    uint32_t* cnt = sm + 2 * CAP;
    __shared__ uint32_t s_min, s_max;
    __shared__ uint32_t s_wsum[32];
    const uint32_t b = starts[t] + uint32_t(seg * CAP);
    const int L = SEG ? min(CAP, int(starts[t + 1] - starts[t]) - seg * CAP) : int(starts[t + 1] - b);
    if (SEG && L <= 0) return;
    const int tid = threadIdx.x;
    if (tid == 0) {
        s_min = 0xFFFFFFFFu;
        s_max = 0u;
    }
    const int nbk = max(1, min(NB, L / TS_SORT_BDIV));
    for (int i = tid; i <= nbk; i += NT) cnt[cpad(i)] = 0;
    uint32_t gg[R], kk[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        gg[r] = i < L ? __ldg(in + b + i) : 0u;
    }
    uint32_t mn = 0xFFFFFFFFu, mx = 0u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        kk[r] = i < L ? __ldg(dkey + gg[r]) : 0u;
        if (i < L) {
            mn = min(mn, kk[r]);
            mx = max(mx, kk[r]);
        }
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    __syncthreads();
    if ((tid & 31) == 0) {
        atomicMin(&s_min, mn);
        atomicMax(&s_max, mx);
    }
    __syncthreads();
    const uint32_t kmin = s_min;
    // bucket = floor(float(key - kmin) * scale): monotone non-decreasing in the key
    const float scale = float(nbk) / (float(s_max - kmin) + 1.0f);
    uint32_t bk[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        bk[r] = min(uint32_t(nbk - 1), uint32_t(float(kk[r] - kmin) * scale));
        if (i < L) atomicAdd(&cnt[cpad(int(bk[r]))], 1u);
    }
    __syncthreads();
    // exclusive scan of the bucket counts: every thread a contiguous segment, block scan of the sums
    {
        const int per = (nbk + NT - 1) / NT;
        const int s0 = min(nbk, tid * per), s1 = min(nbk, s0 + per);
        uint32_t run = 0;
        for (int i = s0; i < s1; ++i) run += cnt[cpad(i)];
        const int lane = tid & 31, wid = tid >> 5;
        uint32_t inc = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        if (lane == 31) s_wsum[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            uint32_t w = lane < NT / 32 ? s_wsum[lane] : 0u;
            uint32_t wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += v;
            }
            if (lane < NT / 32) s_wsum[lane] = wi - w;
        }
        __syncthreads();
        uint32_t acc = inc - run + s_wsum[wid];
        for (int i = s0; i < s1; ++i) {
            const uint32_t c = cnt[cpad(i)];
            cnt[cpad(i)] = acc;
            acc += c;
        }
    }
    __syncthreads();
    // scatter into buckets (order inside a bucket arbitrary); cnt[i] ends as the end of bucket i
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        if (i < L) {
            const uint32_t p = atomicAdd(&cnt[cpad(int(bk[r]))], 1u);
            skv[p] = (static_cast<unsigned long long>(kk[r]) << 32) | gg[r];
        }
    }
    __syncthreads();
    // final position of every element: its bucket's start plus the number of bucket
    // members ordered before it on (key, index); written straight to the tile list
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        if (i < L) {
            const uint32_t bb = bk[r];
            const int e = int(cnt[cpad(int(bb))]);
            const int s = bb == 0 ? 0 : int(cnt[cpad(int(bb) - 1)]);
            const unsigned long long mine = (static_cast<unsigned long long>(kk[r]) << 32) | gg[r];
            int rank = s;
            // buckets hold ~2 members on average: a short rolled loop (the compiler's 8-way
            // unrolling with remainder paths cost more than the loop itself)
#pragma unroll kSortRU
            for (int j = s; j < e; ++j) rank += skv[j] < mine ? 1 : 0;
            out[b + rank] = gg[r];
        }
    }
}

// One CTA per unit (a tile list, or for SEG one of the 4 segments of a long list), grid-stride:
// units u = blockIdx.x, blockIdx.x + gridDim.x, ... of the class.  meta == nullptr: the host
// passes the class's tile list and count; otherwise (graph-captured step) both come from the
// device-side class counts, so the grid is a fixed resident-size grid.
template <int CAP, int NT, bool SEG = false, bool DEV = false>
__global__ void __launch_bounds__(NT) tile_sort_kernel(const uint32_t* __restrict__ starts,
                                                       const uint32_t* __restrict__ in,
                                                       const uint32_t* __restrict__ dkey, uint32_t* __restrict__ out,
                                                       const uint32_t* __restrict__ tiles, uint32_t n_host,
                                                       const uint32_t* __restrict__ meta, int cls) {
    extern __shared__ uint32_t sm[];
    if (!DEV) {  // host path: exactly one unit per CTA
        tile_sort_one<CAP, NT, SEG>(tiles[SEG ? blockIdx.x >> 2 : blockIdx.x], SEG ? int(blockIdx.x & 3u) : 0, starts,
                                    in, dkey, out, sm);
        return;
    }
    uint32_t off = 0, n = n_host;
    class_range(meta, cls, &off, &n);
    const uint32_t units = SEG ? 4u * n : n;
    for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
        const uint32_t t = tiles[off + (SEG ? u >> 2 : u)];
        tile_sort_one<CAP, NT, SEG>(t, SEG ? int(u & 3u) : 0, starts, in, dkey, out, sm);
        __syncthreads();  // shared memory reused by the next unit
    }
}

// Merge level of a long tile list: sorted runs of length RL pair up into runs of 2 RL
// (run 2p with run 2p + 1; an absent partner is an empty run), src -> dst at the same
// offsets.  Merge path: each thread finds how many of its first output's predecessors come
// from the left run by a binary search on (depth key, index), then emits 4 outputs.
constexpr int kMergeT = 256, kMergePer = 4;
__device__ __forceinline__ bool key_less(uint32_t a, uint32_t b, const uint32_t* __restrict__ dkey) {
    const uint32_t ka = __ldg(dkey + a), kb = __ldg(dkey + b);
    return ka < kb || (ka == kb && a < b);
}

__device__ __forceinline__ void merge_one(uint32_t t, const uint32_t* __restrict__ starts,
                                          const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                          const uint32_t* __restrict__ dkey, int RL) {
    const uint32_t b = starts[t];
    const int Ltot = int(starts[t + 1] - b);
    const int o0 = (blockIdx.x * kMergeT + threadIdx.x) * kMergePer;
    if (o0 >= Ltot) return;
    const int pbase = (o0 / (2 * RL)) * (2 * RL);
    const uint32_t* A = src + b + pbase;
    const uint32_t* B = A + RL;
    const int nA = min(RL, Ltot - pbase), nB = max(0, min(RL, Ltot - pbase - RL));
    const int o = o0 - pbase;
    int lo = max(0, o - nB), hi = min(o, nA);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (key_less(A[mid], B[o - 1 - mid], dkey)) lo = mid + 1;
        else hi = mid;
    }
    int i = lo, j = o - lo;
#pragma unroll
    for (int k = 0; k < kMergePer; ++k) {
        if (o + k >= nA + nB) break;
        const bool fromA = j >= nB || (i < nA && key_less(A[i], B[j], dkey));
        dst[b + pbase + o + k] = fromA ? A[i++] : B[j++];
    }
}

__global__ void __launch_bounds__(kMergeT) merge_level_kernel(const uint32_t* __restrict__ starts,
                                                             const uint32_t* __restrict__ tiles,
                                                             const uint32_t* __restrict__ src,
                                                             uint32_t* __restrict__ dst,
                                                             const uint32_t* __restrict__ dkey, int RL,
                                                             uint32_t n_host, const uint32_t* __restrict__ meta) {
    uint32_t off = 0, n = n_host;
    if (meta) class_range(meta, 6, &off, &n);
    for (uint32_t y = blockIdx.y; y < n; y += gridDim.y) merge_one(tiles[off + y], starts, src, dst, dkey, RL);
}

// Blend order of the tiles: longest lists first (a one-CTA counting sort of the tiles on
// length / kOW, descending), so the long-running blend CTAs start in the first
// wave instead of forming the kernel's tail.  Order inside a bin is arbitrary.
#ifndef TS_ORDER_W
#define TS_ORDER_W 32
#endif
constexpr int kOW = TS_ORDER_W;             // list-length width of an order bin
constexpr int kOB = (2 + kCapL / TS_ORDER_W + 31) / 32 * 32;  // bins: empty, single, (L - 1) / kOW
// ascending key of a list length: 0 empty, 1 single, 2 + (L - 1) / kOW; every size-class
// boundary is a multiple of kOW, so in descending key order each class is one contiguous range
__device__ __forceinline__ uint32_t order_key(uint32_t L) {
    return L == 0 ? 0u : L == 1 ? 1u : 2u + (L - 1u) / uint32_t(kOW);
}

// lens == nullptr: lengths from the tile ranges; else lens[t] (the forward's processed lengths)
// gflag != nullptr (graph-captured step, forward order only): the step's capacity check.  If the
// sticky overflow flag is already set, or the lists need more than capI slots or a list is longer
// than kCapL (the host-side paths would reallocate / take the radix sort), the flag is set and
// the view is emptied -- every tile range (starts) and class count zeroed, order = identity -- so
// every later kernel of the step is a no-op on valid memory and K9 / Adam skip on the flag; the
// host replays the step outside the graph (ts_capi.cu graph_settle).
__global__ void __launch_bounds__(1024) tile_order_kernel(uint32_t* __restrict__ starts,
                                                          const uint32_t* __restrict__ lens, int Tn,
                                                          uint32_t* __restrict__ order, uint32_t* __restrict__ gflag,
                                                          uint32_t capI, uint32_t* __restrict__ meta) {
    if (gflag) {
        __shared__ int s_bad;
        if (threadIdx.x == 0) s_bad = (*gflag != 0u) || starts[Tn] > capI || meta[7] > uint32_t(kCapL);
        __syncthreads();
        if (s_bad) {
            for (int t = threadIdx.x; t <= Tn; t += 1024) starts[t] = 0u;
            for (int t = threadIdx.x; t < Tn; t += 1024) order[t] = uint32_t(t);
            if (threadIdx.x < 8) meta[threadIdx.x] = 0u;
            if (threadIdx.x == 0) *gflag = 1u;
            return;
        }
    }
    __shared__ uint32_t hist[kOB];
    for (int i = threadIdx.x; i < kOB; i += 1024) hist[i] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < Tn; t += 1024) atomicAdd(&hist[kOB - 1 - min(uint32_t(kOB - 1), order_key(lens ? lens[t] : starts[t + 1] - starts[t]))], 1u);
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the bins by one warp (kOB / 32 per lane)
        constexpr int PL = kOB / 32;
        uint32_t v[PL], sum = 0;
#pragma unroll
        for (int k = 0; k < PL; ++k) sum += (v[k] = hist[threadIdx.x * PL + k]);
        uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (int(threadIdx.x) >= o) inc += u;
        }
        uint32_t run = inc - sum;
#pragma unroll
        for (int k = 0; k < PL; ++k) {
            hist[threadIdx.x * PL + k] = run;
            run += v[k];
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < Tn; t += 1024) order[atomicAdd(&hist[kOB - 1 - min(uint32_t(kOB - 1), order_key(lens ? lens[t] : starts[t + 1] - starts[t]))], 1u)] = uint32_t(t);
}

// lists of one instance need no sort: copy
__global__ void tile_copy_single_kernel(const uint32_t* __restrict__ starts, const uint32_t* __restrict__ in,
                                        uint32_t* __restrict__ out, const uint32_t* __restrict__ tiles, uint32_t n_host,
                                        const uint32_t* __restrict__ meta) {
    uint32_t off = 0, n = n_host;
    if (meta) class_range(meta, 0, &off, &n);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t b = starts[tiles[off + i]];
        out[b] = in[b];
    }
}

}  // namespace

int bin_sort_cap() { return kCapL; }

bool bin_supported(int Tn) { return size_t(Tn) * 4 <= 200 * 1024; }

bool launch_bin_count(Context& c, const DevCam& cam, const ts_render_config& cfg) {
    (void)cfg;
    const int Tn = cam.tiles_x * cam.tiles_y;
    const int chunk = bin_chunk_for(c.N, c.sm_count);
    const int nch = int(std::max<int64_t>(1, (c.N + chunk - 1) / chunk));
    // bintot: [0, Tn) totals | meta (16: class counts 0..6, max length)
    if (!ensure(c, c.binH, size_t(nch) * Tn) || !ensure(c, c.bintot, size_t(Tn) + 16)) return false;
    set_func_attr(c, reinterpret_cast<const void*>(bin_scatter_kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                  200 * 1024);
    if (!c.bin_host) {
        if (cudaMallocHost(reinterpret_cast<void**>(&c.bin_host), 16 * sizeof(uint32_t)) != cudaSuccess ||
            cudaEventCreateWithFlags(&c.bin_ev, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c.bin_fork, cudaEventDisableTiming) != cudaSuccess)
            return false;
    }
    uint32_t* meta = c.bintot.p + Tn;
    cudaMemsetAsync(meta, 0, 16 * 4, c.stream);
    if (c.N > 0) {
        // H[chunk][tile] was accumulated by K1 (launch_preprocess)
        // column prefixes, tile totals, class counts and (last CTA) the tile ranges
        bin_colscan_kernel<<<(Tn + 63) / 64, 64 * kCS, 0, c.stream>>>(c.binH.p, nch, Tn, c.bintot.p, meta,
                                                                        c.starts.p);
        TS_LAUNCHED(c);
    } else {
        cudaMemsetAsync(c.bintot.p, 0, size_t(Tn) * 4, c.stream);
        launch_exclusive_scan(c, c.bintot.p, nullptr, c.starts.p, Tn);
    }
    // I, the class counts and the longest list to pinned host memory, on a side stream (off the
    // engine stream, where the copies delayed the scatter); the host waits on this event only
    if (c.gmode) return true;  // a captured step never reads the counts back
    cudaEventRecord(c.bin_fork, c.stream);
    cudaStreamWaitEvent(c.side[1], c.bin_fork, 0);
    cudaMemcpyAsync(c.bin_host, c.starts.p + Tn, 4, cudaMemcpyDeviceToHost, c.side[1]);
    cudaMemcpyAsync(c.bin_host + 1, meta, 8 * 4, cudaMemcpyDeviceToHost, c.side[1]);
    cudaEventRecord(c.bin_ev, c.side[1]);
    return true;
}

void launch_tile_order(Context& c, int Tn, cudaStream_t st) {
    if (!ensure(c, c.tile_order, size_t(Tn))) return;
    // graph-captured step: the capacity check of the step runs here (see tile_order_kernel)
    const uint32_t capI = uint32_t(std::min<size_t>(c.ival[1].cap, c.ival[0].cap));
    tile_order_kernel<<<1, 1024, 0, st ? st : c.stream>>>(c.starts.p, nullptr, Tn, c.tile_order.p,
                                                c.gmode ? c.counters.p + kGraphFlag : nullptr, capI,
                                                c.bintot.p + Tn);
    TS_LAUNCHED(c);
}

void launch_bwd_tile_order(Context& c, int Tn, cudaStream_t st) {
    if (!c.tile_proc.p || !ensure(c, c.bwd_order, size_t(Tn))) return;
    tile_order_kernel<<<1, 1024, 0, st ? st : c.stream>>>(c.starts.p, c.tile_proc.p, Tn, c.bwd_order.p, nullptr, 0u, nullptr);
    TS_LAUNCHED(c);
}

int64_t finish_bin_count(Context& c, uint32_t* max_len) {
    if (cudaEventSynchronize(c.bin_ev) != cudaSuccess) return -1;
    for (int k = 0; k < 7; ++k) c.bin_class[k] = c.bin_host[1 + k];
    *max_len = c.bin_host[8];
    return int64_t(c.bin_host[0]);
}

void launch_bin_scatter(Context& c, const DevCam& cam, const ts_render_config& cfg) {
    const int Tn = cam.tiles_x * cam.tiles_y;
    if (c.N == 0) return;  // (may run before this view's I is known on the host)
    const int chunk = bin_chunk_for(c.N, c.sm_count);
    const int nch = int((c.N + chunk - 1) / chunk);
    bin_scatter_kernel<<<nch, kBinThreads, size_t(Tn) * 4, c.stream>>>(c.rect.p, c.splat.p, c.N, cam.w, cam.h,
                                                                       cam.tiles_x, Tn, cfg.cull_mode, c.binH.p,
                                                                       c.starts.p, c.ival[1].p, chunk,
                                                                       uint32_t(std::min<size_t>(c.ival[1].cap, 0xFFFFFFFFu)));
    TS_LAUNCHED(c);
}

// one size class: host mode launches exactly the class's tiles (count known on the host);
// graph mode a resident-size grid that walks the device-side class count (grid-stride)
template <int CAP, int NT, bool SEG = false>
static void sort_variant(Context& c, const uint32_t* tiles, uint32_t n, cudaStream_t st, int cls) {
    if (!c.gmode && !n) return;
    set_func_attr(c, reinterpret_cast<const void*>(tile_sort_kernel<CAP, NT, SEG, false>),
                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(tile_sort_smem(CAP)));
    set_func_attr(c, reinterpret_cast<const void*>(tile_sort_kernel<CAP, NT, SEG, true>),
                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(tile_sort_smem(CAP)));
    const size_t smem = tile_sort_smem(CAP);
    unsigned grid = SEG ? 4 * n : n;
    if (c.gmode) {
        // the class count of the view's last host-path step (+25%, + 8) as the grid: one unit per
        // CTA as on the host path; a class that grew is walked grid-stride
        const unsigned hint = n + n / 4 + 8;
        grid = SEG ? 4 * hint : hint;
    }
    // segments sort in place in the scatter output; whole lists go to the final list buffer
    if (c.gmode)
        tile_sort_kernel<CAP, NT, SEG, true><<<grid, NT, smem, st>>>(c.starts.p, c.ival[1].p, c.dkey[0].p,
                                                                     SEG ? c.ival[1].p : c.ival[0].p, tiles, n,
                                                                     c.bintot.p + c.cur_tn, cls);
    else
        tile_sort_kernel<CAP, NT, SEG, false><<<grid, NT, smem, st>>>(c.starts.p, c.ival[1].p, c.dkey[0].p,
                                                                      SEG ? c.ival[1].p : c.ival[0].p, tiles, n,
                                                                      nullptr, cls);
    TS_LAUNCHED(c);
}

void launch_tile_depth_sort(Context& c, int Tn, uint32_t max_len) {
    (void)max_len;
    if (!c.gmode && c.I == 0) return;
    c.cur_tn = Tn;
    // the size classes are contiguous ranges of the tile order (descending list length), so
    // every class kernel also starts with its longest lists; c.tile_order is built first.
    // Host mode: class offsets from the host-read class counts; graph mode: each kernel
    // derives them from the device-side counts (class_range)
    const uint32_t* ord = c.tile_order.p;
    const uint32_t* meta = c.gmode ? c.bintot.p + Tn : nullptr;
    uint32_t off[7] = {0, 0, 0, 0, 0, 0, 0};
    if (!c.gmode) {
        off[6] = 0;
        off[4] = off[6] + c.bin_class[6];
        off[3] = off[4] + c.bin_class[4];
        off[5] = off[3] + c.bin_class[3];
        off[2] = off[5] + c.bin_class[5];
        off[1] = off[2] + c.bin_class[2];
        off[0] = off[1] + c.bin_class[1];
    }
    if (c.gmode || c.bin_class[0]) {
        const unsigned grid = (c.bin_class[0] + c.bin_class[0] / 4 + 8 + 255) / 256;
        tile_copy_single_kernel<<<grid, 256, 0, c.stream>>>(c.starts.p, c.ival[1].p, c.ival[0].p, ord + off[0],
                                                            c.bin_class[0], meta);
        TS_LAUNCHED(c);
    }
    // the size classes are independent: the two largest run on fork streams so their
    // CTAs share the GPU with the smaller classes instead of queueing behind them
    if (!c.fork_ev) {
        cudaEventCreateWithFlags(&c.fork_ev, cudaEventDisableTiming);
        for (int k = 0; k < 2; ++k) {
            cudaStreamCreateWithFlags(&c.side[k], cudaStreamNonBlocking);
            cudaEventCreateWithFlags(&c.join_ev[k], cudaEventDisableTiming);
        }
    }
    cudaEventRecord(c.fork_ev, c.stream);
    cudaStreamWaitEvent(c.side[0], c.fork_ev, 0);
    cudaStreamWaitEvent(c.side[1], c.fork_ev, 0);
    sort_variant<kCap2, 512>(c, ord + off[3], c.bin_class[3], c.side[0], 3);
    if (c.gmode || c.bin_class[6]) {  // lists longer than kCap3: 4 sorted segments, then 2 merge levels
        const uint32_t* lt = ord + off[6];
        sort_variant<kCap3, 1024, true>(c, lt, c.bin_class[6], c.side[0], 6);
        // c.sortmp holds >= I entries (run_forward sizes it before the fork)
        const dim3 g(kCapL / (kMergeT * kMergePer), c.gmode ? c.bin_class[6] + c.bin_class[6] / 4 + 8 : c.bin_class[6]);
        merge_level_kernel<<<g, kMergeT, 0, c.side[0]>>>(c.starts.p, lt, c.ival[1].p, c.sortmp.p, c.dkey[0].p, kCap3,
                                                        c.bin_class[6], meta);
        merge_level_kernel<<<g, kMergeT, 0, c.side[0]>>>(c.starts.p, lt, c.sortmp.p, c.ival[0].p, c.dkey[0].p,
                                                        2 * kCap3, c.bin_class[6], meta);
        c.launches += 2;
    }
    sort_variant<kCap3, 1024>(c, ord + off[4], c.bin_class[4], c.side[1], 4);
    sort_variant<kCapM, TS_NT_M>(c, ord + off[5], c.bin_class[5], c.side[1], 5);
    sort_variant<kCap1, TS_NT_1>(c, ord + off[2], c.bin_class[2], c.stream, 2);
    sort_variant<kCap0, 256>(c, ord + off[1], c.bin_class[1], c.stream, 1);
    for (int k = 0; k < 2; ++k) {
        cudaEventRecord(c.join_ev[k], c.side[k]);
        cudaStreamWaitEvent(c.stream, c.join_ev[k], 0);
    }
}

}  // namespace ts
