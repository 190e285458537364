// Binning kernels (§B.2):
//   K2 exclusive scan (single-pass, decoupled look-back) of per-Gaussian tile
//      counts in depth-sorted order -> instance offsets and I;
//   K3 duplicate: one (tile key u16, gaussian u32) instance per kept tile,
//      re-running the exact-cull test of K1 (bit-identical);
//   K4 two-stage stable LSD radix sort (8-bit digits): depth keys over N
//      Gaussians (4 passes) BEFORE duplication, then tile keys over I instances
//      (ceil(log2 Tn)/8 passes).  Stable over a depth-ordered Gaussian-major
//      list, the result equals the single stable sort on (tile<<32 | depth)
//       while moving 6 B/instance/pass instead of 12;
//   K5 tile ranges by boundary detection (empty tiles get the lower bound).
// All HBM-bound integer work: coalesced loads, block-local stable ranking in
// shared memory, staged (digit-grouped) coalesced scatter.
#include "ts_internal.cuh"
#include "ts_math.cuh"

#include <algorithm>

namespace ts {
namespace {

// ----------------------------------------------------------------------------
// exclusive scan, decoupled look-back
// ----------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// block-wide exclusive scan of one value per thread (blockDim multiple of 32, <= 1024)
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t inc = warp_incl_scan(v);
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < nw ? s_warp[lane] : 0u;
        uint32_t wi = warp_incl_scan(w);
        if (lane < nw) s_warp[lane] = wi - w;
        if (lane == nw - 1) s_warp[32] = wi;
    }
    __syncthreads();
    uint32_t r = inc - v + s_warp[wid];
    *total = s_warp[32];
    return r;
}

// element i of the scanned sequence is in[perm[i]] (or in[i]); its exclusive
// prefix is written to out[i] and the total to out[n].
__global__ void __launch_bounds__(kScanThreads) scan_kernel(const uint32_t* __restrict__ in,
                                                            const uint32_t* __restrict__ perm,
                                                            uint32_t* __restrict__ out, int64_t n,
                                                            unsigned long long* __restrict__ state,
                                                            uint32_t* __restrict__ ticket) {
    __shared__ uint32_t s_warp[33];
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t base = int64_t(tile) * kScanTile + int64_t(threadIdx.x) * kScanItems;
    uint32_t v[kScanItems], pi[kScanItems];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t i = base + k;
        pi[k] = (perm && i < n) ? __ldg(perm + i) : uint32_t(i);
    }
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t i = base + k;
        uint32_t x = 0;
        if (i < n) x = __ldg(in + pi[k]);
        v[k] = x;
        sum += x;
    }
    uint32_t agg;
    uint32_t excl = block_excl_scan(sum, s_warp, &agg);
    // decoupled look-back by warp 0 over a window of 32 predecessors at a time
    if (threadIdx.x < 32) {
        volatile unsigned long long* st = state;
        const int lane = threadIdx.x;
        if (tile == 0) {
            if (lane == 0) st[0] = (2ull << 32) | agg;
            if (lane == 0) s_prefix = 0;
        } else {
            if (lane == 0) st[tile] = (1ull << 32) | agg;
            uint32_t prefix = 0;
            int64_t j0 = int64_t(tile) - 1;  // window: tiles j0, j0-1, ..., j0-31
            while (true) {
                const int64_t j = j0 - lane;
                unsigned long long s = 2ull << 32;  // before tile 0: inclusive prefix 0
                if (j >= 0) {
                    do {
                        s = st[j];
                    } while ((s >> 32) == 0);
                }
                const unsigned pmask = __ballot_sync(0xffffffffu, (s >> 32) == 2);
                const int first = pmask ? __ffs(pmask) - 1 : 32;  // closest inclusive prefix
                uint32_t v = lane <= first ? uint32_t(s) : 0u;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                prefix += v;
                if (pmask) break;
                j0 -= 32;
            }
            if (lane == 0) {
                st[tile] = (2ull << 32) | (prefix + agg);
                s_prefix = prefix;
            }
        }
    }
    __syncthreads();
    uint32_t run = s_prefix + excl;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t i = base + k;
        if (i < n) out[i] = run;
        run += v[k];
    }
    if (int64_t(tile) == (n - 1) / kScanTile && threadIdx.x == kScanThreads - 1) out[n] = s_prefix + agg;
    if (n == 0 && tile == 0 && threadIdx.x == 0) out[0] = 0;
}

// ----------------------------------------------------------------------------
// LSD radix sort, 8-bit digits, stable.  Per pass: per-tile digit counts
// (tile = 2048 keys) -> one exclusive scan over the digit-major count matrix
// -> rank + scatter: each CTA loads its 2048 keys and values up front (16
// independent loads per thread), ranks them stably in shared memory (warp
// match + per-warp digit counters), and writes digit-grouped runs coalesced.
// ----------------------------------------------------------------------------
constexpr int kRT = 256;             // threads per CTA
constexpr int kRI = 8;               // keys per thread
constexpr int kRTile = kRT * kRI;    // 2048 keys per tile
constexpr int kRW = kRT / 32;        // warps

template <class K>
__global__ void __launch_bounds__(kRT) radix_count_kernel(const K* __restrict__ keys, int64_t n, int shift,
                                                          uint32_t* __restrict__ counts, int ntiles) {
    __shared__ uint32_t h[kRW][256];
    const int wid = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kRW * 256; i += kRT) (&h[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = int64_t(blockIdx.x) * kRTile;
    uint32_t d[kRI];
#pragma unroll
    for (int r = 0; r < kRI; ++r) {
        const int64_t i = base + int64_t(r) * kRT + threadIdx.x;
        d[r] = i < n ? uint32_t((uint64_t(keys[i]) >> shift) & 255u) : 0x100u;
    }
#pragma unroll
    for (int r = 0; r < kRI; ++r)
        if (d[r] < 256u) atomicAdd(&h[wid][d[r]], 1u);
    __syncthreads();
    const int dd = threadIdx.x;
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kRW; ++w) s += h[w][dd];
    counts[int64_t(dd) * ntiles + blockIdx.x] = s;
}

template <class K>
__global__ void __launch_bounds__(kRT) radix_scatter_kernel(const K* __restrict__ kin,
                                                           const uint32_t* __restrict__ vin, K* __restrict__ kout,
                                                           uint32_t* __restrict__ vout, int64_t n, int shift,
                                                           const uint32_t* __restrict__ goff, int ntiles) {
    __shared__ uint32_t wcnt[kRW][256];
    __shared__ uint32_t s_bstart[256];
    __shared__ uint32_t s_goff[256];
    __shared__ uint32_t s_warp[33];
    __shared__ K skey[kRTile];
    __shared__ uint32_t sval[kRTile];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t wbase = int64_t(blockIdx.x) * kRTile + int64_t(wid) * (kRI * 32);
    K kk[kRI];
    uint32_t vv[kRI];
#pragma unroll
    for (int r = 0; r < kRI; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        kk[r] = i < n ? kin[i] : K(0);
        vv[r] = i < n ? vin[i] : 0u;
    }
    for (int i = threadIdx.x; i < kRW * 256; i += kRT) (&wcnt[0][0])[i] = 0;
    s_goff[threadIdx.x] = goff[int64_t(threadIdx.x) * ntiles + blockIdx.x];
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    // peers of every round first (independent MATCH ops overlap), then the
    // sequential per-warp digit counters
    uint32_t dig[kRI], peer[kRI];
#pragma unroll
    for (int r = 0; r < kRI; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        dig[r] = i < n ? uint32_t((uint64_t(kk[r]) >> shift) & 255u) : 0x1FFu;
    }
#pragma unroll
    for (int r = 0; r < kRI; ++r) peer[r] = __match_any_sync(0xffffffffu, dig[r]);
    uint32_t dr[kRI];  // digit | (rank within warp) << 9 ; digit 0x1FF = invalid
#pragma unroll
    for (int r = 0; r < kRI; ++r) {
        const uint32_t d = dig[r];
        const bool valid = d < 256u;
        const uint32_t peers = peer[r];
        const uint32_t pre = valid ? wcnt[wid][d] : 0u;
        __syncwarp();
        if (valid && (peers & lt) == 0) wcnt[wid][d] = pre + __popc(peers);
        __syncwarp();
        dr[r] = d | ((pre + __popc(peers & lt)) << 9);
    }
    __syncthreads();
    const int d = threadIdx.x;
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kRW; ++w) {
        const uint32_t t = wcnt[w][d];
        wcnt[w][d] = tot;
        tot += t;
    }
    uint32_t btot;
    s_bstart[d] = block_excl_scan(tot, s_warp, &btot);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRI; ++r) {
        const uint32_t dd = dr[r] & 0x1FFu;
        if (dd < 256u) {
            const uint32_t lp = s_bstart[dd] + wcnt[wid][dd] + (dr[r] >> 9);
            skey[lp] = kk[r];
            sval[lp] = vv[r];
        }
    }
    __syncthreads();
    const int tile_n = int(tmin<int64_t>(kRTile, n - int64_t(blockIdx.x) * kRTile));
#pragma unroll
    for (int r = 0; r < kRI; ++r) {
        const int i = threadIdx.x + r * kRT;
        if (i < tile_n) {
            const K key = skey[i];
            const uint32_t dd = uint32_t((uint64_t(key) >> shift) & 255u);
            const uint32_t pos = s_goff[dd] + (uint32_t(i) - s_bstart[dd]);
            kout[pos] = key;
            vout[pos] = sval[i];
        }
    }
}

// ----------------------------------------------------------------------------
// K3 duplicate (write pass of build_instances; per depth-sorted Gaussian)
// ----------------------------------------------------------------------------
// Iterates depth-sorted positions j (offsets[j] = exclusive prefix of tile
// counts in depth order, so writes are contiguous across a warp); each
// Gaussian's kept tiles come from the 64-bit mask K1 recorded over its tile
// rect (bit = row-major position in the rect), so the exact-cull test is NOT
// re-evaluated; rects of more than 64 tiles (flag bit) re-run it.
template <class K>
__global__ void duplicate_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ offsets,
                                 const uint4* __restrict__ binrec, const float4* __restrict__ splat, int64_t N, int W,
                                 int H, int tiles_x, int cull_mode, K* __restrict__ tkey,
                                 uint32_t* __restrict__ ival) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= N) return;
    const uint32_t g = perm[j];
    const uint4 rc = binrec[g];
    const int tx0 = rc.x & 0xFFFF, tx1 = (rc.x >> 16) & 0x7FFF, ty0 = rc.y & 0xFFFF, ty1 = (rc.y >> 16) & 0x7FFF;
    if (tx0 > tx1 || ty0 > ty1) return;
    uint32_t o = offsets[j];
    if (!(rc.y & 0x80000000u)) {
        const int wdt = tx1 - tx0 + 1;
        uint64_t m = (uint64_t(rc.w) << 32) | rc.z;
        while (m) {
            const int bit = __ffsll((long long)m) - 1;
            m &= m - 1;
            const int ty = ty0 + bit / wdt, tx = tx0 + bit % wdt;
            tkey[o] = K(ty * tiles_x + tx);
            ival[o] = g;
            ++o;
        }
        return;
    }
    const float4 s0 = splat[3 * g], s1 = splat[3 * g + 1];
    const float nBA = tsx::div(-s1.y, s1.x), nBC = tsx::div(-s1.y, s1.z);
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
            if (cull_mode == 0 || tsx::tile_keep(s0.x, s0.y, s1.x, s1.y, s1.z, s0.z, nBA, nBC, tx, ty, W, H)) {
                tkey[o] = K(ty * tiles_x + tx);
                ival[o] = g;
                ++o;
            }
        }
}

// ----------------------------------------------------------------------------
// K5 tile ranges: starts[t] = #instances with tile < t ; starts[Tn] = I
// ----------------------------------------------------------------------------
template <class K>
__global__ void ranges_kernel(const K* __restrict__ tkey, int64_t I, int Tn, uint32_t* __restrict__ starts) {
    // 8 consecutive keys per thread (one or two 16-byte loads when aligned)
    const int64_t i0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
    if (i0 >= I) return;
    K k[8];
    if (i0 + 8 <= I) {
        const uint4* src = reinterpret_cast<const uint4*>(tkey + i0);
#pragma unroll
        for (int q = 0; q < int(sizeof(K)) / 2; ++q) {
            const uint4 v = src[q];
            const K* pv = reinterpret_cast<const K*>(&v);
#pragma unroll
            for (int u = 0; u < 16 / int(sizeof(K)); ++u) k[q * (16 / int(sizeof(K))) + u] = pv[u];
        }
    } else {
        for (int u = 0; u < 8; ++u) k[u] = i0 + u < I ? tkey[i0 + u] : K(0);
    }
    int prev = i0 == 0 ? -1 : int(tkey[i0 - 1]);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int64_t i = i0 + u;
        if (i >= I) break;
        const int t = int(k[u]);
        for (int tt = prev + 1; tt <= t; ++tt) starts[tt] = uint32_t(i);
        prev = t;
        if (i == I - 1)
            for (int tt = t + 1; tt <= Tn; ++tt) starts[tt] = uint32_t(I);
    }
}

__global__ void fill_u32_kernel(uint32_t* p, int64_t n, uint32_t v) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

}  // namespace

void launch_exclusive_scan(Context& c, const uint32_t* in, const uint32_t* perm, uint32_t* out, int64_t n) {
    const int64_t tiles = std::max<int64_t>(1, (n + kScanTile - 1) / kScanTile);
    ensure(c, c.scan_state, size_t(tiles));
    cudaMemsetAsync(c.scan_state.p, 0, size_t(tiles) * sizeof(unsigned long long), c.stream);
    cudaMemsetAsync(c.counters.p, 0, sizeof(uint32_t), c.stream);
    scan_kernel<<<unsigned(tiles), kScanThreads, 0, c.stream>>>(in, perm, out, n, c.scan_state.p, c.counters.p);
    TS_LAUNCHED(c);
}

// Sorts (keys, vals) stably by the low 8*NPASS key bits, ping-ponging between
// buffers 0 and 1 of the given pairs; the result ends in buffer (NPASS & 1).
template <class K, int NPASS>
void radix_sort(Context& c, K* k0, uint32_t* v0, K* k1, uint32_t* v1, int64_t n) {
    if (n == 0) return;
    const int ntiles = int((n + kRTile - 1) / kRTile);
    const size_t hn = size_t(ntiles) * 256;
    ensure(c, c.rhist, 2 * hn + 1);
    uint32_t* counts = c.rhist.p;
    uint32_t* offs = c.rhist.p + hn;
    K* ks[2] = {k0, k1};
    uint32_t* vs[2] = {v0, v1};
    {  // max shared-memory carveout: 8 resident scatter CTAs per SM instead of 4
        const auto carve = cudaFuncAttributePreferredSharedMemoryCarveout;
        set_func_attr(c, reinterpret_cast<const void*>(radix_scatter_kernel<uint32_t>), carve, 100);
        set_func_attr(c, reinterpret_cast<const void*>(radix_scatter_kernel<uint16_t>), carve, 100);
        set_func_attr(c, reinterpret_cast<const void*>(radix_count_kernel<uint32_t>), carve, 100);
        set_func_attr(c, reinterpret_cast<const void*>(radix_count_kernel<uint16_t>), carve, 100);
        set_func_attr(c, reinterpret_cast<const void*>(radix_scatter_kernel<unsigned long long>), carve, 100);
    }
    for (int p = 0; p < NPASS; ++p) {
        const int s = p & 1;
        radix_count_kernel<K><<<ntiles, kRT, 0, c.stream>>>(ks[s], n, 8 * p, counts, ntiles);
        TS_LAUNCHED(c);
        launch_exclusive_scan(c, counts, nullptr, offs, int64_t(hn));
        radix_scatter_kernel<K><<<ntiles, kRT, 0, c.stream>>>(ks[s], vs[s], ks[s ^ 1], vs[s ^ 1], n, 8 * p, offs,
                                                              ntiles);
        TS_LAUNCHED(c);
    }
}

void launch_depth_sort(Context& c) {
    // stable LSD over 32-bit depth keys; 4 passes end in buffer 0
    radix_sort<uint32_t, 4>(c, c.dkey[0].p, c.dperm[0].p, c.dkey[1].p, c.dperm[1].p, c.N);
}

int64_t launch_scan_counts(Context& c) {
    launch_exclusive_scan(c, c.tcount.p, c.dperm[0].p, c.offsets.p, c.N);
    uint32_t I = 0;
    cudaMemcpyAsync(&I, c.offsets.p + c.N, sizeof(uint32_t), cudaMemcpyDeviceToHost, c.stream);
    cudaStreamSynchronize(c.stream);
    return int64_t(I);
}

void launch_duplicate(Context& c, const DevCam& cam, const ts_render_config& cfg) {
    if (c.N == 0 || c.I == 0) return;
    const int bs = 256;
    const unsigned grid = unsigned((c.N + bs - 1) / bs);
    if (cam.tiles_x * cam.tiles_y >= 65536)  // 32-bit tile keys
        duplicate_kernel<uint32_t><<<grid, bs, 0, c.stream>>>(c.dperm[0].p, c.offsets.p, c.rect.p, c.splat.p, c.N,
                                                              cam.w, cam.h, cam.tiles_x, cfg.cull_mode, c.tkey32[0].p,
                                                              c.ival[0].p);
    else
        duplicate_kernel<uint16_t><<<grid, bs, 0, c.stream>>>(c.dperm[0].p, c.offsets.p, c.rect.p, c.splat.p, c.N,
                                                              cam.w, cam.h, cam.tiles_x, cfg.cull_mode, c.tkey[0].p,
                                                              c.ival[0].p);
    TS_LAUNCHED(c);
}

// ----------------------------------------------------------------------------
// morton_reorder: 63-bit Morton codes of the means quantised
// to 21 bits per axis over their bounding box (inflated by 1e-6), x in the least
// significant interleave position; stable LSD sort of (code, index); every
// per-Gaussian array is then gathered through the permutation.
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint64_t spread3(uint32_t v) {
    uint64_t x = v & 0x1FFFFFu;
    x = (x | (x << 32)) & 0x1F00000000FFFFull;
    x = (x | (x << 16)) & 0x1F0000FF0000FFull;
    x = (x | (x << 8)) & 0x100F00F00F00F00Full;
    x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}

__global__ void bbox_kernel(const float* __restrict__ means, int64_t N, float* __restrict__ box /* 6: min xyz, max xyz */) {
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < N; g += int64_t(gridDim.x) * blockDim.x)
        for (int k = 0; k < 3; ++k) {
            const float v = means[3 * g + k];
            lo[k] = fminf(lo[k], v);
            hi[k] = fmaxf(hi[k], v);
        }
    for (int k = 0; k < 3; ++k) {
        for (int o = 16; o > 0; o >>= 1) {
            lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
            hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
        if ((threadIdx.x & 31) == 0) {
            // order-preserving int images of floats for atomic min/max
            const int a = __float_as_int(lo[k]), b = __float_as_int(hi[k]);
            atomicMin(reinterpret_cast<int*>(box) + k, a >= 0 ? a : int(0x80000000u ^ ~uint32_t(a)));
            atomicMax(reinterpret_cast<int*>(box) + 3 + k, b >= 0 ? b : int(0x80000000u ^ ~uint32_t(b)));
        }
    }
}

__device__ __forceinline__ float unmap_ordered(int v) {
    return v >= 0 ? __int_as_float(v) : __int_as_float(int(~(uint32_t(v) ^ 0x80000000u)));
}

__global__ void morton_code_kernel(const float* __restrict__ means, int64_t N, const float* __restrict__ box,
                                   unsigned long long* __restrict__ code, uint32_t* __restrict__ idx) {
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= N) return;
    uint64_t c = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float lo = unmap_ordered(reinterpret_cast<const int*>(box)[k]);
        const float hi = unmap_ordered(reinterpret_cast<const int*>(box)[3 + k]);
        const float span = tsx::add(tsx::sub(hi, lo), 1e-6f);
        const float t = tsx::mul(tsx::div(tsx::sub(means[3 * g + k], lo), span), 2097152.0f);
        uint32_t q = uint32_t(t);
        q = q > 2097151u ? 2097151u : q;
        c |= spread3(q) << k;
    }
    code[g] = c;
    idx[g] = uint32_t(g);
}

template <int W>
__global__ void gather_rows_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                   const uint32_t* __restrict__ perm, int64_t N) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= N * W) return;
    const int64_t r = i / W, k = i - r * W;
    dst[i] = src[int64_t(perm[r]) * W + k];
}

void launch_tile_sort(Context& c, int tile_bits, bool key32) {
    if (key32) {  // >= 2^16 tiles: 32-bit tile keys, ceil(bits / 8) passes (3 up to 2^24 tiles)
        radix_sort<uint32_t, 3>(c, c.tkey32[0].p, c.ival[0].p, c.tkey32[1].p, c.ival[1].p, c.I);
        std::swap(c.tkey32[0], c.tkey32[1]);  // odd pass count: keep the sorted list in buffer 0
        std::swap(c.ival[0], c.ival[1]);
        ++c.gen;
    } else if (tile_bits <= 8) {
        radix_sort<uint16_t, 1>(c, c.tkey[0].p, c.ival[0].p, c.tkey[1].p, c.ival[1].p, c.I);
        std::swap(c.tkey[0], c.tkey[1]);  // keep the sorted list in buffer 0
        std::swap(c.ival[0], c.ival[1]);
        ++c.gen;
    } else {
        radix_sort<uint16_t, 2>(c, c.tkey[0].p, c.ival[0].p, c.tkey[1].p, c.ival[1].p, c.I);
    }
}

void launch_ranges(Context& c, int n_tiles, bool key32) {
    if (c.I == 0) {
        fill_u32_kernel<<<(n_tiles + 256) / 256, 256, 0, c.stream>>>(c.starts.p, n_tiles + 1, 0u);
        TS_LAUNCHED(c);
        return;
    }
    const unsigned grid = unsigned((c.I + 8 * 256 - 1) / (8 * 256));
    if (key32)
        ranges_kernel<uint32_t><<<grid, 256, 0, c.stream>>>(c.tkey32[0].p, c.I, n_tiles, c.starts.p);
    else
        ranges_kernel<uint16_t><<<grid, 256, 0, c.stream>>>(c.tkey[0].p, c.I, n_tiles, c.starts.p);
    TS_LAUNCHED(c);
}

template <int W>
static void gather_group(Context& c, const float* src, float* dst, const uint32_t* perm, int64_t N) {
    const int64_t n = N * W;
    if (n == 0) return;
    gather_rows_kernel<W><<<unsigned((n + 255) / 256), 256, 0, c.stream>>>(src, dst, perm, N);
    TS_LAUNCHED(c);
}

bool launch_morton_reorder(Context& c, uint32_t* perm_host) {
    const int64_t N = c.N;
    if (N == 0) return true;
    // persistent scratch (codes, permutation, a spare 59*N store): no allocation per call
    if (!ensure_grow(c, c.mcode[0], N) || !ensure_grow(c, c.mcode[1], N) || !ensure_grow(c, c.midx[0], N) ||
        !ensure_grow(c, c.midx[1], N) || !ensure_grow(c, c.spare, std::max(c.params.cap, size_t(59) * N + 8)) ||
        !ensure(c, c.dens, size_t(6) * (N + 1)))
        return false;
    float* boxp = reinterpret_cast<float*>(c.dens.p);  // 6 floats of densify scratch
    const int init[6] = {0x7f800000, 0x7f800000, 0x7f800000, int(0x80000000u ^ ~0xff800000u),
                         int(0x80000000u ^ ~0xff800000u), int(0x80000000u ^ ~0xff800000u)};
    cudaMemcpyAsync(boxp, init, sizeof(init), cudaMemcpyHostToDevice, c.stream);
    bbox_kernel<<<c.sm_count * 2, 256, 0, c.stream>>>(c.params.p, N, boxp);
    morton_code_kernel<<<unsigned((N + 255) / 256), 256, 0, c.stream>>>(c.params.p, N, boxp, c.mcode[0].p,
                                                                        c.midx[0].p);
    c.launches += 2;
    radix_sort<unsigned long long, 8>(c, c.mcode[0].p, c.midx[0].p, c.mcode[1].p, c.midx[1].p, N);
    const uint32_t* perm = c.midx[0].p;  // 8 passes: result in buffer 0
    // permute params and both moments (flat 59*N, per attribute block) into the spare store
    // and swap it in; then the statistics and sampling rates through the spare's head
    const Off o(N);
    DevBuf<float>* bufs[3] = {&c.params, &c.m, &c.v};
    for (DevBuf<float>* bp : bufs) {
        if (!ensure_grow(c, c.spare, bp->cap)) return false;
        const float* b = bp->p;
        float* t = c.spare.p;
        gather_group<3>(c, b + o.means, t + o.means, perm, N);
        gather_group<3>(c, b + o.ls, t + o.ls, perm, N);
        gather_group<4>(c, b + o.q, t + o.q, perm, N);
        gather_group<1>(c, b + o.op, t + o.op, perm, N);
        gather_group<3>(c, b + o.dc, t + o.dc, perm, N);
        gather_group<45>(c, b + o.rest, t + o.rest, perm, N);
        std::swap(*bp, c.spare);
        ++c.gen;
    }
    float* tmp = c.spare.p;
    gather_group<1>(c, c.accum.p, tmp, perm, N);
    cudaMemcpyAsync(c.accum.p, tmp, size_t(N) * 4, cudaMemcpyDeviceToDevice, c.stream);
    gather_group<1>(c, c.vcount.p, tmp, perm, N);
    cudaMemcpyAsync(c.vcount.p, tmp, size_t(N) * 4, cudaMemcpyDeviceToDevice, c.stream);
    // sampling rates follow their rows
    if (c.nu_valid) {
        gather_group<1>(c, c.nu_hat.p, tmp, perm, N);
        cudaMemcpyAsync(c.nu_hat.p, tmp, size_t(N) * 4, cudaMemcpyDeviceToDevice, c.stream);
    }
    if (perm_host) cudaMemcpyAsync(perm_host, perm, size_t(N) * 4, cudaMemcpyDeviceToHost, c.stream);
    return cudaStreamSynchronize(c.stream) == cudaSuccess;
}

}  // namespace ts
