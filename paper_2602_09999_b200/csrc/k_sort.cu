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
    uint32_t v[kScanItems];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t i = base + k;
        uint32_t x = 0;
        if (i < n) x = perm ? __ldg(in + __ldg(perm + i)) : __ldg(in + i);
        v[k] = x;
        sum += x;
    }
    uint32_t agg;
    uint32_t excl = block_excl_scan(sum, s_warp, &agg);
    if (threadIdx.x == 0) {
        volatile unsigned long long* st = state;
        if (tile == 0) {
            st[0] = (2ull << 32) | agg;
            s_prefix = 0;
        } else {
            st[tile] = (1ull << 32) | agg;
            uint32_t prefix = 0;
            int64_t j = int64_t(tile) - 1;
            while (j >= 0) {
                unsigned long long s;
                do {
                    s = st[j];
                } while ((s >> 32) == 0);
                prefix += uint32_t(s);
                if ((s >> 32) == 2) break;
                --j;
            }
            st[tile] = (2ull << 32) | (prefix + agg);
            s_prefix = prefix;
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
// radix pass: histogram + stable rank/scatter (8-bit digit)
// ----------------------------------------------------------------------------
constexpr int kRadixThreads = 256;
constexpr int kRadixItems = 16;
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 4096
constexpr int kWarps = kRadixThreads / 32;

template <class K>
__global__ void __launch_bounds__(kRadixThreads) radix_hist_kernel(const K* __restrict__ keys, int64_t n, int shift,
                                                                   uint32_t* __restrict__ hist, int nblocks) {
    __shared__ uint32_t cnt[kWarps][256];
    const int wid = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarps * 256; i += kRadixThreads) (&cnt[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = int64_t(blockIdx.x) * kRadixTile;
#pragma unroll 4
    for (int k = 0; k < kRadixItems; ++k) {
        const int64_t i = base + int64_t(k) * kRadixThreads + threadIdx.x;
        if (i < n) atomicAdd(&cnt[wid][(uint32_t(keys[i]) >> shift) & 255u], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += kRadixThreads) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += cnt[w][d];
        hist[int64_t(d) * nblocks + blockIdx.x] = s;
    }
}

template <class K>
__global__ void __launch_bounds__(kRadixThreads) radix_scatter_kernel(const K* __restrict__ kin,
                                                                      const uint32_t* __restrict__ vin,
                                                                      K* __restrict__ kout,
                                                                      uint32_t* __restrict__ vout, int64_t n,
                                                                      int shift, const uint32_t* __restrict__ goff,
                                                                      int nblocks) {
    __shared__ uint32_t wcnt[kWarps][256];
    __shared__ uint32_t bstart[256];
    __shared__ uint32_t gstart[256];
    __shared__ uint32_t s_warp[33];
    __shared__ K skey[kRadixTile];
    __shared__ uint32_t sval[kRadixTile];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarps * 256; i += kRadixThreads) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const int64_t wbase = int64_t(blockIdx.x) * kRadixTile + int64_t(wid) * (kRadixItems * 32);
    const uint32_t lt = (1u << lane) - 1u;
    K kk[kRadixItems];
    uint32_t vv[kRadixItems];
    uint32_t dr[kRadixItems];  // digit | rank << 8 ; digit 0x1FF = invalid
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        const bool valid = i < n;
        K key = valid ? kin[i] : K(0);
        uint32_t val = valid ? vin[i] : 0u;
        uint32_t d = valid ? ((uint32_t(key) >> shift) & 255u) : 0x1FFu;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t rank = 0;
        if (valid) {
            const uint32_t pre = wcnt[wid][d];
            rank = pre + __popc(peers & lt);
            __syncwarp(peers);
            if ((peers & lt) == 0) wcnt[wid][d] = pre + __popc(peers);
        }
        __syncwarp();
        kk[r] = key;
        vv[r] = val;
        dr[r] = d | (rank << 9);
    }
    __syncthreads();
    // per digit: exclusive prefix over warps; block totals
    uint32_t tot = 0;
    const int d = threadIdx.x;  // 256 threads == 256 digits
    {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            uint32_t t = wcnt[w][d];
            wcnt[w][d] = run;
            run += t;
        }
        tot = run;
        gstart[d] = goff[int64_t(d) * nblocks + blockIdx.x];
    }
    uint32_t btot;
    const uint32_t bs = block_excl_scan(tot, s_warp, &btot);
    bstart[d] = bs;
    __syncthreads();
    // local stable placement
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
        const uint32_t dd = dr[r] & 0x1FFu;
        if (dd < 256u) {
            const uint32_t lp = bstart[dd] + wcnt[wid][dd] + (dr[r] >> 9);
            skey[lp] = kk[r];
            sval[lp] = vv[r];
        }
    }
    __syncthreads();
    const int64_t tile_n = tmin<int64_t>(kRadixTile, n - int64_t(blockIdx.x) * kRadixTile);
    for (int i = threadIdx.x; i < tile_n; i += kRadixThreads) {
        const K key = skey[i];
        const uint32_t dd = (uint32_t(key) >> shift) & 255u;
        const uint32_t pos = gstart[dd] + (uint32_t(i) - bstart[dd]);
        kout[pos] = key;
        vout[pos] = sval[i];
    }
}

// ----------------------------------------------------------------------------
// K3 duplicate (write pass of build_instances; per depth-sorted Gaussian)
// ----------------------------------------------------------------------------
__global__ void duplicate_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ offsets,
                                 const uint32_t* __restrict__ tcount, const uint2* __restrict__ rect,
                                 const float4* __restrict__ splat, int64_t N, int W, int H, int tiles_x,
                                 int cull_mode, uint16_t* __restrict__ tkey, uint32_t* __restrict__ ival) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= N) return;
    const uint32_t g = perm[j];
    const uint32_t c = tcount[g];
    if (c == 0) return;
    uint32_t o = offsets[j];
    const uint2 rc = rect[g];
    const int tx0 = rc.x & 0xFFFF, tx1 = rc.x >> 16, ty0 = rc.y & 0xFFFF, ty1 = rc.y >> 16;
    const float4 s0 = splat[3 * g], s1 = splat[3 * g + 1];
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
            if (cull_mode == 0 || tsx::tile_keep(s0.x, s0.y, s1.x, s1.y, s1.z, s0.z, tx, ty, W, H)) {
                tkey[o] = uint16_t(ty * tiles_x + tx);
                ival[o] = g;
                ++o;
            }
        }
}

// ----------------------------------------------------------------------------
// K5 tile ranges: starts[t] = #instances with tile < t ; starts[Tn] = I
// ----------------------------------------------------------------------------
__global__ void ranges_kernel(const uint16_t* __restrict__ tkey, int64_t I, int Tn, uint32_t* __restrict__ starts) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= I) return;
    const int t = tkey[i];
    const int tp = i == 0 ? -1 : int(tkey[i - 1]);
    for (int tt = tp + 1; tt <= t; ++tt) starts[tt] = uint32_t(i);
    if (i == I - 1)
        for (int tt = t + 1; tt <= Tn; ++tt) starts[tt] = uint32_t(I);
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

template <class K>
void radix_pass(Context& c, const K* kin, const uint32_t* vin, K* kout, uint32_t* vout, int64_t n, int shift) {
    if (n == 0) return;
    const int nblocks = int((n + kRadixTile - 1) / kRadixTile);
    const size_t hn = size_t(nblocks) * 256;
    ensure(c, c.rhist, 2 * hn + 1);
    uint32_t* hist = c.rhist.p;
    uint32_t* offs = c.rhist.p + hn;
    radix_hist_kernel<K><<<nblocks, kRadixThreads, 0, c.stream>>>(kin, n, shift, hist, nblocks);
    TS_LAUNCHED(c);
    launch_exclusive_scan(c, hist, nullptr, offs, int64_t(hn));
    radix_scatter_kernel<K><<<nblocks, kRadixThreads, 0, c.stream>>>(kin, vin, kout, vout, n, shift, offs, nblocks);
    TS_LAUNCHED(c);
}

template void radix_pass<uint32_t>(Context&, const uint32_t*, const uint32_t*, uint32_t*, uint32_t*, int64_t, int);
template void radix_pass<uint16_t>(Context&, const uint16_t*, const uint32_t*, uint16_t*, uint32_t*, int64_t, int);

void launch_depth_sort(Context& c) {
    // stable LSD over 32-bit depth keys; 4 passes end in buffer 0
    for (int p = 0; p < 4; ++p) {
        const int s = p & 1;
        radix_pass<uint32_t>(c, c.dkey[s].p, c.dperm[s].p, c.dkey[s ^ 1].p, c.dperm[s ^ 1].p, c.N, 8 * p);
    }
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
    duplicate_kernel<<<unsigned((c.N + bs - 1) / bs), bs, 0, c.stream>>>(
        c.dperm[0].p, c.offsets.p, c.tcount.p, c.rect.p, c.splat.p, c.N, cam.w, cam.h, cam.tiles_x,
        cfg.cull_mode, c.tkey[0].p, c.ival[0].p);
    TS_LAUNCHED(c);
}

void launch_tile_sort(Context& c, int tile_bits) {
    const int passes = (tile_bits + 7) / 8;
    for (int p = 0; p < passes; ++p) {
        const int s = p & 1;
        radix_pass<uint16_t>(c, c.tkey[s].p, c.ival[s].p, c.tkey[s ^ 1].p, c.ival[s ^ 1].p, c.I, 8 * p);
    }
    if (passes & 1) {  // keep the sorted list in buffer 0
        std::swap(c.tkey[0], c.tkey[1]);
        std::swap(c.ival[0], c.ival[1]);
    }
}

void launch_ranges(Context& c, int n_tiles) {
    if (c.I == 0) {
        fill_u32_kernel<<<(n_tiles + 256) / 256, 256, 0, c.stream>>>(c.starts.p, n_tiles + 1, 0u);
        TS_LAUNCHED(c);
        return;
    }
    ranges_kernel<<<unsigned((c.I + 255) / 256), 256, 0, c.stream>>>(c.tkey[0].p, c.I, n_tiles, c.starts.p);
    TS_LAUNCHED(c);
}

}  // namespace ts
