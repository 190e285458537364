// K6 blend_fwd and K8 blend_bwd: one CTA of two warps per 16x16 tile, each thread a 1x4 pixel
// column; the two warps (8 rows each) run independently.
//
// Forward (fragment_alpha SPEC.md:316-324, blend_tile :326-334): each warp stages the tile's
// depth-ordered instance list 128 entries at a time into its own shared batch, keeping only the
// splats whose keep ellipse reaches its 8 rows (compacted in list order, 48 B rows gathered by
// Gaussian index); each thread blends its 4 pixels front to back, "blend then stop" at
// T < 1e-4, and the warp leaves as soon as its 128 pixels are done.  The keep decision Q <= k2
// uses the exact-op quadratic form (bit-identical to the oracle); alpha uses MUFU.EX2.
//
// Backward (backward_per_pixel SPEC.md:382-390): front-to-back replay of each pixel up to its
// contributor count, dL/dalpha from the colour still to come (g . U, kept as one scalar) and
// rcp.approx(1 - alpha).  Per fragment a thread sums its 4 pixels' 9 partial
// gradients and parks them in shared memory; every kRF = 3 worked fragments 27 lanes each sum one
// (fragment, value) row of 32 lane partials (16-byte reads) and send it to the per-Gaussian
// 2D-gradient accumulator (scalar REDs) -- ~22 instead of ~60 instructions per worked fragment for
// the transposed shuffle reduction (red9, TS_BWD_SMEMRED=0).  Staging as in the forward (per warp,
// row-culled, up to the warp's last contributor).
#include "ts_internal.cuh"
#include "ts_math.cuh"

namespace ts {
namespace {

constexpr int kT = 64;       // threads per tile CTA (2 warps)
#ifndef TS_BWD_SMEMRED
#define TS_BWD_SMEMRED 1
#endif
#ifndef TS_BWD_RF
#define TS_BWD_RF 3
#endif
constexpr int kRF = TS_BWD_RF;  // K8: worked fragments per deferred-reduction flush (<= 9)
static_assert(kRF >= 1 && kRF <= 9, "flush sums 9 kRF rows, sid / 9 via (sid * 57) >> 9");
constexpr int kRS = 36;      // K8: shared row stride (floats) of the 32 lane partials of one (fragment, value)
constexpr int kPPT = 4;      // pixels per thread (a 1x4 column)
constexpr int kBatch = 128;  // splats staged per round
constexpr float kNegHalfLog2e = -0.72134752044448170368f;  // -0.5 * log2(e)

// the per-warp row cull uses each splat's conservative half-height ry (tsx::ellipse_ry,
// computed once per Gaussian by K1 into c.ryv)
// pixel rows of thread `tid` in a 16x16 tile: warp w owns rows [8w, 8w+8),
// lanes 0-15 rows 8w..8w+3, lanes 16-31 rows 8w+4..8w+7; column = tid % 16.
__device__ __forceinline__ int tile_row0(int tid) { return (tid >> 5) * 8 + ((tid >> 4) & 1) * 4; }

// resident-CTA minimums that cap the registers at 72 (K6: 14 CTAs = 28 warps per SM) and 96 (K8: 10
// CTAs, with 20 KB of shared memory each): K6 0.239 -> 0.217 ms (with the per-warp staging below)
// against 78 uncapped registers, 15-16 CTAs slower again (0.237 ms); K8 (deferred reduction) 0.387 /
// 0.378 / 0.377 ms at 12 / 11 / 10 CTAs
#ifndef TS_FWD_JU
#define TS_FWD_JU 4  // unroll of K6's fragment loop (0: the compiler's choice; 1: +7 us, 2: +0, 4: -2.5 us)
#endif
constexpr int kFwdJU = TS_FWD_JU > 0 ? TS_FWD_JU : 1;
#ifndef TS_BWD_JU
#define TS_BWD_JU 2  // unroll of K8's fragment loop (0: the compiler's choice; 1: +0, 2: -3 us)
#endif
constexpr int kBwdJU = TS_BWD_JU > 0 ? TS_BWD_JU : 1;
#ifndef TS_FWD_CHK
#define TS_FWD_CHK 128  // = kBatch: once per staged batch (16: 0.1985, 32: 0.198, 128: 0.196 ms)
#endif
constexpr int kFwdChk = TS_FWD_CHK;
#ifndef TS_FWD_MINB
#define TS_FWD_MINB 12  // 12: 0.1944, 14: 0.1961, 16: 0.2089 ms (after the per-batch saturation test)
#endif
#ifndef TS_BWD_MINB
#define TS_BWD_MINB 10
#endif
// kCkpt (per-Gaussian backward): the blend state (T, C) of each pixel before list
// positions 32, 64, ... (BlendCheckpoint) goes to ckpt[(starts[t] / 32 + t + k) * 256
// + pixel], written when the warp first reaches a position at or past the boundary (its pixels' state
// cannot change over entries it skips)
template <bool kCompat, bool kCkpt>
__global__ void __launch_bounds__(kT, TS_FWD_MINB) blend_fwd_kernel(const uint32_t* __restrict__ starts,
                                                      const uint32_t* __restrict__ ival,
                                                      const float4* __restrict__ splat, DevCam cam,
                                                      ts_render_config cfg, float* __restrict__ rgb,
                                                      float* __restrict__ Tfin, uint32_t* __restrict__ pcount,
                                                      uint32_t* __restrict__ ip_counter,
                                                      const uint32_t* __restrict__ order,
                                                      uint32_t* __restrict__ tile_proc,
                                                      const float* __restrict__ ryv, float4* __restrict__ ckpt,
                                                      float4* __restrict__ gz, uint32_t nz) {
    // per-warp staged batches: only the splats whose keep ellipse reaches the warp's 8 rows,
    // compacted in list order (the warps of a tile run independently: no CTA barrier in the loop)
    __shared__ float4 sA[2][kBatch];  // mx, my, k2, o
    __shared__ float4 sB[2][kBatch];  // A, 2B, C, -
    __shared__ float4 sC[2][kBatch];  // r, g, b, list position + 1 (uint bits)
    __shared__ uint32_t s_max;
    const int t = order ? int(order[blockIdx.x]) : int(blockIdx.x);
    const int tx = t % cam.tiles_x, ty = t / cam.tiles_x;
    const int px = tx * 16 + (threadIdx.x & 15);
    const int py0 = ty * 16 + tile_row0(threadIdx.x);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float wy0 = float(ty * 16 + warp * 8), wy1 = wy0 + 7.f;
    const uint32_t b = starts[t], e = starts[t + 1];
    const float fpx = float(px);
    // per-pixel state as pixel pairs (rows py0+2h, py0+2h+1) for the packed ops
    float2 Tp[2], C0p[2], C1p[2], C2p[2];
    const float2 pyp[2] = {make_float2(float(py0), float(py0 + 1)), make_float2(float(py0 + 2), float(py0 + 3))};
    uint32_t last[kPPT];
    uint32_t done = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        Tp[h] = make_float2(1.f, 1.f);
        C0p[h] = C1p[h] = C2p[h] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < kPPT; ++k) {
        last[k] = 0;
        if (px >= cam.w || py0 + k >= cam.h) {
            done |= 1u << k;
            if (!kCompat) {  // fast path: a pixel is live while T >= 1e-4 (outside the image: never)
                if (k & 1) Tp[k >> 1].y = 0.f;
                else Tp[k >> 1].x = 0.f;
            }
        }
    }
    // scalar views of the pair state (constant k after unrolling: stays in registers)
#define T(k) (((k) & 1) ? Tp[(k) >> 1].y : Tp[(k) >> 1].x)
#define C0(k) (((k) & 1) ? C0p[(k) >> 1].y : C0p[(k) >> 1].x)
#define C1(k) (((k) & 1) ? C1p[(k) >> 1].y : C1p[(k) >> 1].x)
#define C2(k) (((k) & 1) ? C2p[(k) >> 1].y : C2p[(k) >> 1].x)
    // "blend then stop": the fast path keeps no done mask, a pixel with T < 1e-4 is simply never
    // kept again (T only decreases); the compat path ("stop before blending") keeps the mask
    auto all_done = [&]() -> bool {
        if (kCompat) return done == 0xFu;
        return fmaxf(fmaxf(Tp[0].x, Tp[0].y), fmaxf(Tp[1].x, Tp[1].y)) < 1e-4f;
    };
    uint32_t ckb = 1;  // next checkpoint boundary (kCkpt)
    if (threadIdx.x == 0) s_max = 0;
    for (uint32_t base = b; base < e; base += kBatch) {
        __syncwarp();  // every lane is done reading the previous batch
        if (__all_sync(0xffffffffu, all_done())) break;
        int n = 0;
#pragma unroll
        for (int u = 0; u < kBatch / 32; ++u) {
            const uint32_t i = base + uint32_t(lane + 32 * u);
            float4 s0, s1, s2;
            bool hit = false;
            if (i < e) {
                const uint32_t g = __ldg(ival + i);
                s0 = __ldg(splat + 3 * g);
                s1 = __ldg(splat + 3 * g + 1);
                s2 = __ldg(splat + 3 * g + 2);
                const float ry = __ldg(ryv + g);
                hit = !(s0.y + ry < wy0 || s0.y - ry > wy1);  // keep ellipse reaches this warp's rows
            }
            const uint32_t m = __ballot_sync(0xffffffffu, hit);
            if (hit) {
                const int pos = n + __popc(m & ((1u << lane) - 1u));
                sA[warp][pos] = s0;
                sB[warp][pos] = make_float4(s1.x, tsx::add(s1.y, s1.y), s1.z, 0.f);
                sC[warp][pos] = make_float4(s2.x, s2.y, s2.z, __uint_as_float(i - b + 1u));
            }
            n += __popc(m);
        }
        __syncwarp();
        // the fast path tests for saturation once per kFwdChk entries (a lane leaving the loop
        // early saves issue slots only once its whole warp has left; a saturated pixel keeps
        // nothing, so the test placement does not change results)
        constexpr int kChk = kCompat ? 1 : kFwdChk;
        for (int j0 = 0; j0 < n; j0 += kChk) {
            if (all_done()) break;
            const int j1 = min(n, j0 + kChk);
#if TS_FWD_JU > 0
#pragma unroll kFwdJU
#endif
            for (int j = j0; j < j1; ++j) {
                const float4 q = sB[warp][j];
                const float4 a = sA[warp][j];
                const float dx = tsx::sub(fpx, a.x);
                const float bdx = tsx::mul(q.y, dx), adxdx = tsx::mul(tsx::mul(q.x, dx), dx);
                const float4 col = sC[warp][j];
                // keep decisions of the 4 pixels first (exact Q, branch-free), heavy path only if any is set
                float2 Qp[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    // Q = fma(dy, fma(C, dy, 2B*dx), (A*dx)*dx) (tsx::conic_q), two rows per op
                    const float2 dy = tsx::sub2(pyp[h], tsx::dup2(a.y));
                    Qp[h] = tsx::fma2(dy, tsx::fma2(tsx::dup2(q.z), dy, tsx::dup2(bdx)), tsx::dup2(adxdx));
                }
                const uint32_t idx1 = __float_as_uint(col.w);
                if constexpr (kCkpt) {
                    while (32u * ckb < idx1) {  // entry idx1 - 1 is at or past boundary ckb
                        float4* dst = ckpt + size_t(b / 32u + uint32_t(t) + ckb) * 256u;
                        const int pr = tile_row0(threadIdx.x), pc = threadIdx.x & 15;
#pragma unroll
                        for (int k = 0; k < kPPT; ++k) dst[(pr + k) * 16 + pc] = make_float4(T(k), C0(k), C1(k), C2(k));
                        ++ckb;
                    }
                }
                if constexpr (kCompat) {
                    uint32_t km = 0;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        km |= (Qp[h].x <= a.z) ? (1u << (2 * h)) : 0u;
                        km |= (Qp[h].y <= a.z) ? (2u << (2 * h)) : 0u;
                    }
                    km &= ~done;
                    if (!km) continue;
#pragma unroll
                    for (int k = 0; k < kPPT; ++k) {
                        if (!(km & (1u << k))) continue;
                        const float Qk = (k & 1) ? Qp[k >> 1].y : Qp[k >> 1].x;
                        const float G = tsx::ex2_approx(Qk * kNegHalfLog2e);
                        const float al = fminf(0.99f, a.w * G);
                        const float om = 1.f - al;
                        if (T(k) * om < 1e-4f) {
                            done |= 1u << k;
                            continue;
                        }
                        const float w = al * T(k);
                        C0(k) = fmaf(w, col.x, C0(k));
                        C1(k) = fmaf(w, col.y, C1(k));
                        C2(k) = fmaf(w, col.z, C2(k));
                        T(k) = T(k) * om;
                        last[k] = idx1;
                    }
                    if (done == 0xFu) break;
                } else {
                    bool kp[kPPT];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        kp[2 * h] = Qp[h].x <= a.z && Tp[h].x >= 1e-4f;
                        kp[2 * h + 1] = Qp[h].y <= a.z && Tp[h].y >= 1e-4f;
                    }
                    if (!(kp[0] | kp[1] | kp[2] | kp[3])) continue;
                    // branch-free over the 4 pixels, two pixel pairs in packed fp32x2 ops
                    // (per lane the same IEEE ops as the scalar form): a dropped pixel
                    // blends alpha 0, which leaves C and T bit-identical (fma(0, c, C) = C, T * 1 = T)
                    const float2 cx = tsx::dup2(col.x), cy = tsx::dup2(col.y), cz = tsx::dup2(col.z);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const bool k0 = kp[2 * h], k1 = kp[2 * h + 1];
                        const float2 e = tsx::mul2(Qp[h], tsx::dup2(kNegHalfLog2e));
                        const float2 G = make_float2(tsx::ex2_approx(e.x), tsx::ex2_approx(e.y));
                        const float2 og = tsx::mul2(tsx::dup2(a.w), G);
                        const float2 al = make_float2(k0 ? fminf(0.99f, og.x) : 0.f, k1 ? fminf(0.99f, og.y) : 0.f);
                        const float2 w = tsx::mul2(al, Tp[h]);
                        C0p[h] = tsx::fma2(w, cx, C0p[h]);
                        C1p[h] = tsx::fma2(w, cy, C1p[h]);
                        C2p[h] = tsx::fma2(w, cz, C2p[h]);
                        Tp[h] = tsx::mul2(Tp[h], tsx::sub2(tsx::dup2(1.f), al));
                        last[2 * h] = k0 ? idx1 : last[2 * h];
                        last[2 * h + 1] = k1 ? idx1 : last[2 * h + 1];
                    }
                }
            }
        }
    }
    const int P = cam.w * cam.h;
    uint32_t mymax = 0;
#pragma unroll
    for (int k = 0; k < kPPT; ++k) {
        const int py = py0 + k;
        if (px < cam.w && py < cam.h) {
            const int p = py * cam.w + px;
            rgb[p] = C0(k) + T(k) * cfg.bg[0];
            rgb[P + p] = C1(k) + T(k) * cfg.bg[1];
            rgb[2 * P + p] = C2(k) + T(k) * cfg.bg[2];
            Tfin[p] = T(k);
            pcount[p] = last[k];
        }
        mymax = max(mymax, last[k]);
    }
    // processed list length of this tile (bench counter Ip)
    const uint32_t wm = __reduce_max_sync(0xffffffffu, mymax);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicMax(&s_max, wm);
    __syncthreads();
    if (threadIdx.x == 0 && s_max) atomicAdd(ip_counter, s_max);
    if (threadIdx.x == 0 && tile_proc) tile_proc[t] = s_max;
    // clear the per-Gaussian 2D-gradient accumulator for this view's backward (grid-stride, 16-byte
    // stores): this issue-bound kernel leaves the DRAM idle, the HBM-bound K9 used to do it
    for (uint32_t i = blockIdx.x * kT + threadIdx.x; i < nz; i += gridDim.x * kT) gz[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}
#undef T
#undef C0
#undef C1
#undef C2

// Transposed warp reduction of 9 values: after 5 xor-shuffle steps each even
// lane holds the warp sum of value `slot` (9 distinct slots over the warp).
struct Red9 {
    int slot;  // -1 if this lane holds no slot
};

__device__ __forceinline__ int red9_slot(int lane) {
    const int hi = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1, b1 = (lane >> 1) & 1;
    if (lane & 1) return -1;
    const int xi = b1;
    const int wi = (b2 ? 2 : 0) + xi;
    if (wi > 2) return -1;
    const int ui = (b3 ? 3 : 0) + wi;
    if (ui > 4) return -1;
    const int slot = (hi ? 5 : 0) + ui;
    return slot > 8 ? -1 : slot;
}

__device__ __forceinline__ float red9(const float (&v)[9], int lane) {
    const bool hi = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
    float u[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const float lo_v = v[k];
        const float hi_v = (k + 5 < 9) ? v[k + 5] : 0.f;
        const float keep = hi ? hi_v : lo_v, send = hi ? lo_v : hi_v;
        u[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float w[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float lo_v = u[k];
        const float hi_v = (k + 3 < 5) ? u[k + 3] : 0.f;
        const float keep = b3 ? hi_v : lo_v, send = b3 ? lo_v : hi_v;
        w[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    float x[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float lo_v = w[k];
        const float hi_v = (k + 2 < 3) ? w[k + 2] : 0.f;
        const float keep = b2 ? hi_v : lo_v, send = b2 ? lo_v : hi_v;
        x[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    float y;
    {
        const float keep = b1 ? x[1] : x[0], send = b1 ? x[0] : x[1];
        y = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    y += __shfl_xor_sync(0xffffffffu, y, 1);
    return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// The two warps of a tile run independently: each stages only the splats whose keep ellipse
// reaches its 8 rows (compacted in list order, up to the warp's last contributor), reduces every
// fragment over its 128 pixels and sends the 9 sums straight to the accumulator (one scalar RED
// per slot lane): no shared partial rows, no merge pass and no CTA barrier (round 1 merged the
// two warps' partials in shared memory and sent one vector RED set per (Gaussian, tile):
// 0.436 vs 0.420 ms at H).
__global__ void __launch_bounds__(kT, TS_BWD_MINB) blend_bwd_kernel(const uint32_t* __restrict__ starts,
                                                      const uint32_t* __restrict__ ival,
                                                      const float4* __restrict__ splat, DevCam cam,
                                                      const float* __restrict__ rgb, const uint32_t* __restrict__ pcount,
                                                      const float* __restrict__ dLdC, float4* __restrict__ g2d,
                                                      const uint32_t* __restrict__ order,
                                                      const float* __restrict__ ryv) {
    __shared__ float4 sA[2][kBatch];  // mx, my, k2, o
    __shared__ float4 sB[2][kBatch];  // A, 2B, C, Gaussian index (uint bits)
    __shared__ float4 sC[2][kBatch];  // r, g, b, list position (uint bits)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = order ? int(order[blockIdx.x]) : int(blockIdx.x);
    const int tx = t % cam.tiles_x, ty = t / cam.tiles_x;
    const int px = tx * 16 + (threadIdx.x & 15);
    const int py0 = ty * 16 + tile_row0(threadIdx.x);
    const float wy0 = float(ty * 16 + warp * 8), wy1 = wy0 + 7.f;
    const int P = cam.w * cam.h;
    const float fpx = float(px);
    float2 g0p[2], g1p[2], g2p[2], gUp[2], Tp[2];
    const float2 pyp[2] = {make_float2(float(py0), float(py0 + 1)), make_float2(float(py0 + 2), float(py0 + 3))};
    uint32_t cnt[kPPT];
    uint32_t mymax = 0;
#pragma unroll
    for (int k = 0; k < kPPT; ++k) {
        const int py = py0 + k;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, u = 0.f;
        cnt[k] = 0;
        if (px < cam.w && py < cam.h) {
            const int p = py * cam.w + px;
            a0 = dLdC[p];
            a1 = dLdC[P + p];
            a2 = dLdC[2 * P + p];
            u = a0 * rgb[p] + a1 * rgb[P + p] + a2 * rgb[2 * P + p];
            cnt[k] = pcount[p];
        }
        if (k & 1) {
            g0p[k >> 1].y = a0, g1p[k >> 1].y = a1, g2p[k >> 1].y = a2, gUp[k >> 1].y = u, Tp[k >> 1].y = 1.f;
        } else {
            g0p[k >> 1].x = a0, g1p[k >> 1].x = a1, g2p[k >> 1].x = a2, gUp[k >> 1].x = u, Tp[k >> 1].x = 1.f;
        }
        mymax = max(mymax, cnt[k]);
    }
    const uint32_t wm = __reduce_max_sync(0xffffffffu, mymax);
    const uint32_t b = starts[t];
    const uint32_t e = min(starts[t + 1], b + wm);
    float* const gacc = reinterpret_cast<float*>(g2d);
#if TS_BWD_SMEMRED
    // deferred reduction: the 9 lane partials of kRF worked fragments are parked in shared memory
    // (row (fragment, value) of 32 lanes, stride kRS: conflict-free 16-byte reads) and summed by
    // 9 kRF lanes at once, each reading its row and sending one RED
    __shared__ __align__(16) float sR[2][kRF * 9 * kRS];
    __shared__ uint32_t sRg[2][kRF];
    int nbuf = 0;
    auto flush = [&]() {
        __syncwarp();
        for (int sid = lane; sid < 9 * nbuf; sid += 32) {
            const float4* row = reinterpret_cast<const float4*>(&sR[warp][sid * kRS]);
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4) {
                const float4 x = row[q4];
                acc = tsx::add2(acc, make_float2(x.x, x.y));
                acc = tsx::add2(acc, make_float2(x.z, x.w));
            }
            const float r = acc.x + acc.y;
            const int f = (sid * 57) >> 9;  // sid / 9 (exact for sid < 81)
            if (r != 0.f) atomicAdd(gacc + 12 * size_t(sRg[warp][f]) + (sid - 9 * f), r);
        }
        __syncwarp();
        nbuf = 0;
    };
#else
    const int slot = red9_slot(lane);
#endif
    for (uint32_t base = b; base < e; base += kBatch) {
        __syncwarp();  // every lane is done reading the previous batch
        int n = 0;
#pragma unroll
        for (int u = 0; u < kBatch / 32; ++u) {
            const uint32_t i = base + uint32_t(lane + 32 * u);
            float4 s0, s1, s2;
            uint32_t g = 0;
            bool hit = false;
            if (i < e) {
                g = __ldg(ival + i);
                s0 = __ldg(splat + 3 * g);
                s1 = __ldg(splat + 3 * g + 1);
                s2 = __ldg(splat + 3 * g + 2);
                const float ry = __ldg(ryv + g);
                hit = !(s0.y + ry < wy0 || s0.y - ry > wy1);
            }
            const uint32_t m = __ballot_sync(0xffffffffu, hit);
            if (hit) {
                const int pos = n + __popc(m & ((1u << lane) - 1u));
                sA[warp][pos] = s0;
                sB[warp][pos] = make_float4(s1.x, tsx::add(s1.y, s1.y), s1.z, __uint_as_float(g));
                sC[warp][pos] = make_float4(s2.x, s2.y, s2.z, __uint_as_float(i - b));
            }
            n += __popc(m);
        }
        __syncwarp();
#if TS_BWD_JU > 0
#pragma unroll kBwdJU
#endif
        for (int j = 0; j < n; ++j) {
            const float4 q = sB[warp][j];
            const float4 a = sA[warp][j];
            const float dx = tsx::sub(fpx, a.x);
            const float adx = tsx::mul(q.x, dx);
            const float bdx = tsx::mul(q.y, dx), adxdx = tsx::mul(adx, dx);
            const float4 colw = sC[warp][j];
            const uint32_t li = __float_as_uint(colw.w);
            float2 Qp[2], dyp[2];
            uint32_t km = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                dyp[h] = tsx::sub2(pyp[h], tsx::dup2(a.y));
                Qp[h] = tsx::fma2(dyp[h], tsx::fma2(tsx::dup2(q.z), dyp[h], tsx::dup2(bdx)), tsx::dup2(adxdx));
                km |= (li < cnt[2 * h] && Qp[h].x <= a.z) ? (1u << (2 * h)) : 0u;
                km |= (li < cnt[2 * h + 1] && Qp[h].y <= a.z) ? (2u << (2 * h)) : 0u;
            }
            if (!__any_sync(0xffffffffu, km)) continue;
            const float4 col = colw;
            const float hoa = 0.5f * a.w;
            const float2 ncx = tsx::dup2(-col.x), ncy = tsx::dup2(-col.y), ncz = tsx::dup2(-col.z);
            // per-thread sums over its pixels (pairs, folded at the end): colour / opacity
            // grads and the three moments of dL/dQ that give the mean2d and conic grads
            // (dx is shared).  Branch-free: a dropped pixel has alpha 0 (w = 0, T and g.U
            // unchanged) and a zero dL/dalpha mask.  ng* = negated quantities (ngc = -g.c,
            // ndal = -dL/dalpha) so every update is one FFMA2.
            float2 vr2, vg2, vb2, nvo2, sq2, sqy2, sqyy2;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const bool k0 = km & (1u << (2 * h)), k1 = km & (2u << (2 * h));
                const float2 e = tsx::mul2(Qp[h], tsx::dup2(kNegHalfLog2e));
                // G of a dropped pixel is 0: alpha, w, the opacity and conic terms vanish with it
                const float2 G = make_float2(k0 ? tsx::ex2_approx(e.x) : 0.f, k1 ? tsx::ex2_approx(e.y) : 0.f);
                const float2 og = tsx::mul2(tsx::dup2(a.w), G);
                const float2 al = make_float2(fminf(og.x, 0.99f), fminf(og.y, 0.99f));
                // alpha not clamped: gradient flows through G (SPEC.md clamp rule, App. A.8)
                const float2 Gl = make_float2(og.x <= 0.99f ? G.x : 0.f, og.y <= 0.99f ? G.y : 0.f);
                const float2 w = tsx::mul2(al, Tp[h]);
                const float2 om = tsx::sub2(tsx::dup2(1.f), al);
                const float2 ngc = tsx::fma2(g2p[h], ncz, tsx::fma2(g1p[h], ncy, tsx::mul2(g0p[h], ncx)));
                const float2 after = tsx::fma2(w, ngc, gUp[h]);  // g . (colour after this fragment, incl. bg)
                const float2 r = make_float2(rcp_approx(om.x), rcp_approx(om.y));
                const float2 ndal = tsx::fma2(Tp[h], ngc, tsx::mul2(after, r));
                const float2 nvo = tsx::mul2(Gl, ndal);              // -dL/do contribution
                const float2 dQ = tsx::mul2(nvo, tsx::dup2(hoa));  // dL/dQ = -0.5 o G dL/dalpha
                const float2 dQy = tsx::mul2(dQ, dyp[h]);
                if (h == 0) {
                    vr2 = tsx::mul2(w, g0p[h]);
                    vg2 = tsx::mul2(w, g1p[h]);
                    vb2 = tsx::mul2(w, g2p[h]);
                    nvo2 = nvo;
                    sq2 = dQ;
                    sqy2 = dQy;
                    sqyy2 = tsx::mul2(dQy, dyp[h]);
                } else {
                    vr2 = tsx::fma2(w, g0p[h], vr2);
                    vg2 = tsx::fma2(w, g1p[h], vg2);
                    vb2 = tsx::fma2(w, g2p[h], vb2);
                    nvo2 = tsx::add2(nvo2, nvo);
                    sq2 = tsx::add2(sq2, dQ);
                    sqy2 = tsx::add2(sqy2, dQy);
                    sqyy2 = tsx::fma2(dQy, dyp[h], sqyy2);
                }
                gUp[h] = after;
                Tp[h] = tsx::mul2(Tp[h], om);
            }
            const float vr = vr2.x + vr2.y, vg = vg2.x + vg2.y, vb = vb2.x + vb2.y, vo = -(nvo2.x + nvo2.y);
            const float sq = sq2.x + sq2.y, sqy = sqy2.x + sqy2.y, sqyy = sqyy2.x + sqyy2.y;
            // dQ/dmx = -(2A dx + 2B dy), dQ/dmy = -(2B dx + 2C dy), dQ/dA = dx^2, dQ/dB = 2 dx dy, dQ/dC = dy^2
            float v[9];
            v[0] = -(2.f * adx * sq + q.y * sqy);
            v[1] = -(q.y * dx * sq + 2.f * q.z * sqy);
            v[2] = dx * dx * sq;
            v[3] = 2.f * dx * sqy;
            v[4] = sqyy;
            v[5] = vo;
            v[6] = vr;
            v[7] = vg;
            v[8] = vb;
#if TS_BWD_SMEMRED
#pragma unroll
            for (int k = 0; k < 9; ++k) sR[warp][(nbuf * 9 + k) * kRS + lane] = v[k];
            if (lane == 0) sRg[warp][nbuf] = __float_as_uint(q.w);
            if (++nbuf == kRF) flush();
#else
            const float r = red9(v, lane);
            if (slot >= 0 && r != 0.f) atomicAdd(gacc + 12 * size_t(__float_as_uint(q.w)) + slot, r);
#endif
        }
#if TS_BWD_SMEMRED
        if (nbuf) flush();
#endif
    }
}

// ---------------------------------------------------------------------------
// Per-Gaussian bucket backward (backward_per_gaussian SPEC.md:392-400; option,
// ts_render_config.backward_mode = 1).  A CTA of kGW warps per tile; a warp takes a bucket of 32 list
// entries, one Gaussian per lane.  The tile's per-pixel data (dL/dC, g . C_final, contributor
// count) sit in shared memory; the pixels still active in the bucket (count past its start) form a
// compacted list.  Pixel q flows lane 0 -> 31 (step s, lane i handles pixel s - i): lane 0 restores
// (T, g . U) from the forward's checkpoint at the bucket start, every lane blends its Gaussian into
// the pixel and hands (T, g . U) to the next lane by shuffle; each lane accumulates its Gaussian's
// 9 partial gradients over the tile in registers and sends them with one RED set per bucket.
// Same per-fragment arithmetic as K8 (dL/dalpha from g . U and rcp(1 - alpha)).
// ---------------------------------------------------------------------------
constexpr int kGW = 4;

__global__ void __launch_bounds__(kGW * 32) blend_bwd_gauss_kernel(const uint32_t* __restrict__ starts,
                                                                  const uint32_t* __restrict__ ival,
                                                                  const float4* __restrict__ splat, DevCam cam,
                                                                  const float* __restrict__ rgb,
                                                                  const uint32_t* __restrict__ pcount,
                                                                  const float* __restrict__ dLdC,
                                                                  float4* __restrict__ g2d,
                                                                  const uint32_t* __restrict__ order,
                                                                  const uint32_t* __restrict__ tile_proc,
                                                                  const float4* __restrict__ ckpt) {
    __shared__ float4 sPix[256];  // dL/dC (3), u = g . C_final (incl. background)
    __shared__ uint32_t sCnt[256];
    __shared__ uint8_t sList[kGW][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = order ? int(order[blockIdx.x]) : int(blockIdx.x);
    const int tx = t % cam.tiles_x, ty = t / cam.tiles_x;
    const uint32_t b = starts[t];
    const uint32_t L = min(starts[t + 1] - b, tile_proc[t]);
    if (L == 0) return;
    const int P = cam.w * cam.h;
    for (int pix = threadIdx.x; pix < 256; pix += kGW * 32) {
        const int px = tx * 16 + (pix & 15), py = ty * 16 + (pix >> 4);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        uint32_t cn = 0;
        if (px < cam.w && py < cam.h) {
            const int p = py * cam.w + px;
            v.x = dLdC[p];
            v.y = dLdC[P + p];
            v.z = dLdC[2 * P + p];
            v.w = v.x * rgb[p] + v.y * rgb[P + p] + v.z * rgb[2 * P + p];
            cn = pcount[p];
        }
        sPix[pix] = v;
        sCnt[pix] = cn;
    }
    __syncthreads();
    const uint32_t bbase = b / 32u + uint32_t(t);
    const uint32_t nbk = (L + 31u) / 32u;
    const float fx0 = float(tx * 16), fy0 = float(ty * 16);
    for (uint32_t k = uint32_t(warp); k < nbk; k += kGW) {
        const uint32_t pos = 32u * k + uint32_t(lane);
        const bool has = pos < L;
        float mx = 0.f, my = 0.f, k2 = -1.f, o = 0.f, A = 0.f, B2 = 0.f, C = 0.f, cr = 0.f, cg = 0.f, cb = 0.f;
        uint32_t g = 0;
        if (has) {
            g = __ldg(ival + b + pos);
            const float4 s0 = __ldg(splat + 3 * g), s1 = __ldg(splat + 3 * g + 1), s2 = __ldg(splat + 3 * g + 2);
            mx = s0.x, my = s0.y, k2 = s0.z, o = s0.w;
            A = s1.x, B2 = tsx::add(s1.y, s1.y), C = s1.z;
            cr = s2.x, cg = s2.y, cb = s2.z;
        }
        // pixels with a contributor past the bucket start, compacted
        int npix = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int pix = 32 * r + lane;
            const bool act = sCnt[pix] > 32u * k;
            const uint32_t m = __ballot_sync(0xffffffffu, act);
            if (act) sList[warp][npix + __popc(m & ((1u << lane) - 1u))] = uint8_t(pix);
            npix += __popc(m);
        }
        __syncwarp();
        float a_mx = 0.f, a_my = 0.f, a_A = 0.f, a_B = 0.f, a_C = 0.f, a_o = 0.f, a_r = 0.f, a_g = 0.f, a_b = 0.f;
        float T = 1.f, gU = 0.f;
        const float4* ck = ckpt + size_t(bbase + k) * 256u;
        const float hoa = 0.5f * o;
        for (int s = 0; s < npix + 31; ++s) {
            float Tin = __shfl_up_sync(0xffffffffu, T, 1);
            float gUin = __shfl_up_sync(0xffffffffu, gU, 1);
            const int q = s - lane;
            if (q >= 0 && q < npix) {
                const int pix = sList[warp][q];
                const float4 pv = sPix[pix];
                if (lane == 0) {
                    if (k == 0) {
                        Tin = 1.f;
                        gUin = pv.w;
                    } else {
                        const float4 c4 = ck[pix];
                        Tin = c4.x;
                        gUin = pv.w - (pv.x * c4.y + pv.y * c4.z + pv.z * c4.w);
                    }
                }
                T = Tin;
                gU = gUin;
                if (has && pos < sCnt[pix]) {
                    const float dx = tsx::sub(fx0 + float(pix & 15), mx), dy = tsx::sub(fy0 + float(pix >> 4), my);
                    const float Q = tsx::conic_q(A, B2, C, dx, dy);
                    if (Q <= k2) {
                        const float G = tsx::ex2_approx(Q * kNegHalfLog2e);
                        const float og = o * G;
                        const float al = fminf(og, 0.99f);
                        const float w = al * T;
                        const float om = 1.f - al;
                        const float ngc = fmaf(pv.z, -cb, fmaf(pv.y, -cg, pv.x * -cr));
                        const float after = fmaf(w, ngc, gU);
                        const float ndal = fmaf(T, ngc, after * rcp_approx(om));
                        const float nvo = (og <= 0.99f ? G : 0.f) * ndal;
                        const float dQ = nvo * hoa;
                        a_mx -= dQ * (2.f * A * dx + B2 * dy);
                        a_my -= dQ * (B2 * dx + 2.f * C * dy);
                        a_A += dQ * dx * dx;
                        a_B += 2.f * dQ * dx * dy;
                        a_C += dQ * dy * dy;
                        a_o -= nvo;
                        a_r += w * pv.x;
                        a_g += w * pv.y;
                        a_b += w * pv.z;
                        T = T * om;
                        gU = after;
                    }
                }
            }
        }
        if (has) {
            atomicAdd(g2d + 3 * g, make_float4(a_mx, a_my, a_A, a_B));
            atomicAdd(g2d + 3 * g + 1, make_float4(a_C, a_o, a_r, a_g));
            atomicAdd(reinterpret_cast<float*>(g2d + 3 * g + 2), a_b);
        }
        __syncwarp();  // sList is rebuilt for the next bucket
    }
}

}  // namespace

void launch_blend_fwd(Context& c, const DevCam& cam, const ts_render_config& cfg) {
    const int Tn = cam.tiles_x * cam.tiles_y;
    ensure(c, c.tile_proc, size_t(Tn));
    const uint32_t* ord = c.order_ok ? c.tile_order.p : nullptr;
    const bool ck = cfg.backward_mode == 1 && !cfg.early_stop_compat && !c.gmode &&
                    ensure_grow(c, c.ckpt, (size_t(c.I) / 32 + size_t(Tn) + 1) * 256);
    c.ckpt_valid = ck;
#define TS_FWD(C, K)                                                                                          \
    blend_fwd_kernel<C, K><<<Tn, kT, 0, c.stream>>>(c.starts.p, c.ival[0].p, c.splat.p, cam, cfg, c.rgb.p, c.Tfin.p, \
                                                    c.pcount.p, c.counters.p + 2, ord, c.tile_proc.p, c.ryv.p,   \
                                                    c.ckpt.p, c.g2d.p, uint32_t(3 * c.N))
    if (cfg.early_stop_compat) TS_FWD(true, false);
    else if (ck) TS_FWD(false, true);
    else TS_FWD(false, false);
#undef TS_FWD
    c.g2d_clean = true;
    TS_LAUNCHED(c);
}

void launch_blend_bwd(Context& c, const DevCam& cam, const ts_render_config& cfg) {
    (void)cfg;
    const int Tn = cam.tiles_x * cam.tiles_y;
    const uint32_t* ord = c.bwd_order_ok ? c.bwd_order.p : (c.order_ok ? c.tile_order.p : nullptr);
    if (cfg.backward_mode == 1 && c.ckpt_valid)
        blend_bwd_gauss_kernel<<<Tn, kGW * 32, 0, c.stream>>>(c.starts.p, c.ival[0].p, c.splat.p, cam, c.rgb.p,
                                                               c.pcount.p, c.dLdC.p, c.g2d.p, ord, c.tile_proc.p,
                                                               c.ckpt.p);
    else
        blend_bwd_kernel<<<Tn, kT, 0, c.stream>>>(c.starts.p, c.ival[0].p, c.splat.p, cam, c.rgb.p, c.pcount.p,
                                                  c.dLdC.p, c.g2d.p, ord, c.ryv.p);
    c.g2d_clean = false;  // K9 consumes it without clearing; the next forward's K6 clears it
    TS_LAUNCHED(c);
}

}  // namespace ts
