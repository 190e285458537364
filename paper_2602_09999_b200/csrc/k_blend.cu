// K6 blend_fwd and K8 blend_bwd: one CTA per 16x16 tile, one thread per pixel.
//
// Forward (fragment_alpha SPEC.md:316-324, blend_tile :326-334): the tile's
// depth-ordered instance list is staged 256 splats at a time into shared memory
// (gathered by Gaussian index, 48 B rows), every pixel blends front to back,
// "blend then stop" at T < 1e-4, and the CTA leaves as soon as all 256 pixels
// are done (__syncthreads_count).  The keep decision Q <= k2 uses the exact-op
// quadratic form (bit-identical to the oracle); alpha uses MUFU.EX2.
//
// Backward (backward_per_pixel SPEC.md:382-390): front-to-back replay with the
// suffix-colour recurrence (no division by (1 - alpha) of T).
// Per fragment, the 32 lanes of a warp (32 pixels) reduce their 9 partial
// gradients with a transposed shuffle reduction (12 SHFL instead of 45), the 8
// warps merge in shared memory, and each (Gaussian, tile) pair issues ONE set of
// vector atomics (RED.F32x4) into the per-Gaussian 2D-gradient accumulator.
#include "ts_internal.cuh"
#include "ts_math.cuh"

namespace ts {
namespace {

constexpr int kT = 256;
constexpr float kNegHalfLog2e = -0.72134752044448170368f;  // -0.5 * log2(e)

__global__ void __launch_bounds__(kT) blend_fwd_kernel(const uint32_t* __restrict__ starts,
                                                      const uint32_t* __restrict__ ival,
                                                      const float4* __restrict__ splat, DevCam cam,
                                                      ts_render_config cfg, float* __restrict__ rgb,
                                                      float* __restrict__ Tfin, uint32_t* __restrict__ pcount,
                                                      uint32_t* __restrict__ ip_counter) {
    __shared__ float4 sA[kT];  // mx, my, k2, o
    __shared__ float4 sB[kT];  // A, 2B, C
    __shared__ float4 sC[kT];  // r, g, b
    __shared__ uint32_t s_max;
    const int t = blockIdx.x;
    const int tx = t % cam.tiles_x, ty = t / cam.tiles_x;
    const int px = tx * 16 + (threadIdx.x & 15), py = ty * 16 + (threadIdx.x >> 4);
    const bool inside = px < cam.w && py < cam.h;
    const uint32_t b = starts[t], e = starts[t + 1];
    const float fpx = float(px), fpy = float(py);
    float T = 1.f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
    uint32_t last = 0;
    bool done = !inside;
    const bool compat = cfg.early_stop_compat != 0;
    if (threadIdx.x == 0) s_max = 0;
    for (uint32_t base = b; base < e; base += kT) {
        if (__syncthreads_count(done) == kT) break;
        const uint32_t i = base + threadIdx.x;
        if (i < e) {
            const uint32_t g = __ldg(ival + i);
            const float4 s0 = __ldg(splat + 3 * g), s1 = __ldg(splat + 3 * g + 1), s2 = __ldg(splat + 3 * g + 2);
            sA[threadIdx.x] = s0;
            sB[threadIdx.x] = make_float4(s1.x, tsx::add(s1.y, s1.y), s1.z, 0.f);
            sC[threadIdx.x] = s2;
        }
        __syncthreads();
        const int n = int(tmin<uint32_t>(kT, e - base));
        if (!done) {
            for (int j = 0; j < n; ++j) {
                const float4 a = sA[j];
                const float4 q = sB[j];
                const float dx = tsx::sub(fpx, a.x), dy = tsx::sub(fpy, a.y);
                const float Q = tsx::conic_q(q.x, q.y, q.z, dx, dy);
                if (!(Q <= a.z)) continue;
                const float G = tsx::ex2_approx(Q * kNegHalfLog2e);
                const float al = fminf(0.99f, a.w * G);
                const float om = 1.f - al;
                if (compat && T * om < 1e-4f) {
                    done = true;
                    break;
                }
                const float w = al * T;
                const float4 col = sC[j];
                C0 = fmaf(w, col.x, C0);
                C1 = fmaf(w, col.y, C1);
                C2 = fmaf(w, col.z, C2);
                T = T * om;
                last = base - b + uint32_t(j) + 1u;
                if (!compat && T < 1e-4f) {
                    done = true;
                    break;
                }
            }
        }
    }
    if (inside) {
        const int P = cam.w * cam.h;
        const int p = py * cam.w + px;
        rgb[p] = C0 + T * cfg.bg[0];
        rgb[P + p] = C1 + T * cfg.bg[1];
        rgb[2 * P + p] = C2 + T * cfg.bg[2];
        Tfin[p] = T;
        pcount[p] = last;
    }
    // processed list length of this tile (bench counter Ip)
    const uint32_t wm = __reduce_max_sync(0xffffffffu, last);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicMax(&s_max, wm);
    __syncthreads();
    if (threadIdx.x == 0 && s_max) atomicAdd(ip_counter, s_max);
}

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

constexpr int kGS = 12;  // smem gradient row stride (floats)

__global__ void __launch_bounds__(kT) blend_bwd_kernel(const uint32_t* __restrict__ starts,
                                                      const uint32_t* __restrict__ ival,
                                                      const float4* __restrict__ splat, DevCam cam,
                                                      const float* __restrict__ rgb, const uint32_t* __restrict__ pcount,
                                                      const float* __restrict__ dLdC, float4* __restrict__ g2d) {
    __shared__ float4 sA[kT];  // mx, my, k2, o
    __shared__ float4 sB[kT];  // A, 2B, C
    __shared__ float4 sC[kT];  // r, g, b
    __shared__ uint32_t sIdx[kT];
    __shared__ float sG[kT * kGS];
    __shared__ uint32_t s_max;
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x;
    const int tx = t % cam.tiles_x, ty = t / cam.tiles_x;
    const int px = tx * 16 + (threadIdx.x & 15), py = ty * 16 + (threadIdx.x >> 4);
    const bool inside = px < cam.w && py < cam.h;
    const int P = cam.w * cam.h;
    const int p = py * cam.w + px;
    float g0 = 0.f, g1 = 0.f, g2 = 0.f, R0 = 0.f, R1 = 0.f, R2 = 0.f;
    uint32_t cnt = 0;
    if (inside) {
        g0 = dLdC[p];
        g1 = dLdC[P + p];
        g2 = dLdC[2 * P + p];
        R0 = rgb[p];
        R1 = rgb[P + p];
        R2 = rgb[2 * P + p];
        cnt = pcount[p];
    }
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    const uint32_t wm = __reduce_max_sync(0xffffffffu, cnt);
    if (lane == 0) atomicMax(&s_max, wm);
    __syncthreads();
    const uint32_t b = starts[t];
    const uint32_t e = min(starts[t + 1], b + s_max);
    const int slot = red9_slot(lane);
    const float fpx = float(px), fpy = float(py);
    float T = 1.f, P0 = 0.f, P1 = 0.f, P2 = 0.f;
    for (uint32_t base = b; base < e; base += kT) {
        const uint32_t i = base + threadIdx.x;
        if (i < e) {
            const uint32_t g = __ldg(ival + i);
            const float4 s0 = __ldg(splat + 3 * g), s1 = __ldg(splat + 3 * g + 1), s2 = __ldg(splat + 3 * g + 2);
            sA[threadIdx.x] = s0;
            sB[threadIdx.x] = make_float4(s1.x, tsx::add(s1.y, s1.y), s1.z, 0.f);
            sC[threadIdx.x] = s2;
            sIdx[threadIdx.x] = g;
        }
#pragma unroll
        for (int k = 0; k < kGS; ++k) sG[threadIdx.x * kGS + k] = 0.f;
        __syncthreads();
        const int n = int(tmin<uint32_t>(kT, e - base));
        const uint32_t local0 = base - b;
        for (int j = 0; j < n; ++j) {
            const float4 a = sA[j];
            const float4 q = sB[j];
            float v[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) v[k] = 0.f;
            bool keep = false;
            float dx = 0.f, dy = 0.f, Q = 0.f;
            if (local0 + uint32_t(j) < cnt) {
                dx = tsx::sub(fpx, a.x);
                dy = tsx::sub(fpy, a.y);
                Q = tsx::conic_q(q.x, q.y, q.z, dx, dy);
                keep = Q <= a.z;
            }
            if (!__any_sync(0xffffffffu, keep)) continue;
            if (keep) {
                const float4 col = sC[j];
                const float G = tsx::ex2_approx(Q * kNegHalfLog2e);
                const float og = a.w * G;
                const bool clamped = og > 0.99f;
                const float al = clamped ? 0.99f : og;
                const float w = al * T;
                const float om = 1.f - al;
                const float iom = __frcp_rn(om);
                v[6] = w * g0;
                v[7] = w * g1;
                v[8] = w * g2;
                const float af0 = R0 - P0 - w * col.x;
                const float af1 = R1 - P1 - w * col.y;
                const float af2 = R2 - P2 - w * col.z;
                const float dal = g0 * (T * col.x - af0 * iom) + g1 * (T * col.y - af1 * iom) +
                                  g2 * (T * col.z - af2 * iom);
                if (!clamped) {
                    v[5] = G * dal;
                    const float dQ = -0.5f * G * a.w * dal;
                    v[0] = dQ * -(2.f * q.x * dx + q.y * dy);
                    v[1] = dQ * -(q.y * dx + 2.f * q.z * dy);
                    v[2] = dQ * dx * dx;
                    v[3] = dQ * 2.f * dx * dy;
                    v[4] = dQ * dy * dy;
                }
                P0 = fmaf(w, col.x, P0);
                P1 = fmaf(w, col.y, P1);
                P2 = fmaf(w, col.z, P2);
                T = T * om;
            }
            const float r = red9(v, lane);
            if (slot >= 0) atomicAdd(&sG[j * kGS + slot], r);
        }
        __syncthreads();
        if (int(threadIdx.x) < n) {
            const float* gs = sG + threadIdx.x * kGS;
            const float4 a0 = make_float4(gs[0], gs[1], gs[2], gs[3]);
            const float4 a1 = make_float4(gs[4], gs[5], gs[6], gs[7]);
            const float a2 = gs[8];
            const bool any = (a0.x != 0.f) | (a0.y != 0.f) | (a0.z != 0.f) | (a0.w != 0.f) | (a1.x != 0.f) |
                             (a1.y != 0.f) | (a1.z != 0.f) | (a1.w != 0.f) | (a2 != 0.f);
            if (any) {
                const uint32_t g = sIdx[threadIdx.x];
                atomicAdd(g2d + 3 * g, a0);
                atomicAdd(g2d + 3 * g + 1, a1);
                atomicAdd(reinterpret_cast<float*>(g2d + 3 * g + 2), a2);
            }
        }
        __syncthreads();
    }
}

}  // namespace

void launch_blend_fwd(Context& c, const DevCam& cam, const ts_render_config& cfg) {
    const int Tn = cam.tiles_x * cam.tiles_y;
    blend_fwd_kernel<<<Tn, kT, 0, c.stream>>>(c.starts.p, c.ival[0].p, c.splat.p, cam, cfg, c.rgb.p, c.Tfin.p,
                                              c.pcount.p, c.counters.p + 2);
    TS_LAUNCHED(c);
}

void launch_blend_bwd(Context& c, const DevCam& cam, const ts_render_config& cfg) {
    (void)cfg;
    const int Tn = cam.tiles_x * cam.tiles_y;
    blend_bwd_kernel<<<Tn, kT, 0, c.stream>>>(c.starts.p, c.ival[0].p, c.splat.p, cam, c.rgb.p, c.pcount.p,
                                              c.dLdC.p, c.g2d.p);
    TS_LAUNCHED(c);
}

}  // namespace ts
