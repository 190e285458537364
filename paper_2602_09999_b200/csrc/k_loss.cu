// K7 training_loss: 0.8 L1 + 0.2 (1 - SSIM) with an 11x11
// Gaussian window (sigma 1.5), C1 = 0.01^2, C2 = 0.03^2, reflect padding, and the
// analytic dL/dC, in one kernel per 32x32 tile and colour channel (see
// loss_fused_kernel).  With  mu = W x,  v = W x^2 - mu_x^2,  cov = W xy - mu_x mu_y:
//   dSSIM/dx_p = (W^T a)_p + x_p (W^T b)_p + y_p (W^T c)_p,
//   a = dS/dmu_x - 2 mu_x dS/dv_x - mu_y dS/dcov,  b = 2 dS/dv_x,  c = dS/dcov,
//   dL/dC = (0.8 sign(x - y) - 0.2 dSSIM/dx) / M.
#include <cmath>
#include <type_traits>

#include "ts_internal.cuh"
#include "ts_math.cuh"

namespace ts {
namespace {

__constant__ float c_gw[11];
__device__ __forceinline__ int refl(int i, int n) { return i < 0 ? -i : (i >= n ? 2 * (n - 1) - i : i); }

// ---------------------------------------------------------------------------
// Fused loss kernel: forward moments, SSIM terms and the transposed filter of the
// backward in ONE kernel per 32x32 output tile and colour channel (no map round
// trip through HBM).  Positions relative to the tile origin (x0, y0):
//   input    52x52  [-10, 42)  reflect-indexed image values
//   moments  42x42  [-5, 37)   five window moments, SSIM and (a, b, c); (a, b, c)
//                               are zero outside the image (zero extension)
//   virtual  47     [-5, 42)   positions of the transposed filter: the reflect
//                               padding of the forward folds -p and 2(W-1)-p back
//                               onto p (per axis; separable)
//   output   32x32  [0, 32)
// The transposed filter is the same symmetric window.  Shared memory (floats):
// A = 5 x 52 x 42 horizontal moments (row stride 43), later hb 3 x 42 x 47;
// B = 3 x 42 x 58 (row stride 59) (input 2 x 52 x 52 (row stride 53), then (a, b, c)
// column-padded to [-10, 48), then vb 3 x 47 x 32).
// ---------------------------------------------------------------------------
constexpr int kFT = 32;                   // output tile edge
constexpr int kFI = kFT + 20;             // input region edge (52)
constexpr int kFM = kFT + 10;             // moment region edge (42)
constexpr int kFV = kFT + 15;             // virtual transposed-filter positions (47)
constexpr int kFP = kFV + 11;             // padded (a, b, c) columns / hf rows (58)
// shared row strides padded to odd word counts: the row-parallel passes (lanes on consecutive
// rows) then hit 32 distinct banks (round 1's even strides: ~40% of the shared wavefronts were
// bank conflicts)
constexpr int kXS = kFI + 1;              // input rows (53)
constexpr int kAS = kFM + 1;              // horizontal-moment rows (43)
constexpr int kAP = kFI * kAS;            // one moment plane
constexpr int kBS = kFP + 1;              // (a, b, c) rows (59)
constexpr int kBP = kFM * kBS;            // one (a, b, c) plane
constexpr int kFA = 5 * kAP;              // 11180
constexpr int kFB = 3 * kBP;              // 7434 (also holds the input 2 x 52 x 53 and vb 3 x 47 x 32)
static_assert(kFB >= 2 * kFI * kXS && kFB >= 3 * kFV * kFT && kFA >= 3 * kFM * kFV, "shared layout");
#ifndef TS_LOSS_THREADS
#define TS_LOSS_THREADS 320  // 10 warps: the 312 horizontal-moment items of a tile in one round
#endif
constexpr int kFThreads = TS_LOSS_THREADS;
constexpr int kFRowGroups = kFThreads / 64;                       // input rows per pass
constexpr int kFRowIters = (kFI + kFRowGroups - 1) / kFRowGroups;  // passes
constexpr size_t kFusedSmem = size_t(kFA + kFB) * 4;

__global__ void __launch_bounds__(kFThreads, 3) loss_fused_kernel(const float* __restrict__ X,
                                                              const float* __restrict__ Y, float* __restrict__ dL,
                                                              int W, int H, float inv_m, double* __restrict__ acc) {
    extern __shared__ float fsm[];
    float* A = fsm;
    float* B = fsm + kFA;
    const int ch = blockIdx.z, P = W * H;
    const int x0 = blockIdx.x * kFT, y0 = blockIdx.y * kFT;
    const int tid = threadIdx.x;
    const float* Xc = X + size_t(ch) * P;
    const float* Yc = Y + size_t(ch) * P;
    float wk[11];
#pragma unroll
    for (int k = 0; k < 11; ++k) wk[k] = c_gw[k];
    // 1. input region (reflect; clamped first so far-outside positions of small images stay in range)
    float* xs = B;
    float* ys = B + kFI * kXS;
    {
        // kFRowGroups rows x 64 columns per pass (52 active): the column's reflected index
        // once per thread; all rows' loads issued before any store (latency overlapped)
        const int c = tid & 63;
        if (c < kFI) {
            const int gx = refl(min(max(x0 - 10 + c, -(W - 1)), 2 * (W - 1)), W);
            float xv[kFRowIters], yv[kFRowIters];
#pragma unroll
            for (int k = 0; k < kFRowIters; ++k) {
                const int r = min((tid >> 6) + kFRowGroups * k, kFI - 1);
                const int gy = refl(min(max(y0 - 10 + r, -(H - 1)), 2 * (H - 1)), H);
                xv[k] = __ldg(Xc + gy * W + gx);
                yv[k] = __ldg(Yc + gy * W + gx);
            }
#pragma unroll
            for (int k = 0; k < kFRowIters; ++k) {
                const int r = (tid >> 6) + kFRowGroups * k;
                if (r < kFI) {
                    xs[r * kXS + c] = xv[k];
                    ys[r * kXS + c] = yv[k];
                }
            }
        }
    }
    __syncthreads();
    // 2. horizontal moments: rows [0, 52) x moment cols [0, 42), items of 7 columns
    float l1 = 0.f, ss = 0.f;
    {
        constexpr int S = 7, NS = kFM / S;
        for (int it = tid; it < kFI * NS; it += kFThreads) {
            const int r = it % kFI, c0 = (it / kFI) * S;  // lanes on consecutive rows
            // (x, y) pairs: {mu_x, mu_y} and {x^2, y^2} moments in packed fp32x2 ops
            float2 ab[S + 10];
#pragma unroll
            for (int k = 0; k < S + 10; ++k) ab[k] = make_float2(xs[r * kXS + c0 + k], ys[r * kXS + c0 + k]);
#pragma unroll
            for (int j = 0; j < S; ++j) {
                float2 m01 = make_float2(0.f, 0.f), m23 = m01;
                float m4 = 0.f;
#pragma unroll
                for (int k = 0; k < 11; ++k) {
                    const float2 v = ab[j + k];
                    const float2 wv = tsx::mul2(tsx::dup2(wk[k]), v);
                    m01 = tsx::add2(m01, wv);
                    m23 = tsx::fma2(wv, v, m23);
                    m4 = fmaf(wv.x, v.y, m4);
                }
                const int o = r * kAS + c0 + j;
                A[o] = m01.x;
                A[kAP + o] = m01.y;
                A[2 * kAP + o] = m23.x;
                A[3 * kAP + o] = m23.y;
                A[4 * kAP + o] = m4;
            }
        }
    }
    __syncthreads();
    // 3. vertical moments over moment rows [0, 42) -> SSIM and (a, b, c) into B as
    //    abc[q][r][c + 5] (padded columns [-10, 48) hold zeros)
    {
        constexpr int S = 7, NS = kFM / S;  // 6 x 42 = 252 items: one round of 256 threads
        for (int it = tid; it < kFM * NS; it += kFThreads) {
            const int c = it % kFM, r0 = (it / kFM) * S;
            float m[S][5];
#pragma unroll
            for (int q = 0; q < 4; q += 2) {  // moment pairs (0,1), (2,3) packed
                float2 win[S + 10];
#pragma unroll
                for (int k = 0; k < S + 10; ++k)
                    win[k] = make_float2(A[q * kAP + (r0 + k) * kAS + c], A[(q + 1) * kAP + (r0 + k) * kAS + c]);
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    float2 sacc = make_float2(0.f, 0.f);
#pragma unroll
                    for (int k = 0; k < 11; ++k) sacc = tsx::fma2(tsx::dup2(wk[k]), win[j + k], sacc);
                    m[j][q] = sacc.x;
                    m[j][q + 1] = sacc.y;
                }
            }
            {
                float win[S + 10];
#pragma unroll
                for (int k = 0; k < S + 10; ++k) win[k] = A[4 * kAP + (r0 + k) * kAS + c];
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    float sacc = 0.f;
#pragma unroll
                    for (int k = 0; k < 11; ++k) sacc = fmaf(wk[k], win[j + k], sacc);
                    m[j][4] = sacc;
                }
            }
            const int gx = x0 - 5 + c;
#pragma unroll
            for (int j = 0; j < S; ++j) {
                const int r = r0 + j, gy = y0 - 5 + r;
                float ta = 0.f, tb = 0.f, tc = 0.f;
                if (gx >= 0 && gx < W && gy >= 0 && gy < H) {
                    const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
                    const float ux = m[j][0], uy = m[j][1];
                    const float vx = m[j][2] - ux * ux, vy = m[j][3] - uy * uy, cxy = m[j][4] - ux * uy;
                    const float n1 = 2.f * ux * uy + C1, n2 = 2.f * cxy + C2;
                    const float d1 = ux * ux + uy * uy + C1, d2 = vx + vy + C2;
                    const float iD = __fdividef(1.f, d1 * d2);
                    const float Sv = n1 * n2 * iD;
                    const float dS_dux = (2.f * uy * n2 - Sv * 2.f * ux * d2) * iD;
                    const float dS_dvx = -Sv * d1 * iD;
                    const float dS_dcxy = 2.f * n1 * iD;
                    ta = dS_dux - 2.f * ux * dS_dvx - uy * dS_dcxy;
                    tb = 2.f * dS_dvx;
                    tc = dS_dcxy;
                    if (r >= 5 && r < 5 + kFT && c >= 5 && c < 5 + kFT) ss += Sv;
                }
                B[0 * kBP + r * kBS + c + 5] = ta;
                B[1 * kBP + r * kBS + c + 5] = tb;
                B[2 * kBP + r * kBS + c + 5] = tc;
            }
        }
        // zero the padding columns [0, 5) and [47, 58) of every (a, b, c) row (3 x 42 rows)
        if (tid < 3 * kFM) {
            float* row = B + (tid / kFM) * kBP + (tid % kFM) * kBS;
#pragma unroll
            for (int k = 0; k < 5; ++k) row[k] = 0.f;
#pragma unroll
            for (int k = kFM + 5; k < kFP; ++k) row[k] = 0.f;
        }
    }
    __syncthreads();
    // 4a. horizontal transposed pass at virtual columns [-5, 42): hb[q][r][m] (A, 3 x 42 x 47);
    //     (a, b) packed, c scalar
    {
        constexpr int S = 8, NS = (kFV + S - 1) / S;  // 6 segments (48 columns, last partly unused)
        for (int it = tid; it < kFM * NS; it += kFThreads) {
            const int r = it % kFM, c0 = (it / kFM) * S;  // lanes on consecutive rows
            float2 ab[S + 10];
            float cc[S + 10];
#pragma unroll
            for (int k = 0; k < S + 10; ++k) {
                const bool in = c0 + k < kFP;
                ab[k] = in ? make_float2(B[r * kBS + c0 + k], B[kBP + r * kBS + c0 + k]) : make_float2(0.f, 0.f);
                cc[k] = in ? B[2 * kBP + r * kBS + c0 + k] : 0.f;
            }
#pragma unroll
            for (int j = 0; j < S; ++j) {
                float2 sab = make_float2(0.f, 0.f);
                float sc = 0.f;
#pragma unroll
                for (int k = 0; k < 11; ++k) {
                    sab = tsx::fma2(tsx::dup2(wk[k]), ab[j + k], sab);
                    sc = fmaf(wk[k], cc[j + k], sc);
                }
                if (c0 + j < kFV) {
                    A[r * kFV + c0 + j] = sab.x;
                    A[kFM * kFV + r * kFV + c0 + j] = sab.y;
                    A[2 * kFM * kFV + r * kFV + c0 + j] = sc;
                }
            }
        }
    }
    __syncthreads();
    // 5a. vertical transposed pass at virtual rows [-5, 42) straight from hb, with the
    //     column fold of the reflect padding applied on the fly (tiles at the image's
    //     left/right edge only): vb[q][m][c] (B, 3 x 47 x 32); hb rows outside [0, 42)
    //     and columns beyond the image are zero; (a, b) packed
    {
        constexpr int S = 6, NS = (kFV + S - 1) / S;  // 8 groups (48 rows, last partly unused)
        const bool fold = x0 <= 5 || x0 + kFT - 1 >= W - 6;  // CTA-uniform
        auto pass = [&](auto fold_tag) {
            constexpr bool kFold = decltype(fold_tag)::value;
            for (int it = tid; it < kFT * NS; it += kFThreads) {
                const int c = it % kFT, r0 = (it / kFT) * S;
                const int px = x0 + c;
                const int ml = kFold && px >= 1 && px <= 5 ? -px - x0 + 5 : -1;                       // mirror of -px
                const int mr = kFold && px >= W - 6 && px <= W - 2 ? 2 * (W - 1) - px - x0 + 5 : -1;  // of 2(W-1)-px
                float2 ab[S + 10];
                float cc[S + 10];
#pragma unroll
                for (int k = 0; k < S + 10; ++k) {
                    const int r = r0 + k - 5;
                    const bool in = r >= 0 && r < kFM && px < W;
                    const float* h0 = A + r * kFV;
                    float va = 0.f, vbb = 0.f, vc = 0.f;
                    if (in) {
                        va = h0[c + 5];
                        vbb = h0[kFM * kFV + c + 5];
                        vc = h0[2 * kFM * kFV + c + 5];
                        if (kFold && ml >= 0) {
                            va += h0[ml];
                            vbb += h0[kFM * kFV + ml];
                            vc += h0[2 * kFM * kFV + ml];
                        }
                        if (kFold && mr >= 0) {
                            va += h0[mr];
                            vbb += h0[kFM * kFV + mr];
                            vc += h0[2 * kFM * kFV + mr];
                        }
                    }
                    ab[k] = make_float2(va, vbb);
                    cc[k] = vc;
                }
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    float2 sab = make_float2(0.f, 0.f);
                    float sc = 0.f;
#pragma unroll
                    for (int k = 0; k < 11; ++k) {
                        sab = tsx::fma2(tsx::dup2(wk[k]), ab[j + k], sab);
                        sc = fmaf(wk[k], cc[j + k], sc);
                    }
                    if (r0 + j < kFV) {
                        B[(r0 + j) * kFT + c] = sab.x;
                        B[kFV * kFT + (r0 + j) * kFT + c] = sab.y;
                        B[2 * kFV * kFT + (r0 + j) * kFT + c] = sc;
                    }
                }
            }
        };
        if (fold) pass(std::true_type{});
        else pass(std::false_type{});
    }
    __syncthreads();
    // 5b. fold rows; dL/dC = (0.8 sign(x - y) - 0.2 (Wt a + x Wt b + y Wt c)) / M
    for (int i = tid; i < kFT * kFT; i += kFThreads) {
        const int r = i / kFT, c = i - r * kFT;
        const int px = x0 + c, py = y0 + r;
        if (px >= W || py >= H) continue;
        float t[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const float* vb = B + q * kFV * kFT + c;
            float v = vb[(r + 5) * kFT];
            if (py >= 1 && py <= 5) v += vb[(-py - y0 + 5) * kFT];
            if (py >= H - 6 && py <= H - 2) v += vb[(2 * (H - 1) - py - y0 + 5) * kFT];
            t[q] = v;
        }
        const int p = py * W + px;
        const float xv = __ldg(Xc + p), yv = __ldg(Yc + p);
        const float dS = t[0] + xv * t[1] + yv * t[2];
        const float d = xv - yv;
        l1 += fabsf(d);
        const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
        dL[size_t(ch) * P + p] = (0.8f * sg - 0.2f * dS) * inv_m;
    }
    // block reduction of (L1, SSIM) -> double atomics
    __shared__ float r1[kFThreads / 32], r2[kFThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if ((tid & 31) == 0) {
        r1[tid >> 5] = l1;
        r2[tid >> 5] = ss;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0, b = 0;
        for (int w = 0; w < kFThreads / 32; ++w) {
            a += r1[w];
            b += r2[w];
        }
        atomicAdd(acc, a);
        atomicAdd(acc + 1, b);
    }
}
}  // namespace

void launch_loss(Context& c, const float* target_chw) {
    if (first_on_device(c, reinterpret_cast<const void*>(&c_gw))) {  // __constant__ is per device
        double g[11], s = 0;
        for (int i = 0; i < 11; ++i) {
            const double d = i - 5;
            g[i] = std::exp(-(d * d) / (2.0 * 1.5 * 1.5));
            s += g[i];
        }
        float gf[11];
        for (int i = 0; i < 11; ++i) gf[i] = float(g[i] / s);
        cudaMemcpyToSymbol(c_gw, gf, sizeof(gf));
    }
    const int W = c.fw, H = c.fh, P = W * H;
    cudaMemsetAsync(c.loss_acc.p, 0, 2 * sizeof(double), c.stream);
    set_func_attr(c, reinterpret_cast<const void*>(loss_fused_kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                  int(kFusedSmem));
    const dim3 grid((W + kFT - 1) / kFT, (H + kFT - 1) / kFT, 3);
    loss_fused_kernel<<<grid, kFThreads, kFusedSmem, c.stream>>>(c.rgb.p, target_chw, c.dLdC.p, W, H,
                                                                 float(1.0 / (3.0 * double(P))), c.loss_acc.p);
    TS_LAUNCHED(c);
}

}  // namespace ts
