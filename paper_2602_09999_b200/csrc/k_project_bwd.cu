// K9 preprocess_bwd: one thread per Gaussian.
// backward_project with the J clamp adjoint, the SH colour
// clamp, sigmoid/exp activation adjoints, and
// accumulate_densify_stats: accum += |dL/dmean2d|, count += 1.
//
// Two kernels share the per-Gaussian adjoint (pb_grads):
//  * project_bwd_kernel: gradients written (after a clear) or ACCUMULATED into
//    the flat 59*N buffer (multi-view batches sum);
//  * project_bwd_adam_kernel: fused_backward_update: each
//    Gaussian's complete gradient row is consumed by the fused Adam update in
//    place, and rows of invisible Gaussians get the zero-gradient update in
//    the same sweep (or none in skip-invisible mode) -- the end state is bitwise
//    that of backward + adam_step_fused, without writing or re-reading the
//    gradient buffer.
// Both are HBM-bound: a CTA stages all inputs of its Gaussians (attribute
// blocks of the 59*N layout, SH rows, 2D gradients, statistics; for the fused
// kernel also both Adam moments) with one pass of independent 16-byte loads
// (stage_spans), computes from shared memory, and writes rows back through
// shared memory so every global access is coalesced.  The per-Gaussian 2D
// accumulator is consumed and zeroed.
#include <cmath>

#include "ts_internal.cuh"
#ifndef TS_PB_MINB
#define TS_PB_MINB 5  // 5 resident CTAs (96 registers): more staged rows in flight; measured 0.281 -> 0.268 ms
#endif
#include "ts_math.cuh"
#include "ts_stage.cuh"

namespace ts {
namespace {

// ex2.approx with the scaling multiply pinned (__fmul_rn): the scale activation
// feeds several consumers and must not be contracted differently per kernel
__device__ __forceinline__ float exp2f_approx_(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// staged per-Gaussian rows of one Gaussian
struct Rows {
    const float* mu;   // 3
    const float* ls;   // 3
    const float* q;    // 4
    float op;          // logit
    const float* dc;   // 3
    const float* rest; // 45 (only [0, nrest) read)
    const float* g2;   // 12: dmx dmy dA dB dC do dr dg db
};

// SH-rest gradient consumers: store into a row, or hand to a per-element update
struct RowSink {
    float* a;
    __device__ __forceinline__ void operator()(int k, float g) const { a[k] = g; }
};

// Adjoint of one visible Gaussian.  gs[14] = d{means(3), log_scales(3),
// quats(4), opacity_logit(1), sh_dc(3)}; SH-rest gradient k in [0, nrest) goes
// to sink(k, g) right after rest[k] is last read (so the sink may update the
// row in place).  Returns |dL/dmean2d| for the densification statistics.
template <int DEG, class Sink>
__device__ __forceinline__ float pb_grads(const Rows& r, const Sink& sink, const DevCam& cam,
                                          const ts_render_config& cfg, float nu, float (&gs)[14]) {
    constexpr int nb = (DEG + 1) * (DEG + 1);
    const float* W = cam.W;
    const float dmx = r.g2[0], dmy = r.g2[1], dA = r.g2[2], dB = r.g2[3], dC = r.g2[4], dop = r.g2[5];
    float drc[3] = {r.g2[6], r.g2[7], r.g2[8]};
    // ---- recompute forward quantities ----
    const float mu[3] = {r.mu[0], r.mu[1], r.mu[2]};
    const float xh = W[0] * mu[0] + W[1] * mu[1] + W[2] * mu[2] + W[3];
    const float yh = W[4] * mu[0] + W[5] * mu[1] + W[6] * mu[2] + W[7];
    const float zh = W[8] * mu[0] + W[9] * mu[1] + W[10] * mu[2] + W[11];
    const float q0 = r.q[0], q1 = r.q[1], q2 = r.q[2], q3 = r.q[3];
    const float qn = sqrtf(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
    const float iqn = 1.f / qn;
    const float w = q0 * iqn, x = q1 * iqn, y = q2 * iqn, z = q3 * iqn;
    float R[9];
    // explicit fma order (R feeds the scale gradient directly; both kernels inlining
    // this adjoint must round identically, see test_fused_backward_adam_equals_separate)
    R[0] = fmaf(-2.f, fmaf(y, y, z * z), 1.f);
    R[1] = 2.f * fmaf(x, y, -(w * z));
    R[2] = 2.f * fmaf(x, z, w * y);
    R[3] = 2.f * fmaf(x, y, w * z);
    R[4] = fmaf(-2.f, fmaf(x, x, z * z), 1.f);
    R[5] = 2.f * fmaf(y, z, -(w * x));
    R[6] = 2.f * fmaf(x, z, -(w * y));
    R[7] = 2.f * fmaf(y, z, w * x);
    R[8] = fmaf(-2.f, fmaf(x, x, y * y), 1.f);
    float s[3], s_raw[3], s_h[3], aaf = 0.f, ofac = 1.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) s[k] = s_raw[k] = exp2f_approx_(__fmul_rn(r.ls[k], 1.44269504088896341f));
    if (cfg.aa_mode == 1) {  // 3D filter: s_hat = sqrt(s^2 + kappa/nu^2), opacity factor
        aaf = cfg.kappa3d / (nu * nu);
        float qp = 1.f, hp = 1.f;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float q = s_raw[k] * s_raw[k];
            s_h[k] = q + aaf;
            s[k] = sqrtf(s_h[k]);
            qp *= q;
            hp *= s_h[k];
        }
        ofac = sqrtf(qp / hp);
    }
    float Mm[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) Mm[3 * i + k] = R[3 * i + k] * s[k];
    float Sf[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            Sf[3 * i + j] = Mm[3 * i] * Mm[3 * j] + Mm[3 * i + 1] * Mm[3 * j + 1] + Mm[3 * i + 2] * Mm[3 * j + 2];
    const float limx = 1.3f * (0.5f * float(cam.w) / cam.fx);
    const float limy = 1.3f * (0.5f * float(cam.h) / cam.fy);
    const float iz = 1.f / zh, iz2 = iz * iz, iz3 = iz2 * iz;
    const float txz = xh * iz, tyz = yh * iz;
    const bool clx = (txz < -limx) || (txz > limx);
    const bool cly = (tyz < -limy) || (tyz > limy);
    const float ux = fminf(limx, fmaxf(-limx, txz)), uy = fminf(limy, fmaxf(-limy, tyz));
    const float J00 = cam.fx * iz, J02 = -cam.fx * ux * iz;
    const float J11 = cam.fy * iz, J12 = -cam.fy * uy * iz;
    float Tm[6];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        Tm[j] = J00 * W[j] + J02 * W[8 + j];
        Tm[3 + j] = J11 * W[4 + j] + J12 * W[8 + j];
    }
    float TS[6];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            TS[3 * a + j] = Tm[3 * a] * Sf[j] + Tm[3 * a + 1] * Sf[3 + j] + Tm[3 * a + 2] * Sf[6 + j];
    const float ca0 = TS[0] * Tm[0] + TS[1] * Tm[1] + TS[2] * Tm[2];
    const float cb = TS[0] * Tm[3] + TS[1] * Tm[4] + TS[2] * Tm[5];
    const float cc0 = TS[3] * Tm[3] + TS[4] * Tm[4] + TS[5] * Tm[5];
    const float ca = ca0 + cfg.dilation, cc = cc0 + cfg.dilation;
    if (cfg.aa_mode == 3) {  // Mip compensation factor, detached from Sigma2D
        const float dpre = ca0 * cc0 - cb * cb;
        ofac = dpre > 0.f ? sqrtf(dpre / (ca * cc - cb * cb)) : 0.f;
    }
    const float idet = 1.f / (ca * cc - cb * cb);
    const float A = cc * idet, B = -cb * idet, C = ca * idet;
    const float o = 1.f / (1.f + __expf(-r.op));
    // ---- colour / SH ----
    const float cpx = -(W[0] * W[3] + W[4] * W[7] + W[8] * W[11]);
    const float cpy = -(W[1] * W[3] + W[5] * W[7] + W[9] * W[11]);
    const float cpz = -(W[2] * W[3] + W[6] * W[7] + W[10] * W[11]);
    const float e0 = mu[0] - cpx, e1 = mu[1] - cpy, e2 = mu[2] - cpz;
    const float dl = sqrtf(e0 * e0 + e1 * e1 + e2 * e2);
    const float idl = 1.f / dl;
    const float d0 = e0 * idl, d1 = e1 * idl, d2 = e2 * idl;
    float Y[16];
    float dY[16][3];
    Y[0] = TS_SH_C0;
#pragma unroll
    for (int k = 0; k < 16; ++k) dY[k][0] = dY[k][1] = dY[k][2] = 0.f;
    if (DEG >= 1) {
        Y[1] = -TS_SH_C1 * d1;
        Y[2] = TS_SH_C1 * d2;
        Y[3] = -TS_SH_C1 * d0;
        dY[1][1] = -TS_SH_C1;
        dY[2][2] = TS_SH_C1;
        dY[3][0] = -TS_SH_C1;
    }
    if (DEG >= 2) {
        const float xx = d0 * d0, yy = d1 * d1, zz = d2 * d2;
        Y[4] = TS_SH_C2_0 * d0 * d1;
        Y[5] = TS_SH_C2_1 * d1 * d2;
        Y[6] = TS_SH_C2_2 * (2.f * zz - xx - yy);
        Y[7] = TS_SH_C2_3 * d0 * d2;
        Y[8] = TS_SH_C2_4 * (xx - yy);
        dY[4][0] = TS_SH_C2_0 * d1;
        dY[4][1] = TS_SH_C2_0 * d0;
        dY[5][1] = TS_SH_C2_1 * d2;
        dY[5][2] = TS_SH_C2_1 * d1;
        dY[6][0] = -2.f * TS_SH_C2_2 * d0;
        dY[6][1] = -2.f * TS_SH_C2_2 * d1;
        dY[6][2] = 4.f * TS_SH_C2_2 * d2;
        dY[7][0] = TS_SH_C2_3 * d2;
        dY[7][2] = TS_SH_C2_3 * d0;
        dY[8][0] = 2.f * TS_SH_C2_4 * d0;
        dY[8][1] = -2.f * TS_SH_C2_4 * d1;
        if (DEG >= 3) {
            Y[9] = TS_SH_C3_0 * d1 * (3.f * xx - yy);
            Y[10] = TS_SH_C3_1 * d0 * d1 * d2;
            Y[11] = TS_SH_C3_2 * d1 * (4.f * zz - xx - yy);
            Y[12] = TS_SH_C3_3 * d2 * (2.f * zz - 3.f * xx - 3.f * yy);
            Y[13] = TS_SH_C3_4 * d0 * (4.f * zz - xx - yy);
            Y[14] = TS_SH_C3_5 * d2 * (xx - yy);
            Y[15] = TS_SH_C3_6 * d0 * (xx - 3.f * yy);
            dY[9][0] = TS_SH_C3_0 * 6.f * d0 * d1;
            dY[9][1] = TS_SH_C3_0 * (3.f * xx - 3.f * yy);
            dY[10][0] = TS_SH_C3_1 * d1 * d2;
            dY[10][1] = TS_SH_C3_1 * d0 * d2;
            dY[10][2] = TS_SH_C3_1 * d0 * d1;
            dY[11][0] = -2.f * TS_SH_C3_2 * d0 * d1;
            dY[11][1] = TS_SH_C3_2 * (4.f * zz - xx - 3.f * yy);
            dY[11][2] = 8.f * TS_SH_C3_2 * d1 * d2;
            dY[12][0] = -6.f * TS_SH_C3_3 * d0 * d2;
            dY[12][1] = -6.f * TS_SH_C3_3 * d1 * d2;
            dY[12][2] = TS_SH_C3_3 * (6.f * zz - 3.f * xx - 3.f * yy);
            dY[13][0] = TS_SH_C3_4 * (4.f * zz - 3.f * xx - yy);
            dY[13][1] = -2.f * TS_SH_C3_4 * d0 * d1;
            dY[13][2] = 8.f * TS_SH_C3_4 * d0 * d2;
            dY[14][0] = 2.f * TS_SH_C3_5 * d0 * d2;
            dY[14][1] = -2.f * TS_SH_C3_5 * d1 * d2;
            dY[14][2] = TS_SH_C3_5 * (xx - yy);
            dY[15][0] = TS_SH_C3_6 * (3.f * xx - 3.f * yy);
            dY[15][1] = -6.f * TS_SH_C3_6 * d0 * d1;
        }
    }
    float ddir0 = 0.f, ddir1 = 0.f, ddir2 = 0.f;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        float raw = Y[0] * r.dc[ch];
#pragma unroll
        for (int k = 1; k < nb; ++k) raw += Y[k] * r.rest[3 * (k - 1) + ch];
        raw += 0.5f;
        if (raw < 0.f) drc[ch] = 0.f;
        const float d = drc[ch];
        gs[11 + ch] = Y[0] * d;
#pragma unroll
        for (int k = 1; k < nb; ++k) {
            const float cf = r.rest[3 * (k - 1) + ch] * d;
            sink(3 * (k - 1) + ch, Y[k] * d);
            ddir0 += dY[k][0] * cf;
            ddir1 += dY[k][1] * cf;
            ddir2 += dY[k][2] * cf;
        }
    }
    const float nd = d0 * ddir0 + d1 * ddir1 + d2 * ddir2;
    float dmean0 = (ddir0 - d0 * nd) * idl, dmean1 = (ddir1 - d1 * nd) * idl, dmean2 = (ddir2 - d2 * nd) * idl;
    // ---- opacity ----
    gs[10] = dop * ofac * o * (1.f - o);
    // ---- conic -> dilated cov2d ----
    const float hb = 0.5f * dB;
    const float K00 = A * dA + B * hb, K01 = A * hb + B * dC;
    const float K10 = B * dA + C * hb, K11 = B * hb + C * dC;
    const float da = -(K00 * A + K01 * B);
    const float db = -2.f * (K00 * B + K01 * C);
    const float dc = -(K10 * B + K11 * C);
    // ---- cov2d = Tm S Tm^T ----
    const float G2[4] = {da, 0.5f * db, 0.5f * db, dc};
    float dS[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            dS[3 * i + j] = fmaf(Tm[3 + i], fmaf(G2[2], Tm[j], G2[3] * Tm[3 + j]),
                                 Tm[i] * fmaf(G2[0], Tm[j], G2[1] * Tm[3 + j]));
    float dTm[6];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j) dTm[3 * a + j] = 2.f * (G2[2 * a] * TS[j] + G2[2 * a + 1] * TS[3 + j]);
    const float dJ00 = dTm[0] * W[0] + dTm[1] * W[1] + dTm[2] * W[2];
    const float dJ02 = dTm[0] * W[8] + dTm[1] * W[9] + dTm[2] * W[10];
    const float dJ11 = dTm[3] * W[4] + dTm[4] * W[5] + dTm[5] * W[6];
    const float dJ12 = dTm[3] * W[8] + dTm[4] * W[9] + dTm[5] * W[10];
    // ---- camera point ----
    float dtx = dmx * cam.fx * iz, dty = dmy * cam.fy * iz;
    float dtz = -dmx * cam.fx * xh * iz2 - dmy * cam.fy * yh * iz2;
    dtz += -dJ00 * cam.fx * iz2 - dJ11 * cam.fy * iz2;
    if (!clx) {
        dtx += dJ02 * (-cam.fx * iz2);
        dtz += dJ02 * (2.f * cam.fx * xh * iz3);
    } else {
        dtz += dJ02 * (cam.fx * ux * iz2);
    }
    if (!cly) {
        dty += dJ12 * (-cam.fy * iz2);
        dtz += dJ12 * (2.f * cam.fy * yh * iz3);
    } else {
        dtz += dJ12 * (cam.fy * uy * iz2);
    }
    gs[0] = dmean0 + W[0] * dtx + W[4] * dty + W[8] * dtz;
    gs[1] = dmean1 + W[1] * dtx + W[5] * dty + W[9] * dtz;
    gs[2] = dmean2 + W[2] * dtx + W[6] * dty + W[10] * dtz;
    // ---- Sigma = M M^T, M = R diag(s) ----
    float dM[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            dM[3 * i + k] = 2.f * fmaf(dS[3 * i + 2], Mm[6 + k], fmaf(dS[3 * i + 1], Mm[3 + k], dS[3 * i] * Mm[k]));
    float dR[9];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        // explicit fma order: both kernels that inline this adjoint (gradient-writing and
        // fused-Adam) must produce the same bits (fused_backward_update == separate pair)
        const float ds = fmaf(R[6 + k], dM[6 + k], fmaf(R[3 + k], dM[3 + k], R[k] * dM[k]));
#pragma unroll
        for (int i = 0; i < 3; ++i) dR[3 * i + k] = dM[3 * i + k] * s[k];
        if (cfg.aa_mode == 1)  // through s_hat = sqrt(s^2 + kappa/nu^2) and the opacity factor
            gs[3 + k] = fmaf(ds, s_raw[k] * s_raw[k] / s[k], dop * o * ofac * (aaf / s_h[k]));
        else
            gs[3 + k] = __fmul_rn(ds, s[k]);
    }
    const float dqw = 2.f * (-z * dR[1] + y * dR[2] + z * dR[3] - x * dR[5] - y * dR[6] + x * dR[7]);
    const float dqx = 2.f * (y * dR[1] + z * dR[2] + y * dR[3] - 2.f * x * dR[4] - w * dR[5] + z * dR[6] + w * dR[7] -
                             2.f * x * dR[8]);
    const float dqy = 2.f * (-2.f * y * dR[0] + x * dR[1] + w * dR[2] + x * dR[3] + z * dR[5] - w * dR[6] +
                             z * dR[7] - 2.f * y * dR[8]);
    const float dqz = 2.f * (-2.f * z * dR[0] - w * dR[1] + x * dR[2] + w * dR[3] - 2.f * z * dR[4] + y * dR[5] +
                             x * dR[6] + y * dR[7]);
    const float dot = w * dqw + x * dqx + y * dqy + z * dqz;
    gs[6] = (dqw - w * dot) * iqn;
    gs[7] = (dqx - x * dot) * iqn;
    gs[8] = (dqy - y * dot) * iqn;
    gs[9] = (dqz - z * dot) * iqn;
    return sqrtf(dmx * dmx + dmy * dmy);
}

// ---------------------------------------------------------------------------
// gradient-writing kernel
// ---------------------------------------------------------------------------
constexpr int kBlock = 128;

// shared-memory layout of one CTA (floats; every segment a multiple of 4)
template <int DEG, bool ACCUM>
struct PbLayout {
    static constexpr int kMu = 0;
    static constexpr int kLs = kMu + 3 * kBlock + 4;
    static constexpr int kQ = kLs + 3 * kBlock + 4;
    static constexpr int kOp = kQ + 4 * kBlock + 4;
    static constexpr int kDc = kOp + kBlock + 4;
    static constexpr int kG2 = kDc + 3 * kBlock + 4;
    static constexpr int kAc = kG2 + 12 * kBlock + 4;
    static constexpr int kVc = kAc + kBlock + 4;
    static constexpr int kRest = kVc + kBlock + 4;
    static constexpr int kGRest = kRest + (DEG > 0 ? 45 * kBlock + 4 : 0);
    static constexpr int kTotal = kGRest + (DEG > 0 && ACCUM ? 45 * kBlock + 4 : 0);
};

template <int DEG, bool ACCUM>
__global__ void __launch_bounds__(kBlock, TS_PB_MINB) project_bwd_kernel(const float* __restrict__ P, float* __restrict__ G,
                                                             float4* __restrict__ g2d,
                                                             const uint32_t* __restrict__ tcount,
                                                             float* __restrict__ accum, float* __restrict__ vcount,
                                                             uint8_t* __restrict__ vis, int64_t N, DevCam cam,
                                                             ts_render_config cfg, int zero_inactive,
                                                             const float* __restrict__ nu_hat,
                                                             const uint32_t* __restrict__ gflag) {
    extern __shared__ __align__(16) float smem[];
    using L = PbLayout<DEG, ACCUM>;
    if (gflag && *gflag) return;  // graph-captured step voided by its capacity check (replayed by the host)
    constexpr int nrest = 3 * ((DEG + 1) * (DEG + 1) - 1);
    const Off off(N);
    const int64_t g0 = int64_t(blockIdx.x) * kBlock;
    const int64_t g = g0 + threadIdx.x;
    const int rows = int(tmin<int64_t>(kBlock, N - g0));
    const bool active = g < N && tcount[g] != 0;
    // a stale (consumed, uncleared) buffer needs zeros on inactive rows too
    if (!__syncthreads_or(active || (zero_inactive && g < N))) return;
    int sh[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    {
        const Span base[8] = {{smem + L::kMu, P + off.means + 3 * g0, 3 * rows},
                              {smem + L::kLs, P + off.ls + 3 * g0, 3 * rows},
                              {smem + L::kQ, P + off.q + 4 * g0, 4 * rows},
                              {smem + L::kOp, P + off.op + g0, rows},
                              {smem + L::kDc, P + off.dc + 3 * g0, 3 * rows},
                              {smem + L::kG2, reinterpret_cast<const float*>(g2d + 3 * g0), 12 * rows},
                              {smem + L::kAc, accum + g0, rows},
                              {smem + L::kVc, vcount + g0, rows}};
        __shared__ unsigned long long bar;
        if constexpr (DEG == 0) {
            int s8[8];
            stage_spans_tma(base, s8, &bar);
            for (int k = 0; k < 8; ++k) sh[k] = s8[k];
        } else if constexpr (!ACCUM) {
            const Span sp[9] = {base[0], base[1], base[2], base[3], base[4], base[5], base[6], base[7],
                                {smem + L::kRest, P + off.rest + g0 * 45, 45 * rows}};
            int s9[9];
            stage_spans_tma(sp, s9, &bar);
            for (int k = 0; k < 9; ++k) sh[k] = s9[k];
        } else {
            const Span sp[10] = {base[0], base[1], base[2], base[3], base[4], base[5], base[6], base[7],
                                 {smem + L::kRest, P + off.rest + g0 * 45, 45 * rows},
                                 {smem + L::kGRest, G + off.rest + g0 * 45, 45 * rows}};
            stage_spans_tma(sp, sh, &bar);
        }
    }
    const int tid = threadIdx.x;
    float* rest_row = smem + L::kRest + sh[8] + tid * 45;
    if (active) {
        float dummy[4] = {0.f, 0.f, 0.f, 0.f};
        const Rows rw{smem + L::kMu + sh[0] + 3 * tid, smem + L::kLs + sh[1] + 3 * tid, smem + L::kQ + sh[2] + 4 * tid,
                      smem[L::kOp + sh[3] + tid],      smem + L::kDc + sh[4] + 3 * tid,
                      DEG > 0 ? rest_row : dummy,      smem + L::kG2 + sh[5] + 12 * tid};
        float gs[14];
        float nrm;
        if constexpr (ACCUM && nrest > 0) {
            float grest[nrest];
            nrm = pb_grads<DEG>(rw, RowSink{grest}, cam, cfg, nu_hat ? nu_hat[g] : 1.f, gs);
            float* grow = smem + L::kGRest + sh[9] + tid * 45;
#pragma unroll
            for (int k = 0; k < nrest; ++k) grow[k] += grest[k];
        } else {
            // overwrite mode: gradients replace the parameter row in place (each
            // element is read by pb_grads before it is written)
            nrm = pb_grads<DEG>(rw, RowSink{DEG > 0 ? rest_row : dummy}, cam, cfg, nu_hat ? nu_hat[g] : 1.f, gs);
        }
        const int64_t idx[14] = {off.means + 3 * g,  off.means + 3 * g + 1, off.means + 3 * g + 2, off.ls + 3 * g,
                                 off.ls + 3 * g + 1, off.ls + 3 * g + 2,    off.q + 4 * g,         off.q + 4 * g + 1,
                                 off.q + 4 * g + 2,  off.q + 4 * g + 3,     off.op + g,            off.dc + 3 * g,
                                 off.dc + 3 * g + 1, off.dc + 3 * g + 2};
#pragma unroll
        for (int k = 0; k < 14; ++k) {
            if constexpr (ACCUM) G[idx[k]] += gs[k];
            else G[idx[k]] = gs[k];
        }
        accum[g] = smem[L::kAc + sh[6] + tid] + nrm;
        vcount[g] = smem[L::kVc + sh[7] + tid] + 1.f;
        vis[g] = 1;
    } else if (!ACCUM && zero_inactive && g < N) {
        const int64_t idx[14] = {off.means + 3 * g,  off.means + 3 * g + 1, off.means + 3 * g + 2, off.ls + 3 * g,
                                 off.ls + 3 * g + 1, off.ls + 3 * g + 2,    off.q + 4 * g,         off.q + 4 * g + 1,
                                 off.q + 4 * g + 2,  off.q + 4 * g + 3,     off.op + g,            off.dc + 3 * g,
                                 off.dc + 3 * g + 1, off.dc + 3 * g + 2};
#pragma unroll
        for (int k = 0; k < 14; ++k) G[idx[k]] = 0.f;
        if constexpr (nrest == 0) {
            for (int k = 0; k < 45; ++k) G[off.rest + 45 * g + k] = 0.f;
        }
    }
    if constexpr (!ACCUM && nrest > 0) {
        // overwrite mode: rows of inactive Gaussians and inactive SH degrees carry zeros
        if (tid < rows) {
            if (!active) {
                for (int k = 0; k < 45; ++k) rest_row[k] = 0.f;
            } else {
                for (int k = nrest; k < 45; ++k) rest_row[k] = 0.f;
            }
        }
    }
    __syncthreads();
    if constexpr (nrest > 0) {
        store_span<kBlock>(G + off.rest + g0 * 45, (ACCUM ? smem + L::kGRest + sh[9] : smem + L::kRest + sh[8]),
                           rows * 45);
    }
}

// ---------------------------------------------------------------------------
// fused backward + Adam kernel
// ---------------------------------------------------------------------------
constexpr int kFB = 128;  // Gaussians (= threads) per CTA
#ifndef TS_FB_UNROLL
#define TS_FB_UNROLL 4
#endif
#ifndef TS_FB_MINB
#define TS_FB_MINB 4
#endif
#ifndef TS_FB_QUADS
#define TS_FB_QUADS 2
#endif

struct FusedAdam {
    float lr[6];  // per group
    float b1, b2, omb1, omb2, eps, bc1, bc2;
};

// Adam element: the reference op sequence (ts_math.cuh adam_elem)
__device__ __forceinline__ void adam_fused_elem(float& th, float g, float& m, float& v, float lr, const FusedAdam& a,
                                                tsx::RcpConst c1, tsx::RcpConst c2) {
    tsx::adam_elem(th, g, m, v, lr, a.b1, a.b2, a.omb1, a.omb2, a.eps, c1, c2);
}

// shared layout (floats): staged parameters (6 attribute segments of the CTA's
// rows, each with 4 words of alignment room; overwritten in place by the
// gradient rows), the 2D gradients, the statistics and per-row active flags.
struct FbLayout {
    static constexpr int kP = 0;
    static constexpr int kG2 = kP + 59 * kFB + 24;
    static constexpr int kAc = kG2 + 12 * kFB + 4;
    static constexpr int kVc = kAc + kFB + 4;
    static constexpr int kAct = kVc + kFB + 4;
    static constexpr int kTotal = kAct + kFB;
};

// Two phases per CTA of 128 Gaussians:
//  1. per thread (one Gaussian): the adjoint from the TMA-staged parameter rows;
//     the 59-float gradient row replaces the staged parameter row in shared
//     memory (zeros for invisible rows and inactive SH degrees), the 2D
//     accumulator is cleared, the statistics updated;
//  2. per CTA: one coalesced sweep over each attribute segment of the CTA's
//     rows -- g from shared memory, theta (an L2 hit: just staged), m and v
//     streamed from HBM with 8 independent element groups in flight per thread
//     -- applying the fused Adam element update and writing theta, m, v back.
//     The gradient never touches HBM.
template <int DEG, bool kSkipInvisible>
__global__ void __launch_bounds__(kFB, TS_FB_MINB) project_bwd_adam_kernel(float* __restrict__ P, float* __restrict__ Mo,
                                                                  float* __restrict__ Vo, float4* __restrict__ g2d,
                                                                  const uint32_t* __restrict__ tcount,
                                                                  float* __restrict__ accum,
                                                                  float* __restrict__ vcount,
                                                                  uint8_t* __restrict__ vis, int64_t N, DevCam cam,
                                                                  ts_render_config cfg, FusedAdam fa,
                                                                  const float* __restrict__ nu_hat) {
    extern __shared__ __align__(16) float smem[];
    using L = FbLayout;
    constexpr int width[6] = {3, 3, 4, 1, 3, 45};
    constexpr int segoff[6] = {0, 3 * kFB + 4, 6 * kFB + 8, 10 * kFB + 12, 11 * kFB + 16, 14 * kFB + 20};
    constexpr int nrest = 3 * ((DEG + 1) * (DEG + 1) - 1);
    const Off off(N);
    const int64_t goff[6] = {off.means, off.ls, off.q, off.op, off.dc, off.rest};
    const int64_t g0 = int64_t(blockIdx.x) * kFB;
    const int tid = threadIdx.x;
    const int64_t g = g0 + tid;
    const int rows = int(tmin<int64_t>(kFB, N - g0));
    const bool active = g < N && tcount[g] != 0;
    if (kSkipInvisible && !__syncthreads_or(active)) return;
    int sh[9];
    {
        Span sp[9];
#pragma unroll
        for (int s = 0; s < 6; ++s) sp[s] = Span{smem + L::kP + segoff[s], P + goff[s] + width[s] * g0, width[s] * rows};
        sp[6] = Span{smem + L::kG2, reinterpret_cast<const float*>(g2d + 3 * g0), 12 * rows};
        sp[7] = Span{smem + L::kAc, accum + g0, rows};
        sp[8] = Span{smem + L::kVc, vcount + g0, rows};
        // pull this CTA's Adam moments toward L2 now (bulk prefetch, no shared
        // memory), so the HBM reads overlap the adjoint phase below
        if (tid == 0) {
#pragma unroll
            for (int s = 0; s < 6; ++s) {
                prefetch_l2(Mo + goff[s] + width[s] * g0, width[s] * rows);
                prefetch_l2(Vo + goff[s] + width[s] * g0, width[s] * rows);
            }
        }
        __shared__ unsigned long long bar;
        stage_spans_tma(sp, sh, &bar);
    }
    float* act = smem + L::kAct;
    if (tid < rows) {
        float* pr[6];
#pragma unroll
        for (int s = 0; s < 6; ++s) pr[s] = smem + L::kP + segoff[s] + sh[s] + width[s] * tid;
        act[tid] = active ? 1.f : 0.f;
        float gs[14];
        if (active) {
            const Rows rw{pr[0], pr[1], pr[2], pr[3][0], pr[4], pr[5], smem + L::kG2 + sh[6] + 12 * tid};
            // in place: every SH-rest element is read before its gradient is written
            const float nrm = pb_grads<DEG>(rw, RowSink{pr[5]}, cam, cfg, nu_hat ? nu_hat[g] : 1.f, gs);
            accum[g] = smem[L::kAc + sh[7] + tid] + nrm;
            vcount[g] = smem[L::kVc + sh[8] + tid] + 1.f;
            vis[g] = 1;
        } else {
#pragma unroll
            for (int k = 0; k < 14; ++k) gs[k] = 0.f;
        }
        for (int k = active ? nrest : 0; k < 45; ++k) pr[5][k] = 0.f;
        int k = 0;
#pragma unroll
        for (int s = 0; s < 5; ++s)
#pragma unroll
            for (int j = 0; j < width[s]; ++j, ++k) pr[s][j] = gs[k];
    }
    __syncthreads();
    const tsx::RcpConst c1 = tsx::rcp_const(fa.bc1), c2 = tsx::rcp_const(fa.bc2);
    // a rolled segment loop and 4 element groups in flight keep the sweep's code small (the
    // unrolled 6 x 12 sweep thrashed the instruction cache: 38% "no instruction" stalls)
#pragma unroll 1
    for (int s = 0; s < 6; ++s) {
        constexpr int kU = TS_FB_UNROLL;
        const int n = width[s] * rows;
        const float* gr_s = smem + L::kP + segoff[s] + sh[s];
        float* Pg = P + goff[s] + width[s] * g0;
        float* Mg = Mo + goff[s] + width[s] * g0;
        float* Vg = Vo + goff[s] + width[s] * g0;
        const float lr = fa.lr[s];
        int done = 0;
        if (((goff[s] + width[s] * g0) & 3) == 0) {
            // segment on a 16-byte boundary (N % 4 == 0): float4 sweep, kQ quads per array in flight
            const int n4 = n >> 2;
            const float4* g4 = reinterpret_cast<const float4*>(gr_s);
            float4* P4 = reinterpret_cast<float4*>(Pg);
            float4* M4 = reinterpret_cast<float4*>(Mg);
            float4* V4 = reinterpret_cast<float4*>(Vg);
            constexpr int kQ = TS_FB_QUADS;
            for (int q0 = tid; q0 < n4; q0 += kQ * kFB) {
                float4 tq[kQ], mq[kQ], vq[kQ];
#pragma unroll
                for (int u = 0; u < kQ; ++u) {
                    const int q = q0 + u * kFB;
                    if (q < n4) {
                        tq[u] = P4[q];
                        mq[u] = M4[q];
                        vq[u] = V4[q];
                    }
                }
#pragma unroll
                for (int u = 0; u < kQ; ++u) {
                    const int q = q0 + u * kFB;
                    if (q < n4) {
                        const float4 gq = g4[q];
                        float* tp = &tq[u].x;
                        float* mp = &mq[u].x;
                        float* vp = &vq[u].x;
                        const float* gp = &gq.x;
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (!kSkipInvisible || act[(4 * q + k) / width[s]] != 0.f)
                                adam_fused_elem(tp[k], gp[k], mp[k], vp[k], lr, fa, c1, c2);
                        P4[q] = tq[u];
                        M4[q] = mq[u];
                        V4[q] = vq[u];
                    }
                }
            }
            done = n4 << 2;
        }
        for (int i0 = done + tid; i0 < n; i0 += kU * kFB) {
            float tr[kU], mr[kU], vr[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int i = i0 + u * kFB;
                if (i < n) {
                    tr[u] = Pg[i];
                    mr[u] = Mg[i];
                    vr[u] = Vg[i];
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int i = i0 + u * kFB;
                if (i < n && (!kSkipInvisible || act[i / width[s]] != 0.f)) {
                    adam_fused_elem(tr[u], gr_s[i], mr[u], vr[u], lr, fa, c1, c2);
                    Pg[i] = tr[u];
                    Mg[i] = mr[u];
                    Vg[i] = vr[u];
                }
            }
        }
    }
}


}  // namespace

void launch_project_bwd(Context& c, const DevCam& cam, const ts_render_config& cfg, bool accumulate,
                        bool zero_inactive) {
    if (c.N == 0) return;
    const int64_t blocks = (c.N + kBlock - 1) / kBlock;
    const uint32_t* gf = c.gmode ? c.counters.p + kGraphFlag : nullptr;
#define TS_PB(D)                                                                                      \
    if (accumulate) {                                                                                 \
        constexpr int sm = PbLayout<D, true>::kTotal * 4;                                             \
        set_func_attr(c, reinterpret_cast<const void*>(project_bwd_kernel<D, true>), cudaFuncAttributeMaxDynamicSharedMemorySize, sm); \
        project_bwd_kernel<D, true><<<unsigned(blocks), kBlock, sm, c.stream>>>(                      \
            c.params.p, c.grads.p, c.g2d.p, c.tcount.p, c.accum.p, c.vcount.p, c.vis.p, c.N, cam, cfg, 0, c.nu_hat.p, gf); \
    } else {                                                                                          \
        constexpr int sm = PbLayout<D, false>::kTotal * 4;                                            \
        set_func_attr(c, reinterpret_cast<const void*>(project_bwd_kernel<D, false>), cudaFuncAttributeMaxDynamicSharedMemorySize, sm); \
        project_bwd_kernel<D, false><<<unsigned(blocks), kBlock, sm, c.stream>>>(                     \
            c.params.p, c.grads.p, c.g2d.p, c.tcount.p, c.accum.p, c.vcount.p, c.vis.p, c.N, cam, cfg,   \
            int(zero_inactive), c.nu_hat.p, gf);                                                                 \
    }
    switch (cfg.sh_degree) {
        case 0: TS_PB(0); break;
        case 1: TS_PB(1); break;
        case 2: TS_PB(2); break;
        default: TS_PB(3); break;
    }
#undef TS_PB
    TS_LAUNCHED(c);
}

void launch_project_bwd_adam(Context& c, const DevCam& cam, const ts_render_config& cfg, const ts_adam_config& a) {
    if (c.N == 0) return;
    FusedAdam fa;
    for (int k = 0; k < 6; ++k) fa.lr[k] = a.lr[k];
    fa.b1 = a.beta1;
    fa.b2 = a.beta2;
    fa.omb1 = 1.0f - a.beta1;
    fa.omb2 = 1.0f - a.beta2;
    fa.eps = a.eps;
    fa.bc1 = a.bc1;
    fa.bc2 = a.bc2;
    const int64_t blocks = (c.N + kFB - 1) / kFB;
    constexpr int sm = FbLayout::kTotal * 4;
    const bool skip = a.mode == 4;
#define TS_FB(D)                                                                                          \
    if (skip) {                                                                                           \
        set_func_attr(c, reinterpret_cast<const void*>(project_bwd_adam_kernel<D, true>), cudaFuncAttributeMaxDynamicSharedMemorySize, sm); \
        project_bwd_adam_kernel<D, true><<<unsigned(blocks), kFB, sm, c.stream>>>(                        \
            c.params.p, c.m.p, c.v.p, c.g2d.p, c.tcount.p, c.accum.p, c.vcount.p, c.vis.p, c.N, cam, cfg, fa, c.nu_hat.p); \
    } else {                                                                                              \
        set_func_attr(c, reinterpret_cast<const void*>(project_bwd_adam_kernel<D, false>), cudaFuncAttributeMaxDynamicSharedMemorySize, sm); \
        project_bwd_adam_kernel<D, false><<<unsigned(blocks), kFB, sm, c.stream>>>(                       \
            c.params.p, c.m.p, c.v.p, c.g2d.p, c.tcount.p, c.accum.p, c.vcount.p, c.vis.p, c.N, cam, cfg, fa, c.nu_hat.p); \
    }
    switch (cfg.sh_degree) {
        case 0: TS_FB(0); break;
        case 1: TS_FB(1); break;
        case 2: TS_FB(2); break;
        default: TS_FB(3); break;
    }
#undef TS_FB
    TS_LAUNCHED(c);
}

}  // namespace ts
