// K9 preprocess_bwd: one thread per Gaussian (visible ones do work).
// backward_project with the J clamp adjoint, the SH colour
// clamp, sigmoid/exp activation adjoints, and
// accumulate_densify_stats: accum += |dL/dmean2d|, count += 1.
// Gradients are ACCUMULATED into the flat 59*N buffer (multi-view batches sum,
// SPEC.md:735); the per-Gaussian 2D accumulator is consumed and zeroed here.
// HBM-bound: a CTA stages all inputs of its 128 Gaussians (6 attribute blocks,
// SH rows, 2D gradients, statistics) with one pass of independent 16-byte
// loads (stage_spans), computes from shared memory, and writes SH gradient
// rows back through shared memory so every global access is coalesced.
#include "ts_internal.cuh"
#include "ts_math.cuh"
#include "ts_stage.cuh"

namespace ts {
namespace {

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
__global__ void __launch_bounds__(kBlock) project_bwd_kernel(const float* __restrict__ P, float* __restrict__ G,
                                                             float4* __restrict__ g2d,
                                                             const uint32_t* __restrict__ tcount,
                                                             float* __restrict__ accum, float* __restrict__ vcount,
                                                             uint8_t* __restrict__ vis, int64_t N, DevCam cam,
                                                             ts_render_config cfg) {
    extern __shared__ __align__(16) float smem[];
    using L = PbLayout<DEG, ACCUM>;
    const Off off(N);
    const int64_t g0 = int64_t(blockIdx.x) * kBlock;
    const int64_t g = g0 + threadIdx.x;
    constexpr int deg = DEG;
    constexpr int nb = (deg + 1) * (deg + 1);
    constexpr int nrest = 3 * (nb - 1);
    const int rows = int(tmin<int64_t>(kBlock, N - g0));
    const bool active = g < N && tcount[g] != 0;
    // does any Gaussian of this block need work?
    if (!__syncthreads_or(active)) return;
    // ---- stage every per-Gaussian input of the CTA in one pass (max MLP) ----
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
        if constexpr (DEG == 0) {
            int s8[8];
            stage_spans<kBlock>(base, s8);
            for (int k = 0; k < 8; ++k) sh[k] = s8[k];
        } else if constexpr (!ACCUM) {
            const Span sp[9] = {base[0], base[1], base[2], base[3], base[4], base[5], base[6], base[7],
                                {smem + L::kRest, P + off.rest + g0 * 45, 45 * rows}};
            int s9[9];
            stage_spans<kBlock>(sp, s9);
            for (int k = 0; k < 9; ++k) sh[k] = s9[k];
        } else {
            const Span sp[10] = {base[0], base[1], base[2], base[3], base[4], base[5], base[6], base[7],
                                 {smem + L::kRest, P + off.rest + g0 * 45, 45 * rows},
                                 {smem + L::kGRest, G + off.rest + g0 * 45, 45 * rows}};
            stage_spans<kBlock>(sp, sh);
        }
    }
    __syncthreads();
#define GW(idx, val)                          \
    do {                                      \
        if constexpr (ACCUM) G[idx] += (val); \
        else G[idx] = (val);                  \
    } while (0)
    const int tid = threadIdx.x;
    if (active) {
        const float* W = cam.W;
        const float* g2s = smem + L::kG2 + sh[5] + 12 * tid;
        reinterpret_cast<float4*>(g2d)[3 * g] = make_float4(0.f, 0.f, 0.f, 0.f);
        reinterpret_cast<float4*>(g2d)[3 * g + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
        reinterpret_cast<float4*>(g2d)[3 * g + 2] = make_float4(0.f, 0.f, 0.f, 0.f);
        const float dmx = g2s[0], dmy = g2s[1], dA = g2s[2], dB = g2s[3], dC = g2s[4], dop = g2s[5];
        float drc[3] = {g2s[6], g2s[7], g2s[8]};
        // ---- recompute forward quantities (from the staged rows) ----
        const float* mus = smem + L::kMu + sh[0] + 3 * tid;
        const float mu[3] = {mus[0], mus[1], mus[2]};
        const float xh = W[0] * mu[0] + W[1] * mu[1] + W[2] * mu[2] + W[3];
        const float yh = W[4] * mu[0] + W[5] * mu[1] + W[6] * mu[2] + W[7];
        const float zh = W[8] * mu[0] + W[9] * mu[1] + W[10] * mu[2] + W[11];
        const float* qs = smem + L::kQ + sh[2] + 4 * tid;
        const float q0 = qs[0], q1 = qs[1], q2 = qs[2], q3 = qs[3];
        const float qn = sqrtf(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
        const float iqn = 1.f / qn;
        const float w = q0 * iqn, x = q1 * iqn, y = q2 * iqn, z = q3 * iqn;
        float R[9];
        R[0] = 1.f - 2.f * (y * y + z * z);
        R[1] = 2.f * (x * y - w * z);
        R[2] = 2.f * (x * z + w * y);
        R[3] = 2.f * (x * y + w * z);
        R[4] = 1.f - 2.f * (x * x + z * z);
        R[5] = 2.f * (y * z - w * x);
        R[6] = 2.f * (x * z - w * y);
        R[7] = 2.f * (y * z + w * x);
        R[8] = 1.f - 2.f * (x * x + y * y);
        const float* lss = smem + L::kLs + sh[1] + 3 * tid;
        float s[3];
        for (int k = 0; k < 3; ++k) s[k] = __expf(lss[k]);
        float Mm[9];
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < 3; ++k) Mm[3 * i + k] = R[3 * i + k] * s[k];
        float Sf[9];
        for (int i = 0; i < 3; ++i)
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
        for (int j = 0; j < 3; ++j) {
            Tm[j] = J00 * W[j] + J02 * W[8 + j];
            Tm[3 + j] = J11 * W[4 + j] + J12 * W[8 + j];
        }
        float TS[6];
        for (int r = 0; r < 2; ++r)
            for (int j = 0; j < 3; ++j)
                TS[3 * r + j] = Tm[3 * r] * Sf[j] + Tm[3 * r + 1] * Sf[3 + j] + Tm[3 * r + 2] * Sf[6 + j];
        const float a = TS[0] * Tm[0] + TS[1] * Tm[1] + TS[2] * Tm[2] + cfg.dilation;
        const float bb = TS[0] * Tm[3] + TS[1] * Tm[4] + TS[2] * Tm[5];
        const float c = TS[3] * Tm[3] + TS[4] * Tm[4] + TS[5] * Tm[5] + cfg.dilation;
        const float idet = 1.f / (a * c - bb * bb);
        const float A = c * idet, B = -bb * idet, C = a * idet;
        const float o = 1.f / (1.f + __expf(-smem[L::kOp + sh[3] + tid]));
        const float* dcs = smem + L::kDc + sh[4] + 3 * tid;
        // ---- colour / SH ----
        const float cpx = -(W[0] * W[3] + W[4] * W[7] + W[8] * W[11]);
        const float cpy = -(W[1] * W[3] + W[5] * W[7] + W[9] * W[11]);
        const float cpz = -(W[2] * W[3] + W[6] * W[7] + W[10] * W[11]);
        const float e0 = mu[0] - cpx, e1 = mu[1] - cpy, e2 = mu[2] - cpz;
        const float dl = sqrtf(e0 * e0 + e1 * e1 + e2 * e2);
        const float idl = 1.f / dl;
        const float d0 = e0 * idl, d1 = e1 * idl, d2 = e2 * idl;
        float* rs = smem + L::kRest + sh[8] + tid * 45;
        float* rg = ACCUM ? smem + L::kGRest + sh[9] + tid * 45 : rs;  // overwrite mode reuses the param row
        float Y[16];
        float dY[16][3];
        Y[0] = TS_SH_C0;
        for (int k = 0; k < 16; ++k) dY[k][0] = dY[k][1] = dY[k][2] = 0.f;
        if (deg >= 1) {
            Y[1] = -TS_SH_C1 * d1;
            Y[2] = TS_SH_C1 * d2;
            Y[3] = -TS_SH_C1 * d0;
            dY[1][1] = -TS_SH_C1;
            dY[2][2] = TS_SH_C1;
            dY[3][0] = -TS_SH_C1;
        }
        if (deg >= 2) {
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
            if (deg >= 3) {
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
        for (int ch = 0; ch < 3; ++ch) {
            float raw = Y[0] * dcs[ch];
            _Pragma("unroll") for (int k = 1; k < nb; ++k) raw += Y[k] * rs[3 * (k - 1) + ch];
            raw += 0.5f;
            if (raw < 0.f) drc[ch] = 0.f;
            const float d = drc[ch];
            GW(off.dc + 3 * g + ch, Y[0] * d);
            _Pragma("unroll") for (int k = 1; k < nb; ++k) {
                const float cf = rs[3 * (k - 1) + ch] * d;
                if constexpr (ACCUM) rg[3 * (k - 1) + ch] += Y[k] * d;
                else rg[3 * (k - 1) + ch] = Y[k] * d;
                ddir0 += dY[k][0] * cf;
                ddir1 += dY[k][1] * cf;
                ddir2 += dY[k][2] * cf;
            }
        }
        const float nd = d0 * ddir0 + d1 * ddir1 + d2 * ddir2;
        float dmean0 = (ddir0 - d0 * nd) * idl, dmean1 = (ddir1 - d1 * nd) * idl, dmean2 = (ddir2 - d2 * nd) * idl;
        // ---- opacity ----
        GW(off.op + g, dop * o * (1.f - o));
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
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                dS[3 * i + j] = Tm[i] * (G2[0] * Tm[j] + G2[1] * Tm[3 + j]) +
                                Tm[3 + i] * (G2[2] * Tm[j] + G2[3] * Tm[3 + j]);
        float dTm[6];
        for (int r = 0; r < 2; ++r)
            for (int j = 0; j < 3; ++j) dTm[3 * r + j] = 2.f * (G2[2 * r] * TS[j] + G2[2 * r + 1] * TS[3 + j]);
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
        dmean0 += W[0] * dtx + W[4] * dty + W[8] * dtz;
        dmean1 += W[1] * dtx + W[5] * dty + W[9] * dtz;
        dmean2 += W[2] * dtx + W[6] * dty + W[10] * dtz;
        GW(off.means + 3 * g, dmean0);
        GW(off.means + 3 * g + 1, dmean1);
        GW(off.means + 3 * g + 2, dmean2);
        // ---- Sigma = M M^T, M = R diag(s) ----
        float dM[9];
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < 3; ++k)
                dM[3 * i + k] = 2.f * (dS[3 * i] * Mm[k] + dS[3 * i + 1] * Mm[3 + k] + dS[3 * i + 2] * Mm[6 + k]);
        float dR[9];
        for (int k = 0; k < 3; ++k) {
            const float ds = R[k] * dM[k] + R[3 + k] * dM[3 + k] + R[6 + k] * dM[6 + k];
            for (int i = 0; i < 3; ++i) dR[3 * i + k] = dM[3 * i + k] * s[k];
            GW(off.ls + 3 * g + k, ds * s[k]);
        }
        const float dqw = 2.f * (-z * dR[1] + y * dR[2] + z * dR[3] - x * dR[5] - y * dR[6] + x * dR[7]);
        const float dqx = 2.f * (y * dR[1] + z * dR[2] + y * dR[3] - 2.f * x * dR[4] - w * dR[5] + z * dR[6] +
                                 w * dR[7] - 2.f * x * dR[8]);
        const float dqy = 2.f * (-2.f * y * dR[0] + x * dR[1] + w * dR[2] + x * dR[3] + z * dR[5] - w * dR[6] +
                                 z * dR[7] - 2.f * y * dR[8]);
        const float dqz = 2.f * (-2.f * z * dR[0] - w * dR[1] + x * dR[2] + w * dR[3] - 2.f * z * dR[4] +
                                 y * dR[5] + x * dR[6] + y * dR[7]);
        const float dot = w * dqw + x * dqx + y * dqy + z * dqz;
        GW(off.q + 4 * g, (dqw - w * dot) * iqn);
        GW(off.q + 4 * g + 1, (dqx - x * dot) * iqn);
        GW(off.q + 4 * g + 2, (dqy - y * dot) * iqn);
        GW(off.q + 4 * g + 3, (dqz - z * dot) * iqn);
        // ---- densification statistics ----
        accum[g] = smem[L::kAc + sh[6] + tid] + sqrtf(dmx * dmx + dmy * dmy);
        vcount[g] = smem[L::kVc + sh[7] + tid] + 1.f;
        vis[g] = 1;
    }
#undef GW
    if constexpr (!ACCUM && nrest > 0) {
        // overwrite mode: rows of inactive Gaussians and inactive SH degrees carry zeros
        if (int(threadIdx.x) < rows) {
            float* row = smem + L::kRest + sh[8] + threadIdx.x * 45;
            if (!active) {
                for (int k = 0; k < 45; ++k) row[k] = 0.f;
            } else {
                for (int k = nrest; k < 45; ++k) row[k] = 0.f;
            }
        }
    }
    __syncthreads();
    if constexpr (nrest > 0) {
        store_span<kBlock>(G + off.rest + g0 * 45,
                           (ACCUM ? smem + L::kGRest + sh[9] : smem + L::kRest + sh[8]), rows * 45);
    }
}

}  // namespace

void launch_project_bwd(Context& c, const DevCam& cam, const ts_render_config& cfg, bool accumulate) {
    if (c.N == 0) return;
    const int64_t blocks = (c.N + kBlock - 1) / kBlock;
#define TS_PB(D)                                                                                      \
    if (accumulate) {                                                                                 \
        constexpr int sm = PbLayout<D, true>::kTotal * 4;                                             \
        cudaFuncSetAttribute(project_bwd_kernel<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); \
        project_bwd_kernel<D, true><<<unsigned(blocks), kBlock, sm, c.stream>>>(                      \
            c.params.p, c.grads.p, c.g2d.p, c.tcount.p, c.accum.p, c.vcount.p, c.vis.p, c.N, cam, cfg); \
    } else {                                                                                          \
        constexpr int sm = PbLayout<D, false>::kTotal * 4;                                            \
        cudaFuncSetAttribute(project_bwd_kernel<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); \
        project_bwd_kernel<D, false><<<unsigned(blocks), kBlock, sm, c.stream>>>(                     \
            c.params.p, c.grads.p, c.g2d.p, c.tcount.p, c.accum.p, c.vcount.p, c.vis.p, c.N, cam, cfg); \
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

}  // namespace ts
