// K7 training_loss: 0.8 L1 + 0.2 (1 - SSIM) with an 11x11
// Gaussian window (sigma 1.5), C1 = 0.01^2, C2 = 0.03^2, reflect padding, and the
// analytic dL/dC.  Two shared-memory-tiled kernels per 32x32 pixel tile and
// colour channel, both register-blocked (sliding windows: a thread filters 8
// consecutive columns of one row, then 4 consecutive rows of one column, so
// every staged value is loaded once per window instead of once per tap):
//   loss_fwd: reflect-padded 42x42 patch of rendered and target colour, the 5
//     separable window moments, the SSIM map and its partial derivatives
//     (a, b, c below), block-reduced L1 / SSIM sums;
//   loss_bwd: the transposed filter of (a, b, c): separable correlation of the
//     zero-extended maps, plus, for pixels within 5 of the image border, the
//     terms folded back through the reflect padding; then
//     dL/dC = (0.8 sign(x-y) - 0.2 (W^T a + x W^T b + y W^T c)) / M.
// With  mu = W x,  v = W x^2 - mu_x^2,  cov = W xy - mu_x mu_y  (per pixel):
//   dSSIM/dx_p = (W^T a)_p + x_p (W^T b)_p + y_p (W^T c)_p,
//   a = dS/dmu_x - 2 mu_x dS/dv_x - mu_y dS/dcov,  b = 2 dS/dv_x,  c = dS/dcov.
#include <cmath>

#include "ts_internal.cuh"

namespace ts {
namespace {

__constant__ float c_gw[11];
constexpr int kT = 32;           // output tile edge
constexpr int kP = kT + 10;      // padded patch edge (42)
constexpr int kPS = kP + 1;      // smem row stride
constexpr int kThreads = 256;
constexpr int kSeg = 8;          // columns per horizontal work item
constexpr int kRows = 4;         // rows per vertical work item

__device__ __forceinline__ int refl(int i, int n) { return i < 0 ? -i : (i >= n ? 2 * (n - 1) - i : i); }

__global__ void __launch_bounds__(kThreads) loss_fwd_kernel(const float* __restrict__ X, const float* __restrict__ Y,
                                                            float* __restrict__ maps, int W, int H,
                                                            double* __restrict__ acc) {
    __shared__ float sx[kP][kPS], sy[kP][kPS];
    __shared__ float hm[5][kP][kT + 1];
    const int ch = blockIdx.z, P = W * H;
    const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;
    const int tid = threadIdx.x;
    const float* Xc = X + size_t(ch) * P;
    const float* Yc = Y + size_t(ch) * P;
    for (int i = tid; i < kP * kP; i += kThreads) {
        const int r = i / kP, c = i - r * kP;
        const int gi = refl(y0 - 5 + r, H) * W + refl(x0 - 5 + c, W);
        sx[r][c] = __ldg(Xc + gi);
        sy[r][c] = __ldg(Yc + gi);
    }
    __syncthreads();
    // horizontal: (row, 8-column segment) items, sliding window of 18 inputs
    for (int it = tid; it < kP * (kT / kSeg); it += kThreads) {
        const int r = it / (kT / kSeg), c0 = (it - r * (kT / kSeg)) * kSeg;
        float a[kSeg + 10], b[kSeg + 10];
#pragma unroll
        for (int k = 0; k < kSeg + 10; ++k) {
            a[k] = sx[r][c0 + k];
            b[k] = sy[r][c0 + k];
        }
#pragma unroll
        for (int j = 0; j < kSeg; ++j) {
            float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f, m4 = 0.f;
#pragma unroll
            for (int k = 0; k < 11; ++k) {
                const float w = c_gw[k], xa = a[j + k], yb = b[j + k];
                const float wx = w * xa, wy = w * yb;
                m0 += wx;
                m1 += wy;
                m2 = fmaf(wx, xa, m2);
                m3 = fmaf(wy, yb, m3);
                m4 = fmaf(wx, yb, m4);
            }
            hm[0][r][c0 + j] = m0, hm[1][r][c0 + j] = m1, hm[2][r][c0 + j] = m2, hm[3][r][c0 + j] = m3,
            hm[4][r][c0 + j] = m4;
        }
    }
    __syncthreads();
    // vertical: (column, 4-row group) items, sliding window of 14 rows; SSIM per pixel
    const int c = tid % kT, rg = (tid / kT) * kRows;  // 32 columns x 8 groups = 256 threads
    float l1 = 0.f, ss = 0.f;
    {
        float m[kRows][5];
#pragma unroll
        for (int j = 0; j < kRows; ++j)
#pragma unroll
            for (int q = 0; q < 5; ++q) m[j][q] = 0.f;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            float win[kRows + 10];
#pragma unroll
            for (int k = 0; k < kRows + 10; ++k) win[k] = hm[q][rg + k][c];
#pragma unroll
            for (int j = 0; j < kRows; ++j)
#pragma unroll
                for (int k = 0; k < 11; ++k) m[j][q] = fmaf(c_gw[k], win[j + k], m[j][q]);
        }
        const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
        float* mp = maps + size_t(ch) * 3 * P;
#pragma unroll
        for (int j = 0; j < kRows; ++j) {
            const int x = x0 + c, y = y0 + rg + j;
            if (x >= W || y >= H) continue;
            const float ux = m[j][0], uy = m[j][1];
            const float vx = m[j][2] - ux * ux, vy = m[j][3] - uy * uy, cxy = m[j][4] - ux * uy;
            const float n1 = 2.f * ux * uy + C1, n2 = 2.f * cxy + C2;
            const float d1 = ux * ux + uy * uy + C1, d2 = vx + vy + C2;
            const float iD = 1.f / (d1 * d2);
            const float S = n1 * n2 * iD;
            const float dS_dux = (2.f * uy * n2 - S * 2.f * ux * d2) * iD;
            const float dS_dvx = -S * d1 * iD;
            const float dS_dcxy = 2.f * n1 * iD;
            const int p = y * W + x;
            mp[p] = dS_dux - 2.f * ux * dS_dvx - uy * dS_dcxy;
            mp[P + p] = 2.f * dS_dvx;
            mp[2 * P + p] = dS_dcxy;
            ss += S;
            l1 += fabsf(sx[rg + j + 5][c + 5] - sy[rg + j + 5][c + 5]);
        }
    }
    // block reduction of (L1, SSIM) -> double atomics
    __shared__ float r1[kThreads / 32], r2[kThreads / 32];
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
        for (int w = 0; w < kThreads / 32; ++w) {
            a += r1[w];
            b += r2[w];
        }
        atomicAdd(acc, a);
        atomicAdd(acc + 1, b);
    }
}

// sum over the 11x11 window of the zero-extended map f around (jx, jy)
__device__ __forceinline__ float window_sum(const float* __restrict__ f, int jx, int jy, int W, int H) {
    float s = 0.f;
    for (int oy = -5; oy <= 5; ++oy) {
        const int yy = jy + oy;
        if (yy < 0 || yy >= H) continue;
        float r = 0.f;
#pragma unroll
        for (int ox = -5; ox <= 5; ++ox) {
            const int xx = jx + ox;
            if (xx >= 0 && xx < W) r = fmaf(c_gw[ox + 5], __ldg(f + yy * W + xx), r);
        }
        s = fmaf(c_gw[oy + 5], r, s);
    }
    return s;
}

__global__ void __launch_bounds__(kThreads) loss_bwd_kernel(const float* __restrict__ X, const float* __restrict__ Y,
                                                            const float* __restrict__ maps, float* __restrict__ dL,
                                                            int W, int H, float inv_m) {
    __shared__ float sf[3][kP][kPS];
    __shared__ float hm[3][kP][kT + 1];
    const int ch = blockIdx.z, P = W * H;
    const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;
    const int tid = threadIdx.x;
    const float* mp = maps + size_t(ch) * 3 * P;
    for (int i = tid; i < kP * kP; i += kThreads) {
        const int r = i / kP, c = i - r * kP;
        const int gy = y0 - 5 + r, gx = x0 - 5 + c;
        const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
        const int gi = gy * W + gx;
#pragma unroll
        for (int q = 0; q < 3; ++q) sf[q][r][c] = in ? __ldg(mp + q * P + gi) : 0.f;
    }
    __syncthreads();
    for (int it = tid; it < kP * (kT / kSeg); it += kThreads) {
        const int r = it / (kT / kSeg), c0 = (it - r * (kT / kSeg)) * kSeg;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            float a[kSeg + 10];
#pragma unroll
            for (int k = 0; k < kSeg + 10; ++k) a[k] = sf[q][r][c0 + k];
#pragma unroll
            for (int j = 0; j < kSeg; ++j) {
                float s = 0.f;
#pragma unroll
                for (int k = 0; k < 11; ++k) s = fmaf(c_gw[k], a[j + k], s);
                hm[q][r][c0 + j] = s;
            }
        }
    }
    __syncthreads();
    const int c = tid % kT, rg = (tid / kT) * kRows;
    float t[kRows][3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        float win[kRows + 10];
#pragma unroll
        for (int k = 0; k < kRows + 10; ++k) win[k] = hm[q][rg + k][c];
#pragma unroll
        for (int j = 0; j < kRows; ++j) {
            float s = 0.f;
#pragma unroll
            for (int k = 0; k < 11; ++k) s = fmaf(c_gw[k], win[j + k], s);
            t[j][q] = s;
        }
    }
    const bool border_tile = x0 <= 5 || y0 <= 5 || x0 + kT - 1 >= W - 6 || y0 + kT - 1 >= H - 6;
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
        const int x = x0 + c, y = y0 + rg + j;
        if (x >= W || y >= H) continue;
        if (border_tile && (x <= 5 || x >= W - 6 || y <= 5 || y >= H - 6)) {
            // reflect-padding fold terms of the transposed filter
            int jx[3], jy[3], nx = 0, ny = 0;
            jx[nx++] = x;
            if (x >= 1 && x <= 5) jx[nx++] = -x;
            if (x >= W - 6 && x <= W - 2) jx[nx++] = 2 * (W - 1) - x;
            jy[ny++] = y;
            if (y >= 1 && y <= 5) jy[ny++] = -y;
            if (y >= H - 6 && y <= H - 2) jy[ny++] = 2 * (H - 1) - y;
            for (int a = 0; a < nx; ++a)
                for (int b = 0; b < ny; ++b) {
                    if (a == 0 && b == 0) continue;
                    for (int q = 0; q < 3; ++q) t[j][q] += window_sum(mp + q * P, jx[a], jy[b], W, H);
                }
        }
        const int p = y * W + x;
        const float xv = X[size_t(ch) * P + p], yv = Y[size_t(ch) * P + p];
        const float dS = t[j][0] + xv * t[j][1] + yv * t[j][2];
        const float d = xv - yv;
        const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
        dL[size_t(ch) * P + p] = (0.8f * sg - 0.2f * dS) * inv_m;
    }
}

}  // namespace

void launch_loss(Context& c, const float* target_chw) {
    static bool init = false;
    if (!init) {
        double g[11], s = 0;
        for (int i = 0; i < 11; ++i) {
            const double d = i - 5;
            g[i] = std::exp(-(d * d) / (2.0 * 1.5 * 1.5));
            s += g[i];
        }
        float gf[11];
        for (int i = 0; i < 11; ++i) gf[i] = float(g[i] / s);
        cudaMemcpyToSymbol(c_gw, gf, sizeof(gf));
        init = true;
    }
    const int W = c.fw, H = c.fh, P = W * H;
    cudaMemsetAsync(c.loss_acc.p, 0, 2 * sizeof(double), c.stream);
    const dim3 grid((W + kT - 1) / kT, (H + kT - 1) / kT, 3);
    loss_fwd_kernel<<<grid, kThreads, 0, c.stream>>>(c.rgb.p, target_chw, c.loss_tmp.p, W, H, c.loss_acc.p);
    loss_bwd_kernel<<<grid, kThreads, 0, c.stream>>>(c.rgb.p, target_chw, c.loss_tmp.p, c.dLdC.p, W, H,
                                                     float(1.0 / (3.0 * double(P))));
    c.launches += 2;
}

}  // namespace ts
