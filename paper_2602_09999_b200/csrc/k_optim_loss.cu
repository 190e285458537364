// K10 fused Adam, K7 training loss and
// layout helpers.
//
// Adam: one linear float4 sweep over the flat 59*N buffer; per element a fixed
// sequence of explicit round-to-nearest ops (reference = SPEC literal formula,
// fused = bias corrections folded into host constants: one IEEE sqrt and one
// IEEE division per element), bitwise equal to the oracle's restatement.
// Reads theta, g, m, v and writes theta, m, v (28 B/element, HBM-bound); with
// zero_grads the gradient is cleared in the same pass (+4 B).
//
// Loss: 0.8 L1 + 0.2 (1 - SSIM), 11x11 Gaussian window (sigma 1.5), reflect
// padding; analytic dL/dC via the transposed (fold) separable filter.
#include <cmath>

#include "ts_internal.cuh"
#include "ts_math.cuh"

namespace ts {
namespace {

struct AdamArgs {
    float lr[6];      // reference: lr ; fused: lr / (1 - b1^t) (host double -> float)
    float b1, b2, omb1, omb2, eps, bc1, bc2;
    float rsb2;       // fused: 1 / sqrt(1 - b2^t) (host double -> float)
    int mode, zero;
};

// reference (SPEC.md:466 literal): theta -= lr * (m / bc1) / (sqrt(v / bc2) + eps)
// fused:         theta -= (lr/bc1) * m / (sqrt(v) * (1/sqrt(bc2)) + eps)
// Both fixed op sequences with explicit round-to-nearest ops; the oracle
// restates each bit for bit.
template <bool kFused>
__device__ __forceinline__ void adam_one(float& th, float& g, float& m, float& v, float lr, const AdamArgs& a) {
    using namespace tsx;
    m = add(mul(a.b1, m), mul(a.omb1, g));
    v = add(mul(a.b2, v), mul(mul(a.omb2, g), g));
    if (kFused) {
        const float den = add(mul(sqrt_(v), a.rsb2), a.eps);
        th = sub(th, div(mul(lr, m), den));
    } else {
        const float mh = div(m, a.bc1);
        const float vh = div(v, a.bc2);
        const float den = add(sqrt_(vh), a.eps);
        th = sub(th, div(mul(lr, mh), den));
    }
}

// flat-buffer group boundaries (elements): means | scales | quats | opacity | sh_dc | sh_rest
struct Bounds {
    uint32_t b1, b2, b3, b4, b5;
};

template <int MODE>
__device__ __forceinline__ bool visible_of(uint32_t i, const Bounds& b, const uint8_t* __restrict__ vis) {
    if (MODE != 2) return true;
    uint32_t gi;
    if (i < b.b1) gi = i / 3u;
    else if (i < b.b2) gi = (i - b.b1) / 3u;
    else if (i < b.b3) gi = (i - b.b2) >> 2;
    else if (i < b.b4) gi = i - b.b3;
    else if (i < b.b5) gi = (i - b.b4) / 3u;
    else gi = (i - b.b5) / 45u;
    return vis[gi] != 0;
}

// One float4 (4 consecutive elements) per thread; elements outside [begin, end)
// are written back unchanged.  Buffers are padded to a multiple of 4 floats.
template <int MODE, bool ZERO>
__global__ void __launch_bounds__(256) adam_kernel(float4* __restrict__ th, float4* __restrict__ g,
                                                   float4* __restrict__ m, float4* __restrict__ v, uint32_t q0,
                                                   uint32_t q1, uint32_t begin, uint32_t end, Bounds bd, AdamArgs a,
                                                   const uint8_t* __restrict__ vis) {
    const uint32_t q = q0 + blockIdx.x * 256u + threadIdx.x;
    if (q >= q1) return;
    float4 t4 = th[q], g4 = g[q], m4 = m[q], v4 = v[q];
    float* tp = &t4.x;
    float* gp = &g4.x;
    float* mp = &m4.x;
    float* vp = &v4.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t i = 4u * q + k;
        if (i < begin || i >= end) continue;
        const float lr = i < bd.b1 ? a.lr[0]
                         : i < bd.b2 ? a.lr[1]
                         : i < bd.b3 ? a.lr[2]
                         : i < bd.b4 ? a.lr[3]
                         : i < bd.b5 ? a.lr[4]
                                     : a.lr[5];
        if (visible_of<MODE>(i, bd, vis)) adam_one<MODE != 0>(tp[k], gp[k], mp[k], vp[k], lr, a);
        if (ZERO) gp[k] = 0.f;
    }
    th[q] = t4;
    m[q] = m4;
    v[q] = v4;
    if (ZERO) g[q] = g4;
}

__global__ void hwc_to_chw_kernel(const float* __restrict__ hwc, float* __restrict__ chw, int P) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    chw[p] = hwc[3 * p];
    chw[P + p] = hwc[3 * p + 1];
    chw[2 * P + p] = hwc[3 * p + 2];
}

__global__ void chw_to_hwc_kernel(const float* __restrict__ chw, float* __restrict__ hwc, int P) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    hwc[3 * p] = chw[p];
    hwc[3 * p + 1] = chw[P + p];
    hwc[3 * p + 2] = chw[2 * P + p];
}

__global__ void opacity_reset_kernel(float* __restrict__ op, int64_t N, float lmax) {
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g < N) op[g] = op[g] < lmax ? op[g] : lmax;
}

// ---------------------------------------------------------------------------
// loss
// ---------------------------------------------------------------------------
__constant__ float c_gw[11];
constexpr int kNPL = 11;  // temp planes per channel

__device__ __forceinline__ int refl(int i, int n) { return i < 0 ? -i : (i >= n ? 2 * (n - 1) - i : i); }

// horizontal pass: 5 window moments of x, y
__global__ void loss_h_kernel(const float* __restrict__ X, const float* __restrict__ Y, float* __restrict__ tmp,
                              int W, int H) {
    const int P = W * H;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const int ch = blockIdx.y;
    if (p >= P) return;
    const int y = p / W, x = p - y * W;
    const float* xr = X + ch * P + y * W;
    const float* yr = Y + ch * P + y * W;
    float sx = 0.f, sy = 0.f, sxx = 0.f, syy = 0.f, sxy = 0.f;
#pragma unroll
    for (int o = -5; o <= 5; ++o) {
        const int j = refl(x + o, W);
        const float a = xr[j], b = yr[j], w = c_gw[o + 5];
        sx += w * a;
        sy += w * b;
        sxx += w * a * a;
        syy += w * b * b;
        sxy += w * a * b;
    }
    float* t = tmp + size_t(ch) * kNPL * P;
    t[p] = sx;
    t[P + p] = sy;
    t[2 * P + p] = sxx;
    t[3 * P + p] = syy;
    t[4 * P + p] = sxy;
}

// vertical pass + SSIM map + partial derivatives + loss sums
__global__ void loss_v_kernel(const float* __restrict__ X, const float* __restrict__ Y, float* __restrict__ tmp,
                              int W, int H, double* __restrict__ acc) {
    const int P = W * H;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const int ch = blockIdx.y;
    float l1 = 0.f, ss = 0.f;
    if (p < P) {
        const int y = p / W, x = p - y * W;
        float* t = tmp + size_t(ch) * kNPL * P;
        float m[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int o = -5; o <= 5; ++o) {
            const int r = refl(y + o, H) * W + x;
            const float w = c_gw[o + 5];
#pragma unroll
            for (int k = 0; k < 5; ++k) m[k] += w * t[k * P + r];
        }
        const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
        const float ux = m[0], uy = m[1];
        const float vx = m[2] - ux * ux, vy = m[3] - uy * uy, cxy = m[4] - ux * uy;
        const float n1 = 2.f * ux * uy + C1, n2 = 2.f * cxy + C2;
        const float d1 = ux * ux + uy * uy + C1, d2 = vx + vy + C2;
        const float iD = 1.f / (d1 * d2);
        const float S = n1 * n2 * iD;
        const float dS_dux = (2.f * uy * n2 - S * 2.f * ux * d2) * iD;
        const float dS_dvx = -S / d2;
        const float dS_dcxy = 2.f * n1 * iD;
        t[5 * P + p] = dS_dux - 2.f * ux * dS_dvx - uy * dS_dcxy;
        t[6 * P + p] = 2.f * dS_dvx;
        t[7 * P + p] = dS_dcxy;
        ss = S;
        l1 = fabsf(X[ch * P + p] - Y[ch * P + p]);
    }
    // block reduction -> double atomics
    __shared__ float r1[32], r2[32];
    for (int o = 16; o > 0; o >>= 1) {
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        r1[wid] = l1;
        r2[wid] = ss;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) {
            a += r1[w];
            b += r2[w];
        }
        atomicAdd(acc, a);
        atomicAdd(acc + 1, b);
    }
}

// transposed filter along one axis: z(j) = sum_o g f(j - o) (f zero outside),
// folded back through the reflect padding
template <bool kVertical>
__device__ __forceinline__ float zfold(const float* f, int x, int y, int W, int H, int pos, int n) {
    auto zval = [&](int j) {
        float s = 0.f;
#pragma unroll
        for (int o = -5; o <= 5; ++o) {
            const int k = j - o;
            if (k >= 0 && k < n) s += c_gw[o + 5] * (kVertical ? f[k * W + x] : f[y * W + k]);
        }
        return s;
    };
    float r = zval(pos);
    if (pos >= 1 && pos <= 5) r += zval(-pos);
    if (pos >= n - 6 && pos <= n - 2) r += zval(2 * (n - 1) - pos);
    return r;
}

__global__ void loss_ht_kernel(float* __restrict__ tmp, int W, int H) {
    const int P = W * H;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const int ch = blockIdx.y;
    if (p >= P) return;
    const int y = p / W, x = p - y * W;
    float* t = tmp + size_t(ch) * kNPL * P;
#pragma unroll
    for (int k = 0; k < 3; ++k) t[(8 + k) * P + p] = zfold<false>(t + (5 + k) * P, x, y, W, H, x, W);
}

__global__ void loss_vt_kernel(const float* __restrict__ X, const float* __restrict__ Y, const float* __restrict__ tmp,
                               float* __restrict__ dL, int W, int H, float inv_m) {
    const int P = W * H;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const int ch = blockIdx.y;
    if (p >= P) return;
    const int y = p / W, x = p - y * W;
    const float* t = tmp + size_t(ch) * kNPL * P;
    const float ta = zfold<true>(t + 8 * P, x, y, W, H, y, H);
    const float tb = zfold<true>(t + 9 * P, x, y, W, H, y, H);
    const float tc = zfold<true>(t + 10 * P, x, y, W, H, y, H);
    const float xv = X[ch * P + p], yv = Y[ch * P + p];
    const float dS = ta + xv * tb + yv * tc;
    const float d = xv - yv;
    const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
    dL[ch * P + p] = (0.8f * sg - 0.2f * dS) * inv_m;
}

}  // namespace

void launch_adam(Context& c, const ts_adam_config& a, int64_t begin, int64_t end) {
    if (end <= begin) return;
    AdamArgs x;
    const bool fused = a.mode != 0;
    for (int k = 0; k < 6; ++k) x.lr[k] = fused ? float(double(a.lr[k]) / double(a.bc1)) : a.lr[k];
    x.b1 = a.beta1;
    x.b2 = a.beta2;
    x.omb1 = 1.0f - a.beta1;
    x.omb2 = 1.0f - a.beta2;
    x.eps = a.eps;
    x.bc1 = a.bc1;
    x.bc2 = a.bc2;
    x.rsb2 = float(1.0 / std::sqrt(double(a.bc2)));
    x.mode = a.mode;
    x.zero = a.zero_grads;
    const uint32_t N = uint32_t(c.N);
    const Bounds bd{3u * N, 6u * N, 10u * N, 11u * N, 14u * N};
    const uint32_t q0 = uint32_t(begin / 4), q1 = uint32_t((end + 3) / 4);
    const unsigned blocks = (q1 - q0 + 255u) / 256u;
    auto* th = reinterpret_cast<float4*>(c.params.p);
    auto* g = reinterpret_cast<float4*>(c.grads.p);
    auto* m = reinterpret_cast<float4*>(c.m.p);
    auto* v = reinterpret_cast<float4*>(c.v.p);
    const uint32_t b = uint32_t(begin), e = uint32_t(end);
#define TS_ADAM(MODE, Z) adam_kernel<MODE, Z><<<blocks, 256, 0, c.stream>>>(th, g, m, v, q0, q1, b, e, bd, x, c.vis.p)
    if (a.mode == 2) {
        if (a.zero_grads) TS_ADAM(2, true);
        else TS_ADAM(2, false);
    } else if (a.mode == 1) {
        if (a.zero_grads) TS_ADAM(1, true);
        else TS_ADAM(1, false);
    } else {
        if (a.zero_grads) TS_ADAM(0, true);
        else TS_ADAM(0, false);
    }
#undef TS_ADAM
    TS_LAUNCHED(c);
}

void launch_hwc_to_chw(Context& c, const float* hwc, float* chw, int P) {
    hwc_to_chw_kernel<<<(P + 255) / 256, 256, 0, c.stream>>>(hwc, chw, P);
    TS_LAUNCHED(c);
}

void launch_chw_to_hwc(Context& c, const float* chw, float* hwc, int P) {
    chw_to_hwc_kernel<<<(P + 255) / 256, 256, 0, c.stream>>>(chw, hwc, P);
    TS_LAUNCHED(c);
}

void launch_opacity_reset(Context& c, float lmax) {
    if (c.N == 0) return;
    opacity_reset_kernel<<<unsigned((c.N + 255) / 256), 256, 0, c.stream>>>(c.params.p + 10 * c.N, c.N, lmax);
    TS_LAUNCHED(c);
}

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
    const dim3 grid((P + 255) / 256, 3);
    loss_h_kernel<<<grid, 256, 0, c.stream>>>(c.rgb.p, target_chw, c.loss_tmp.p, W, H);
    loss_v_kernel<<<grid, 256, 0, c.stream>>>(c.rgb.p, target_chw, c.loss_tmp.p, W, H, c.loss_acc.p);
    loss_ht_kernel<<<grid, 256, 0, c.stream>>>(c.loss_tmp.p, W, H);
    loss_vt_kernel<<<grid, 256, 0, c.stream>>>(c.rgb.p, target_chw, c.loss_tmp.p, c.dLdC.p, W, H,
                                               float(1.0 / (3.0 * double(P))));
    c.launches += 4;
}

}  // namespace ts
