// K10 fused Adam and layout helpers.
//
// Adam: one linear float4 sweep over the flat 59*N buffer; per element the SPEC's
// literal op sequence with explicit round-to-nearest ops, so every
// mode is bitwise equal to adam_step_reference and to the
// oracle's restatement.  "fused" is the single sweep itself (moments and update in
// one pass); the per-element arithmetic is the reference's.
// Reads theta, g, m, v and writes theta, m, v (28 B/element, HBM-bound); with
// zero_grads the gradient is cleared in the same pass (+4 B).
#include <cmath>
#include <cstring>

#include "ts_internal.cuh"
#include "ts_math.cuh"

namespace ts {
namespace {

struct AdamArgs {
    float lr[6];
    float b1, b2, omb1, omb2, eps, bc1, bc2;
    int mode, zero;
};

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
// DEV (graph-captured step): the per-step arguments come from device memory (written before each
// launch) and a voided step (capacity check) does nothing; the host path keeps them in the
// kernel's parameter bank
template <int MODE, bool ZERO, bool DEV>
__global__ void __launch_bounds__(256) adam_kernel(float4* __restrict__ th, float4* __restrict__ g,
                                                   float4* __restrict__ m, float4* __restrict__ v, uint32_t q0,
                                                   uint32_t q1, uint32_t begin, uint32_t end, Bounds bd, AdamArgs a_host,
                                                   const uint8_t* __restrict__ vis,
                                                   const AdamArgs* __restrict__ a_dev,
                                                   const uint32_t* __restrict__ gflag) {
    const uint32_t q = q0 + blockIdx.x * 256u + threadIdx.x;
    if (q >= q1) return;
    if (DEV && *gflag) return;
    const AdamArgs& a = DEV ? *a_dev : a_host;
    float4 t4 = th[q], g4 = g[q], m4 = m[q], v4 = v[q];
    float* tp = &t4.x;
    float* gp = &g4.x;
    float* mp = &m4.x;
    float* vp = &v4.x;
    const tsx::RcpConst c1 = tsx::rcp_const(a.bc1), c2 = tsx::rcp_const(a.bc2);
    const float b1 = a.b1, b2 = a.b2, omb1 = a.omb1, omb2 = a.omb2, eps = a.eps;
    auto lr_of = [&](uint32_t i) {
        return i < bd.b1 ? a.lr[0] : i < bd.b2 ? a.lr[1] : i < bd.b3 ? a.lr[2] : i < bd.b4 ? a.lr[3] : i < bd.b5 ? a.lr[4] : a.lr[5];
    };
    const uint32_t i0 = 4u * q;
    // the quad inside [begin, end) and inside one parameter group (all but a handful of quads
    // when N % 4 != 0): one learning rate, no per-element range tests
    const bool uniform = i0 >= begin && i0 + 3u < end && lr_of(i0) == lr_of(i0 + 3u);
    if (uniform && MODE != 2) {
        const float lr = lr_of(i0);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            tsx::adam_elem(tp[k], gp[k], mp[k], vp[k], lr, b1, b2, omb1, omb2, eps, c1, c2);
            if (ZERO) gp[k] = 0.f;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t i = i0 + k;
            if (i < begin || i >= end) continue;
            if (visible_of<MODE>(i, bd, vis))
                tsx::adam_elem(tp[k], gp[k], mp[k], vp[k], lr_of(i), b1, b2, omb1, omb2, eps, c1, c2);
            if (ZERO) gp[k] = 0.f;
        }
    }
    th[q] = t4;
    m[q] = m4;
    v[q] = v4;
    if (ZERO) g[q] = g4;
}

// compute_sampling_rates: per Gaussian the max over cameras whose
// J-clamp frustum contains the mean of max(fx, fy) / z; 1 / extent when none.  Same
// op order as the oracle's tso_compute_sampling_rates (project_mean, exact ops).
__global__ void sampling_rate_kernel(const float* __restrict__ means, int64_t N, const DevCam* __restrict__ cams,
                                     int ncams, float fallback, float* __restrict__ nu) {
    using namespace tsx;
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= N) return;
    const float m0 = means[3 * g], m1 = means[3 * g + 1], m2 = means[3 * g + 2];
    float best = 0.f;
    bool any = false;
    for (int k = 0; k < ncams; ++k) {
        const DevCam& cam = cams[k];
        const float* W = cam.W;
        const float xh = add(add(add(mul(W[0], m0), mul(W[1], m1)), mul(W[2], m2)), W[3]);
        const float yh = add(add(add(mul(W[4], m0), mul(W[5], m1)), mul(W[6], m2)), W[7]);
        const float zh = add(add(add(mul(W[8], m0), mul(W[9], m1)), mul(W[10], m2)), W[11]);
        if (!(zh > cam.nearp)) continue;
        const float limx = mul(1.3f, div(mul(0.5f, float(cam.w)), cam.fx));
        const float limy = mul(1.3f, div(mul(0.5f, float(cam.h)), cam.fy));
        const float tx = div(xh, zh), ty = div(yh, zh);
        if (tx < -limx || tx > limx || ty < -limy || ty > limy) continue;
        const float v = div(cam.fx > cam.fy ? cam.fx : cam.fy, zh);
        best = any ? (v > best ? v : best) : v;
        any = true;
    }
    nu[g] = any ? best : fallback;
}

// apply_3d_filter_clip: log_scales <- max(log_scales, log(sqrt(kappa) / nu))
__global__ void filter3d_clip_kernel(float* __restrict__ ls, const float* __restrict__ nu, int64_t N, float sk) {
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= N) return;
    const float fl = tsx::logf_det(tsx::div(sk, nu[g]));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float l = ls[3 * g + k];
        ls[3 * g + k] = l < fl ? fl : l;
    }
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

AdamArgs adam_args(const ts_adam_config& a) {
    AdamArgs x;
    for (int k = 0; k < 6; ++k) x.lr[k] = a.lr[k];
    x.b1 = a.beta1;
    x.b2 = a.beta2;
    x.omb1 = 1.0f - a.beta1;
    x.omb2 = 1.0f - a.beta2;
    x.eps = a.eps;
    x.bc1 = a.bc1;
    x.bc2 = a.bc2;
    x.mode = a.mode;
    x.zero = a.zero_grads;
    return x;
}

}  // namespace

// per-step Adam arguments for a captured graph: copied to c.adam_dev before each launch
size_t adam_args_bytes(const ts_adam_config& a, void* out) {
    const AdamArgs x = adam_args(a);
    std::memcpy(out, &x, sizeof(x));
    return sizeof(x);
}

void launch_adam(Context& c, const ts_adam_config& a, int64_t begin, int64_t end) {
    if (end <= begin) return;
    const AdamArgs x = adam_args(a);
    const uint32_t N = uint32_t(c.N);
    const Bounds bd{3u * N, 6u * N, 10u * N, 11u * N, 14u * N};
    const uint32_t q0 = uint32_t(begin / 4), q1 = uint32_t((end + 3) / 4);
    const unsigned blocks = (q1 - q0 + 255u) / 256u;
    auto* th = reinterpret_cast<float4*>(c.params.p);
    auto* g = reinterpret_cast<float4*>(c.grads.p);
    auto* m = reinterpret_cast<float4*>(c.m.p);
    auto* v = reinterpret_cast<float4*>(c.v.p);
    const uint32_t b = uint32_t(begin), e = uint32_t(end);
    const AdamArgs* xd = nullptr;
    if (c.gmode) {  // the graph reads this step's arguments from device memory (graph_step writes them)
        static_assert(sizeof(AdamArgs) <= sizeof(c.adam_dev_bytes), "adam args");
        xd = reinterpret_cast<const AdamArgs*>(c.adam_dev);
    }
    const uint32_t* gf = c.gmode ? c.counters.p + kGraphFlag : nullptr;
#define TS_ADAM(MODE, Z)                                                                                      \
    if (c.gmode)                                                                                              \
        adam_kernel<MODE, Z, true><<<blocks, 256, 0, c.stream>>>(th, g, m, v, q0, q1, b, e, bd, x, c.vis.p, xd, gf); \
    else                                                                                                      \
        adam_kernel<MODE, Z, false><<<blocks, 256, 0, c.stream>>>(th, g, m, v, q0, q1, b, e, bd, x, c.vis.p, xd, gf)
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

bool launch_sampling_rates(Context& c, const DevCam* cams_host, int ncams, float extent) {
    if (c.N == 0) return true;
    if (!ensure_grow(c, c.cams, size_t(ncams))) return false;
    cudaMemcpyAsync(c.cams.p, cams_host, sizeof(DevCam) * ncams, cudaMemcpyHostToDevice, c.stream);
    sampling_rate_kernel<<<unsigned((c.N + 255) / 256), 256, 0, c.stream>>>(c.params.p, c.N, c.cams.p, ncams,
                                                                            1.0f / extent, c.nu_hat.p);
    TS_LAUNCHED(c);
    // cams_host is the caller's (pageable) array: the copy has completed when this returns
    return cudaStreamSynchronize(c.stream) == cudaSuccess;
}

void launch_filter3d_clip(Context& c, float kappa3d) {
    if (c.N == 0) return;
    filter3d_clip_kernel<<<unsigned((c.N + 255) / 256), 256, 0, c.stream>>>(c.params.p + 3 * c.N, c.nu_hat.p, c.N,
                                                                            std::sqrt(kappa3d));
    TS_LAUNCHED(c);
}

void launch_hwc_to_chw(Context& c, const float* hwc, float* chw, int P, cudaStream_t st) {
    hwc_to_chw_kernel<<<(P + 255) / 256, 256, 0, st ? st : c.stream>>>(hwc, chw, P);
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

}  // namespace ts
