// K11 densify_compact (order DESIGN.md App. A.10).
// predicate (per Gaussian) -> three exclusive scans (survivors | clones |
// split children) -> stable scatter of params / moments into freshly sized
// buffers.  Moments of new rows start at zero; statistics and
// gradients are reset.  Thresholds compare in log/logit space against host
// double constants, so selection masks are bit-identical to the oracle.
#include <algorithm>

#include "ts_internal.cuh"
#include "ts_math.cuh"

namespace ts {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ float u01(uint64_t seed, int64_t iter, int64_t parent, int code) {
    const uint64_t h = mix64(mix64(mix64(seed ^ mix64(uint64_t(iter))) ^ uint64_t(parent)) ^ uint64_t(code));
    return tsx::mul(tsx::add(float(h >> 40), 0.5f), 0x1.0p-24f);
}

struct DensArgs {
    float thresh, log_small, log_big, logit_min;
};

__device__ __forceinline__ float qnorm(const float* q) {
    using namespace tsx;
    return sqrt_(add(add(add(mul(q[0], q[0]), mul(q[1], q[1])), mul(q[2], q[2])), mul(q[3], q[3])));
}

__global__ void densify_flags_kernel(const float* __restrict__ P, const float* __restrict__ accum,
                                     const float* __restrict__ vcount, int64_t N, DensArgs a,
                                     uint32_t* __restrict__ fA, uint32_t* __restrict__ fB,
                                     uint32_t* __restrict__ fC, uint32_t* __restrict__ st) {
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= N) return;
    const Off off(N);
    const float* ls = P + off.ls + 3 * g;
    float q[4] = {P[off.q + 4 * g], P[off.q + 4 * g + 1], P[off.q + 4 * g + 2], P[off.q + 4 * g + 3]};
    const float mls = fmaxf(ls[0], fmaxf(ls[1], ls[2]));
    const float qn = qnorm(q);
    const bool sel = vcount[g] > 0.f && tsx::div(accum[g], vcount[g]) > a.thresh;
    const bool small = mls <= a.log_small;
    const bool prc = (P[off.op + g] < a.logit_min) || !(qn >= 1e-4f);
    const bool prn = prc || (mls > a.log_big);
    const float mlc = tsx::sub(mls, 0x1.e148a2p-2f);
    const bool pchild = prc || (mlc > a.log_big);
    const bool split = sel && !small;
    fA[g] = (!split && !prn) ? 1u : 0u;
    fB[g] = (sel && small && !prn) ? 1u : 0u;
    fC[g] = (split && !pchild) ? 2u : 0u;
    // pruned rows of the post-densify set: the original, its clone, or both children
    uint32_t pruned = (!split && prn) ? 1u : 0u;
    if (sel && small && prn) pruned += 1u;
    if (split && pchild) pruned += 2u;
    if (sel && small) atomicAdd(st + 0, 1u);
    if (split) atomicAdd(st + 1, 1u);
    if (pruned) atomicAdd(st + 2, pruned);
}

// Element-parallel copy, one pass per array (WHICH 0 = parameters, 1 / 2 = first / second
// Adam moment) into a fresh 59*NA buffer: thread i reads element i of the source store
// (coalesced over every attribute block) and writes it to the rows of its Gaussian in the
// compacted layout -- the kept row (runs of consecutive survivors stay coalesced), the clone
// row and the two split-child rows (moments of new rows are zero).  Every
// destination row is written exactly once, so the output needs no clear.
template <int WD, int WHICH>
__device__ __forceinline__ void copy_elem(float x, uint32_t r, uint32_t dbase, const uint32_t* __restrict__ fA,
                                          const uint32_t* __restrict__ fB, const uint32_t* __restrict__ fC,
                                          const uint32_t* __restrict__ oA, const uint32_t* __restrict__ oB,
                                          const uint32_t* __restrict__ oC, uint32_t nA, uint32_t nB,
                                          float* __restrict__ O) {
    const uint32_t g = r / uint32_t(WD), j = r - g * uint32_t(WD);
    if (__ldg(fA + g)) O[dbase + uint32_t(WD) * __ldg(oA + g) + j] = x;
    const float y = WHICH == 0 ? x : 0.f;
    if (__ldg(fB + g)) O[dbase + uint32_t(WD) * (nA + __ldg(oB + g)) + j] = y;
    if (__ldg(fC + g)) {
        const uint32_t c0 = nA + nB + __ldg(oC + g);
        O[dbase + uint32_t(WD) * c0 + j] = y;        // children start as copies of the parent;
        O[dbase + uint32_t(WD) * (c0 + 1) + j] = y;  // densify_children_kernel sets means / scales
    }
}

template <int WHICH>
__global__ void __launch_bounds__(256) densify_copy_kernel(const float* __restrict__ src, uint32_t N,
                                                           const uint32_t* __restrict__ fA,
                                                           const uint32_t* __restrict__ fB,
                                                           const uint32_t* __restrict__ fC,
                                                           const uint32_t* __restrict__ oA,
                                                           const uint32_t* __restrict__ oB,
                                                           const uint32_t* __restrict__ oC, uint32_t nA, uint32_t nB,
                                                           uint32_t NA, float* __restrict__ O) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 59u * N) return;
    const float x = src[i];
    if (i < 3u * N) copy_elem<3, WHICH>(x, i, 0u, fA, fB, fC, oA, oB, oC, nA, nB, O);
    else if (i < 6u * N) copy_elem<3, WHICH>(x, i - 3u * N, 3u * NA, fA, fB, fC, oA, oB, oC, nA, nB, O);
    else if (i < 10u * N) copy_elem<4, WHICH>(x, i - 6u * N, 6u * NA, fA, fB, fC, oA, oB, oC, nA, nB, O);
    else if (i < 11u * N) copy_elem<1, WHICH>(x, i - 10u * N, 10u * NA, fA, fB, fC, oA, oB, oC, nA, nB, O);
    else if (i < 14u * N) copy_elem<3, WHICH>(x, i - 11u * N, 11u * NA, fA, fB, fC, oA, oB, oC, nA, nB, O);
    else copy_elem<45, WHICH>(x, i - 14u * N, 14u * NA, fA, fB, fC, oA, oB, oC, nA, nB, O);
}

// Split children: mean = parent mean + R (s * z), z ~ N(0, I) by Box-Muller from
// a counter-based hash of (seed, iteration, parent, code), with the deterministic log / cos
// (ts_math.cuh), so children equal the oracle's bit for bit; log-scales = parent - ln 1.6.
__global__ void densify_children_kernel(const float* __restrict__ P, uint32_t N, const uint32_t* __restrict__ fC,
                                        const uint32_t* __restrict__ oC, uint32_t nA, uint32_t nB, uint32_t NA,
                                        float* __restrict__ O, uint64_t seed, int64_t iter) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= N || !fC[g]) return;
    using namespace tsx;
    const Off so(N), d(NA);
    const float* ls = P + so.ls + 3 * int64_t(g);
    float q[4] = {P[so.q + 4 * int64_t(g)], P[so.q + 4 * int64_t(g) + 1], P[so.q + 4 * int64_t(g) + 2],
                  P[so.q + 4 * int64_t(g) + 3]};
    const float qn = qnorm(q);
    const float w = div(q[0], qn), x = div(q[1], qn), y = div(q[2], qn), z = div(q[3], qn);
    const float R[9] = {sub(1.f, mul(2.f, add(mul(y, y), mul(z, z)))), mul(2.f, sub(mul(x, y), mul(w, z))),
                        mul(2.f, add(mul(x, z), mul(w, y))),           mul(2.f, add(mul(x, y), mul(w, z))),
                        sub(1.f, mul(2.f, add(mul(x, x), mul(z, z)))), mul(2.f, sub(mul(y, z), mul(w, x))),
                        mul(2.f, sub(mul(x, z), mul(w, y))),           mul(2.f, add(mul(y, z), mul(w, x))),
                        sub(1.f, mul(2.f, add(mul(x, x), mul(y, y))))};
    for (int child = 0; child < 2; ++child) {
        const int64_t r = int64_t(nA) + nB + oC[g] + child;
        float zs[3];
        for (int k = 0; k < 3; ++k) {
            const float a1 = u01(seed, iter, g, child * 8 + k * 2);
            const float a2 = u01(seed, iter, g, child * 8 + k * 2 + 1);
            zs[k] = mul(sqrt_(mul(-2.0f, logf_det(a1))), cos2pi_det(a2));
            zs[k] = mul(zs[k], expf_det(ls[k]));
        }
        for (int i = 0; i < 3; ++i)
            O[d.means + 3 * r + i] = add(P[so.means + 3 * int64_t(g) + i],
                                         add(add(mul(R[3 * i], zs[0]), mul(R[3 * i + 1], zs[1])), mul(R[3 * i + 2], zs[2])));
        for (int k = 0; k < 3; ++k) O[d.ls + 3 * r + k] = sub(ls[k], 0x1.e148a2p-2f);
    }
}

}  // namespace

int64_t launch_densify(Context& c, float thresh, float log_small, float log_big, float logit_min, uint64_t seed,
                       int64_t iter, int64_t stats[3]) {
    const int64_t N = c.N;
    c.err.clear();
    if (!ensure(c, c.dens, size_t(6) * (N + 1))) return -1;
    uint32_t* fA = c.dens.p;
    uint32_t* fB = fA + (N + 1);
    uint32_t* fC = fB + (N + 1);
    uint32_t* oA = fC + (N + 1);
    uint32_t* oB = oA + (N + 1);
    uint32_t* oC = oB + (N + 1);
    cudaMemsetAsync(c.counters.p + 4, 0, 3 * sizeof(uint32_t), c.stream);
    DensArgs a{thresh, log_small, log_big, logit_min};
    const int bs = 256;
    const unsigned blocks = unsigned(std::max<int64_t>(1, (N + bs - 1) / bs));
    if (N) {
        densify_flags_kernel<<<blocks, bs, 0, c.stream>>>(c.params.p, c.accum.p, c.vcount.p, N, a, fA, fB, fC,
                                                         c.counters.p + 4);
        TS_LAUNCHED(c);
    }
    launch_exclusive_scan(c, fA, nullptr, oA, N);
    launch_exclusive_scan(c, fB, nullptr, oB, N);
    launch_exclusive_scan(c, fC, nullptr, oC, N);
    uint32_t tot[3], st[3];
    cudaMemcpyAsync(&tot[0], oA + N, 4, cudaMemcpyDeviceToHost, c.stream);
    cudaMemcpyAsync(&tot[1], oB + N, 4, cudaMemcpyDeviceToHost, c.stream);
    cudaMemcpyAsync(&tot[2], oC + N, 4, cudaMemcpyDeviceToHost, c.stream);
    cudaMemcpyAsync(st, c.counters.p + 4, sizeof(st), cudaMemcpyDeviceToHost, c.stream);
    if (cudaStreamSynchronize(c.stream) != cudaSuccess) return -1;
    const int64_t nA = tot[0], nB = tot[1], nC = tot[2], NA = nA + nB + nC;
    if (NA > kMaxGaussians) {  // nothing has been modified yet
        c.err = "densify would exceed the 32-bit flat-index limit (~72.8M Gaussians)";
        return -2;
    }
    const size_t L = (size_t(59) * std::max<int64_t>(NA, 1) + 7) & ~size_t(3);
    // three passes through one spare 59*NA buffer, swapped in after each pass (no per-call
    // allocation of the new store; capacities grow with slack, so growth reallocates rarely)
    float** arrs[3] = {&c.params.p, &c.m.p, &c.v.p};
    DevBuf<float>* bufs[3] = {&c.params, &c.m, &c.v};
    for (int w = 0; w < 3; ++w) {
        if (!ensure_grow(c, c.spare, L)) return -1;
        if (N) {
            const float* src = *arrs[w];
            const unsigned eb = unsigned((59 * N + 255) / 256);
            const uint32_t n32 = uint32_t(N), a32 = uint32_t(nA), b32 = uint32_t(nB), NA32 = uint32_t(NA);
            if (w == 0) {
                densify_copy_kernel<0><<<eb, 256, 0, c.stream>>>(src, n32, fA, fB, fC, oA, oB, oC, a32, b32, NA32,
                                                                 c.spare.p);
                densify_children_kernel<<<blocks, bs, 0, c.stream>>>(src, n32, fC, oC, a32, b32, NA32, c.spare.p,
                                                                     seed, iter);
                TS_LAUNCHED(c);
            } else if (w == 1) {
                densify_copy_kernel<1><<<eb, 256, 0, c.stream>>>(src, n32, fA, fB, fC, oA, oB, oC, a32, b32, NA32,
                                                                 c.spare.p);
            } else {
                densify_copy_kernel<2><<<eb, 256, 0, c.stream>>>(src, n32, fA, fB, fC, oA, oB, oC, a32, b32, NA32,
                                                                 c.spare.p);
            }
            TS_LAUNCHED(c);
        } else {
            cudaMemsetAsync(c.spare.p, 0, L * 4, c.stream);
        }
        std::swap(*bufs[w], c.spare);
        ++c.gen;  // buffer addresses changed (captured graphs are stale)
    }
    c.N = NA;
    // resize the remaining per-Gaussian buffers and reset gradients / statistics
    const size_t n1 = size_t(std::max<int64_t>(NA, 1));
    if (!ensure_grow(c, c.grads, L) || !ensure_grow(c, c.accum, n1 + 4) || !ensure_grow(c, c.vcount, n1 + 4) ||
        !ensure_grow(c, c.splat, 3 * n1) || !ensure_grow(c, c.rect, n1) || !ensure_grow(c, c.tcount, n1) ||
        !ensure_grow(c, c.dkey[0], n1) || !ensure_grow(c, c.dkey[1], n1) || !ensure_grow(c, c.dperm[0], n1) ||
        !ensure_grow(c, c.dperm[1], n1) || !ensure_grow(c, c.offsets, n1 + 1) || !ensure_grow(c, c.g2d, 3 * n1 + 1) ||
        !ensure_grow(c, c.vis, n1) || !ensure_grow(c, c.nu_hat, n1) || !ensure_grow(c, c.ryv, n1))
        return -1;
    c.nu_valid = false;  // new rows: the sampling rates must be recomputed (SPEC.md:614 interval)
    cudaMemsetAsync(c.grads.p, 0, c.grads.cap * 4, c.stream);
    cudaMemsetAsync(c.accum.p, 0, n1 * 4, c.stream);
    cudaMemsetAsync(c.vcount.p, 0, n1 * 4, c.stream);
    cudaMemsetAsync(c.g2d.p, 0, 3 * n1 * 16, c.stream);
    cudaMemsetAsync(c.vis.p, 0, n1, c.stream);
    stats[0] = st[0];
    stats[1] = st[1];
    stats[2] = st[2];
    return NA;
}

}  // namespace ts
