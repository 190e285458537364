// ts_stage.cuh — cooperative global->shared staging of contiguous float runs.
//
// Per-Gaussian SH rows are 45 floats (180 B): one thread per Gaussian reading
// its own row strides 180 B across a warp and keeps only ~4 B per thread in
// flight.  Instead a CTA copies the contiguous span of its rows with 16-byte
// vector loads, 4 independent loads per thread per round (memory-level
// parallelism), into shared memory; each thread then reads its row there
// (row stride 45 words is bank-conflict free).  The span need not be 16-byte
// aligned: the copy starts at the aligned address below it and the returned
// shift locates element 0 (callers' buffers are padded at both ends).
#pragma once
#include <cstdint>

namespace ts {

// dst must hold count + 4 floats (16-byte aligned).  Returns shift s with
// dst[s + i] == src[i] for 0 <= i < count.
template <int kThreads>
__device__ __forceinline__ int stage_span(float* __restrict__ dst, const float* __restrict__ src, int count) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    const int shift = int((a & 15u) >> 2);
    const float4* s4 = reinterpret_cast<const float4*>(a - uintptr_t(shift) * 4u);
    float4* d4 = reinterpret_cast<float4*>(dst);
    const int n4 = (count + shift + 3) >> 2;
    for (int base = threadIdx.x; base < n4; base += 4 * kThreads) {
        float4 r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = base + u * kThreads;
            if (i < n4) r[u] = __ldg(s4 + i);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = base + u * kThreads;
            if (i < n4) d4[i] = r[u];
        }
    }
    return shift;
}

// coalesced scalar store of a staged span back to global memory
template <int kThreads>
__device__ __forceinline__ void store_span(float* __restrict__ dst, const float* __restrict__ src, int count) {
    for (int i = threadIdx.x; i < count; i += kThreads) dst[i] = src[i];
}

}  // namespace ts
