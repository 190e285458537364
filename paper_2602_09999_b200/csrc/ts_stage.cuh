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

namespace ts {

// A contiguous run of 4-byte words to stage: src (global, 4-byte aligned) ->
// dst (shared, 16-byte aligned, count + 4 words of room).
struct Span {
    float* dst;
    const float* src;
    int count;
};

// Stage NS spans with ONE barrier-free pass: every thread issues up to
// kUnroll independent 16-byte loads across all spans before storing any of
// them, so a CTA has its whole working set in flight at once (the per-Gaussian
// attribute blocks of the flat 59*N layout are separate contiguous runs).
// shift[s] locates element 0 of span s in its dst (see stage_span).
template <int kThreads, int NS, int kUnroll = 8>
__device__ __forceinline__ void stage_spans(const Span (&sp)[NS], int (&shift)[NS]) {
    int start[NS + 1];
    const float4* s4[NS];
    start[0] = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(sp[s].src);
        shift[s] = int((a & 15u) >> 2);
        s4[s] = reinterpret_cast<const float4*>(a - uintptr_t(shift[s]) * 4u);
        const int n4 = sp[s].count > 0 ? (sp[s].count + shift[s] + 3) >> 2 : 0;
        start[s + 1] = start[s] + n4;
    }
    const int total = start[NS];
    for (int base = threadIdx.x; base < total; base += kUnroll * kThreads) {
        float4 r[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int i = base + u * kThreads;
            if (i < total) {
                const float4* p = s4[0] + i;
#pragma unroll
                for (int s = 1; s < NS; ++s)
                    if (i >= start[s]) p = s4[s] + (i - start[s]);
                r[u] = __ldg(p);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int i = base + u * kThreads;
            if (i < total) {
                float4* d = reinterpret_cast<float4*>(sp[0].dst) + i;
#pragma unroll
                for (int s = 1; s < NS; ++s)
                    if (i >= start[s]) d = reinterpret_cast<float4*>(sp[s].dst) + (i - start[s]);
                *d = r[u];
            }
        }
    }
}

}  // namespace ts
