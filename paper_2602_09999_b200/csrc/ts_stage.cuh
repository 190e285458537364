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

namespace ts {

// ---------------------------------------------------------------------------
// TMA bulk staging (cp.async.bulk global -> shared, completion on an mbarrier).
// One elected thread issues one bulk copy per span; the copy engine moves the
// bytes, so staging costs a handful of instructions per CTA instead of a loop
// per 16-byte chunk.  Spans are copied from the 16-byte-aligned address at or
// below src (shift as in stage_span); callers' global buffers are padded so the
// rounded-up tail stays in bounds.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// bulk L2 prefetch of count floats at src (16-byte granularity; rounded outward,
// callers' buffers are padded)
__device__ __forceinline__ void prefetch_l2(const float* src, int count) {
    if (count <= 0) return;
    const uintptr_t a = reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15);
    const uintptr_t e = (reinterpret_cast<uintptr_t>(src + count) + 15) & ~uintptr_t(15);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(uint32_t(e - a)) : "memory");
}

// wait for phase 0 of an mbarrier
__device__ __forceinline__ void mbar_wait0(unsigned long long* bar) {
    uint32_t ready = 0;
    while (!ready) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ready)
            : "r"(smem_u32(bar))
            : "memory");
    }
}

// issue the bulk copies of NS spans on an (initialised, visible) mbarrier; thread 0 only
template <int NS>
__device__ __forceinline__ void tma_issue_spans(const Span (&sp)[NS], int (&shift)[NS], unsigned long long* bar) {
    uint32_t bytes[NS];
    const char* src[NS];
    uint32_t total = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(sp[s].src);
        shift[s] = int((a & 15u) >> 2);
        src[s] = reinterpret_cast<const char*>(a - uintptr_t(shift[s]) * 4u);
        bytes[s] = sp[s].count > 0 ? uint32_t(((sp[s].count + shift[s]) * 4 + 15) & ~15) : 0u;
        total += bytes[s];
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(total)
                     : "memory");
#pragma unroll
        for (int s = 0; s < NS; ++s)
            if (bytes[s])
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(sp[s].dst)),
                    "l"(src[s]), "r"(bytes[s]), "r"(smem_u32(bar))
                    : "memory");
    }
}

__device__ __forceinline__ void mbar_init_all(unsigned long long* bars, int n) {
    if (threadIdx.x == 0) {
        for (int k = 0; k < n; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + k)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
}

template <int NS>
__device__ __forceinline__ void stage_spans_tma(const Span (&sp)[NS], int (&shift)[NS], unsigned long long* bar) {
    mbar_init_all(bar, 1);
    tma_issue_spans(sp, shift, bar);
    mbar_wait0(bar);
}

}  // namespace ts
