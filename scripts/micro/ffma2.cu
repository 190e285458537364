// Microbenchmark: issue throughput of FFMA (3-reg) vs FFMA2 (packed f32x2) on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2(float a, float b) {
    unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
template <int ILP>
__global__ void k_ffma(float* out, int iters, float s) {
    float x[ILP], y = s * 1.0001f, z = s * 0.9999f;
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(y), "f"(z));
    float acc = 0; for (int i = 0; i < ILP; ++i) acc += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int ILP>
__global__ void k_ffma2(float* out, int iters, float s) {
    unsigned long long x[ILP], y = f2(s * 1.0001f, s * 1.0002f), z = f2(s * 0.9999f, s * 0.9998f);
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = f2(threadIdx.x + i, threadIdx.x - i);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(y), "l"(z));
    float acc = 0; for (int i = 0; i < ILP; ++i) { acc += __int_as_float(int(x[i])) + __int_as_float(int(x[i] >> 32)); }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int ILP>
__global__ void k_mix(float* out, int iters, float s) {   // FFMA2 interleaved with integer ALU ops
    unsigned long long x[ILP], y = f2(s * 1.0001f, s * 1.0002f), z = f2(s * 0.9999f, s * 0.9998f);
    unsigned u[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) { x[i] = f2(threadIdx.x + i, threadIdx.x - i); u[i] = threadIdx.x * (i + 3); }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(y), "l"(z));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[i]) : "r"(it), "r"(i));
        }
    float acc = 0; for (int i = 0; i < ILP; ++i) { acc += __int_as_float(int(x[i])) + __int_as_float(int(x[i] >> 32)) + u[i]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int ILP>
__global__ void k_ex2(float* out, int iters, float s) {
    float x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = (threadIdx.x + i) * 1e-3f;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
    float acc = 0; for (int i = 0; i < ILP; ++i) acc += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4 * 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096, blocks = sms * 8, threads = 256;
    auto run = [&](const char* name, void (*kern)(float*, int, float), double ops_per_inner) {
        kern<<<blocks, threads>>>(out, iters, 1.f);
        cudaEventRecord(a);
        kern<<<blocks, threads>>>(out, iters, 1.f);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double warp_instr = double(blocks) * threads / 32 * iters * ops_per_inner;
        double per_sm_clk = warp_instr / sms / (ms * 1e-3 * clk * 1e3);
        printf("%-8s %.3f ms  warp-instr/SM/clk = %.2f (at %d MHz nominal)\n", name, ms, per_sm_clk, clk / 1000);
    };
    run("ffma", k_ffma<8>, 8);
    run("ffma2", k_ffma2<8>, 8);
    run("mix", k_mix<8>, 16);
    run("ex2", k_ex2<8>, 8);
    return 0;
}
