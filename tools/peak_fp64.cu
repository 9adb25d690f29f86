// Measured fp64 tensor-core (DMMA.8x8x4) and fp64 FMA peaks of this B200:
// the roofline denominator for the K3 scorer (MEASURED_PEAKS.json has only
// HBM and bf16).  Every warp runs 16 independent accumulator chains.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double *out, int iters) {
    double acc[16][2];
    for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 16; ++i) s += acc[i][0] + acc[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double *out, int iters) {
    double acc[16];
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x;
    const double a = 1.0000001, b = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 16; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int n_sm = 0;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, sizeof(double) * n_sm * 8 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096, blocks = n_sm * 4, threads = 256;
    float best_dmma = 1e30f, best_dfma = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        k_dmma<<<blocks, threads>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) best_dmma = ms < best_dmma ? ms : best_dmma;
        cudaEventRecord(a);
        k_dfma<<<blocks, threads>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (rep) best_dfma = ms < best_dfma ? ms : best_dfma;
    }
    const double warps = (double)blocks * threads / 32;
    const double dmma_flop = warps * iters * 16 * 512.0;             // 8x8x4 MACs x 2 per DMMA
    const double dfma_flop = (double)blocks * threads * iters * 16 * 2.0;
    printf("{\"fp64_dmma_tflops\": %.2f, \"fp64_fma_tflops\": %.2f, \"sms\": %d, "
           "\"how\": \"tools/peak_fp64.cu: %d blocks x %d threads, 16 independent DMMA.8x8x4 (resp. DFMA) chains "
           "per thread x %d iterations, best of 4 CUDA-event timings\"}\n",
           dmma_flop / best_dmma / 1e9, dfma_flop / best_dfma / 1e9, n_sm, blocks, threads, iters);
    return 0;
}
