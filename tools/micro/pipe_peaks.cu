// Pipe-throughput microbenchmarks for the roofline denominators that
// MEASURED_PEAKS.json does not carry: FP64 DFMA (the FFT stages) and 32-bit
// IMAD (the candidate-hash dot products).  8 independent chains per thread,
// 4 blocks x 256 threads per SM, timed with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 pipe_peaks.cu -o pipe_peaks
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;
}

__global__ void imad_kernel(unsigned* out, unsigned a, unsigned b) {
    unsigned x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = x[k] * a + b;
    }
    unsigned s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= x[k];
    if (s == 0x12345678u) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 4, threads = 256;
    double* dout;
    cudaMalloc(&dout, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double ops = (double)blocks * threads * kIters * 8;
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(dout, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    printf("{\"fp64_fma_tflops\": %.2f, ", 2 * ops / (best * 1e-3) / 1e12);
    best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        imad_kernel<<<blocks, threads>>>((unsigned*)dout, 2654435761u, 12345u);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double imad_per_s = ops / (best * 1e-3);
    printf("\"imad_tops\": %.2f, \"imad_lanes_per_clk_per_sm\": %.1f, \"sms\": %d, "
           "\"clock_mhz\": %d}\n",
           imad_per_s / 1e12, imad_per_s / (sms * (clk * 1e3)), sms, clk / 1000);
    return 0;
}
