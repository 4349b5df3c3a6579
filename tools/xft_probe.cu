// FP64 peak probe for bench.py's FP64 roofline -- MEASUREMENT INFRASTRUCTURE ONLY.
//
// B200's FP64 pipe has no published per-SKU figure in this image's guides, so
// bench.py measures it: a grid of 148 x 8 CTAs x 256 threads, each thread
// running 8 independent DFMA dependency chains (enough ILP to cover the
// DFMA latency), timed with CUDA events, best of 5.  2 flops per DFMA.
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dfma_chains(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;  // keeps the chains live
}

extern "C" double xft_probe_fp64_tflops(int device) {
    if (cudaSetDevice(device) != cudaSuccess) return -1.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return -1.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 2048;
    dfma_chains<<<blocks, threads>>>(out, 16, 0.999999, 1e-7);  // warm-up
    double best = 0.0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dfma_chains<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
        double tf = flops / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? best : -1.0;
}
