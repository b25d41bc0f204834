// fp64_peak.cu -- measured FP64 DFMA throughput of this B200 (roofline denominator for the
// FP64 CUDA-core kernels; MEASURED_PEAKS.json carries only HBM and bf16).  8 independent DFMA
// chains per thread, 148 x 8 CTAs of 256 threads, CUDA events, best of 5.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double *out, int iters, double a, double b)
{
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1.2345) out[0] = s;
}
int main()
{
    int dev = 0, nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double *d;
    cudaMalloc(&d, 8);
    const int iters = 1 << 16, threads = 256, blocks = nsm * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_loop<<<blocks, threads>>>(d, 1024, 0.999999, 1e-7);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * (double)iters * threads * blocks;
    double tf = flops / (best * 1e-3) / 1e12;
    double per_sm_clk = flops / 2 / (best * 1e-3) / nsm / (clk * 1e3);
    printf("{\"fp64_dfma_tflops\": %.3f, \"sms\": %d, \"clock_attr_mhz\": %.0f, "
           "\"dfma_per_sm_per_clk_at_attr_clock\": %.2f, \"ms\": %.4f}\n", tf, nsm, clk / 1e3,
           per_sm_clk, best);
    return 0;
}
