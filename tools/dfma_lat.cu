#include <cstdio>
__global__ void chain(double *out, long long *cyc, int n, double a, double b)
{
    double x = threadIdx.x * 1e-3, y = x + 1.0, z = x + 2.0, w = x + 3.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        x = fma(x, a, b);
    }
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) {
        x = fma(x, a, b); y = fma(y, a, b); z = fma(z, a, b); w = fma(w, a, b);
    }
    long long t2 = clock64();
    out[threadIdx.x] = x + y + z + w;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
int main()
{
    double *o; long long *c, h[2];
    cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 16);
    for (int warps = 1; warps <= 4; warps *= 2) {
        chain<<<1, 32 * warps>>>(o, c, 4096, 0.999999, 1e-7);
        cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
        printf("warps/CTA %d: 1 chain %.2f cyc/dfma, 4 chains %.2f cyc per step (4 dfma)\n", warps, h[0] / 4096.0, h[1] / 4096.0);
    }
    return 0;
}
