// Latency probes on sm_100a: dependent DFMA chain, fp64 reciprocal, __syncthreads, shfl, LDS.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *o, long long *c, double x0) {
    __shared__ double s[256];
    s[threadIdx.x] = x0 + threadIdx.x;
    __syncthreads();
    double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) x = fma(x, y, 1e-12);
    long long t1 = clock64();
    for (int i = 0; i < 256; ++i) x = 1.0 / (x + 1.0);
    long long t2 = clock64();
    for (int i = 0; i < 256; ++i) __syncthreads();
    long long t3 = clock64();
    for (int i = 0; i < 256; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1) * 1e-30;
    long long t4 = clock64();
    int idx = threadIdx.x;
    for (int i = 0; i < 256; ++i) { x += s[idx]; idx = (idx + (x > 1e300)) & 255; }
    long long t5 = clock64();
    float f = (float)x;
    for (int i = 0; i < 256; ++i) f = fmaf(f, 1.0000001f, 1e-12f);
    long long t6 = clock64();
    o[blockIdx.x * blockDim.x + threadIdx.x] = x + f;
    if (threadIdx.x == 0) { c[0] = t1 - t0; c[1] = t2 - t1; c[2] = t3 - t2; c[3] = t4 - t3; c[4] = t5 - t4; c[5] = t6 - t5; }
}
int main() {
    double *o; long long *c, h[6];
    cudaMalloc(&o, 8 * 256 * 148); cudaMalloc(&c, 64);
    for (int r = 0; r < 3; ++r) k<<<1, 256>>>(o, c, 0.5);
    cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    const char *n[6] = {"dfma dep", "fp64 1/x dep", "syncthreads(256thr)", "shfl dep", "lds dep", "ffma dep"};
    for (int i = 0; i < 6; ++i) printf("%-22s %.1f cycles/op\n", n[i], h[i] / 256.0);
    return 0;
}
