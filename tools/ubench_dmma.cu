// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) peak micro-benchmark (run under gpurun):
// every warp issues ACC independent accumulator chains of mma for ITER iterations.
// Prints TFLOP/s (512 flops per warp-level m8n8k4 mma) for several CTA counts per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void dmma_loop(double *out, int iters) {
    double c[ACC][2];
    const int l = threadIdx.x & 31;
    double a = 1.0 + 1e-9 * l, b = 1.0 - 1e-9 * l;
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ACC; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;
}

template <int ACC>
static void run(int sms, int per_sm, int threads) {
    double *out;
    cudaMalloc(&out, 8);
    const int iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
        cudaEventRecord(a);
        dmma_loop<ACC><<<sms * per_sm, threads>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r > 0 && ms < best) best = ms;
    }
    const double flops = 512.0 * ACC * (double)iters * (threads / 32) * sms * per_sm;
    printf("acc %d  ctas/SM %d  threads %d: %.2f TFLOP/s (%s)\n", ACC, per_sm, threads,
           flops / best / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<4>(sms, 1, 256);
    run<4>(sms, 2, 256);
    run<8>(sms, 1, 256);
    run<8>(sms, 2, 256);
    run<8>(sms, 4, 256);
    run<16>(sms, 2, 256);
    return 0;
}
