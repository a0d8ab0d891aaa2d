// Standalone timing of the speculative leaf-LU loop (64 x 64, one barrier per column), to
// separate its intrinsic cost from the executor: nvcc -arch=sm_100a -O3 -o tools/ubench_getrf
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) lu2_kernel(const double *G, double *out, long long *cyc) {
    __shared__ __align__(16) double Tw[128];
    const int tr = threadIdx.x >> 2, tc = threadIdx.x & 3, lane = threadIdx.x & 31;
    const int m = 64;
    double b[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) b[q] = G[tr + (tc + 4 * q) * 64 + blockIdx.x * 4096];
    __syncthreads();
    long long t0 = clock64();
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int j = 4 * k + jj;
            if (j < m) {
                double *Pj = Tw + (j & 1) * 64;
                if (tr == j) {
#pragma unroll
                    for (int q = k; q < 16; q += 2)
                        *reinterpret_cast<double2 *>(Pj + tc * 16 + q - (q & 1)) =
                            make_double2((q & 1) ? b[q - 1] : b[q], (q & 1) ? b[q] : b[q + 1]);
                }
                __syncthreads();
                const double lv = __shfl_sync(0xffffffffu, b[k], (lane & ~3) | jj);
                if (tr > j && tr < m) {
                    const double d = Pj[jj * 16 + k];
                    ok = ok && (d != 0.0 ? fabs(lv) <= fabs(d) : lv == 0.0);
                    const double l = d != 0.0 ? lv * (1.0 / d) : lv;
                    const double pk = Pj[tc * 16 + k];
                    if (tc > jj) b[k] -= l * pk;
                    else if (tc == jj) b[k] = l;
#pragma unroll
                    for (int q = (k + 1) & ~1; q < 16; q += 2) {
                        const double2 pr = *reinterpret_cast<const double2 *>(Pj + tc * 16 + q);
                        if (q > k) b[q] -= l * pr.x;
                        b[q + 1] -= l * pr.y;
                    }
                }
            }
        }
    }
    ok = __syncthreads_and(ok);
    long long t1 = clock64();
#pragma unroll
    for (int q = 0; q < 16; ++q) out[tr + (tc + 4 * q) * 64 + blockIdx.x * 4096] = b[q] + ok;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(256) lu_kernel(const double *G, double *out, long long *cyc, int variant) {
    __shared__ double Tw[128];
    const int tr = threadIdx.x >> 2, tc = threadIdx.x & 3, lane = threadIdx.x & 31;
    const int m = 64;
    double b[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) b[q] = G[tr + (tc + 4 * q) * 64 + blockIdx.x * 4096];
    __syncthreads();
    long long t0 = clock64();
    bool ok = true;
    for (int j = 0; j < m; ++j) {
        double *Pj = Tw + (j & 1) * 64;
        if (tr == j) {
#pragma unroll
            for (int q = 0; q < 16; ++q) Pj[tc + 4 * q] = b[q];
        }
        __syncthreads();
        const int jt = j & 3, jq = j >> 2;
        double mine = 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if (q == jq) mine = b[q];
        const double lv = __shfl_sync(0xffffffffu, mine, (lane & ~3) | jt);
        if (tr > j) {
            const double d = Pj[j];
            ok = ok && fabs(lv) <= fabs(d);
            const double l = variant == 1 ? lv * __drcp_rn(d) : lv * (1.0 / d);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int c = tc + 4 * q;
                if (c > j) b[q] -= l * Pj[c];
                else if (c == j) b[q] = l;
            }
        }
    }
    ok = __syncthreads_and(ok);
    long long t1 = clock64();
#pragma unroll
    for (int q = 0; q < 16; ++q) out[tr + (tc + 4 * q) * 64 + blockIdx.x * 4096] = b[q] + ok;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    const int B = 148;
    double *G, *O;
    long long *C;
    cudaMalloc(&G, sizeof(double) * 4096 * B);
    cudaMalloc(&O, sizeof(double) * 4096 * B);
    cudaMalloc(&C, sizeof(long long) * B);
    double *h = new double[4096 * B];
    for (int b = 0; b < B; ++b)
        for (int e = 0; e < 4096; ++e) h[b * 4096 + e] = ((e * 7919 + b) % 1000) / 1000.0 - 0.5 + ((e % 65) == 0 ? 20.0 : 0.0);
    cudaMemcpy(G, h, sizeof(double) * 4096 * B, cudaMemcpyHostToDevice);
    for (int variant = 0; variant < 2; ++variant) {
        for (int rep = 0; rep < 3; ++rep) lu_kernel<<<B, 256>>>(G, O, C, variant);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        lu_kernel<<<B, 256>>>(G, O, C, variant);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long c;
        cudaMemcpy(&c, C, sizeof(long long), cudaMemcpyDeviceToHost);
        printf("variant %d: kernel %.2f us, loop %lld cycles (%.1f per column)\n", variant, ms * 1e3, c, c / 64.0);
    }
    for (int rep = 0; rep < 3; ++rep) lu2_kernel<<<B, 256>>>(G, O, C);
    long long c;
    cudaMemcpy(&c, C, sizeof(long long), cudaMemcpyDeviceToHost);
    printf("unrolled: loop %lld cycles (%.1f per column)\n", c, c / 64.0);
    return 0;
}
