// Standalone micro-benchmark of the 64-row register-tiled TRSM/SEGMUL body (not part of
// the library).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench_tile.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NT, int NQ>
__global__ void __launch_bounds__(NT) tile_kernel(const double *P, const double *B, double *O, int tiles, int k) {
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
    constexpr int G = NT / 64;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const double *Pm = P + (size_t)t * 4096;
        const double *Bm = B + (size_t)t * 4096;
        double acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
        for (int j = 0; j < 64; j += 2) {
            const double a0 = Pm[tx + j * 64], a1 = Pm[tx + (j + 1) * 64];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                int c = min(ty + G * q, k - 1);
                acc[q] += a0 * Bm[j + c * 64] + a1 * Bm[j + 1 + c * 64];
            }
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            int c = ty + G * q;
            if (c < k) O[(size_t)t * 4096 + tx + c * 64] = acc[q];
        }
        __syncthreads();
    }
}

template <int NT, int NQ>
void run(const char *name, const double *P, const double *B, double *O, int tiles, int k, int grid) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    tile_kernel<NT, NQ><<<grid, NT>>>(P, B, O, tiles, k);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) tile_kernel<NT, NQ><<<grid, NT>>>(P, B, O, tiles, k);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double per_tile_per_cta = ms / 5 * 1e3 / ((double)tiles / grid);
    printf("%-28s grid %5d: %8.3f ms/launch, %7.2f us per tile per CTA\n", name, grid, ms / 5, per_tile_per_cta);
}

int main() {
    const int tiles = 148 * 64;
    double *P, *B, *O;
    cudaMalloc(&P, sizeof(double) * 4096 * tiles);
    cudaMalloc(&B, sizeof(double) * 4096 * tiles);
    cudaMalloc(&O, sizeof(double) * 4096 * tiles);
    cudaMemset(P, 0, sizeof(double) * 4096 * tiles);
    cudaMemset(B, 0, sizeof(double) * 4096 * tiles);
    run<256, 2>("NT256 k=7 (1 CTA/SM)", P, B, O, tiles, 7, 148);
    run<256, 2>("NT256 k=7 (4 CTA/SM)", P, B, O, tiles, 7, 148 * 4);
    run<1024, 1>("NT1024 k=7 (1 CTA/SM)", P, B, O, tiles, 7, 148);
    run<256, 16>("NT256 k=64 (1 CTA/SM)", P, B, O, tiles, 64, 148);
    run<1024, 4>("NT1024 k=64 (1 CTA/SM)", P, B, O, tiles, 64, 148);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
