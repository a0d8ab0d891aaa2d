// Read-bandwidth micro-benchmark for the H-matvec access patterns (run under gpurun):
//   contiguous  : grid-stride double2 loads over a 4 GiB buffer, U loads in flight per thread
//   chunk512    : each warp reads 512 B chunks (64 doubles = one 64-row column slice of a
//                 block, as seg_kernel does) at scattered chunk indices
// Prints GB/s (bytes read / CUDA-event time, best of 5).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void read_contig(const double2 *__restrict__ p, long long n2, double *out) {
    double acc = 0.0;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (; i + (U - 1) * stride < n2; i += U * stride) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = p[i + u * stride];
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
    }
    for (; i < n2; i += stride) acc += p[i].x + p[i].y;
    if (acc == 1234.5) out[0] = acc;
}

// 64-double chunks (512 B); warp w reads chunks w, w + W, ... in a permuted order; each lane
// loads 2 doubles per chunk, U chunks in flight
template <int U>
__global__ void read_chunks(const double *__restrict__ p, long long nchunk, double *out) {
    const int lane = threadIdx.x & 31;
    const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
    double acc = 0.0;
    for (long long c = w; c < nchunk; c += U * W) {
        double a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long long cc = c + u * W;
            if (cc < nchunk) {
                long long q = (cc * 2654435761ll) % nchunk;  // scatter chunk order
                a[u] = p[q * 64 + lane];
                b[u] = p[q * 64 + 32 + lane];
            } else {
                a[u] = b[u] = 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += a[u] + b[u];
    }
    if (acc == 1234.5) out[0] = acc;
}

template <typename K>
static float timeit(K launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r > 0 && ms < best) best = ms;
    }
    return best;
}

int main() {
    const long long bytes = 4ll << 30;
    double *p, *out;
    cudaMalloc(&p, bytes);
    cudaMalloc(&out, 64);
    cudaMemset(p, 0, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long long n2 = bytes / 16, nch = bytes / 512;
    for (int bps : {4, 8, 16}) {
        int grid = sms * bps;
        float t4 = timeit([&] { read_contig<4><<<grid, 256>>>((const double2 *)p, n2, out); });
        float t8 = timeit([&] { read_contig<8><<<grid, 256>>>((const double2 *)p, n2, out); });
        float c4 = timeit([&] { read_chunks<4><<<grid, 256>>>(p, nch, out); });
        float c8 = timeit([&] { read_chunks<8><<<grid, 256>>>(p, nch, out); });
        printf("blocks/SM %2d: contig U4 %.0f GB/s  U8 %.0f GB/s | chunk512 U4 %.0f GB/s  U8 %.0f GB/s\n",
               bps, bytes / t4 / 1e6, bytes / t8 / 1e6, bytes / c4 / 1e6, bytes / c8 / 1e6);
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
