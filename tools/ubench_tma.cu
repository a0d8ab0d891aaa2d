// Bulk-copy (cp.async.bulk) streaming micro-benchmark (run under gpurun): one CTA per SM,
// one producer lane streaming BATCH-byte copies of a contiguous 4 GiB buffer into a
// STAGES-deep shared-memory ring (full/empty mbarriers), 8 consumer warps summing the slot.
// Variant `extra`: each batch also issues 3 small (512 B) copies, like the descriptor /
// t-span / x-slice copies of seg_tma_kernel.  Prints GB/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t par) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(b)),
                 "r"(par)
                 : "memory");
}
__device__ __forceinline__ void bulk(void *d, const void *s, uint32_t n, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)),
                 "l"(s), "r"(n), "r"(sa(b))
                 : "memory");
}

template <int STAGES, int BATCH>
__global__ void __launch_bounds__(288, 1) stream(const double *p, long long nbatch, int extra, double *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    double *ring = (double *)sm;
    double *aux = ring + STAGES * (BATCH / 8);
    uint64_t *full = (uint64_t *)(aux + STAGES * 256);
    uint64_t *empty = full + STAGES;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long per = (nbatch + gridDim.x - 1) / gridDim.x;
    const long long b0 = blockIdx.x * per, b1 = min(nbatch, b0 + per);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0;
            for (long long b = b0; b < b1; ++b) {
                mbar_wait(&empty[st], ph ^ 1);
                mbar_expect(&full[st], BATCH + (extra ? 3 * 512 : 0));
                bulk(ring + st * (BATCH / 8), p + b * (BATCH / 8), BATCH, &full[st]);
                if (extra)
                    for (int k = 0; k < 3; ++k)
                        bulk(aux + st * 256 + k * 64, p + ((b * 7919 + k * 104729) % nbatch) * (BATCH / 8), 512, &full[st]);
                if (++st == STAGES) {
                    st = 0;
                    ph ^= 1;
                }
            }
        }
        return;
    }
    const int tid = threadIdx.x - 32;
    double acc = 0.0;
    int st = 0;
    uint32_t ph = 0;
    for (long long b = b0; b < b1; ++b) {
        mbar_wait(&full[st], ph);
        const double *s = ring + st * (BATCH / 8);
        for (int i = tid; i < BATCH / 8; i += 256) acc += s[i];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++st == STAGES) {
            st = 0;
            ph ^= 1;
        }
    }
    if (acc == 1234.5) out[0] = acc;
}

template <int STAGES, int BATCH>
static void run(const double *p, long long bytes, double *out, int sms) {
    const size_t smem = STAGES * BATCH + STAGES * 2048 + 2 * STAGES * 8 + 256;
    cudaFuncSetAttribute(stream<STAGES, BATCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long nb = bytes / BATCH;
    for (int extra = 0; extra < 2; ++extra) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            stream<STAGES, BATCH><<<sms, 288, smem>>>(p, nb, extra, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r > 0 && ms < best) best = ms;
        }
        printf("stages %d batch %6d extra %d: %.0f GB/s  (%s)\n", STAGES, BATCH, extra,
               (double)nb * BATCH / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
}

int main() {
    const long long bytes = 4ll << 30;
    double *p, *out;
    cudaMalloc(&p, bytes);
    cudaMalloc(&out, 64);
    cudaMemset(p, 0, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<4, 32768>(p, bytes, out, sms);
    run<6, 32768>(p, bytes, out, sms);
    run<12, 16384>(p, bytes, out, sms);
    run<3, 65536>(p, bytes, out, sms);
    return 0;
}
