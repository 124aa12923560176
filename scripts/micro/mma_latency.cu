// Microbenchmark: issue-to-commit-arrival latency of n back-to-back tcgen05.mma
// (kind::i8, M=128, A from TMEM) as seen by the issuing warp (commit + try_wait).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__global__ void k(int N, int n, int reps, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t holder;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = holder;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        long long tot = 0, tiss = 0;
        for (int r = 0; r < reps; ++r) {
            const long long t0 = clock64();
            for (int i = 0; i < n; ++i) {
                const uint64_t bd = desc(su32(sm) + (i & 3) * 8192, N * 16, 128);
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}" ::"r"(tmem),
                             "r"(tmem + 384 + (i & 3) * 8), "l"(bd), "r"(idesc), "r"(i) : "memory");
            }
            const long long t_issue = clock64();
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
            uint32_t ok = 0;
            do {
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(ok) : "r"(su32(&bar)), "r"((uint32_t)(r & 1)) : "memory");
            } while (!ok);
            tot += clock64() - t0;
            tiss += t_issue - t0;
        }
        out[blockIdx.x] = tot / reps;
        out[148 + blockIdx.x] = tiss / reps;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
    long long* d;
    cudaMalloc(&d, 296 * 8);
    long long h[296];
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int N : {96, 256})
        for (int n : {1, 4, 8, 16, 32, 64}) {
            k<<<148, 128, 64 * 1024>>>(N, n, 200, d);
            cudaDeviceSynchronize();
            cudaMemcpy(h, d, 296 * 8, cudaMemcpyDeviceToHost);
            printf("N=%3d n=%2d: issue of n MMAs %6lld cycles, issue->commit arrival %6lld cycles (%s)\n", N, n, h[148], h[0],
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
