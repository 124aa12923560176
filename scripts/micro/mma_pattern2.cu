// Microbenchmark: the conv MMA warp's per-stage pattern — NK k-step MMAs (kind::i8,
// M=128, A from TMEM, one N-wide B from smem), then optional fence / commits / ring
// wait — issued by a converged warp with elect.sync (as the kernel does), or by one
// thread.  Prints cycles per MMA.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma_e(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{.reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit_e(uint32_t bar) {
    asm volatile(
        "{ .reg .pred e; elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
    uint32_t ok = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(bar), "r"(ph)
                     : "memory");
    } while (!ok);
}
// FLAGS: 1 fence/stage, 2 commit/stage, 4 second commit/stage, 8 ring wait (S=4) on the commit,
//        16 per-tile accumulator commit every T stages + wait NB=2 back
template <int FLAGS, int NKC = 0, bool TZ = false>
__global__ void k(int N, int NK_, int stages, long long* out) {
    const int NK = NKC ? NKC : NK_;
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t holder;
    __shared__ uint64_t bars[16];
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0)
        for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = TZ ? 0u : holder;
    if (warp == 0) {
        const int S = 4, KS = 128;
        const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t b_base = su32(sm);
        const uint32_t bstage = (uint32_t)N * KS, bchunk = (uint32_t)N * 16;
        const int T = 3;  // stages per tile
        long long t0 = clock64();
        for (int st = 0; st < stages; ++st) {
            const int s = st % S;
            if ((FLAGS & 8) && st >= S) wait(su32(&bars[s]), (uint32_t)(((st / S) - 1) & 1));
            if ((FLAGS & 16) && st % T == 0 && st >= 2 * T) {
                const int tile = st / T;
                wait(su32(&bars[12 + (tile & 1)]), (uint32_t)(((tile / 2) - 1) & 1));
            }
            if (FLAGS & 1) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dacc = tmem + ((FLAGS & 16) ? ((st / T) & 1) * 192u : 0u);
#pragma unroll
            for (int kk = 0; kk < (NKC ? NKC : NK); ++kk) {
                const uint32_t at = tmem + 384 + s * 32 + kk * 8;
                const uint64_t bd = desc(b_base + (s % 2) * bstage + kk * 2 * bchunk, bchunk, 128);
                mma_e(dacc, at, bd, idesc, (st % T || kk) ? 1u : 0u);
            }
            if (FLAGS & 2) commit_e(su32(&bars[s]));
            if (FLAGS & 4) commit_e(su32(&bars[4 + s]));
            if ((FLAGS & 16) && st % T == T - 1) commit_e(su32(&bars[12 + ((st / T) & 1)]));
        }
        commit_e(su32(&bars[15]));
        if ((threadIdx.x & 31) == 0) wait(su32(&bars[15]), 0);
        __syncwarp();
        if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    long long h[148];
    const int stages = 3000;
    auto run = [&](auto kern, const char* name, int N, int NK) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        kern<<<148, 128, 160 * 1024>>>(N, NK, stages, d);
        cudaDeviceSynchronize();
        kern<<<148, 128, 160 * 1024>>>(N, NK, stages, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        printf("%-40s N=%3d NK=%d  cycles/MMA %6.1f  (%s)\n", name, N, NK, (double)h[0] / (stages * (double)NK),
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int N : {96, 192}) {
        for (int NK : {4, 1}) {
            run(k<0>, "bare", N, NK);
            run(k<1>, "fence", N, NK);
            run(k<2>, "commit", N, NK);
            run(k<3>, "fence+commit", N, NK);
            run(k<7>, "fence+2 commits", N, NK);
            run(k<15>, "fence+2 commits+ring wait", N, NK);
            run(k<31>, "... + tile acc commit/wait", N, NK);
            if (NK == 4) {
                run(k<0, 4>, "bare, unrolled", N, NK);
                run(k<0, 4, true>, "bare, unrolled, tmem=0", N, NK);
                run(k<15, 4, true>, "fence+2 commits+ring, unrolled, tmem=0", N, NK);
                run(k<31, 4, true>, "... + tile acc, unrolled, tmem=0", N, NK);
            } else {
                run(k<0, 1, true>, "bare, unrolled, tmem=0", N, NK);
                run(k<15, 1, true>, "fence+2 commits+ring, unrolled, tmem=0", N, NK);
            }
        }
    }
    return 0;
}
