// Microbenchmark: the conv kernel's MMA issue pattern (3 digit planes x 2 k-steps per
// stage, A from TMEM, per-stage tcgen05.commit to an mbarrier, fence) — cycles per MMA
// for several variants, one CTA per SM, single issuing thread.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar));
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
    uint32_t ok = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(bar), "r"(ph));
    } while (!ok);
}
// VAR: 0 = stage pattern with commit per stage; 1 = no commits; 2 = same B address always;
//      3 = one accumulator (no digit planes); 4 = commit + wait for the stage 4 back (ring of 4)
template <int VAR>
__global__ void k(int Nt, int stages, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t holder;
    __shared__ uint64_t bars[8];
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0)
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tmem = holder;
    if (threadIdx.x == 0) {
        const int S = 4, KS = 64;
        uint32_t idesc = (2u << 4) | ((uint32_t)(Nt >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        uint32_t b_base = su32(sm);
        uint32_t bstage = 3u * Nt * KS, bdig = (uint32_t)Nt * KS, bchunk = (uint32_t)Nt * 16;
        long long t0 = clock64();
        for (int st = 0; st < stages; ++st) {
            int s = st % S;
            if (VAR == 4 && st >= S) wait(su32(&bars[s]), (uint32_t)(((st / S) - 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            uint32_t bst = b_base + (VAR == 2 ? 0 : s * bstage);
            for (int kk = 0; kk < 2; ++kk) {
                uint32_t at = tmem + 448 + s * 16 + kk * 8;
                for (int d = 0; d < 3; ++d) {
                    uint64_t bd = desc(bst + (VAR == 2 ? 0 : d * bdig + kk * 2 * bchunk), bchunk, 128);
                    mma(tmem + (VAR == 3 ? 0 : d * Nt), at, bd, idesc, (st | kk) ? 1u : 0u);
                }
            }
            if (VAR != 1) commit(su32(&bars[s]));
        }
        commit(su32(&bars[7]));
        wait(su32(&bars[7]), 0);
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    long long h[148];
    const int stages = 2000;
    auto run = [&](auto kern, const char* name, int Nt) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        kern<<<148, 128, 160 * 1024>>>(Nt, stages, d);
        cudaDeviceSynchronize();
        kern<<<148, 128, 160 * 1024>>>(Nt, stages, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        printf("%-34s Nt=%3d  cycles/MMA %6.1f  (%s)\n", name, Nt, (double)h[0] / (stages * 6.0),
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int Nt : {32, 112, 128}) {
        run(k<0>, "stage pattern, commit/stage", Nt);
        run(k<1>, "no commits", Nt);
        run(k<2>, "same B address", Nt);
        run(k<3>, "single accumulator", Nt);
        run(k<4>, "commit + ring wait (S=4)", Nt);
    }
    return 0;
}
