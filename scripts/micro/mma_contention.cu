// Microbenchmark: tcgen05.mma (kind::i8, M=128, A from TMEM) issue rate while other warps
// of the CTA hammer TMEM with tcgen05.ld (like the conv epilogue) or tcgen05.st (like
// the producers), or just spin.  Prints cycles per MMA seen by the issuing thread.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ volatile int g_stop;
// MODE: 0 idle helpers, 1 helpers tcgen05.ld, 2 helpers tcgen05.st, 3 helpers ALU spin
template <int MODE>
__global__ void k(int N, int iters, int helpers, long long* out, uint32_t* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t holder;
    __shared__ uint64_t bar;
    __shared__ volatile int done;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        done = 0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = holder;
    if (threadIdx.x == 0) {
        uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        uint32_t b = su32(sm);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            uint64_t bd = desc(b + (i & 7) * 4096, N * 16, 128);
            asm volatile(
                "{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}" ::"r"(tmem),
                "r"(tmem + 384 + (i & 7) * 8), "l"(bd), "r"(idesc), "r"(i));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        uint32_t ok = 0;
        do {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok)
                         : "r"(su32(&bar)), "r"(0u));
        } while (!ok);
        out[blockIdx.x] = clock64() - t0;
        done = 1;
    } else if (warp >= 1 && warp <= helpers) {
        uint32_t r[16], acc = 0;
        for (int q = 0; q < 16; ++q) r[q] = q;
        const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (MODE == 2 ? 384u + 64u : 256u);
        while (!done) {
            if (MODE == 1) {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                    : "r"(ta));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                acc += r[0] ^ r[15];
            } else if (MODE == 2) {
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
                    "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
                    "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            } else if (MODE == 3) {
                for (int q = 0; q < 64; ++q) acc = acc * 1664525u + 1013904223u;
            }
        }
        sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    uint32_t* sink;
    cudaMalloc(&sink, 148 * 1024 * 4);
    long long h[148];
    const int iters = 4000;
    auto run = [&](auto kern, const char* name, int N, int helpers) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        kern<<<148, 640, 64 * 1024>>>(N, iters, helpers, d, sink);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        printf("%-26s N=%3d helpers=%2d  cycles/MMA %7.1f  (%s)\n", name, N, helpers, (double)h[0] / iters,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int N : {96, 112}) {
        run(k<0>, "idle helpers", N, 19);
        run(k<1>, "helpers tcgen05.ld", N, 8);
        run(k<1>, "helpers tcgen05.ld", N, 16);
        run(k<2>, "helpers tcgen05.st", N, 8);
        run(k<2>, "helpers tcgen05.st", N, 16);
        run(k<3>, "helpers ALU spin", N, 19);
    }
    return 0;
}
