// Microbenchmark: round-trip latency of an mbarrier hand-off between two warps of a CTA
// (arrive by one, wait by the other, and back), for different wait flavours.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
    uint32_t ok = 0;
    do {
        if (MODE == 0)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
        else if (MODE == 1)
            asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
        else
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(bar), "r"(ph), "r"(MODE) : "memory");
    } while (!ok);
}
template <int MODE>
__global__ void k(int iters, long long* out, int busy_warps) {
    __shared__ uint64_t bars[2];
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[1])));
        stop = 0;
    }
    __syncthreads();
    if (warp == 0 && lane == 0) {
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bars[0])) : "memory");
            wait<MODE>(su32(&bars[1]), (uint32_t)(i & 1));
        }
        out[blockIdx.x] = clock64() - t0;
        stop = 1;
    } else if (warp == 1 && lane == 0) {
        for (int i = 0; i < iters; ++i) {
            wait<MODE>(su32(&bars[0]), (uint32_t)(i & 1));
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bars[1])) : "memory");
        }
    } else if (warp >= 2 && warp < 2 + busy_warps) {  // other warps keep the schedulers busy
        uint32_t x = threadIdx.x;
        while (!stop) {
#pragma unroll 16
            for (int q = 0; q < 64; ++q) x = x * 1664525u + 1013904223u;
        }
        if (x == 7) out[1000] = x;
    }
}
int main() {
    long long* d;
    cudaMalloc(&d, 2048 * 8);
    long long h[1];
    const int iters = 10000;
    auto run = [&](auto kern, const char* name, int busy) {
        kern<<<148, 672, 0>>>(iters, d, busy);
        cudaDeviceSynchronize();
        kern<<<148, 672, 0>>>(iters, d, busy);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("%-32s busy warps %2d: round trip %7.1f cycles (%s)\n", name, busy, (double)h[0] / iters,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int busy : {0, 8, 19}) {
        run(k<0>, "try_wait", busy);
        run(k<1>, "test_wait spin", busy);
        run(k<32>, "try_wait hint 32ns", busy);
        run(k<1000>, "try_wait hint 1us", busy);
    }
    return 0;
}
