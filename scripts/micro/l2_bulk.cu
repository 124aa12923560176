// Microbenchmark: L2 -> shared memory streaming with cp.async.bulk (the conv B loader's
// pattern): every CTA (one per SM) cycles through a W-byte weight block in chunks of
// C bytes into a ring of R smem buffers.  Prints aggregate GB/s and bytes/clk/SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const uint8_t* __restrict__ src, int W, int C, int R, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bars[8];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nch = W / C;
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int r = i % R;
            const uint32_t bar = su32(&bars[r]);
            if (i >= R) {  // wait for the chunk issued R iterations ago
                uint32_t ok = 0, ph = (uint32_t)(((i / R) - 1) & 1);
                do {
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
                } while (!ok);
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(C) : "memory");
            const uint8_t* g = src + (size_t)(i % nch) * C;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(sm + (size_t)r * C)),
                         "l"(g), "r"(C), "r"(bar)
                         : "memory");
        }
        for (int i = iters; i < iters + R; ++i) {
            const int r = i % R;
            uint32_t ok = 0, ph = (uint32_t)(((i / R) - 1) & 1);
            do {
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(ok) : "r"(su32(&bars[r])), "r"(ph) : "memory");
            } while (!ok);
        }
        out[blockIdx.x] = clock64() - t0;
    }
}
int main() {
    uint8_t* src;
    cudaMalloc(&src, 64 << 20);
    cudaMemset(src, 1, 64 << 20);
    long long* d;
    cudaMalloc(&d, 148 * 8);
    long long h[148];
    for (int C : {8192, 16384, 24576, 49152}) {
        for (int R : {2, 4}) {
            const int W = 12 * 24576;  // ~295 KB weight block (C2 conv1 B per M tile)
            const int iters = 2000;
            if ((size_t)C * R > 200 * 1024) continue;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            k<<<148, 32, C * R>>>(src, W, C, R, 100, d);
            cudaEventRecord(e0);
            k<<<148, 32, C * R>>>(src, W, C, R, iters, d);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
            const double bytes = 148.0 * iters * C;
            printf("chunk %6d ring %d: %8.1f GB/s aggregate, %6.1f B/clk/SM (%s)\n", C, R, bytes / ms / 1e6,
                   (double)iters * C / h[0], cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
