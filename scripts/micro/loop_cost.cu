// Microbenchmark: per-iteration cost of the conv MMA warp's bookkeeping without MMAs —
// (a) lane-0 try_wait on an already-completed mbarrier + __syncwarp, (b) + elected
// tcgen05.commit, (c) commit only, (d) + tcgen05.fence::after_thread_sync.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
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
                     : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
    } while (!ok);
}
template <int V>
__global__ void k(int iters, long long* out) {
    __shared__ uint32_t holder;
    __shared__ uint64_t bars[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bars[0])) : "memory");  // phase 0 done
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) {
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (V & 1) {
                if (lane == 0) wait(su32(&bars[0]), 0u);
                __syncwarp();
            }
            if (V & 8) wait(su32(&bars[0]), 0u);  // all lanes
            if (V & 16) {  // lane 0 test_wait loop
                if (lane == 0) {
                    uint32_t ok = 0;
                    do {
                        asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                     : "=r"(ok) : "r"(su32(&bars[0])), "r"(0u) : "memory");
                    } while (!ok);
                }
                __syncwarp();
            }
            if (V & 32) {  // all lanes test_wait
                uint32_t ok = 0;
                do {
                    asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(ok) : "r"(su32(&bars[0])), "r"(0u) : "memory");
                } while (!ok);
            }
            if (V & 64) {  // lane 0 only, no syncwarp
                if (lane == 0) wait(su32(&bars[0]), 0u);
            }
            if (V & 4) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (V & 2) commit_e(su32(&bars[1 + (i & 3)]));
        }
        if (lane == 0) out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(holder));
}
int main() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    long long h[1];
    const int iters = 4000;
    auto run = [&](auto kern, const char* name) {
        kern<<<148, 128>>>(iters, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("%-44s %7.1f cycles/iter (%s)\n", name, (double)h[0] / iters, cudaGetErrorString(cudaGetLastError()));
    };
    run(k<0>, "empty loop");
    run(k<1>, "try_wait(done) + syncwarp");
    run(k<2>, "elected commit");
    run(k<3>, "try_wait + commit");
    run(k<7>, "try_wait + fence + commit");
    run(k<4>, "fence");
    run(k<8>, "try_wait all lanes");
    run(k<16>, "test_wait lane0 + syncwarp");
    run(k<32>, "test_wait all lanes");
    run(k<64>, "try_wait lane0, no syncwarp");
    run(k<10>, "try_wait all lanes + commit");
    return 0;
}
