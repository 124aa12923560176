// Microbenchmark: tcgen05.ld (TMEM -> registers) and tcgen05.st bandwidth per SM
// with 4 / 8 / 16 warps, 32x32b.x16 shape (64 B per thread per instruction).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <bool ST>
__global__ void k(int iters, long long* out, uint32_t* sink) {
    __shared__ uint32_t holder;
    int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tmem = holder + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 32);
    uint32_t acc = 0;
    long long t0 = clock64();
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = i * threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        uint32_t a = tmem + (uint32_t)((i & 7) * 16);
        if (ST) {
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(a),
                "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
                "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
        } else {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                  "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                : "r"(a));
            if ((i & 3) == 3) {
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                acc += r[0] ^ r[15];
            }
        }
    }
    if (ST) asm volatile("tcgen05.wait::st.sync.aligned;");
    else asm volatile("tcgen05.wait::ld.sync.aligned;");
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc + r[3];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(holder));
}
int main() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    uint32_t* sink;
    cudaMalloc(&sink, 148 * 1024 * 4);
    long long h[148];
    int iters = 4096;
    for (int st = 0; st < 2; ++st)
        for (int warps : {4, 8, 16}) {
            if (st) k<true><<<148, warps * 32>>>(iters, d, sink);
            else k<false><<<148, warps * 32>>>(iters, d, sink);
            cudaDeviceSynchronize();
            cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
            double bytes = (double)warps * 32 * 64 * iters;
            printf("%s warps=%2d  %.1f bytes/clk/SM  (%s)\n", st ? "tcgen05.st" : "tcgen05.ld", warps, bytes / h[0],
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
