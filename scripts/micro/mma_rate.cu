// Microbenchmark: issue rate of tcgen05.mma (cta_group::1, M=128) on one CTA per SM,
// A from TMEM or SMEM, B from SMEM, for kind::i8 and kind::f16.  Prints cycles per MMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
template <int KIND, bool ATMEM>
__global__ void k(int N, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder; __shared__ uint64_t bar;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar))); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = holder;
  if (threadIdx.x == 0) {
    uint32_t idesc = (KIND == 0 ? (2u << 4) : (1u << 4)) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint32_t b = su32(sm), a = su32(sm + 65536);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint64_t bd = desc(b, N * 16, 128);
      if (ATMEM) {
        if (KIND == 0) asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}" :: "r"(tmem), "r"(tmem + 384), "l"(bd), "r"(idesc), "r"(i));
        else asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" :: "r"(tmem), "r"(tmem + 384), "l"(bd), "r"(idesc), "r"(i));
      } else {
        uint64_t ad = desc(a, 2048, 128);
        if (KIND == 0) asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}" :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(i));
        else asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(i));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)));
    uint32_t ok = 0;
    do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(su32(&bar)), "r"(0u)); } while (!ok);
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}
int main() {
  long long* d; cudaMalloc(&d, 148 * 8); long long h[148];
  int iters = 20000;
  auto run = [&](auto kern, const char* name, int N, double macs_per) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    kern<<<148, 128, 200 * 1024>>>(N, iters, d); cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); kern<<<148, 128, 200 * 1024>>>(N, iters, d); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    double cyc = (double)h[0] / iters;
    double tops = 2.0 * macs_per * iters * 148 / (ms * 1e-3) / 1e12;
    printf("%-22s N=%3d  cycles/MMA %7.1f   chip %7.1f TOPS  (err %s)\n", name, N, cyc, tops, cudaGetErrorString(cudaGetLastError()));
  };
  for (int N : {32, 64, 96, 112, 128, 144, 192, 224, 256}) {
    run(k<0, true>, "i8  A=tmem  B=smem", N, 128.0 * N * 32);
    run(k<0, false>, "i8  A=smem  B=smem", N, 128.0 * N * 32);
    run(k<1, true>, "f16 A=tmem  B=smem", N, 128.0 * N * 16);
    run(k<1, false>, "f16 A=smem  B=smem", N, 128.0 * N * 16);
  }
  return 0;
}
