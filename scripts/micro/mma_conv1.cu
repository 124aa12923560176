// Microbenchmark: the conv1 MMA warp loop in isolation — per tile 3 K stages (4,4,1 MMAs of
// N=192, A from a 3-slot TMEM ring, B from a 4-stage smem ring), per stage one batched probe of
// the A/B barriers and two commits, per tile an accumulator commit and a 2-buffer ring wait.
// FLAGS: 1 = a B-loader warp streams real 24.6 KB cp.async.bulk copies (else it only arrives),
//        2 = an epilogue warp releases accumulators (else the MMA warp waits on its own commit),
//        4 = skip the A/B probes.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ bool mtry(uint32_t a, uint32_t p) {
    uint32_t ok;
    asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                 : "=r"(ok) : "r"(a), "r"(p) : "memory");
    return ok;
}
__device__ __forceinline__ void commit_e(uint32_t bar) {
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }" ::"r"(bar) : "memory");
}
template <int NK>
__device__ __forceinline__ void stage(uint32_t d, uint32_t a0, uint64_t b0, uint64_t inck, uint32_t idesc, uint32_t acc0) {
#pragma unroll
    for (int kk = 0; kk < NK; ++kk)
        asm volatile("{ .reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p; }" ::"r"(d),
                     "r"(a0 + 8u * kk), "l"(b0 + inck * kk), "r"(idesc), "r"(kk ? 1u : acc0) : "memory");
}
template <int FLAGS>
__global__ void k(const uint8_t* __restrict__ wsrc, int tiles, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t holder;
    __shared__ uint64_t bars[16];  // 0-3 bfull, 4-7 bempty, 8-9 accf, 10-11 acce
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NS = 4;
    constexpr uint32_t BST = 3 * 64 * 128;  // 24576 B per B stage
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t bfull = su32(&bars[0]), bempty = su32(&bars[4]), accf = su32(&bars[8]), acce = su32(&bars[10]);
    const int nst = tiles * 3;
    if (warp == 0) {  // MMA warp
        const uint32_t idesc = (2u << 4) | ((uint32_t)(192 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t bchunk = 192 * 16;
        const uint64_t d0 = desc(su32(sm), bchunk, 128), inck = (2u * bchunk) >> 4;
        int bs = 0, buf = 0;
        uint32_t bph = 0, aph = 0;
        const long long t0 = clock64();
        for (int tile = 0; tile < tiles; ++tile) {
            for (int ks = 0; ks < 3; ++ks) {
                bool d1 = (FLAGS & 4) || mtry(bfull + 8 * bs, bph);
                bool d2 = ks != 0 || tile < 2 || mtry(acce + 8 * buf, aph ^ 1u);
                while (!d1) d1 = mtry(bfull + 8 * bs, bph);
                while (!d2) d2 = mtry(acce + 8 * buf, aph ^ 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t dst = d0 + ((bs * BST) >> 4);
                const uint32_t at = 384 + ks * 32, dacc = buf * 192;
                if (ks < 2) stage<4>(dacc, at, dst, inck, idesc, ks ? 1u : 0u);
                else stage<1>(dacc, at, dst, inck, idesc, 1u);
                commit_e(bempty + 8 * bs);
                if (++bs == NS) bs = 0, bph ^= 1u;
            }
            commit_e(accf + 8 * buf);
            if (!(FLAGS & 2)) {  // no epilogue: the MMA warp's own commit releases the buffer
            }
            if (++buf == 2) buf = 0, aph ^= 1u;
        }
        commit_e(su32(&bars[15]));
        while (!mtry(su32(&bars[15]), 0u)) {
        }
        if (lane == 0) out[blockIdx.x] = (clock64() - t0) / nst;
    } else if (warp == 1) {  // B loader
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int st = 0; st < nst; ++st) {
                while (!mtry(bempty + 8 * s, ph ^ 1u)) {
                }
                if (FLAGS & 1) {
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bfull + 8 * s), "r"(BST) : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     su32(sm + s * BST)), "l"(wsrc + (size_t)(st % 12) * BST), "r"(BST), "r"(bfull + 8 * s) : "memory");
                } else {
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bfull + 8 * s) : "memory");
                }
                if (++s == NS) s = 0, ph ^= 1u;
            }
        }
    } else if (warp == 2) {  // accumulator consumer
        if (lane == 0) {
            int buf = 0;
            uint32_t ph = 0;
            for (int tile = 0; tile < tiles; ++tile) {
                while (!mtry(accf + 8 * buf, ph)) {
                }
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(acce + 8 * buf) : "memory");
                if (++buf == 2) buf = 0, ph ^= 1u;
            }
        }
    }
    else if (FLAGS & 8) {  // other warps poll a barrier that completes only at the end
        if (lane == 0)
            while (!mtry(su32(&bars[14]), 0u)) {
            }
    } else if (FLAGS & 16) {  // other warps run ALU work
        uint32_t x = threadIdx.x;
        for (int i = 0; i < tiles * 200; ++i) x = x * 1664525u + 1013904223u;
        if (x == 7) out[1] = x;
    } else if (FLAGS & 32) {  // other warps: TMEM loads from their lane quadrant (epilogue-like)
        const uint32_t ta = ((uint32_t)((warp & 3) * 32) << 16) + 192u;
        uint32_t acc = 0;
        for (int i = 0; i < tiles * 8; ++i) {
            uint32_t r[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                           "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                         : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc += r[0] ^ r[15];
        }
        if (acc == 7) out[1] = acc;
    }
    if (warp == 0 && (FLAGS & 8) && lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bars[14])) : "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(holder));
}
int main() {
    uint8_t* w;
    cudaMalloc(&w, 12 * 24576);
    cudaMemset(w, 1, 12 * 24576);
    long long* d;
    cudaMalloc(&d, 148 * 8);
    long long h[1];
    auto run = [&](auto kern, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
        kern<<<148, 672, 4 * 24576>>>(w, 400, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("%-40s %6lld cycles per stage (%s)\n", name, h[0], cudaGetErrorString(cudaGetLastError()));
    };
    run(k<0>, "arrive-only B, self acc");
    run(k<1>, "bulk B copies");
    run(k<4>, "no A/B probes (B arrive-only)");
    run(k<5>, "no probes, bulk B");
    run(k<1 | 8>, "bulk B + 18 polling warps");
    run(k<1 | 16>, "bulk B + 18 ALU warps");
    run(k<1 | 32>, "bulk B + 18 TMEM-load warps");
    return 0;
}
