// neuron.cu — bandwidth-bound per-neuron stages on latency maps:
//   a4 spk_fire (IF on materialised potentials), a5 spk_pool (Eq. 3,
//   P:L140-149), a6 spk_inhibit, a8 spk_rstdp_route (Eq. 7),
//   a9 spk_gather and the dense <-> latency boundary conversions.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace {

constexpr int kT = 256;

// ---------------------------------------------------------------- fire
// One thread per neuron; the T potentials of a neuron are a stride-N column of
// BTCHW, so a warp reads 32 consecutive floats per step (coalesced).
__global__ void fire_kernel(const float* __restrict__ pot, int B, int T, size_t N, float theta,
                            uint8_t* __restrict__ lat, float* __restrict__ pstar) {
    spk_pdl_wait();
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (size_t)B * N) return;
    const size_t b = q / N, i = q % N;
    const float* p = pot + b * (size_t)T * N + i;
    int l = T;
    float ps = 0.0f;
    for (int t = 0; t < T; ++t) {
        const float v = __ldg(p + (size_t)t * N);
        if (v > theta) {  // strict "higher than" (R-STRICT)
            l = t;
            ps = v;
            break;
        }
    }
    lat[q] = (uint8_t)l;
    if (pstar) pstar[q] = ps;
}

// Four consecutive neurons per thread (N % 4 == 0, 16-byte aligned rows): the potentials of 8
// steps are loaded as float4s before any is tested, so 128 bytes per thread are in flight instead
// of one dependent 4-byte load per step; the thread stops at the first chunk after which all four
// neurons have crossed.  Same strict first-crossing test and P* as fire_kernel.
constexpr int kFireChunk = 8;
__global__ void __launch_bounds__(kT) fire4_kernel(const float4* __restrict__ pot, int B, int T, size_t N4, float theta,
                                                   uchar4* __restrict__ lat, float4* __restrict__ pstar) {
    spk_pdl_wait();
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (size_t)B * N4) return;
    const size_t b = q / N4, i = q % N4;
    const float4* p = pot + b * (size_t)T * N4 + i;
    int l[4] = {T, T, T, T};
    float ps[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int t0 = 0; t0 < T; t0 += kFireChunk) {
        float4 v[kFireChunk];
#pragma unroll
        for (int u = 0; u < kFireChunk; ++u)
            v[u] = t0 + u < T ? __ldcs(p + (size_t)(t0 + u) * N4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = kFireChunk - 1; u >= 0; --u) {  // descending: the earliest crossing is written last
            if (t0 + u >= T) continue;
            const float e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (l[k] >= t0 && e[k] > theta) {  // strict "higher than" (R-STRICT); not yet fired earlier
                    l[k] = t0 + u;
                    ps[k] = e[k];
                }
        }
        if (l[0] < T && l[1] < T && l[2] < T && l[3] < T) break;
    }
    lat[q] = make_uchar4((uint8_t)l[0], (uint8_t)l[1], (uint8_t)l[2], (uint8_t)l[3]);
    if (pstar) pstar[q] = make_float4(ps[0], ps[1], ps[2], ps[3]);
}

// ---------------------------------------------------------------- pool
// Per-step window max of cumulative trains == window min of latencies; padded
// cells never fire.  Grid: x = chunks of one output plane, (y, z) = plane index
// (32-bit index math inside a plane).
__global__ void __launch_bounds__(kT) pool_kernel(const uint8_t* __restrict__ lat, long long BC, int ppy, int H, int W,
                                                  int T, spk_pool_geom g, int Ho, int Wo, uint8_t* __restrict__ out) {
    spk_pdl_wait();
    // blockIdx.y selects a slice of ppy planes; inside it all index math is 32-bit
    const int plane_out = Ho * Wo;
    const int q = blockIdx.x * kT + threadIdx.x;  // < ppy * plane_out <= 2^30
    const long long bc = (long long)blockIdx.y * ppy + q / plane_out;
    if (bc >= BC || q >= ppy * plane_out) return;
    const int r = q % plane_out, y = r / Wo, x = r - y * Wo;
    const int y0 = y * g.Sh - g.Ph, x0 = x * g.Sw - g.Pw;
    const int i0 = max(0, -y0), i1 = min(g.Lh, H - y0), j0 = max(0, -x0), j1 = min(g.Lw, W - x0);
    const uint8_t* p = lat + (size_t)bc * H * W + (long long)y0 * W + x0;
    int m = T;
    for (int i = i0; i < i1; ++i)
        for (int j = j0; j < j1; ++j) m = min(m, (int)__ldg(p + (size_t)i * W + j));
    out[(size_t)bc * plane_out + r] = (uint8_t)min(m, T);
}


// Unpadded square windows of compile-time size L (C2 pool 2: 3x3/3): every window lies
// inside the plane, so the L*L loads of an output are unrolled and issued together
// instead of one dependent load per runtime loop iteration.
template <int L>
__global__ void __launch_bounds__(kT) pool_fixed_kernel(const uint8_t* __restrict__ lat, long long BC, int ppy, int H,
                                                        int W, int T, int S, int Ho, int Wo,
                                                        uint8_t* __restrict__ out) {
    spk_pdl_wait();
    const int plane_out = Ho * Wo;
    const int q = blockIdx.x * kT + threadIdx.x;
    const long long bc = (long long)blockIdx.y * ppy + q / plane_out;
    if (bc >= BC || q >= ppy * plane_out) return;
    const int r = q % plane_out, y = r / Wo, x = r - y * Wo;
    const uint8_t* p = lat + (size_t)bc * H * W + (size_t)(y * S) * W + x * S;
    uint32_t v[L * L];
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int j = 0; j < L; ++j) v[i * L + j] = __ldg(p + (size_t)i * W + j);
    uint32_t m = (uint32_t)T;
#pragma unroll
    for (int e = 0; e < L * L; ++e) m = min(m, v[e]);
    out[(size_t)bc * plane_out + r] = (uint8_t)m;
}

// Planes that fit shared memory (every config's pooling): a CTA copies a run of
// whole input planes — one contiguous byte range — with 16-byte loads, takes the
// window minima from shared memory and writes its contiguous run of output planes
// with 16-byte stores: one HBM read of the input and one write of the output.
constexpr int kPoolSmem = 96 * 1024;

__device__ __forceinline__ void copy_bytes(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, size_t n) {
    if ((((uintptr_t)dst | (uintptr_t)src | n) & 15) == 0) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        for (size_t q = threadIdx.x; q < n / 16; q += blockDim.x) d4[q] = s4[q];
    } else if ((((uintptr_t)dst | (uintptr_t)src | n) & 3) == 0) {
        const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
        uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
        for (size_t q = threadIdx.x; q < n / 4; q += blockDim.x) d4[q] = s4[q];
    } else {
        for (size_t q = threadIdx.x; q < n; q += blockDim.x) dst[q] = src[q];
    }
}

template <bool BULK>
__global__ void __launch_bounds__(kT) pool_smem_kernel(const uint8_t* __restrict__ lat, long long BC, int ppc, int H,
                                                       int W, int T, spk_pool_geom g, int Ho, int Wo,
                                                       uint8_t* __restrict__ out) {
    spk_pdl_wait();
    extern __shared__ __align__(128) uint8_t psm[];
    __shared__ __align__(8) unsigned long long bar;
    const int HW = H * W, HWo = Ho * Wo;
    const long long bc0 = (long long)blockIdx.x * ppc;
    const int np = (int)min((long long)ppc, BC - bc0);
    uint8_t* sin = psm;
    uint8_t* sout = psm + (((size_t)ppc * HW + 127) & ~(size_t)127);
    const uint32_t nin = (uint32_t)np * HW;
    if (BULK) {  // one TMA bulk copy of the run of planes (16-byte multiples, checked on the host)
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nin) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    (uint32_t)__cvta_generic_to_shared(sin)),
                "l"(lat + bc0 * HW), "r"(nin), "r"(b)
                : "memory");
        }
        __syncthreads();  // barrier initialised before anyone polls it
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done)
                         : "r"(b)
                         : "memory");
    } else {
        copy_bytes(sin, lat + bc0 * HW, nin);
        __syncthreads();
    }
    const int n = np * HWo;
    // one output row per warp iteration (divisions amortised over the row)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool p2 = g.Lh == 2 && g.Lw == 2 && g.Sh == 2 && g.Sw == 2 && g.Ph == 0 && g.Pw == 0;
    const uint32_t tt = 0x01010101u * (uint32_t)T;
    // narrow output rows (C2 pool 2: 4 x 4 planes) would idle most lanes of a row-per-warp
    // loop: there every thread takes whole outputs instead
    const bool narrow = Wo < 16;
    for (int o = narrow ? (int)threadIdx.x : n; o < n; o += kT) {
        const int pl = o / HWo, r = o - pl * HWo, y = r / Wo, x = r - y * Wo;
        const int y0 = y * g.Sh - g.Ph, x0 = x * g.Sw - g.Pw;
        const int i0 = max(0, -y0), i1 = min(g.Lh, H - y0), j0 = max(0, -x0), j1 = min(g.Lw, W - x0);
        const uint8_t* r0 = sin + pl * HW + y0 * W + x0;
        int m = T;
        for (int i = i0; i < i1; ++i)
            for (int j = j0; j < j1; ++j) m = min(m, (int)r0[i * W + j]);
        sout[o] = (uint8_t)m;
    }
    for (int row = warp; row < (narrow ? 0 : np * Ho); row += kT / 32) {
        const int pl = row / Ho, y = row - pl * Ho;
        const uint8_t* r0 = sin + pl * HW + (y * g.Sh - g.Ph) * W;
        uint8_t* orow = sout + row * Wo;
        if (p2 && (W & 7) == 0 && (Wo & 3) == 0) {  // 2x2/2: four outputs from two 8-byte reads
            for (int xq = lane; xq < (Wo >> 2); xq += 32) {
                const uint2 a = *reinterpret_cast<const uint2*>(r0 + 8 * xq);
                const uint2 b = *reinterpret_cast<const uint2*>(r0 + W + 8 * xq);
                const uint32_t m0 = __vminu4(a.x, b.x), m1 = __vminu4(a.y, b.y);
                const uint32_t h0 = __vminu4(m0 & 0x00ff00ffu, (m0 >> 8) & 0x00ff00ffu);  // bytes 0, 2
                const uint32_t h1 = __vminu4(m1 & 0x00ff00ffu, (m1 >> 8) & 0x00ff00ffu);
                const uint32_t v = (h0 & 0xffu) | ((h0 >> 8) & 0xff00u) | ((h1 & 0xffu) << 16) | ((h1 << 8) & 0xff000000u);
                *reinterpret_cast<uint32_t*>(orow + 4 * xq) = __vminu4(v, tt);
            }
        } else if (p2 && (W & 1) == 0) {  // 2x2/2: one output from two 2-byte reads
            for (int x = lane; x < Wo; x += 32) {
                const uint32_t a = *reinterpret_cast<const uint16_t*>(r0 + 2 * x);
                const uint32_t b = *reinterpret_cast<const uint16_t*>(r0 + W + 2 * x);
                const uint32_t m = __vminu4(a, b);
                orow[x] = (uint8_t)min(min(m & 0xffu, m >> 8), (uint32_t)T);
            }
        } else {
            const int y0 = y * g.Sh - g.Ph;
            const int i0 = max(0, -y0), i1 = min(g.Lh, H - y0);
            for (int x = lane; x < Wo; x += 32) {
                const int x0 = x * g.Sw - g.Pw;
                const int j0 = max(0, -x0), j1 = min(g.Lw, W - x0);
                int m = T;
                for (int i = i0; i < i1; ++i)
                    for (int j = j0; j < j1; ++j) m = min(m, (int)r0[i * W + x0 + j]);
                orow[x] = (uint8_t)min(m, T);
            }
        }
    }
    if (BULK) {  // TMA bulk store of the run of output planes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + bc0 * HWo),
                         "r"((uint32_t)__cvta_generic_to_shared(sout)), "r"((uint32_t)n)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    } else {
        __syncthreads();
        copy_bytes(out + bc0 * HWo, sout, (size_t)n);
    }
}

// ---------------------------------------------------------------- inhibit
// One CTA per (sample, chunk of <= kInhPix pixels); threads stride over the
// chunk's (channel, pixel) cells so that a sample with few pixels and many maps
// still fills the CTA.  Pass 1: per pixel, shared-memory atomicMin of the unique
// key (lat asc, P* desc, c asc) over firing cells; pass 2: every other firing
// cell of the pixel is set to never.
constexpr int kInhPix = 256;

__global__ void __launch_bounds__(kT) inhibit_kernel(uint8_t* __restrict__ lat, float* __restrict__ pstar, int C,
                                                     int HW, int T, int pc) {
    spk_pdl_wait();
    __shared__ unsigned long long best[kInhPix];
    const int b = blockIdx.y, p0 = blockIdx.x * pc;  // pc <= kInhPix pixels per CTA
    const int np = min(pc, HW - p0);
    uint8_t* L = lat + (size_t)b * C * HW + p0;
    float* P = pstar + (size_t)b * C * HW + p0;
    for (int q = threadIdx.x; q < np; q += kT) best[q] = ~0ull;
    __syncthreads();
    const int n = C * np;
    for (int e = threadIdx.x; e < n; e += kT) {
        const int c = e / np, pl = e - c * np;
        const int l = L[(size_t)c * HW + pl];
        if (l >= T) continue;
        const float ps = P[(size_t)c * HW + pl] + 0.0f;  // -0 -> +0: equal potentials tie on c
        const uint32_t pd = ~spk_float_order_u32(ps);        // larger P* -> smaller key
        atomicMin(&best[pl], ((unsigned long long)l << 56) | ((unsigned long long)pd << 24) | (unsigned)c);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += kT) {
        const int c = e / np, pl = e - c * np;
        const size_t o = (size_t)c * HW + pl;
        if (L[o] < T && (unsigned)c != (unsigned)(best[pl] & 0xFFFFFFu)) {
            L[o] = (uint8_t)T;
            P[o] = 0.0f;
        }
    }
}


// Large maps (HW >= 4096, HW % 4 == 0: C4): a thread owns 4 adjacent pixels of one sample
// and walks every channel twice — first keeping the 4 least keys in registers (4-byte
// latency loads, P* read only where something fired), then writing "never" to every
// other firing cell.  Latencies are read once from HBM (the second walk hits L2),
// potentials once where alive.
__global__ void __launch_bounds__(kT) inhibit_wide_kernel(uint8_t* __restrict__ lat, float* __restrict__ pstar,
                                                          int C, int HW, int T) {
    spk_pdl_wait();
    const int b = blockIdx.y;
    const int p = 4 * (blockIdx.x * kT + threadIdx.x);
    if (p >= HW) return;
    uint8_t* L = lat + (size_t)b * C * HW + p;
    float* P = pstar + (size_t)b * C * HW + p;
    unsigned long long best[4] = {~0ull, ~0ull, ~0ull, ~0ull};
    const uint32_t tt = 0x01010101u * (uint32_t)T;
    constexpr int U = 8;  // channels whose latency words are loaded before any is used
    auto consider = [&](int c, uint32_t l4) {
        if (__vcmpltu4(l4, tt) == 0u) return;  // nothing fired at these 4 pixels
        const float4 p4 = *reinterpret_cast<const float4*>(P + (size_t)c * HW);
        const float pv[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t l = (l4 >> (8 * j)) & 0xffu;
            if (l < (uint32_t)T) {
                const uint32_t pd = ~spk_float_order_u32(pv[j] + 0.0f);  // -0 -> +0: equal potentials tie on c
                const unsigned long long key = ((unsigned long long)l << 56) | ((unsigned long long)pd << 24) | (unsigned)c;
                best[j] = key < best[j] ? key : best[j];
            }
        }
    };
    int c = 0;
    for (; c + U <= C; c += U) {
        uint32_t l4[U];
#pragma unroll
        for (int u = 0; u < U; ++u) l4[u] = *reinterpret_cast<const uint32_t*>(L + (size_t)(c + u) * HW);
#pragma unroll
        for (int u = 0; u < U; ++u) consider(c + u, l4[u]);
    }
    for (; c < C; ++c) consider(c, *reinterpret_cast<const uint32_t*>(L + (size_t)c * HW));
    const uint32_t wc[4] = {(uint32_t)(best[0] & 0xFFFFFFu), (uint32_t)(best[1] & 0xFFFFFFu),
                            (uint32_t)(best[2] & 0xFFFFFFu), (uint32_t)(best[3] & 0xFFFFFFu)};
    auto suppress = [&](int c, uint32_t l4) {
        uint32_t kill = __vcmpltu4(l4, tt);  // 0xff per firing byte
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (wc[j] == (uint32_t)c) kill &= ~(0xffu << (8 * j));
        if (kill == 0u) return;
        *reinterpret_cast<uint32_t*>(L + (size_t)c * HW) = (l4 & ~kill) | (tt & kill);
        float* pp = P + (size_t)c * HW;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (kill & (0xffu << (8 * j))) pp[j] = 0.0f;
    };
    for (c = 0; c + U <= C; c += U) {
        uint32_t l4[U];
#pragma unroll
        for (int u = 0; u < U; ++u) l4[u] = *reinterpret_cast<const uint32_t*>(L + (size_t)(c + u) * HW);
#pragma unroll
        for (int u = 0; u < U; ++u) suppress(c + u, l4[u]);
    }
    for (; c < C; ++c) suppress(c, *reinterpret_cast<const uint32_t*>(L + (size_t)c * HW));
}

// Small maps (HW <= 32: C2 layer 3, 200 maps of 4 x 4): one CTA per sample, thread
// (pixel, channel group) keeps its least key in a register, groups reduced through shared
// memory — no 200-way atomics on one pixel's slot.
__global__ void __launch_bounds__(kT) inhibit_small_kernel(uint8_t* __restrict__ lat, float* __restrict__ pstar,
                                                           int C, int HW, int T) {
    spk_pdl_wait();
    __shared__ unsigned long long part[kT];
    __shared__ uint32_t win_c[32];
    const int b = blockIdx.x;
    const int ngrp = kT / HW, p = threadIdx.x % HW, grp = threadIdx.x / HW;
    uint8_t* L = lat + (size_t)b * C * HW;
    float* P = pstar + (size_t)b * C * HW;
    unsigned long long best = ~0ull;
    // four channels per trip: their latency loads (and the P* loads of those that fired)
    // are in flight together instead of one dependent load per loop trip
    if (grp < ngrp)
        for (int c0 = grp; c0 < C; c0 += 4 * ngrp) {
            int l[4];
            float pv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = c0 + u * ngrp;
                l[u] = c < C ? (int)L[c * HW + p] : T;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) pv[u] = l[u] < T ? P[(c0 + u * ngrp) * HW + p] : 0.0f;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (l[u] >= T) continue;
                const uint32_t pd = ~spk_float_order_u32(pv[u] + 0.0f);  // -0 -> +0: equal potentials tie on c
                const unsigned long long key =
                    ((unsigned long long)l[u] << 56) | ((unsigned long long)pd << 24) | (unsigned)(c0 + u * ngrp);
                best = key < best ? key : best;
            }
        }
    part[threadIdx.x] = best;
    __syncthreads();
    if (threadIdx.x < HW) {
        unsigned long long m = ~0ull;
        for (int g2 = 0; g2 < ngrp; ++g2) m = part[g2 * HW + threadIdx.x] < m ? part[g2 * HW + threadIdx.x] : m;
        win_c[threadIdx.x] = m == ~0ull ? 0xffffffffu : (uint32_t)(m & 0xFFFFFFu);
    }
    __syncthreads();
    if (grp < ngrp) {
        const uint32_t wc = win_c[p];
        for (int c0 = grp; c0 < C; c0 += 4 * ngrp) {
            int l[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = c0 + u * ngrp;
                l[u] = c < C ? (int)L[c * HW + p] : T;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = c0 + u * ngrp;
                if (l[u] < T && (uint32_t)c != wc) {
                    L[c * HW + p] = (uint8_t)T;
                    P[c * HW + p] = 0.0f;
                }
            }
        }
    }
}

// ---------------------------------------------------------------- gather
__global__ void gather_kernel(const uint8_t* __restrict__ lat, size_t n, int T, float* __restrict__ f) {
    spk_pdl_wait();
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int l = min((int)lat[q], T);
    f[q] = __fdiv_rn((float)(T - l), (float)T);
}

// Word per lane: a warp reads 4 x 128 contiguous latency bytes and writes 4 x 512 contiguous
// feature bytes (every store instruction one contiguous run; a 16-latencies-per-thread form
// scattered each store over 2 KB and reached 0.64 of HBM against 0.86 for this one at C5); the
// T+1 possible features come from a shared table of the same IEEE divisions (R-GATHER)
__global__ void __launch_bounds__(kT) gather4_kernel(const uint32_t* __restrict__ lat, size_t n4, int T,
                                                     float4* __restrict__ f) {
    spk_pdl_wait();
    __shared__ float tab[256];
    tab[threadIdx.x] = __fdiv_rn((float)(T - min((int)threadIdx.x, T)), (float)T);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const size_t wid = ((size_t)blockIdx.x * kT + threadIdx.x) >> 5, nw = ((size_t)gridDim.x * kT) >> 5;
    constexpr int U = 4;
    for (size_t w0 = wid * (32 * U); w0 < n4; w0 += nw * (32 * U)) {
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t q = w0 + u * 32 + lane;
            v[u] = q < n4 ? __ldcs(lat + q) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t q = w0 + u * 32 + lane;
            if (q < n4)
                __stcs(f + q, make_float4(tab[v[u] & 0xffu], tab[(v[u] >> 8) & 0xffu], tab[(v[u] >> 16) & 0xffu],
                                          tab[v[u] >> 24]));
        }
    }
}

// ---------------------------------------------------------------- pool, 2x2 stride 2 streaming form
// Unpadded 2x2/2 windows on planes whose width is a multiple of 16 (C4, C5 conv layers):
// a thread reads 16 bytes of each of the window's two input rows and writes the 8 pooled
// bytes; two items per trip keep four 16-byte loads in flight.  No shared-memory staging:
// every input byte is read once and the loads stream straight from HBM.
__global__ void __launch_bounds__(kT) pool2_vec_kernel(const uint4* __restrict__ lat, long long n_items, int cw,
                                                       int W16, int T, uint2* __restrict__ out) {
    spk_pdl_wait();
    // item i: chunk c = i % cw of output row r = i / cw (rows of all planes concatenated:
    // output row r reads input rows 2r, 2r + 1 because H is even)
    const uint32_t tt = 0x01010101u * (uint32_t)T;
    auto pool8 = [&](uint4 a, uint4 b) {
        const uint32_t m[4] = {__vminu4(a.x, b.x), __vminu4(a.y, b.y), __vminu4(a.z, b.z), __vminu4(a.w, b.w)};
        uint32_t h[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) h[k] = __vminu4(m[k] & 0x00ff00ffu, (m[k] >> 8) & 0x00ff00ffu);  // bytes 0, 2
        const uint32_t lo = (h[0] & 0xffu) | ((h[0] >> 8) & 0xff00u) | ((h[1] & 0xffu) << 16) | ((h[1] << 8) & 0xff000000u);
        const uint32_t hi = (h[2] & 0xffu) | ((h[2] >> 8) & 0xff00u) | ((h[3] & 0xffu) << 16) | ((h[3] << 8) & 0xff000000u);
        return make_uint2(__vminu4(lo, tt), __vminu4(hi, tt));
    };
    const long long stride = (long long)gridDim.x * kT;
    long long i = (long long)blockIdx.x * kT + threadIdx.x;
    for (; i + stride < n_items; i += 2 * stride) {
        const long long j = i + stride;
        const long long r0 = i / cw, r1 = j / cw;
        const long long a0 = 2 * r0 * W16 + (i - r0 * cw), a1 = 2 * r1 * W16 + (j - r1 * cw);
        const uint4 x0 = __ldcs(lat + a0), y0 = __ldcs(lat + a0 + W16);
        const uint4 x1 = __ldcs(lat + a1), y1 = __ldcs(lat + a1 + W16);
        __stcs(out + i, pool8(x0, y0));
        __stcs(out + j, pool8(x1, y1));
    }
    if (i < n_items) {
        const long long r0 = i / cw;
        const long long a0 = 2 * r0 * W16 + (i - r0 * cw);
        __stcs(out + i, pool8(__ldcs(lat + a0), __ldcs(lat + a0 + W16)));
    }
}

// ---------------------------------------------------------------- boundary conversions
__global__ void lat_to_dense_kernel(const uint8_t* __restrict__ lat, int B, int T, size_t N,
                                    uint8_t* __restrict__ dense) {
    spk_pdl_wait();
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t total = (size_t)B * T * N;
    if (q >= total) return;
    const size_t i = q % N, t = (q / N) % T, b = q / ((size_t)N * T);
    dense[q] = (uint8_t)(lat[b * N + i] <= t);
}

__global__ void dense_to_lat_kernel(const uint8_t* __restrict__ dense, int B, int T, size_t N,
                                    uint8_t* __restrict__ lat, unsigned int* __restrict__ bad) {
    spk_pdl_wait();
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (size_t)B * N) return;
    const size_t b = q / N, i = q % N;
    int l = T;
    bool ok = true;
    for (int t = 0; t < T; ++t) {
        const uint8_t v = dense[(b * T + t) * N + i];
        if (v > 1) ok = false;
        if (v && l == T) l = t;
        if (!v && l < T) ok = false;  // a 1 followed by a 0: not cumulative
    }
    lat[q] = (uint8_t)l;
    if (!ok) atomicMin(bad, (unsigned int)q);
}

// ---------------------------------------------------------------- R-STDP routing
__global__ void rstdp_route_kernel(spk_winner* __restrict__ win, const int32_t* __restrict__ nwin, int B,
                                   int k, const int32_t* __restrict__ labels, int mpc) {
    spk_pdl_wait();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= B * k) return;
    const int b = q / k, s = q % k;
    if (s >= nwin[b]) return;
    spk_winner& w = win[q];
    w.cfg = (w.c / mpc == labels[w.b]) ? 0 : 1;  // reward : punish (R-CLASSMAP)
}

// ---------------------------------------------------------------- data-parallel STDP
__global__ void winners_rebase_kernel(spk_winner* __restrict__ win, const int32_t* __restrict__ nwin, int B, int k,
                                      int b0) {
    spk_pdl_wait();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= B * k) return;
    const int b = q / k, s = q % k;
    if (s < nwin[b]) win[q].b += b0;  // local sample index -> index in the global mini-batch
}

}  // namespace

extern "C" spk_status spk_fire(const float* pot, int B, int T, int C, int H, int W, float theta,
                               uint8_t* lat, float* pstar, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(pot);
    SPK_CHECK_PTR(lat);
    SPK_CHECK(B >= 1 && T >= 1 && C >= 1 && H >= 1 && W >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK(T <= 254, SPK_ERR_UNSUPPORTED, "T > 254");
    const size_t N = (size_t)C * H * W;
    const bool vec = (N & 3) == 0 && (reinterpret_cast<uintptr_t>(pot) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(lat) & 3) == 0 && (reinterpret_cast<uintptr_t>(pstar) & 15) == 0;
    if (vec) {
        spk::launch(fire4_kernel, spk::ceil_div((size_t)B * (N / 4), kT), kT, 0, spk::as_cuda(stream),
            reinterpret_cast<const float4*>(pot), B, T, N / 4, theta, reinterpret_cast<uchar4*>(lat),
            reinterpret_cast<float4*>(pstar));
        return spk::launched("fire4_kernel");
    }
    spk::launch(fire_kernel, spk::ceil_div((size_t)B * N, kT), kT, 0, spk::as_cuda(stream), pot, B, T, N, theta, lat,
                                                                                 pstar);
    return spk::launched("fire_kernel");
}

extern "C" spk_status spk_pool(const uint8_t* lat, int B, int C, int H, int W, int T,
                               const spk_pool_geom* p, uint8_t* out, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(p);
    SPK_CHECK_PTR(out);
    SPK_CHECK(B >= 1 && C >= 1 && H >= 1 && W >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK(T >= 1 && T <= 254, SPK_ERR_UNSUPPORTED, "T=%d outside 1..254", T);
    SPK_CHECK(p->Lh >= 1 && p->Lw >= 1 && p->Sh >= 1 && p->Sw >= 1 && p->Ph >= 0 && p->Pw >= 0, SPK_ERR_ARG,
              "bad pool geometry");
    const int Ho = (H + 2 * p->Ph - p->Lh) / p->Sh + 1, Wo = (W + 2 * p->Pw - p->Lw) / p->Sw + 1;
    SPK_CHECK(H + 2 * p->Ph >= p->Lh && W + 2 * p->Pw >= p->Lw && Ho >= 1 && Wo >= 1, SPK_ERR_SHAPE,
              "pool window larger than padded input (Eq. 3)");
    SPK_CHECK((long long)H * W < (1ll << 31), SPK_ERR_SHAPE, "input plane too large");
    SPK_CHECK((long long)Ho * Wo <= (1 << 30), SPK_ERR_SHAPE, "output plane too large");
    const long long BC = (long long)B * C;
    const int plane_out = Ho * Wo;
    const size_t per_plane = (size_t)H * W + (size_t)plane_out;
    // large planes (C4, C5): whole planes through shared memory, by TMA bulk copies when
    // every run is 16-byte aligned; small planes (C1-C3, L2-resident) take the direct kernel
    static const long long smem_min = [] {  // A/B knob: smallest plane staged through smem
        const char* e = std::getenv("SPK_POOL_SMEM_MIN");
        return e ? std::atoll(e) : 2048ll;
    }();
    // 2x2/2 on even-height planes 16 bytes wide (C5): streaming kernel, no staging
    if (p->Lh == 2 && p->Lw == 2 && p->Sh == 2 && p->Sw == 2 && p->Ph == 0 && p->Pw == 0 && H % 2 == 0 &&
        W % 16 == 0 && (long long)H * W >= smem_min &&
        ((reinterpret_cast<uintptr_t>(lat) & 15) | (reinterpret_cast<uintptr_t>(out) & 7)) == 0) {
        const int cw = W / 16;
        const long long n_items = BC * Ho * cw;
        const unsigned blocks = (unsigned)std::min<long long>((n_items + 2 * kT - 1) / (2 * kT), (long long)spk::sm_count() * 8);
        spk::launch(pool2_vec_kernel, blocks, kT, 0, spk::as_cuda(stream), reinterpret_cast<const uint4*>(lat), n_items, cw,
                                                                  cw, T, reinterpret_cast<uint2*>(out));
        return spk::launched("pool2_vec_kernel");
    }
    if ((long long)H * W >= smem_min && per_plane + 256 <= (size_t)kPoolSmem) {
        const int ppc = (int)std::min<long long>(BC, std::max<long long>(1, (24 * 1024) / (long long)per_plane));  // ~24 KB per CTA
        const size_t smem = (((size_t)ppc * H * W + 127) & ~(size_t)127) + (size_t)ppc * plane_out;
        const long long nblk = (BC + ppc - 1) / ppc;
        SPK_CHECK(nblk < (1ll << 31), SPK_ERR_SHAPE, "B*C too large");
        const bool bulk = ((H * W) % 16 == 0) && (plane_out % 16 == 0) &&
                          ((reinterpret_cast<uintptr_t>(lat) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
        static std::atomic<uint64_t> attr{0};
        if (spk::first_on_device(attr)) {
            cudaFuncSetAttribute(pool_smem_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPoolSmem);
            cudaFuncSetAttribute(pool_smem_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPoolSmem);
        }
        if (bulk) {
            spk::launch(pool_smem_kernel<true>, (unsigned)nblk, kT, smem, spk::as_cuda(stream), lat, BC, ppc, H, W, T, *p, Ho, Wo, out);
            return spk::launched("pool_smem_kernel<bulk>");
        }
        spk::launch(pool_smem_kernel<false>, (unsigned)nblk, kT, smem, spk::as_cuda(stream), lat, BC, ppc, H, W, T, *p, Ho, Wo, out);
        return spk::launched("pool_smem_kernel");
    }
    const long long ppy = std::min<long long>(BC, std::max(1, (1 << 30) / plane_out));
    const long long gy = (BC + ppy - 1) / ppy;
    SPK_CHECK(gy <= 65535, SPK_ERR_SHAPE, "B*C too large");
    const dim3 grid(spk::ceil_div((size_t)ppy * plane_out, kT), (unsigned)gy);
    static const bool fixed_ok = [] {  // A/B knob: SPK_POOL_FIXED=0 keeps the generic kernel
        const char* e = std::getenv("SPK_POOL_FIXED");
        return !(e && e[0] == '0');
    }();
    if (fixed_ok && p->Ph == 0 && p->Pw == 0 && p->Lh == p->Lw && p->Sh == p->Sw && (p->Lh == 2 || p->Lh == 3)) {
        if (p->Lh == 2)
            spk::launch(pool_fixed_kernel<2>, grid, kT, 0, spk::as_cuda(stream), lat, BC, (int)ppy, H, W, T, p->Sh, Ho, Wo, out);
        else
            spk::launch(pool_fixed_kernel<3>, grid, kT, 0, spk::as_cuda(stream), lat, BC, (int)ppy, H, W, T, p->Sh, Ho, Wo, out);
        return spk::launched("pool_fixed_kernel");
    }
    spk::launch(pool_kernel, grid, kT, 0, spk::as_cuda(stream), lat, BC, (int)ppy, H, W, T, *p, Ho, Wo, out);
    return spk::launched("pool_kernel");
}

extern "C" spk_status spk_inhibit(uint8_t* lat, float* pstar, int B, int C, int H, int W, int T,
                                  spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(pstar);
    SPK_CHECK(B >= 1 && C >= 1 && H >= 1 && W >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK(T >= 1 && T <= 254, SPK_ERR_UNSUPPORTED, "T=%d outside 1..254", T);
    SPK_CHECK(C < (1 << 24), SPK_ERR_UNSUPPORTED, "C=%d >= 2^24", C);
    SPK_CHECK((long long)H * W < (1ll << 31) && (long long)C * kInhPix < (1ll << 31), SPK_ERR_SHAPE, "map too large");
    SPK_CHECK(B <= 65535, SPK_ERR_SHAPE, "B=%d > 65535", B);
    const int HW = H * W;
    if (HW <= 32) {
        spk::launch(inhibit_small_kernel, (unsigned)B, kT, 0, spk::as_cuda(stream), lat, pstar, C, HW, T);
        return spk::launched("inhibit_small_kernel");
    }
    if (HW >= 4096 && (HW & 3) == 0 && ((reinterpret_cast<uintptr_t>(lat) | reinterpret_cast<uintptr_t>(pstar)) & 15) == 0) {
        const dim3 grid(spk::ceil_div((size_t)HW / 4, kT), (unsigned)B);
        spk::launch(inhibit_wide_kernel, grid, kT, 0, spk::as_cuda(stream), lat, pstar, C, HW, T);
        return spk::launched("inhibit_wide_kernel");
    }
    // fewer pixels per CTA when the grid would not cover the SMs (C1: one 28x28 sample),
    // so each thread walks a few cells instead of a long chain of dependent loads
    int pc = kInhPix;
    if ((long long)B * spk::ceil_div((size_t)HW, kInhPix) < 148) {
        const int want = (296 + B - 1) / B;  // CTAs per sample
        pc = std::max(1, std::min(kInhPix, (HW + want - 1) / want));
    }
    const dim3 grid(spk::ceil_div((size_t)HW, pc), (unsigned)B);
    spk::launch(inhibit_kernel, grid, kT, 0, spk::as_cuda(stream), lat, pstar, C, HW, T, pc);
    return spk::launched("inhibit_kernel");
}

extern "C" spk_status spk_gather(const uint8_t* lat, size_t n, int T, float* feat, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(feat);
    SPK_CHECK(T >= 1 && T <= 254, SPK_ERR_UNSUPPORTED, "T=%d outside 1..254", T);
    if (n == 0) return SPK_OK;
    if (n % 4 == 0 && (reinterpret_cast<uintptr_t>(lat) & 3) == 0 && (reinterpret_cast<uintptr_t>(feat) & 15) == 0) {
        const size_t n4 = n / 4;
        const unsigned blocks = (unsigned)std::min<size_t>(spk::ceil_div(n4, (size_t)kT * 4), (size_t)spk::sm_count() * 8);
        spk::launch(gather4_kernel, blocks, kT, 0, spk::as_cuda(stream), reinterpret_cast<const uint32_t*>(lat), n4, T,
                                                                reinterpret_cast<float4*>(feat));
        return spk::launched("gather4_kernel");
    }
    spk::launch(gather_kernel, spk::ceil_div(n, kT), kT, 0, spk::as_cuda(stream), lat, n, T, feat);
    return spk::launched("gather_kernel");
}

extern "C" spk_status spk_lat_to_dense(const uint8_t* lat, int B, int T, size_t N, uint8_t* dense,
                                       spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(dense);
    SPK_CHECK(B >= 1 && N >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK(T >= 1 && T <= 254, SPK_ERR_UNSUPPORTED, "T=%d outside 1..254", T);
    const size_t n = (size_t)B * T * N;
    spk::launch(lat_to_dense_kernel, spk::ceil_div(n, kT), kT, 0, spk::as_cuda(stream), lat, B, T, N, dense);
    return spk::launched("lat_to_dense_kernel");
}

extern "C" spk_status spk_dense_to_lat(const uint8_t* dense, int B, int T, size_t N, uint8_t* lat,
                                       int32_t* bad_index, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(dense);
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(bad_index);
    SPK_CHECK(B >= 1 && N >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK(T >= 1 && T <= 254, SPK_ERR_UNSUPPORTED, "T=%d outside 1..254", T);
    SPK_CHECK((size_t)B * N < 0x7fffffffull, SPK_ERR_SHAPE, "B*N too large for the i32 bad_index");
    cudaStream_t s = spk::as_cuda(stream);
    if (cudaMemsetAsync(bad_index, 0xff, sizeof(int32_t), s) != cudaSuccess)
        return spk::launched("memset(bad_index)");
    const size_t n = (size_t)B * N;
    spk::launch(dense_to_lat_kernel, spk::ceil_div(n, kT), kT, 0, s, dense, B, T, N, lat,
                                                            reinterpret_cast<unsigned int*>(bad_index));
    return spk::launched("dense_to_lat_kernel");
}

extern "C" spk_status spk_rstdp_route(spk_winner* win, const int32_t* nwin, int B, int k,
                                      const int32_t* labels, int maps_per_class, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(win);
    SPK_CHECK_PTR(nwin);
    SPK_CHECK_PTR(labels);
    SPK_CHECK(B >= 1 && k >= 1, SPK_ERR_ARG, "B=%d k=%d", B, k);
    SPK_CHECK(maps_per_class >= 1, SPK_ERR_ARG, "maps_per_class < 1");
    spk::launch(rstdp_route_kernel, spk::ceil_div((size_t)B * k, kT), kT, 0, spk::as_cuda(stream), win, nwin, B, k, labels,
                                                                                        maps_per_class);
    return spk::launched("rstdp_route_kernel");
}

extern "C" spk_status spk_winners_rebase(spk_winner* win, const int32_t* nwin, int B, int k, int b0,
                                         spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(win);
    SPK_CHECK_PTR(nwin);
    SPK_CHECK(B >= 1 && k >= 1 && b0 >= 0, SPK_ERR_ARG, "B=%d k=%d b0=%d", B, k, b0);
    SPK_CHECK((long long)B * k < (1ll << 31), SPK_ERR_ARG, "B*k too large");
    spk::launch(winners_rebase_kernel, spk::ceil_div((size_t)B * k, kT), kT, 0, spk::as_cuda(stream), win, nwin, B, k, b0);
    return spk::launched("winners_rebase_kernel");
}
