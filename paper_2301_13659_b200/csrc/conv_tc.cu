// conv_tc.cu — a3 + a4: the spiking convolution (Eq. 2) as ONE
// implicit GEMM on the sm_100a 5th-generation tensor cores, with the IF fire
// fused into the TMEM epilogue.
//
//   rows  M = (pixel, t)  — every time step of every output pixel ("Spyker
//                           processes all the time steps at once");
//                           t is padded to TP in {16, 32} so one pixel's steps
//                           are TP consecutive TMEM lanes of one warp.  An
//                           M tile (128 rows = 128/TP pixels) never crosses a
//                           sample.
//   cols  N = output map o (tile Nt <= 160)
//   depth K = synapse (c, i, j), in the kernel's [Co][Ci][Kh][Kw] order.
//   A[(p,t), k] = [lat_in(p, k) <= t]   — the cumulative spike train, built on
//                 the fly in shared memory from the u8 latency map (never
//                 materialised in HBM), u8 {0,1};
//   B[k, o]     = weight digit planes: w = s * sum_d q_d 2^(8d-23), q_d in u8
//                 (23-bit fixed point, s = power of two >= w_max).
//   D_d = A x B_d with tcgen05.mma kind::i8 (s32 accumulators in TMEM, exact);
//   X = D_2 2^16 + D_1 2^8 + D_0 is the exact integer potential in units of
//   s 2^-23; fire iff X > floor(theta 2^23 / s); P = X s 2^-23 rounded once.
//
// Persistent, warp-specialised CTA (one per SM), 16 warps:
//   warps 0-7   producers: im2col gather of latencies from the staged input
//               band -> expand to the A tile of each K stage
//   warps 8-11  epilogue: tcgen05.ld -> integer threshold test, warp ballot,
//               first-crossing time (popcount: potentials are monotone in t),
//               potential at the crossing
//   warp  12    MMA issuer (one thread), TMEM allocator
//   warp  13    B loader: cp.async.bulk of pre-packed digit planes
//   warps 14-15 band loaders: copy the input rows a tile needs into smem
// Pipelines (mbarriers): input band (1-2 buffers), smem K stages (4), TMEM
// accumulators (1-2 buffers).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "conv.cuh"

namespace {

constexpr int KS = kTcKS;          // synapses per stage (2 MMAs of K=32)
constexpr int S = kTcStages;       // pipeline depth
constexpr int kThreads = 512;      // 16 warps
constexpr int kProd = 256;         // warps 0-7
constexpr int kLoaders = 64;       // warps 14-15
constexpr int kLoadBatch = 8;      // independent loads in flight per band-loader thread
constexpr uint32_t kNever = 0xFFFFFFFFu;

// Optional per-role cycle accounting (SPK_CONV_PROF=1): [block][role][total, wait]
constexpr int kProfRoles = 5;  // producer, epilogue, mma, b-loader, band-loader
__device__ unsigned long long g_conv_prof[1024][kProfRoles][2];

struct TcArgs {
    const uint8_t* lat_in;
    const uint8_t* wpk;  // packed digit planes
    void* out0;
    float* out1;
    spk_conv_geom g;
    int Ho, Wo, HWo, K, nks, TP, logTP, PPT, Nt, n_ntiles, NB, tps, NR, band, nrb, rb_stride;
    long long total_tiles;
    long long theta_q;  // fire iff X > theta_q
    float out_scale;
    uint32_t a_off, b_off, lc_off, kt_off, rg_off, bar_off;  // smem carve-up
    int prof;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t a, uint32_t bytes) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(a), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accum) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
// K-major, no swizzle: 8-row x 16-byte core matrices; LBO = stride between the
// two 16-byte K chunks of one MMA, SBO = stride between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// bytes of a: 1 where a <= t (t < 128), else 0  (SWAR, no cross-byte borrow)
__device__ __forceinline__ uint32_t le_bytes(uint32_t a, uint32_t tt /* t * 0x01010101 | 0x80808080 */) {
    const uint32_t hi = a & 0x80808080u;
    const uint32_t r = tt - (a & 0x7F7F7F7Fu);
    return ((r & ~hi) & 0x80808080u) >> 7;
}

struct TileCoord {
    int b, p0, r0;  // sample, first pixel of the tile (within the sample), first staged input row
};

__device__ __forceinline__ TileCoord tile_coord(const TcArgs& a, long long mt) {
    TileCoord tc;
    tc.b = (int)(mt / a.tps);
    tc.p0 = (int)(mt - (long long)tc.b * a.tps) * a.PPT;
    const int lo = (tc.p0 / a.Wo) * a.g.Sh - a.g.Ph;  // first input row the tile's receptive fields touch
    tc.r0 = max(0, min(lo, a.g.Hi - a.NR));
    return tc;
}

struct RoleClock {
    long long t0 = 0, wait = 0;
    bool on;
    __device__ RoleClock(bool p) : on(p) {
        if (on) t0 = clock64();
    }
    __device__ __forceinline__ void wait_on(uint32_t bar, uint32_t parity) {
        if (!on) {
            mbar_wait(bar, parity);
            return;
        }
        const long long w0 = clock64();
        mbar_wait(bar, parity);
        wait += clock64() - w0;
    }
    // one lane polls, the warp then proceeds together (no smem polling storm)
    __device__ __forceinline__ void wait_warp(uint32_t bar, uint32_t parity) {
        if ((threadIdx.x & 31) == 0) wait_on(bar, parity);
        __syncwarp();
    }
    __device__ void store(int role) {
        if (on && blockIdx.x < 1024) {
            g_conv_prof[blockIdx.x][role][0] = (unsigned long long)(clock64() - t0);
            g_conv_prof[blockIdx.x][role][1] = (unsigned long long)wait;
        }
    }
};

// Contiguous range of tiles of this CTA (consecutive tiles share a sample, so
// the staged input map is reused across them).
__device__ __forceinline__ void tile_range(const TcArgs& a, long long& t0, long long& t1) {
    t0 = (long long)blockIdx.x * a.total_tiles / gridDim.x;
    t1 = (long long)(blockIdx.x + 1) * a.total_tiles / gridDim.x;
}
// Identity of the staged input region a tile reads: the sample when whole
// sample maps are staged (NR == Hi), else the M tile.
__device__ __forceinline__ long long region_key(const TcArgs& a, long long tile) {
    const long long mt = tile / a.n_ntiles;
    return a.NR == a.g.Hi ? mt / a.tps : mt;
}

// ------------------------------------------------------------------ the kernel
template <int EPI, bool PSTAR, int TP>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(const TcArgs a) {
    constexpr int LOGTP = TP == 16 ? 4 : 5;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* As = smem + a.a_off;
    uint8_t* Bs = smem + a.b_off;
    uint8_t* LC = smem + a.lc_off;  // latcol double buffer: [2][PPT][KS]
    const uint32_t* ktab = reinterpret_cast<const uint32_t*>(smem + a.kt_off);
    uint8_t* RG = smem + a.rg_off;  // staged input band(s): [nrb][Ci][NR][Wi]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.bar_off);
    // barrier map: full[S] empty[S] accf[2] acce[2] rgf[2] rge[2], then the TMEM address
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * S + 8);
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S);
    const uint32_t accf0 = smem_u32(bars + 2 * S), acce0 = smem_u32(bars + 2 * S + 2);
    const uint32_t rgf0 = smem_u32(bars + 2 * S + 4), rge0 = smem_u32(bars + 2 * S + 6);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const spk_conv_geom& g = a.g;

    {  // synapse table: (c*NR*Wi + i*Wi + j) << 8 | i << 4 | j, or kNever for padding k >= K
        uint32_t* kt = reinterpret_cast<uint32_t*>(smem + a.kt_off);
        const int KhKw = g.Kh * g.Kw;
        for (int k = threadIdx.x; k < a.nks * KS; k += kThreads) {
            uint32_t e = kNever;
            if (k < a.K) {
                const int c = k / KhKw, r = k - c * KhKw, i = r / g.Kw, j = r - i * g.Kw;
                e = ((uint32_t)(c * a.band + i * g.Wi + j) << 8) | ((uint32_t)i << 4) | (uint32_t)j;
            }
            kt[k] = e;
        }
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, kProd / 32 + 1);  // producer warps + B-loader arrive.expect_tx
            mbar_init(empty0 + 8 * s, 1);       // tcgen05.commit
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(accf0 + 8 * b, 1);          // tcgen05.commit
            mbar_init(acce0 + 8 * b, 4);               // epilogue warps
            mbar_init(rgf0 + 8 * b, kLoaders / 32);    // band loader warps
            mbar_init(rge0 + 8 * b, kProd / 32);       // producer warps
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 12) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp < 8) {
        // ======================= producers (warps 0-7) =======================
        RoleClock rc(a.prof != 0);
        // Warp w builds row groups w and w+8 of every A stage (pixels pA, pB),
        // gathering exactly the latencies those rows need: no cross-warp barrier.
        const int pA = (warp * 8) >> LOGTP, pB = ((warp + 8) * 8) >> LOGTP;
        const int gsel = lane >> 4;            // gather: 0 -> pA, 1 -> pB
        const int gk0 = (lane & 15) * 4;       // 4 synapses per lane
        const int q = lane >> 3, rl = lane & 7;
        uint8_t* lcw = LC + warp * 256;        // per-warp latcol: [2 bufs][2 pixels][KS]
        long long t0, t1;
        tile_range(a, t0, t1);
        long long sidx = 0, prev_key = -1;
        int rcount = 0, rb = 0;
        for (long long tile = t0; tile < t1; ++tile) {
            const long long key = region_key(a, tile);
            if (key != prev_key) {
                prev_key = key;
                rb = rcount % a.nrb;
                rc.wait_warp(rgf0 + 8 * rb, (uint32_t)((rcount / a.nrb) & 1));
                ++rcount;
            }
            const bool last_use = (tile + 1 >= t1) || region_key(a, tile + 1) != key;
            const TileCoord tc = tile_coord(a, tile / a.n_ntiles);
            const uint8_t* region = RG + rb * a.rb_stride;
            const int p = tc.p0 + (gsel ? pB : pA);
            const bool pvalid = p < a.HWo;
            int y0 = 0, x0 = 0, pixbase = 0;
            if (pvalid) {
                const int yo = p / a.Wo, xo = p - yo * a.Wo;
                y0 = yo * g.Sh - g.Ph;
                x0 = xo * g.Sw - g.Pw;
                pixbase = (y0 - tc.r0) * g.Wi + x0;
            }
            auto gather = [&](int ks) -> uint32_t {
                uint32_t packed = 0;
                const uint4 te4 = *reinterpret_cast<const uint4*>(ktab + ks * KS + gk0);
                const uint32_t te[4] = {te4.x, te4.y, te4.z, te4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    uint32_t v = 0xFFu;
                    if (pvalid && te[e] != kNever) {
                        const int iy = y0 + (int)((te[e] >> 4) & 15u), ix = x0 + (int)(te[e] & 15u);
                        if ((unsigned)iy < (unsigned)g.Hi && (unsigned)ix < (unsigned)g.Wi)
                            v = region[pixbase + (int)(te[e] >> 8)];
                    }
                    packed |= v << (8 * e);
                }
                return packed;
            };
            uint32_t cur = gather(0);
            for (int ks = 0; ks < a.nks; ++ks, ++sidx) {
                const int s = (int)(sidx % S);
                const uint32_t ph = (uint32_t)((sidx / S) & 1);
                uint8_t* lc = lcw + (sidx & 1) * 128;
                *reinterpret_cast<uint32_t*>(lc + gsel * KS + gk0) = cur;
                __syncwarp();
                if (ks + 1 < a.nks) cur = gather(ks + 1);  // next stage's loads overlap this expansion
                else if (last_use) {  // staged region no longer read by this warp
                    __syncwarp();
                    if (lane == 0) mbar_arrive(rge0 + 8 * rb);
                }
                // --- wait for the MMAs that last read this A stage, then expand
                rc.wait_warp(empty0 + 8 * s, ph ^ 1u);
                uint8_t* A = As + s * (128 * KS);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int grp = u * 8 + warp;  // 8-row group; chunk c = q
                    const int t = (grp * 8 + rl) & (TP - 1);
                    const uint4 L = *reinterpret_cast<const uint4*>(lc + u * KS + q * 16);
                    const uint32_t tt = 0x80808080u | ((uint32_t)t * 0x01010101u);
                    uint4 o;
                    o.x = le_bytes(L.x, tt);
                    o.y = le_bytes(L.y, tt);
                    o.z = le_bytes(L.z, tt);
                    o.w = le_bytes(L.w, tt);
                    *reinterpret_cast<uint4*>(A + q * 2048 + grp * 128 + rl * 16) = o;
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(full0 + 8 * s);
            }
        }
        if (threadIdx.x == 0) rc.store(0);
    } else if (warp < 12) {
        // ======================= epilogue (warps 8-11) =======================
        RoleClock rc(a.prof != 0);
        const int qd = warp & 3;                  // TMEM lane quadrant
        const int row = qd * 32 + lane;           // accumulator row = (pixel, t)
        const int pix = row >> LOGTP, t = row & (TP - 1);
        const int segbase = lane & ~(TP - 1);
        const uint32_t segmask = (TP == 32) ? 0xffffffffu : ((1u << TP) - 1u);
        long long t0, t1, it = 0;
        tile_range(a, t0, t1);
        for (long long tile = t0; tile < t1; ++tile, ++it) {
            const int buf = (int)(it % a.NB);
            const long long mt = tile / a.n_ntiles;
            const int nt = (int)(tile % a.n_ntiles);
            const int b = (int)(mt / a.tps);
            const int p = (int)(mt - (long long)b * a.tps) * a.PPT + pix;
            const bool pvalid = p < a.HWo;
            const bool rvalid = pvalid && t < g.T;
            const bool writer = pvalid && t == 0;
            rc.wait_warp(accf0 + 8 * buf, (uint32_t)((it / a.NB) & 1));
            tc_fence_after();
            const uint32_t tbase = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(buf * 3 * a.Nt);
            for (int n0 = 0; n0 < a.Nt; n0 += 16) {
                uint32_t d0[16], d1[16], d2[16];
                tmem_ld16(tbase + n0, d0);
                tmem_ld16(tbase + a.Nt + n0, d1);
                tmem_ld16(tbase + 2 * a.Nt + n0, d2);
                tmem_wait_ld();
                const int obase = nt * a.Nt + n0;
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    const int o = obase + jj;
                    const int L = (int)d1[jj] * 256 + (int)d0[jj];
                    const long long X = (long long)(int)d2[jj] * 65536ll + (long long)L;
                    if (EPI == SPK_EPI_POTENTIAL) {
                        if (rvalid && o < g.Co)
                            static_cast<float*>(a.out0)[(((size_t)b * g.T + t) * g.Co + o) * a.HWo + p] =
                                __fmul_rn(__ll2float_rn(X), a.out_scale);
                    } else {
                        const unsigned bal = __ballot_sync(0xffffffffu, rvalid && X > a.theta_q);
                        const unsigned bits = (bal >> segbase) & segmask;
                        const int l = g.T - __popc(bits);  // fired steps are exactly t = lat .. T-1
                        float ps = 0.0f;
                        if (PSTAR) {
                            const long long Xs = __shfl_sync(0xffffffffu, X, segbase + min(l, TP - 1));
                            ps = bits ? __fmul_rn(__ll2float_rn(Xs), a.out_scale) : 0.0f;
                        }
                        if (writer && o < g.Co) {
                            const size_t oi = ((size_t)b * g.Co + o) * a.HWo + p;
                            static_cast<uint8_t*>(a.out0)[oi] = (uint8_t)l;
                            if (PSTAR) a.out1[oi] = ps;
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acce0 + 8 * buf);
        }
        if (warp == 8 && lane == 0) rc.store(1);
    } else if (warp == 12) {
        // ======================= MMA issuer =======================
        RoleClock rc(a.prof != 0);
        if (lane == 0) {
            const uint32_t idesc = (2u << 4) | ((uint32_t)(a.Nt >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            const uint32_t a_base = smem_u32(As), b_base = smem_u32(Bs);
            const uint32_t bstage = 3u * a.Nt * KS, bdig = (uint32_t)a.Nt * KS, bchunk = (uint32_t)a.Nt * 16;
            long long sidx = 0, it = 0, t0, t1;
            tile_range(a, t0, t1);
            for (long long tile = t0; tile < t1; ++tile, ++it) {
                const int buf = (int)(it % a.NB);
                rc.wait_on(acce0 + 8 * buf, (uint32_t)(((it / a.NB) & 1) ^ 1));
                tc_fence_after();
                const uint32_t dbase = tmem + (uint32_t)(buf * 3 * a.Nt);
                for (int ks = 0; ks < a.nks; ++ks, ++sidx) {
                    const int s = (int)(sidx % S);
                    rc.wait_on(full0 + 8 * s, (uint32_t)((sidx / S) & 1));
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < KS / 32; ++kk) {
                        const uint64_t ad = smem_desc(a_base + s * (128 * KS) + kk * 2 * 2048, 2048, 128);
#pragma unroll
                        for (int d = 0; d < 3; ++d) {
                            const uint64_t bd =
                                smem_desc(b_base + s * bstage + d * bdig + kk * 2 * bchunk, bchunk, 128);
                            tc_mma_i8(dbase + d * a.Nt, ad, bd, idesc, (ks | kk) ? 1u : 0u);
                        }
                    }
                    tc_commit(empty0 + 8 * s);
                }
                tc_commit(accf0 + 8 * buf);
            }
            rc.store(2);
        }
        __syncwarp();
    } else if (warp == 13) {
        // ======================= B loader =======================
        RoleClock rc(a.prof != 0);
        if (lane == 0) {
            const uint32_t bstage = 3u * a.Nt * KS;
            const uint32_t b_base = smem_u32(Bs);
            long long sidx = 0, t0, t1;
            tile_range(a, t0, t1);
            for (long long tile = t0; tile < t1; ++tile) {
                const int nt = (int)(tile % a.n_ntiles);
                for (int ks = 0; ks < a.nks; ++ks, ++sidx) {
                    const int s = (int)(sidx % S);
                    rc.wait_on(empty0 + 8 * s, (uint32_t)(((sidx / S) & 1) ^ 1));
                    mbar_arrive_tx(full0 + 8 * s, bstage);
                    bulk_g2s(b_base + s * bstage, a.wpk + ((size_t)nt * a.nks + ks) * bstage, bstage, full0 + 8 * s);
                }
            }
            rc.store(3);
        }
        __syncwarp();
    } else {
        // ======================= input band loaders (warps 14-15) =======================
        RoleClock rc(a.prof != 0);
        const int lt = threadIdx.x - (kThreads - kLoaders);  // 0..63
        const size_t plane = (size_t)g.Hi * g.Wi;
        long long t0, t1, prev_key = -1;
        tile_range(a, t0, t1);
        int rcount = 0;
        for (long long tile = t0; tile < t1; ++tile) {
            const long long key = region_key(a, tile);
            if (key == prev_key) continue;  // same staged region as the previous tile
            prev_key = key;
            const TileCoord tc = tile_coord(a, tile / a.n_ntiles);
            const int rb = rcount % a.nrb;
            uint8_t* dst = RG + rb * a.rb_stride;
            rc.wait_warp(rge0 + 8 * rb, (uint32_t)(((rcount / a.nrb) & 1) ^ 1));
            ++rcount;
            const uint8_t* src = a.lat_in + (size_t)tc.b * g.Ci * plane + (size_t)tc.r0 * g.Wi;
            const int total = g.Ci * a.band;
            if (a.NR == g.Hi && (reinterpret_cast<uintptr_t>(src) & 3) == 0) {
                // whole sample map, 4-byte aligned: one contiguous block of Ci*Hi*Wi bytes
                const int n4 = total >> 2;
                const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
                uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
                for (int q0 = 0; q0 < n4; q0 += kLoaders * kLoadBatch) {
                    uint32_t v[kLoadBatch];
#pragma unroll
                    for (int u = 0; u < kLoadBatch; ++u) {
                        const int q = q0 + u * kLoaders + lt;
                        v[u] = q < n4 ? __ldg(s4 + q) : 0u;
                    }
#pragma unroll
                    for (int u = 0; u < kLoadBatch; ++u) {
                        const int q = q0 + u * kLoaders + lt;
                        if (q < n4) d4[q] = v[u];
                    }
                }
                for (int q = (n4 << 2) + lt; q < total; q += kLoaders) dst[q] = __ldg(src + q);
            } else {
                // Ci bands of NR*Wi contiguous bytes (channel planes are Hi*Wi apart)
                int c = lt / a.band, off = lt - (lt / a.band) * a.band;  // running (channel, offset)
                for (int q0 = 0; q0 < total; q0 += kLoaders * kLoadBatch) {
                    uint8_t v[kLoadBatch];
                    int d[kLoadBatch];
#pragma unroll
                    for (int u = 0; u < kLoadBatch; ++u) {
                        const bool ok = q0 + u * kLoaders + lt < total;
                        v[u] = ok ? __ldg(src + (size_t)c * plane + off) : (uint8_t)0;
                        d[u] = ok ? c * a.band + off : -1;
                        off += kLoaders;
                        while (off >= a.band) {
                            off -= a.band;
                            ++c;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kLoadBatch; ++u)
                        if (d[u] >= 0) dst[d[u]] = v[u];
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(rgf0 + 8 * rb);
        }
        if (lt == 0) rc.store(4);
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 12) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// ------------------------------------------------------------------ weight packing
// Digit planes in the exact smem image of each (n-tile, K-stage) block:
//   block (nt, ks): [digit 0..2][chunk 0..KS/16-1][Nt/8 row groups][8 rows][16 bytes]
__global__ void pack_weights_kernel(const float* __restrict__ w, int Co, int K, int Nt, int n_ntiles, int nks,
                                    float inv_scale23, uint8_t* __restrict__ wpk, int* __restrict__ flag) {
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // over (nt, ks, c, n, e)
    const size_t per_block = (size_t)Nt * KS;
    if (q >= (size_t)n_ntiles * nks * per_block) return;
    const size_t blk = q / per_block, r = q % per_block;
    const int nt = (int)(blk / nks), ks = (int)(blk % nks);
    const int c = (int)(r / ((size_t)Nt * 16)), r2 = (int)(r % ((size_t)Nt * 16));
    const int n = r2 / 16, e = r2 % 16;
    const int k = ks * KS + c * 16 + e, o = nt * Nt + n;
    float v = 0.0f;
    if (o < Co && k < K) v = w[(size_t)o * K + k];
    float x = __fmul_rn(v, inv_scale23);  // exact: inv_scale23 is a power of two
    if (!(x >= 0.0f) || x > 8388608.0f) {  // negative, NaN or above the scale: clamp and flag
        atomicOr(flag, 1);
        x = (x > 8388608.0f) ? 8388608.0f : 0.0f;
    }
    const uint32_t qv = (uint32_t)__float2int_rn(x);  // 0 .. 2^23
    const size_t dst = blk * 3 * per_block + (size_t)c * Nt * 16 + (size_t)(n >> 3) * 128 + (n & 7) * 16 + e;
    wpk[dst] = (uint8_t)(qv & 255u);
    wpk[dst + per_block] = (uint8_t)((qv >> 8) & 255u);
    wpk[dst + 2 * per_block] = (uint8_t)(qv >> 16);
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <int EPI, bool PSTAR, int TP>
void launch(const TcArgs& a, unsigned grid, size_t smem, cudaStream_t s) {
    static bool done = false;
    if (!done) {
        cudaFuncSetAttribute(conv_tc_kernel<EPI, PSTAR, TP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        done = true;
    }
    conv_tc_kernel<EPI, PSTAR, TP><<<grid, kThreads, smem, s>>>(a);
}

template <int TP>
void launch_tp(const TcArgs& a, spk_epilogue epi, bool pstar, unsigned grid, size_t smem, cudaStream_t s) {
    if (epi == SPK_EPI_POTENTIAL) launch<SPK_EPI_POTENTIAL, false, TP>(a, grid, smem, s);
    else if (pstar) launch<SPK_EPI_FIRE, true, TP>(a, grid, smem, s);
    else launch<SPK_EPI_FIRE, false, TP>(a, grid, smem, s);
}

}  // namespace

bool tc_plan(const spk_conv_geom& g, TcPlan& p) {
    p.Ho = (g.Hi + 2 * g.Ph - g.Kh) / g.Sh + 1;
    p.Wo = (g.Wi + 2 * g.Pw - g.Kw) / g.Sw + 1;
    p.K = g.Ci * g.Kh * g.Kw;
    if (g.T > 32 || p.K > kTcMaxK || g.Kh > 16 || g.Kw > 16) return false;
    p.KS = KS;
    p.nks = (p.K + KS - 1) / KS;
    p.TP = g.T <= 16 ? 16 : 32;
    p.PPT = 128 / p.TP;
    int nn = 1;
    while (true) {
        const int per = (g.Co + nn - 1) / nn;
        const int Nt = ((per + 15) / 16) * 16;
        if (3 * Nt <= 480) {
            p.Nt = Nt;
            break;
        }
        ++nn;
    }
    p.n_ntiles = (g.Co + p.Nt - 1) / p.Nt;
    p.NB = (6 * p.Nt <= 512) ? 2 : 1;
    const int HWo = p.Ho * p.Wo;
    p.tps = (HWo + p.PPT - 1) / p.PPT;
    // input rows one tile needs: (rows its pixels span) * Sh + Kh - Sh, at most Hi
    int span = 0;
    for (int j = 0; j < p.tps; ++j) {
        const int y0 = (j * p.PPT) / p.Wo, y1 = (std::min(j * p.PPT + p.PPT, HWo) - 1) / p.Wo;
        span = std::max(span, (y1 - y0) * g.Sh + g.Kh);
    }
    p.NR = std::min(g.Hi, span);
    p.band = p.NR * g.Wi;
    p.NP = (long long)g.B * HWo;
    p.n_mtiles = (long long)g.B * p.tps;
    p.total_tiles = p.n_mtiles * p.n_ntiles;
    p.packed_bytes = (size_t)p.n_ntiles * p.nks * 3 * p.Nt * KS;
    p.ws_bytes = 256 + p.packed_bytes;
    const size_t a = (size_t)S * 128 * KS, b = (size_t)S * 3 * p.Nt * KS, lc = 8 * 256,
                 kt = 4 * (size_t)p.nks * KS;
    const size_t region = ((size_t)g.Ci * p.band + 15) & ~(size_t)15;
    const size_t fixed = a + b + lc + kt + 512;
    const size_t cap = 227 * 1024;
    if (fixed + region > cap || (size_t)g.Ci * p.band >= (1u << 24)) return false;
    p.nrb = (fixed + 2 * region <= cap) ? 2 : 1;
    p.rb_stride = region;
    p.smem_bytes = fixed + p.nrb * region;
    return true;
}

spk_status spk_conv_tc(const uint8_t* lat_in, const float* w, const spk_conv_geom& g, const TcPlan& p,
                       spk_epilogue epi, float theta, float w_max, void* out0, void* out1, void* ws,
                       cudaStream_t s) {
    // scale s = smallest power of two >= w_max; digits of w * 2^23 / s
    int ex = 0;
    std::frexp((double)w_max, &ex);  // w_max = f * 2^ex, f in [0.5, 1)
    double scale = std::ldexp(1.0, ex);
    if (std::ldexp(1.0, ex - 1) >= (double)w_max) scale = std::ldexp(1.0, ex - 1);
    const float inv_scale23 = (float)(8388608.0 / scale);
    const float out_scale = (float)(scale / 8388608.0);

    int* flag = static_cast<int*>(ws);
    uint8_t* wpk = static_cast<uint8_t*>(ws) + 256;
    if (cudaMemsetAsync(flag, 0, sizeof(int), s) != cudaSuccess) return spk::launched("memset(flag)");
    const size_t nthreads = (size_t)p.n_ntiles * p.nks * p.Nt * KS;
    pack_weights_kernel<<<spk::ceil_div(nthreads, 256), 256, 0, s>>>(w, g.Co, p.K, p.Nt, p.n_ntiles, p.nks,
                                                                    inv_scale23, wpk, flag);
    spk_status st = spk::launched("pack_weights_kernel");
    if (st != SPK_OK) return st;

    TcArgs a{};
    a.lat_in = lat_in;
    a.wpk = wpk;
    a.out0 = out0;
    a.out1 = static_cast<float*>(out1);
    a.g = g;
    a.Ho = p.Ho;
    a.Wo = p.Wo;
    a.HWo = p.Ho * p.Wo;
    a.K = p.K;
    a.nks = p.nks;
    a.TP = p.TP;
    a.logTP = p.TP == 16 ? 4 : 5;
    a.PPT = p.PPT;
    a.Nt = p.Nt;
    a.n_ntiles = p.n_ntiles;
    a.NB = p.NB;
    a.tps = p.tps;
    a.NR = p.NR;
    a.band = p.band;
    a.nrb = p.nrb;
    a.rb_stride = (int)p.rb_stride;
    a.total_tiles = p.total_tiles;
    // fire iff X * s 2^-23 > theta  <=>  X > floor(theta 2^23 / s)   (X integer, scaling exact)
    a.theta_q = (long long)std::floor((double)theta * (8388608.0 / scale));
    a.out_scale = out_scale;
    static const int prof_env = [] {
        const char* e = std::getenv("SPK_CONV_PROF");
        return e && e[0] == '1' ? 1 : 0;
    }();
    a.prof = prof_env;
    a.a_off = 0;
    a.b_off = (uint32_t)(S * 128 * KS);
    a.lc_off = a.b_off + (uint32_t)(S * 3 * p.Nt * KS);
    a.kt_off = a.lc_off + 8u * 256u;  // per-producer-warp latcol buffers
    a.rg_off = (a.kt_off + (uint32_t)(4 * p.nks * KS) + 15u) & ~15u;
    a.bar_off = (a.rg_off + (uint32_t)(p.nrb * p.rb_stride) + 15u) & ~15u;
    const long long grid = p.total_tiles < sm_count() ? p.total_tiles : sm_count();
    if (p.TP == 16) launch_tp<16>(a, epi, out1 != nullptr, (unsigned)grid, p.smem_bytes, s);
    else launch_tp<32>(a, epi, out1 != nullptr, (unsigned)grid, p.smem_bytes, s);
    return spk::launched("conv_tc_kernel");
}

// Debug: copy the per-role cycle counters of the last profiled conv (SPK_CONV_PROF=1)
// into host memory [1024][5][2] (u64).  Not part of the public ABI.
extern "C" __attribute__((visibility("default"))) int spk_debug_conv_prof(void* host) {
    return (int)cudaMemcpyFromSymbol(host, g_conv_prof, sizeof(g_conv_prof));
}
