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
//   cols  N = output map o (tile Nt <= 128); the 3 digit planes are stacked
//                           along N (one MMA of N = 3 Nt) when 3 Nt <= 256
//   depth K = synapse (c, i, j), in the kernel's [Co][Ci][Kh][Kw] order.
//   A[(p,t), k] = [lat_in(p, k) <= t]   — the cumulative spike train, built on
//                 the fly from the u8 latency map (never materialised in HBM)
//                 and written straight into TENSOR MEMORY (u8 {0,1}); the MMA
//                 reads A from TMEM, so shared-memory bandwidth is spent on B only;
//   B[k, o]     = weight digit planes: w = s * sum_d q_d 2^(8d-23), q_d in u8
//                 (23-bit fixed point, s = power of two >= w_max), in shared
//                 memory — resident for the whole kernel when it fits, else
//                 streamed per K stage by cp.async.bulk;
//   D_d = A x B_d with tcgen05.mma kind::i8 (s32 accumulators in TMEM, exact);
//   X = D_2 2^16 + D_1 2^8 + D_0 is the exact integer potential in units of
//   s 2^-30 (A carries the spike as 128 = 2^7); fire iff X > floor(theta 2^30 / s);
//   P = X s 2^-30 rounded once.
//
// Persistent, warp-specialised CTA (one per SM), 20 warps (5 per scheduler: 96 registers each):
//   warps 0-7   producers: im2col gather of latencies from the staged input
//               band, expand to A rows, tcgen05.st into the TMEM A stage
//               (warp w writes lane quadrant w%4, K half w/4); A = 128 [lat <= t]
//   warps 8-15  epilogue (2 per TMEM lane quadrant): tcgen05.ld -> integer
//               threshold test, warp ballot,
//               first-crossing time (popcount: potentials are monotone in t),
//               potential at the crossing, staged in smem and written as one
//               run of 128/TP pixels per output map
//   warp  16    MMA issuer (one thread), TMEM allocator
//   warp  17    B loader: cp.async.bulk of pre-packed digit planes
//   warp  18    band loader: copies the input rows a tile needs into smem
//   warp  19    flusher: writes each staged output tile, one run per output map
// Pipelines (mbarriers): input band (1-2 buffers), K stages (8; A in TMEM,
// B in smem), TMEM accumulators (1-2 buffers).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "conv.cuh"

#ifndef SPK_MMA_FAST
#define SPK_MMA_FAST 1  // retained-A N tiles after the first issue all K stages after one wait (C2 conv1 1.08 -> 1.01 ms)
#endif
#ifndef SPK_EXP
#define SPK_EXP 0  // timing experiments only: 1 no wait::st, 2 no gather, 4 no tcgen05.st, 8 no epilogue stores,
                   // 16 no epilogue tcgen05.ld, 32 no MMA, 512 no fire-epilogue TMEM loads,
                   // 1024 fire epilogue without threshold work
#endif

namespace {

constexpr int KS = kTcKS;          // synapses per stage (4 MMAs of K=32)
static_assert(KS == 128, "an A slot holds 4 k-steps of 32 synapses");
constexpr int S = kTcStages;       // pipeline depth
constexpr int kProdWarps = 8;      // warps 0-7: producers
#ifndef SPK_EPI_WARPS
#define SPK_EPI_WARPS 8
#endif
constexpr int kEpiWarps = SPK_EPI_WARPS;  // warps 8..: epilogue (kEpiWarps / 4 per TMEM lane quadrant)
constexpr int kEpiStride = 16 * (kEpiWarps / 4);  // column stride of one epilogue warp's 16-column chunks
constexpr int kMmaWarp = kProdWarps + kEpiWarps;  // warp 16: MMA issuer; 17: B loader; 18: band loader
constexpr int kLoaders = 32;  // one band-loader warp: 20 warps keep 96 registers per thread
constexpr int kFlushWarp = kMmaWarp + 3;           // warp 19: writes staged output tiles to HBM
constexpr int kThreads = (kFlushWarp + 1) * 32;   // 640
constexpr int kNOB = 4;                            // output staging ring (tiles)
constexpr int kLoadBatch = 8;      // independent loads in flight per band-loader thread
constexpr int kACols = KS / 4;     // TMEM columns of one A stage (4 u8 per 32-bit column)
constexpr int kMaxA = 8;           // TMEM A ring slots (<= 8; the rest of the 512 columns hold accumulators)

// Optional per-role cycle accounting (SPK_CONV_PROF=1): [block][role][total, wait]
constexpr int kProfRoles = 25;  // producer, epilogue, mma, b-loader, band-loader, mma:fence/issue/commit, producer sections x9, epilogue sections x6
__device__ unsigned long long g_conv_prof[1024][kProfRoles][2];
#ifdef SPK_CONV_TRACE
// event timestamps of CTA 0's first kTrace tiles (debug aid)
constexpr int kTrace = 256;
__device__ long long g_trace[12][kTrace];
#define TRACE(ev, it)                                                        \
    do {                                                                     \
        if (blockIdx.x == 0 && (it) < kTrace) g_trace[ev][(it)] = clock64(); \
    } while (0)
#else
#define TRACE(ev, it) \
    do {              \
    } while (0)
#endif

struct TcArgs {
    const uint8_t* lat_in;
    const uint8_t* wpk;  // packed digit planes
    const int* wflag;    // pack flags: bit 0 clamp, bit 1 + d = digit plane d has a non-zero digit
    void* out0;
    float* out1;
    spk_conv_geom g;
    int Ho, Wo, HWo, K, nks, Nt, n_ntiles, NB, tps, NR, band, nrb, rb_stride, bres, stack, NS;
    int retain;  // the A stages of an M tile stay in TMEM for all its N tiles (nks <= NA)
    int NA, aCol0;  // TMEM A ring: NA slots of kACols columns from column aCol0 = 512 - NA * kACols
    int G;          // K slots per hand-off (1 or 2): one mbarrier round trip per G * KS synapses
    int kt16;       // synapse offsets fit 16 bits: the table is u16 (half the smem)
    int GB;         // K slots per streamed B hand-off (a multiple of G; = nks: one B copy per tile)
    int WiP, HiP;  // padded input width/height: the staged region includes the zero-padding halo
    long long total_tiles;
    long long theta_q;  // fire iff X > theta_q
    // small reductions (digit sums < 2^24): fire iff d2 + ((d1*256 + d0 + thC) >> 16) > thH,
    // the same test in 32-bit arithmetic (thH = theta_q >> 16, thC = 65535 - (theta_q & 65535))
    int small_x, thH;
    uint32_t thC;
    float out_scale;
    uint32_t b_off, lc_off, kt_off, rg_off, ob_off, bar_off;  // smem carve-up
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
#ifndef SPK_WAIT_TEST
#define SPK_WAIT_TEST 0  // 1: poll with mbarrier.test_wait (never suspends) instead of try_wait
#endif
__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t parity) {
    uint32_t ok;
    if (SPK_WAIT_TEST)
        asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(a), "r"(parity)
                     : "memory");
    else
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(a), "r"(parity)
                     : "memory");
    return ok != 0;
}
#ifndef SPK_WAIT_HINT
#define SPK_WAIT_HINT 20000  // > 0: blocking waits suspend in try_wait for up to this many ns per probe
#endif
#ifndef SPK_WAIT_HINT_ALL
#define SPK_WAIT_HINT_ALL 1  // 1: also the MMA issuer's and the slack roles' waits
#endif
// try_wait with a suspend-time hint: the thread sleeps in the barrier unit until the phase
// completes (or the hint elapses) instead of re-issuing probes
__device__ __forceinline__ bool mbar_try_hint(uint32_t a, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity), "n"(SPK_WAIT_HINT > 0 ? SPK_WAIT_HINT : 1)
        : "memory");
    return ok != 0;
}
// critical-path waits (producers, MMA issuer) poll
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    if (SPK_WAIT_HINT > 0) {
        while (!mbar_try_hint(a, parity)) {
        }
        return;
    }
    while (!mbar_try(a, parity)) {
    }
}
#ifndef SPK_IDLE_NS
#define SPK_IDLE_NS 256
#endif
// Wait on up to three barriers with their first probes in flight together (an mbarrier
// probe costs ~120 cycles of latency even when the phase is already complete).
__device__ __forceinline__ void mbar_wait3(uint32_t a0, uint32_t p0, bool w0, uint32_t a1, uint32_t p1, bool w1,
                                           uint32_t a2 = 0, uint32_t p2 = 0, bool w2 = false) {
    bool d0 = !w0 || mbar_try(a0, p0);
    bool d1 = !w1 || mbar_try(a1, p1);
    bool d2 = !w2 || mbar_try(a2, p2);
    if (SPK_WAIT_HINT_ALL && SPK_WAIT_HINT > 0) {
        while (!d0) d0 = mbar_try_hint(a0, p0);
        while (!d1) d1 = mbar_try_hint(a1, p1);
        while (!d2) d2 = mbar_try_hint(a2, p2);
        return;
    }
    while (!d0) d0 = mbar_try(a0, p0);
    while (!d1) d1 = mbar_try(a1, p1);
    while (!d2) d2 = mbar_try(a2, p2);
}
// A warp group waiting for one event: a single leader thread polls, the others
// sleep in a named hardware barrier (no issue slots spent on polling).
template <int ID, int NTHREADS>
__device__ __forceinline__ void group_wait(uint32_t a, uint32_t parity, bool leader) {
    if (leader) mbar_wait(a, parity);
    asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(NTHREADS) : "memory");
}
// named barrier ids (0 is __syncthreads)
constexpr int kBarProd = 1, kBarEpi = 2, kBarBand = 3;
// waits of roles with slack (epilogue, loaders, flusher) back off between polls so that
// their spinning does not take issue slots from the producers on the same scheduler
__device__ __forceinline__ void mbar_wait_idle(uint32_t a, uint32_t parity) {
    if (SPK_WAIT_HINT_ALL && SPK_WAIT_HINT > 0) {
        while (!mbar_try_hint(a, parity)) {
        }
        return;
    }
    while (!mbar_try(a, parity)) {
        if (SPK_IDLE_NS > 0) __nanosleep(SPK_IDLE_NS);
    }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// the same from a converged warp: one elected lane commits
__device__ __forceinline__ void tc_commit_elect(uint32_t bar) {
    asm volatile(
        "{ .reg .pred e; elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }" ::"r"(bar)
        : "memory");
}

// One K stage of MMAs (NK <= KS/32 = 4 k-steps) from a single asm block: digit
// planes separate (3 accumulators, 3 NK MMAs) or stacked along N (one accumulator
// span, NK MMAs).  bdesc: B descriptor of k-step 0 / digit 0; inck: descriptor
// increment per k-step; incd: per digit plane; acc0: accumulate on the first k-step.
// one k-step of the three digit planes (separate accumulators d0, d1, d2)
// Issued by the whole (converged) MMA warp with warp-uniform operands, one elected
// lane executing the MMAs: the operands then live in uniform registers and each
// tcgen05.mma is a single UTCIMMA (no per-thread operand broadcast loop).
__device__ __forceinline__ void tc_kstep3(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t a, uint64_t x0,
                                          uint64_t incd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p, e;\n.reg .b64 x1, x2;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 p, %7, 0;\n add.s64 x1, %4, %5;\n add.s64 x2, x1, %5;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%3], %4, %6, p;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%1], [%3], x1, %6, p;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%2], [%3], x2, %6, p;\n}\n" ::"r"(d0),
        "r"(d1), "r"(d2), "r"(a), "l"(x0), "l"(incd), "r"(idesc), "r"(acc)
        : "memory");
}
template <int NK>
__device__ __forceinline__ void tc_stage_sep(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t a0, uint64_t bdesc,
                                             uint64_t inck, uint64_t incd, uint32_t idesc, uint32_t acc0) {
    static_assert(NK >= 1 && NK <= 8, "k-steps per hand-off");
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) tc_kstep3(d0, d1, d2, a0 + 8u * kk, bdesc + inck * kk, incd, idesc, kk ? 1u : acc0);
}
// One k-step of the live digit planes as one or two MMAs: MMA A covers planes [pA, pA + nA)
// (accumulators dA, B descriptor bA, N = nA Nt in idA), MMA B (only when `two`) likewise.
// Digit planes that are all zero for every weight of the layer are never issued (exact: they
// would add zero) — C5's fp16-representable weights have no digit 0, binary quantized weights
// (Listing 4) only digit 2.
__device__ __forceinline__ void tc_kstep_gen(uint32_t dA, uint32_t dB, uint32_t a, uint64_t bA, uint64_t bB,
                                             uint32_t idA, uint32_t idB, uint32_t acc, uint32_t two) {
    asm volatile(
        "{\n.reg .pred p, e, q, eq;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 p, %7, 0;\n setp.ne.b32 q, %8, 0;\n and.pred eq, e, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%2], %3, %5, p;\n"
        "@eq tcgen05.mma.cta_group::1.kind::i8 [%1], [%2], %4, %6, p;\n}\n" ::"r"(dA),
        "r"(dB), "r"(a), "l"(bA), "l"(bB), "r"(idA), "r"(idB), "r"(acc), "r"(two)
        : "memory");
}
template <int NK>
__device__ __forceinline__ void tc_stage_gen(uint32_t dA, uint32_t dB, uint32_t a0, uint64_t bA, uint64_t bB,
                                             uint64_t inck, uint32_t idA, uint32_t idB, uint32_t acc0, uint32_t two) {
#pragma unroll
    for (int kk = 0; kk < NK; ++kk)
        tc_kstep_gen(dA, dB, a0 + 8u * kk, bA + inck * kk, bB + inck * kk, idA, idB, kk ? 1u : acc0, two);
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
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// bytes of a: 0x80 where a <= t, else 0, for byte values a, t < 128 (the staged
// region clamps latencies to <= 0x7F): no cross-byte borrow since 0x80|t > a.
__device__ __forceinline__ uint32_t le_bytes80(uint32_t a, uint32_t tt /* t * 0x01010101 | 0x80808080 */) {
    return (tt - a) & 0x80808080u;
}

// Tile bookkeeping without divisions in the loops: a CTA owns the contiguous
// tile range [t0, t1); tile = (b * tps + j) * n_ntiles + nt.
struct TileIter {
    int tile, t1, nt, j, b;
    __device__ __forceinline__ void init(const TcArgs& a) {
        if (a.retain) {  // whole M tiles per CTA: A is produced once for all N tiles
            const long long nm = a.total_tiles / a.n_ntiles;
            tile = (int)((long long)blockIdx.x * nm / gridDim.x) * a.n_ntiles;
            t1 = (int)((long long)(blockIdx.x + 1) * nm / gridDim.x) * a.n_ntiles;
        } else {
            tile = (int)((long long)blockIdx.x * a.total_tiles / gridDim.x);
            t1 = (int)((long long)(blockIdx.x + 1) * a.total_tiles / gridDim.x);
        }
        const int mt = tile / a.n_ntiles;
        nt = tile - mt * a.n_ntiles;
        b = mt / a.tps;
        j = mt - b * a.tps;
    }
    __device__ __forceinline__ bool valid() const { return tile < t1; }
    __device__ __forceinline__ void next(const TcArgs& a) {
        ++tile;
        if (++nt == a.n_ntiles) {
            nt = 0;
            if (++j == a.tps) {
                j = 0;
                ++b;
            }
        }
    }
    // the next tile stages a different input region (or there is no next tile)
    // (band mode: the next M tile of the sample keeps the band when its first row is the same)
    template <int PPT>
    __device__ __forceinline__ bool next_m_same_region(const TcArgs& a) const {
        if (j + 1 == a.tps) return false;  // next sample
        if (a.NR == a.HiP) return true;
        const int lo0 = ((j * PPT) / a.Wo) * a.g.Sh, lo1 = (((j + 1) * PPT) / a.Wo) * a.g.Sh;
        return max(0, min(lo0, a.HiP - a.NR)) == max(0, min(lo1, a.HiP - a.NR));
    }
    template <int PPT>
    __device__ __forceinline__ bool region_ends(const TcArgs& a) const {
        if (tile + 1 >= t1) return true;
        if (nt + 1 < a.n_ntiles) return false;
        return !next_m_same_region<PPT>(a);
    }
    // same, asked at the first N tile of an M tile about the whole M tile (retained A)
    template <int PPT>
    __device__ __forceinline__ bool region_ends_m(const TcArgs& a) const {
        if (tile + (a.n_ntiles - nt) >= t1) return true;
        return !next_m_same_region<PPT>(a);
    }
    // first staged row of this tile, in padded-image rows (input row + Ph)
    template <int PPT>
    __device__ __forceinline__ int r0(const TcArgs& a) const {
        const int lo = ((j * PPT) / a.Wo) * a.g.Sh;  // first padded row the tile's receptive fields touch
        return max(0, min(lo, a.HiP - a.NR));
    }
};

#ifdef SPK_CONV_PROF_BUILD
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
    __device__ __forceinline__ void wait_idle(uint32_t bar, uint32_t parity) {
        const long long w0 = on ? clock64() : 0;
        mbar_wait_idle(bar, parity);
        if (on) wait += clock64() - w0;
    }
    // one lane polls, the warp then proceeds together
    __device__ __forceinline__ void wait_warp(uint32_t bar, uint32_t parity) {
        if ((threadIdx.x & 31) == 0) wait_on(bar, parity);
        __syncwarp();
    }
    __device__ __forceinline__ void wait_warp_idle(uint32_t bar, uint32_t parity) {
        if ((threadIdx.x & 31) == 0) wait_idle(bar, parity);
        __syncwarp();
    }
    __device__ __forceinline__ void wait3(uint32_t a0, uint32_t p0, bool w0_, uint32_t a1, uint32_t p1, bool w1,
                                          uint32_t a2 = 0, uint32_t p2 = 0, bool w2 = false) {
        const long long w0 = on ? clock64() : 0;
        mbar_wait3(a0, p0, w0_, a1, p1, w1, a2, p2, w2);
        if (on) wait += clock64() - w0;
    }
    template <int ID, int N>
    __device__ __forceinline__ void group_wait(uint32_t bar, uint32_t parity, bool leader) {
        const long long w0 = on ? clock64() : 0;
        if (leader) mbar_wait(bar, parity);
        asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory");
        if (on) wait += clock64() - w0;
    }
    __device__ void store(int role) {
        if (on && blockIdx.x < 1024) {
            g_conv_prof[blockIdx.x][role][0] = (unsigned long long)(clock64() - t0);
            g_conv_prof[blockIdx.x][role][1] = (unsigned long long)wait;
        }
    }
};
#else
// production build: no clock reads at all (the instrumented build is a debug aid)
struct RoleClock {
    static constexpr bool on = false;
    __device__ RoleClock(bool) {}
    __device__ __forceinline__ void wait_on(uint32_t bar, uint32_t parity) { mbar_wait(bar, parity); }
    __device__ __forceinline__ void wait_idle(uint32_t bar, uint32_t parity) { mbar_wait_idle(bar, parity); }
    __device__ __forceinline__ void wait_warp(uint32_t bar, uint32_t parity) {
        if ((threadIdx.x & 31) == 0) mbar_wait(bar, parity);
        __syncwarp();
    }
    __device__ __forceinline__ void wait_warp_idle(uint32_t bar, uint32_t parity) {
        if ((threadIdx.x & 31) == 0) mbar_wait_idle(bar, parity);
        __syncwarp();
    }
    __device__ __forceinline__ void wait3(uint32_t a0, uint32_t p0, bool w0, uint32_t a1, uint32_t p1, bool w1,
                                          uint32_t a2 = 0, uint32_t p2 = 0, bool w2 = false) {
        mbar_wait3(a0, p0, w0, a1, p1, w1, a2, p2, w2);
    }
    template <int ID, int N>
    __device__ __forceinline__ void group_wait(uint32_t bar, uint32_t parity, bool leader) {
        if (leader) mbar_wait(bar, parity);
        asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory");
    }
    __device__ void store(int) {}
};
#endif

// MMAs of one k-step over the layer's live digit planes (pack flag bits 1..3): MMA A covers
// planes [pA, pA + nA), MMA B (nB = 1) plane pB.  Stacked layouts (3 Nt <= 256) take the live
// span in one MMA; otherwise (N <= 256 per MMA) planes 0-1 and plane 2 are separate MMAs.
// Planes outside the MMAs are never written: the epilogue reads them as zero (live_cols).
__device__ __forceinline__ void plane_plan(const TcArgs& a, uint32_t& pA, uint32_t& nA, uint32_t& pB, uint32_t& nB) {
    uint32_t pm = a.wflag ? ((uint32_t)__ldcg(a.wflag) >> 1) & 7u : 7u;
    if (pm == 0) pm = 4u;  // all-zero weights: one plane of zeros
    const uint32_t lo = __ffs(pm) - 1, hi = 31 - __clz(pm);
    pB = 0;
    nB = 0;
    if (a.stack == 1 || lo >= 1) {
        pA = lo;
        nA = hi - lo + 1;
    } else {  // plane 0 live, 3 Nt > 256: planes 0-1 (N = 2 Nt) [+ plane 2 (N = Nt)]
        pA = 0;
        nA = hi >= 1 ? 2 : 1;
        if (hi == 2) pB = 2, nB = 1;
    }
}
__device__ __forceinline__ uint32_t live_planes(const TcArgs& a) {
    if (a.stack == 0) return 7u;
    uint32_t pA, nA, pB, nB;
    plane_plan(a, pA, nA, pB, nB);
    return (((1u << nA) - 1u) << pA) | (nB ? 1u << pB : 0u);
}

// ------------------------------------------------------------------ the kernel
template <int EPI, bool PSTAR, int TP>
// 20 warps: 5 per scheduler, whose 16K-register file then allows 96 registers per thread
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(const TcArgs a) {
    constexpr int LOGTP = TP == 1 ? 0 : TP == 16 ? 4 : 5;
    constexpr int PPT = 128 / TP;  // pixels per M tile (TP = 1: one time step, rows = 128 pixels)
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* Bs = smem + a.b_off;
    uint8_t* LC = smem + a.lc_off;  // per-producer-warp latcol: [8 warps][2 bufs][2 pixels][KS/2]
    const uint32_t* ktab = reinterpret_cast<const uint32_t*>(smem + a.kt_off);
    uint8_t* RG = smem + a.rg_off;  // staged input band(s): [nrb][Ci][NR][Wi]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.bar_off);
    // barrier map: full[kMaxA] empty[kMaxA] (A ring in TMEM) accf[4] acce[4] rgf[2] rge[2] bres stg[4]
    // fls[4] bfull[S] bempty[S] (streamed B stages in smem), then the TMEM address
    constexpr int A2 = 2 * kMaxA;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + A2 + 21 + 2 * S);
    const uint32_t bfull0 = smem_u32(bars + A2 + 21), bempty0 = smem_u32(bars + A2 + 21 + S);
    const uint32_t stg0 = smem_u32(bars + A2 + 13), fls0 = smem_u32(bars + A2 + 17);
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kMaxA);
    const uint32_t accf0 = smem_u32(bars + A2), acce0 = smem_u32(bars + A2 + 4);
    const uint32_t rgf0 = smem_u32(bars + A2 + 8), rge0 = smem_u32(bars + A2 + 10);
    const uint32_t bresb = smem_u32(bars + A2 + 12);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const spk_conv_geom& g = a.g;

    {  // synapse table: offset c*NR*WiP + i*WiP + j into the halo'd staged region;
       // padding synapses k >= K point at the "never" sentinel block after the region
        uint32_t* kt = reinterpret_cast<uint32_t*>(smem + a.kt_off);
        uint16_t* kt16 = reinterpret_cast<uint16_t*>(smem + a.kt_off);
        const int KhKw = g.Kh * g.Kw;
        for (int k = threadIdx.x; k < a.nks * KS; k += kThreads) {
            uint32_t e = (uint32_t)(g.Ci * a.band);  // sentinel (reads 0x7F there)
            if (k < a.K) {
                const int c = k / KhKw, r = k - c * KhKw, i = r / g.Kw, j = r - i * g.Kw;
                e = (uint32_t)(c * a.band + i * a.WiP + j);
            }
            if (a.kt16) kt16[k] = (uint16_t)e;
            else kt[k] = e;
        }
    }
    if (a.NR == a.HiP) {  // whole padded samples: the halo never changes, fill it (and all) once
        uint32_t* r4 = reinterpret_cast<uint32_t*>(RG);
        for (int q = threadIdx.x; q < a.nrb * a.rb_stride / 4; q += kThreads) r4[q] = 0x7F7F7F7Fu;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMaxA; ++s) {
            mbar_init(full0 + 8 * s, kProdWarps);  // producer warps
            mbar_init(empty0 + 8 * s, 1);          // tcgen05.commit
        }
        for (int s = 0; s < S; ++s) {
            mbar_init(bfull0 + 8 * s, 1);          // B loader arrive.expect_tx
            mbar_init(bempty0 + 8 * s, 1);         // tcgen05.commit
        }
        for (int b = 0; b < 4; ++b) {
            mbar_init(accf0 + 8 * b, 1);              // tcgen05.commit
            mbar_init(acce0 + 8 * b, kEpiWarps);      // epilogue warps
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(rgf0 + 8 * b, kLoaders / 32);   // band loader warps
            mbar_init(rge0 + 8 * b, kProdWarps);      // producer warps
        }
        mbar_init(bresb, a.nks);  // resident B: one arrive.expect_tx per K stage
        for (int b = 0; b < kNOB; ++b) {
            mbar_init(stg0 + 8 * b, kEpiWarps);  // output tile staged by every epilogue warp
            mbar_init(fls0 + 8 * b, 1);          // staged tile written out by the flusher
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // the setup above (synapse table, barriers, TMEM allocation) reads only kernel parameters and
    // shared memory, so under programmatic dependent launch it overlaps the previous kernel's tail;
    // every role reads the previous kernels' outputs only after this wait
    spk_pdl_wait();
#ifndef SPK_TMEM0
#define SPK_TMEM0 1
#endif
#if SPK_TMEM0
    // the kernel owns all 512 TMEM columns of its SM, so the allocation starts at 0: a
    // compile-time base keeps every TMEM operand warp-uniform (checked once)
    constexpr uint32_t tmem = 0;
    if (threadIdx.x == 0 && *tmem_holder != 0u) __trap();
#else
    const uint32_t tmem = *tmem_holder;
#endif

    if (warp < kProdWarps && (SPK_EXP & 32768)) {  // timing experiment: no producers (MMA skips A waits)
    } else if (TP == 1 && warp < kProdWarps) {
        // ======================= producers, one time step (TP = 1) =======================
        // T = 1 (e.g. rate-coded trains as one-step latency maps, B' = B T): row r of an M tile is
        // pixel j*128 + r, A[r][k] = 0x80 [in(r, k) == 0]; each lane gathers its own pixel's
        // receptive field (64 synapses of its K half per stage) — the synapse-table entries are
        // the same for every lane (broadcast reads), the staged-band bytes are neighbouring pixels'.
        RoleClock rc(a.prof != 0);
        const int quad = warp & 3, half = warp >> 2;
        constexpr int HK = KS / 2;
        const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(a.aCol0 + half * (HK / 4));
        TileIter ti;
        ti.init(a);
        int rb = 0, rbn = 0, sA = 0;
        uint32_t phA = 0, rgph = 0;
        bool need_region = true;
        long long pq[4] = {0, 0, 0, 0};  // SPK_CONV_PROF_BUILD: region wait, gather, slot wait, store+hand-off
        for (; ti.valid(); ti.next(a)) {
            if (a.retain && ti.nt != 0) continue;
            const long long q0 = rc.on ? clock64() : 0;
            if (need_region) {
                rb = rbn;
                rc.template group_wait<kBarProd, kProdWarps * 32>(rgf0 + 8 * rb, rgph, threadIdx.x == 0);
                if (++rbn == a.nrb) rbn = 0, rgph ^= 1u;
            }
            if (rc.on) pq[0] += clock64() - q0;
            const bool last_use = a.retain ? ti.template region_ends_m<PPT>(a) : ti.template region_ends<PPT>(a);
            need_region = last_use;
            const uint8_t* region = RG + rb * a.rb_stride;
            const int p = ti.j * PPT + quad * 32 + lane;
            const bool pvalid = p < a.HWo;
            int pixbase = 0;
            if (pvalid) {
                const int yo = p / a.Wo, xo = p - yo * a.Wo;
                pixbase = (yo * g.Sh - ti.r0<PPT>(a)) * a.WiP + xo * g.Sw;
            }
            for (int ks = 0; ks < a.nks; ++ks) {
                const int kin = a.G == 1 ? 0 : (ks & 1);
                const bool gfirst = kin == 0, glast = kin == a.G - 1 || ks + 1 == a.nks;
                const int s = sA * a.G + kin;
                const uint32_t ph = phA;
                const uint32_t gbar = 8u * (uint32_t)sA;
                if (glast && ++sA == a.NA / a.G) sA = 0, phA ^= 1u;
                uint32_t r[16];
                const long long q1 = rc.on ? clock64() : 0;
                const int kb = ks * KS + half * HK;
                // the stage's 64 table entries first (broadcast reads, all in flight), then the
                // band bytes: one dependent load deep instead of one per 8 synapses
                uint32_t tw[32];  // kt16: 2 entries per word; else 1 entry per word (first 32 synapses)
                if (a.kt16) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const uint4 v = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(ktab) + kb + 8 * q);
                        tw[4 * q] = v.x, tw[4 * q + 1] = v.y, tw[4 * q + 2] = v.z, tw[4 * q + 3] = v.w;
                    }
                }
#pragma unroll
                for (int q8 = 0; q8 < HK / 8; ++q8) {  // 8 synapses per step
                    uint32_t te[8];
                    if (a.kt16) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) te[2 * e] = tw[4 * q8 + e] & 0xFFFFu, te[2 * e + 1] = tw[4 * q8 + e] >> 16;
                    } else {
                        const uint4 v0 = *reinterpret_cast<const uint4*>(ktab + kb + 8 * q8);
                        const uint4 v1 = *reinterpret_cast<const uint4*>(ktab + kb + 8 * q8 + 4);
                        te[0] = v0.x, te[1] = v0.y, te[2] = v0.z, te[3] = v0.w;
                        te[4] = v1.x, te[5] = v1.y, te[6] = v1.z, te[7] = v1.w;
                    }
                    uint32_t w0 = 0x7F7F7F7Fu, w1 = 0x7F7F7F7Fu;  // never (invalid pixel)
                    if (pvalid) {
                        uint32_t bt[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) bt[e] = region[pixbase + (int)te[e]];
                        w0 = __byte_perm(__byte_perm(bt[0], bt[1], 0x0040), __byte_perm(bt[2], bt[3], 0x0040), 0x5410);
                        w1 = __byte_perm(__byte_perm(bt[4], bt[5], 0x0040), __byte_perm(bt[6], bt[7], 0x0040), 0x5410);
                    }
                    r[2 * q8] = le_bytes80(w0, 0x80808080u);  // 0x80 where the input spikes at the step
                    r[2 * q8 + 1] = le_bytes80(w1, 0x80808080u);
                }
                if (ks + 1 == a.nks && last_use) {  // staged band no longer read by this warp
                    __syncwarp();
                    if (lane == 0) mbar_arrive(rge0 + 8 * rb);
                }
                const long long q2 = rc.on ? clock64() : 0;
                if (gfirst) rc.template group_wait<kBarProd, kProdWarps * 32>(empty0 + gbar, ph ^ 1u, threadIdx.x == 0);
                const long long q3 = rc.on ? clock64() : 0;
                tc_fence_after();
                tmem_st16(trow + (uint32_t)(s * kACols), r);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0 && glast) mbar_arrive(full0 + gbar);
                if (rc.on) {
                    const long long q4 = clock64();
                    pq[1] += q2 - q1, pq[2] += q3 - q2, pq[3] += q4 - q3;
                }
            }
        }
        if (threadIdx.x == 0) {
            rc.store(0);
            if (rc.on && blockIdx.x < 1024)
                for (int q = 0; q < 4; ++q) g_conv_prof[blockIdx.x][8 + q][0] = pq[q];
        }
    } else if (TP != 1 && warp < kProdWarps) {
        // ======================= producers =======================
        RoleClock rc(a.prof != 0);
        const int quad = warp & 3, half = warp >> 2;
        const int row = quad * 32 + lane;            // A row this thread writes
        const int t = row & (TP - 1);
        const int pslot = (row >> LOGTP) - ((quad * 32) >> LOGTP);  // 0..PPT/4-1
        // A = 0x80 * [lat <= t]  (bit 7 of  (0x80|t) - (lat & 0x7f), masked by ~lat's bit 7)
        const uint32_t tt = 0x80808080u | ((uint32_t)t * 0x01010101u);
        // gather: this warp's pixels ((quad*32)>>LOGTP ..) x its KS/2 synapses of each stage
        constexpr int HK = KS / 2;                   // synapses per warp per stage (K half)
        constexpr int GPIX = 32 / TP;                // pixels per warp (2 or 1)
        constexpr int GB = HK * GPIX / 32;           // bytes gathered per lane (4 or 2)
        const int gslot = (GPIX == 2) ? (lane >> 4) : 0;
        const int gk = half * HK + ((GPIX == 2) ? (lane & 15) : lane) * GB;
        const int gpix_in_tile = ((quad * 32) >> LOGTP) + gslot;
        uint8_t* lcw = LC + warp * (4 * HK);         // [2 bufs][2 pixels][HK]
        const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(a.aCol0 + half * (HK / 4));
        long long pt[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        TileIter ti;
        ti.init(a);
        int sidx = 0, rb = 0, rbn = 0;
        int sA = 0;           // A ring slot of the next stage
        uint32_t phA = 0;     // and its phase
        uint32_t rgph = 0;
        bool need_region = true;
        long long tprev = rc.on ? clock64() : 0;
        for (; ti.valid(); ti.next(a)) {
            if (a.retain && ti.nt != 0) continue;  // A of this M tile is already in TMEM
            const long long tt0 = rc.on ? clock64() : 0;
            if (rc.on) pt[7] += tt0 - tprev;
            if (need_region) {
                rb = rbn;
                rc.template group_wait<kBarProd, kProdWarps * 32>(rgf0 + 8 * rb, rgph, threadIdx.x == 0);
                if (++rbn == a.nrb) rbn = 0, rgph ^= 1u;
            }
            const long long tt1 = rc.on ? clock64() : 0;
            if (rc.on) pt[8] += tt1 - tt0;
            const bool last_use = a.retain ? ti.template region_ends_m<PPT>(a) : ti.template region_ends<PPT>(a);
            need_region = last_use;
            const uint8_t* region = RG + rb * a.rb_stride;
            const int p = ti.j * PPT + gpix_in_tile;
            const bool pvalid = p < a.HWo;
            int pixbase = 0;  // region offset of this pixel's receptive-field origin (padded coords)
            if (pvalid) {
                const int yo = p / a.Wo, xo = p - yo * a.Wo;
                pixbase = (yo * g.Sh - ti.r0<PPT>(a)) * a.WiP + xo * g.Sw;
            }
            auto gather = [&](int ks) -> uint32_t {
#if (SPK_EXP & 2)
                return 0x01010101u * (uint32_t)ks;
#endif
                if (!pvalid) return 0x7F7F7F7Fu;
                uint32_t te[GB];
                if (a.kt16) {
                    const uint16_t* k16 = reinterpret_cast<const uint16_t*>(ktab) + ks * KS + gk;
                    if (GB == 4) {
                        const uint2 v = *reinterpret_cast<const uint2*>(k16);
                        te[0] = v.x & 0xFFFFu;
                        te[1] = v.x >> 16;
                        te[2] = v.y & 0xFFFFu;
                        te[3] = v.y >> 16;
                    } else {
                        const uint32_t v = *reinterpret_cast<const uint32_t*>(k16);
                        te[0] = v & 0xFFFFu;
                        te[1] = v >> 16;
                    }
                } else if (GB == 4) {
                    const uint4 t4 = *reinterpret_cast<const uint4*>(ktab + ks * KS + gk);
                    te[0] = t4.x;
                    te[1] = t4.y;
                    te[2] = t4.z;
                    te[3] = t4.w;
                } else {
                    const uint2 t2 = *reinterpret_cast<const uint2*>(ktab + ks * KS + gk);
                    te[0] = t2.x;
                    te[1] = t2.y;
                }
                uint32_t packed = 0;
#pragma unroll
                for (int e = 0; e < GB; ++e) packed |= (uint32_t)region[pixbase + (int)te[e]] << (8 * e);
                return packed;
            };
            uint32_t cur = gather(0);
            if (rc.on) pt[6] += clock64() - tt1;
            for (int ks = 0; ks < a.nks; ++ks, ++sidx) {
                long long q0 = rc.on ? clock64() : 0;
                // slot group sA (G consecutive slots, one hand-off) holds stages gi*G .. gi*G+G-1
                const int kin = a.G == 1 ? 0 : (ks & 1);
                const bool gfirst = kin == 0, glast = kin == a.G - 1 || ks + 1 == a.nks;
                const int s = sA * a.G + kin;  // TMEM slot
                const uint32_t ph = phA;
                const uint32_t gbar = 8u * (uint32_t)sA;
                if (glast && ++sA == a.NA / a.G) sA = 0, phA ^= 1u;
#if (SPK_EXP & 64)  // timing experiment: producers only hand stages over
                if (!(SPK_EXP & 16896) && gfirst)
                    rc.template group_wait<kBarProd, kProdWarps * 32>(empty0 + gbar, ph ^ 1u, threadIdx.x == 0);
                if (threadIdx.x == 0) TRACE(6, sidx);
                if (ks + 1 == a.nks && last_use) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(rge0 + 8 * rb);
                }
                __syncwarp();
                if (lane == 0 && !(SPK_EXP & 16384) && glast) mbar_arrive(full0 + gbar);
                continue;
#endif
                uint8_t* lc = lcw + (sidx & 1) * (2 * HK);
                if (GB == 4) *reinterpret_cast<uint32_t*>(lc + gslot * HK + (gk - half * HK)) = cur;
                else *reinterpret_cast<uint16_t*>(lc + gslot * HK + (gk - half * HK)) = (uint16_t)cur;
                __syncwarp();
                long long q1 = rc.on ? clock64() : 0;
                if (ks + 1 < a.nks) {
                    cur = gather(ks + 1);  // next stage's loads overlap this expansion
                } else if (last_use) {     // staged region no longer read by this warp
                    __syncwarp();
                    if (lane == 0) mbar_arrive(rge0 + 8 * rb);
                }
                long long q2 = rc.on ? clock64() : 0;
                // my row of this A stage: HK synapses of K half `half`
                uint32_t r[16];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const uint4 L = *reinterpret_cast<const uint4*>(lc + pslot * HK + q4 * 16);
                    r[4 * q4 + 0] = le_bytes80(L.x, tt);
                    r[4 * q4 + 1] = le_bytes80(L.y, tt);
                    r[4 * q4 + 2] = le_bytes80(L.z, tt);
                    r[4 * q4 + 3] = le_bytes80(L.w, tt);
                }
                long long q3 = rc.on ? clock64() : 0;
                // wait for the MMAs that last read this TMEM A stage, then overwrite it
                if (gfirst) rc.template group_wait<kBarProd, kProdWarps * 32>(empty0 + gbar, ph ^ 1u, threadIdx.x == 0);
                if (threadIdx.x == 0) TRACE(6, sidx);
                long long q4 = rc.on ? clock64() : 0;
                tc_fence_after();
#if !(SPK_EXP & 4)
                tmem_st16(trow + (uint32_t)(s * kACols), r);
#endif
#if !(SPK_EXP & 1)
                tmem_wait_st();
#endif
                tc_fence_before();
                long long q5 = rc.on ? clock64() : 0;
                __syncwarp();
                if (lane == 0 && glast) mbar_arrive(full0 + gbar);
                if (rc.on) {
                    const long long q6 = clock64();
                    pt[0] += q1 - q0;  // latcol store + syncwarp
                    pt[1] += q2 - q1;  // next gather issue
                    pt[2] += q3 - q2;  // expansion (LDS + SWAR)
                    pt[3] += q4 - q3;  // empty wait (incl. warp sync)
                    pt[4] += q5 - q4;  // fence + tcgen05.st + wait::st + fence
                    pt[5] += q6 - q5;  // sync + arrive
                }
            }
            tprev = rc.on ? clock64() : 0;
        }
        if (threadIdx.x == 0) {
            rc.store(0);
            if (rc.on && blockIdx.x < 1024)
                for (int q = 0; q < 9; ++q) g_conv_prof[blockIdx.x][8 + q][0] = pt[q];
        }
    } else if (warp < kProdWarps + kEpiWarps) {
        // ======================= epilogue =======================
        // two warps per TMEM lane quadrant; warp `eh` of a quadrant takes every other 16-column chunk
        RoleClock rc(a.prof != 0);
        long long ep_t[6] = {0, 0, 0, 0, 0, 0};  // SPK_CONV_PROF_BUILD: wait, bar.sync, work, tail (leader); sync, work (warp 5)
        long long ep_w = 0;                      // SPK_CONV_PROF_BUILD: cycles in tcgen05.wait::ld of the fire path
        const int qd = warp & 3;                  // TMEM lane quadrant
        const int eh = (warp - kProdWarps) >> 2;  // 0 or 1
        const int row = qd * 32 + lane;           // accumulator row = (pixel, t)
        const int pix = row >> LOGTP, t = row & (TP - 1);
        const int segbase = lane & ~(TP - 1);
        const uint32_t segmask = (TP == 32) ? 0xffffffffu : ((1u << TP) - 1u);
        // store ownership after a 16-column chunk: lane -> (column lane&15, pixel segment lane>>4)
        const int own_col = lane & 15;
        const int own_seg = (TP == 16) ? (lane >> 4) : 0;
        const bool own_lane = (TP == 16) || lane < 16;
        const int own_pix = ((qd * 32) >> LOGTP) + own_seg;
        // output staging ring: [kNOB tiles][Nt][PPT] lat bytes, then [kNOB][Nt][PPT] P* floats
        uint8_t* ob_lat = smem + a.ob_off;
        float* ob_ps = reinterpret_cast<float*>(smem + a.ob_off + kNOB * a.Nt * PPT);
        {  // digit planes no MMA writes (all-zero digits) hold zeros for the whole kernel: the
           // epilogue then reads every plane unconditionally
            const uint32_t lp = live_planes(a);
            if (lp != 7u) {
                const uint32_t z[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                for (int b = 0; b < a.NB; ++b)
                    for (int d = 0; d < 3; ++d)
                        if (!((lp >> d) & 1u))
                            for (int c = eh * 16; c < a.Nt; c += kEpiStride)
                                tmem_st16(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(b * 3 * a.Nt + d * a.Nt + c), z);
                tmem_wait_st();
            }
        }
        TileIter ti;
        ti.init(a);
        int buf = 0, ob = 0, ep_it = 0;
        uint32_t acc_ph = 0, ob_ph = 0;  // phase bits of the accumulator / staging rings
        for (; ti.valid(); ti.next(a)) {
            const int b = ti.b, nt = ti.nt;
            const int p0 = ti.j * PPT;
            const bool rvalid = p0 + pix < a.HWo && t < g.T;
            // padded rows never fire: fold the row mask into the threshold
            const long long thq = rvalid ? a.theta_q : 0x7fffffffffffffffll;
            const int thh = rvalid ? a.thH : 0x7fffffff;
            // the leader probes the staging slot and the accumulator together, the group sleeps
            const long long ec0 = rc.on ? clock64() : 0;
            if (threadIdx.x == kProdWarps * 32)
                rc.wait3(fls0 + 8 * ob, ob_ph ^ 1u, EPI != SPK_EPI_POTENTIAL && !(SPK_EXP & 65536), accf0 + 8 * buf, acc_ph,
                         !(SPK_EXP & 8704));
            const long long ec1 = rc.on ? clock64() : 0;
            asm volatile("bar.sync %0, %1;" ::"n"(kBarEpi), "n"(kEpiWarps * 32) : "memory");
            const long long ec2 = rc.on ? clock64() : 0;
            if (threadIdx.x == kProdWarps * 32) TRACE(1, ep_it);
            tc_fence_after();
            const uint32_t tbase = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(buf * 3 * a.Nt);
            for (int n0 = eh * 16; n0 < ((SPK_EXP & 128) || EPI != SPK_EPI_POTENTIAL ? 0 : a.Nt); n0 += kEpiStride) {
                uint32_t d0[16], d1[16], d2[16];
#if (SPK_EXP & 16)
#pragma unroll
                for (int q = 0; q < 16; ++q) d0[q] = d1[q] = d2[q] = (uint32_t)(n0 + q + lane);
#else
                tmem_ld16(tbase + n0, d0);
                tmem_ld16(tbase + a.Nt + n0, d1);
                tmem_ld16(tbase + 2 * a.Nt + n0, d2);
                tmem_wait_ld();
#endif
                const int obase = nt * a.Nt + n0;
                if (EPI == SPK_EPI_POTENTIAL) {
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        const int o = obase + jj;
                        const long long X =
                            (long long)(int)d2[jj] * 65536ll + ((long long)(int)d1[jj] * 256ll + (long long)(int)d0[jj]);
                        if (rvalid && o < g.Co)
                            static_cast<float*>(a.out0)[(((size_t)b * g.T + t) * g.Co + o) * a.HWo + p0 + pix] =
                                __fmul_rn(__ll2float_rn(X), a.out_scale);
                    }
                } else {
                    uint32_t mine = 0;
                    float mine_ps = 0.0f;
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        // digit accumulators are >= 0 (u8 x u8): two wide multiply-adds
                        const long long X = (long long)((unsigned long long)d2[jj] * 65536ull +
                                                        ((unsigned long long)d1[jj] * 256ull + d0[jj]));
                        const unsigned bal = __ballot_sync(0xffffffffu, X > thq);
                        if (jj == own_col) mine = bal;
                        if (PSTAR) {
                            const unsigned bits = (bal >> segbase) & segmask;
                            const int l = g.T - __popc(bits);  // fired steps are exactly t = lat .. T-1
                            const long long Xs = __shfl_sync(0xffffffffu, X, segbase + min(l, TP - 1));
                            if (jj == own_col) mine_ps = bits ? __fmul_rn(__ll2float_rn(Xs), a.out_scale) : 0.0f;
                        }
                    }
                    if (own_lane) {  // stage (map, pixel) -> smem
                        const unsigned bits = (mine >> (own_seg * TP)) & segmask;
                        const int ol = (n0 + own_col) * PPT + own_pix;
                        ob_lat[ob * a.Nt * PPT + ol] = (uint8_t)(g.T - __popc(bits));
                        if (PSTAR) ob_ps[ob * a.Nt * PPT + ol] = mine_ps;
                    }
                }
            }
            bool released = false;
            if (TP == 1 && EPI != SPK_EPI_POTENTIAL) {
                // one time step: row = pixel, fire iff X > theta (lat 0, else T = 1); P* = potential
                for (int n0 = eh * 16; n0 < a.Nt; n0 += kEpiStride) {
#pragma unroll
                    for (int h8 = 0; h8 < 16; h8 += 8) {
                        uint32_t r[24];
                        tmem_ld8(tbase + n0 + h8, r);
                        tmem_ld8(tbase + a.Nt + n0 + h8, r + 8);
                        tmem_ld8(tbase + 2 * a.Nt + n0 + h8, r + 16);
                        tmem_wait_ld();
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const long long X = (long long)((unsigned long long)r[16 + j] * 65536ull +
                                                            ((unsigned long long)r[8 + j] * 256ull + r[j]));
                            const bool fire = X > thq;
                            const int ol = ob * a.Nt * PPT + (n0 + h8 + j) * PPT + pix;
                            ob_lat[ol] = fire ? (uint8_t)0 : (uint8_t)g.T;
                            if (PSTAR) ob_ps[ol] = fire ? __fmul_rn(__ll2float_rn(X), a.out_scale) : 0.0f;
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(acce0 + 8 * buf);
                released = true;
            } else if (EPI != SPK_EPI_POTENTIAL && !(SPK_EXP & 128)) {
                // 16-column chunks n0 = eh*16 + 32 i, each read as two 8-column halves; the
                // TMEM loads of the next half overlap the threshold work on the current one,
                // and the accumulator is released as soon as its last load has landed
                uint32_t ra[24], rb[24];
                auto ld8 = [&](int n0, uint32_t* r) {
#if (SPK_EXP & 512)  // timing experiment: fire epilogue without TMEM loads (synthetic digits)
#pragma unroll
                    for (int q = 0; q < 24; ++q) r[q] = (uint32_t)(n0 * 7 + q + lane);
#else
                    tmem_ld8(tbase + n0, r);
                    tmem_ld8(tbase + a.Nt + n0, r + 8);
                    tmem_ld8(tbase + 2 * a.Nt + n0, r + 16);
#endif
                };
                uint32_t mine = 0;
                // P*: the lane holding a (pixel, map)'s first crossing (its bit set, the previous
                // step's clear) writes the potential straight into the staging tile — no shuffle
                const unsigned segstart = (TP == 16) ? 0x00010001u : 0x1u;
                float* ps_tile = ob_ps + ob * a.Nt * PPT + pix;
                auto half = [&](const uint32_t* r, int j0, int c0) {  // c0: tile column of r[0]
#if (SPK_EXP & 1024)  // timing experiment: TMEM loads kept, threshold work reduced to one ballot
                    {
                        const unsigned bal = __ballot_sync(0xffffffffu, (r[0] ^ r[8] ^ r[16] ^ r[23]) > 7u);
                        if (j0 == own_col) mine = bal;
                        return;
                    }
#endif
                    if (a.small_x) {  // 32-bit form of X > theta_q (see TcArgs)
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const uint32_t tl = r[8 + j] * 256u + r[j] + a.thC;
                            const unsigned bal = __ballot_sync(0xffffffffu, (int)(r[16 + j] + (tl >> 16)) > thh);
                            if (j0 + j == own_col) mine = bal;
                            if (PSTAR && ((bal & ~((bal << 1) & ~segstart)) >> lane) & 1u) {
                                const long long X = (long long)r[16 + j] * 65536ll + (long long)(tl - a.thC);
                                ps_tile[(c0 + j) * PPT] = __fmul_rn(__ll2float_rn(X), a.out_scale);
                            }
                        }
                        return;
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        // digit accumulators are >= 0 (u8 x u8): two wide multiply-adds
                        const long long X = (long long)((unsigned long long)r[16 + j] * 65536ull +
                                                        ((unsigned long long)r[8 + j] * 256ull + r[j]));
                        const unsigned bal = __ballot_sync(0xffffffffu, X > thq);
                        if (j0 + j == own_col) mine = bal;
                        if (PSTAR && ((bal & ~((bal << 1) & ~segstart)) >> lane) & 1u)
                            ps_tile[(c0 + j) * PPT] = __fmul_rn(__ll2float_rn(X), a.out_scale);
                    }
                };
                int n0 = eh * 16;
                if (n0 < a.Nt) {
                    ld8(n0, ra);
                    { const long long w0_ = rc.on ? clock64() : 0; tmem_wait_ld(); if (rc.on) ep_w += clock64() - w0_; }
                }
                for (; n0 < a.Nt; n0 += kEpiStride) {
                    ld8(n0 + 8, rb);
                    half(ra, 0, n0);
                    { const long long w0_ = rc.on ? clock64() : 0; tmem_wait_ld(); if (rc.on) ep_w += clock64() - w0_; }
                    const bool more = n0 + kEpiStride < a.Nt;
                    if (more) {
                        ld8(n0 + kEpiStride, ra);
                    } else if (!(SPK_EXP & 8192)) {  // every TMEM read of this buffer has landed
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(acce0 + 8 * buf);
                        released = true;
                    }
                    half(rb, 8, n0 + 8);
                    if (more) { const long long w0_ = rc.on ? clock64() : 0; tmem_wait_ld(); if (rc.on) ep_w += clock64() - w0_; }
                    if (own_lane) {  // stage (map, pixel) -> smem
                        const unsigned bits = (mine >> (own_seg * TP)) & segmask;
                        const int ol = (n0 + own_col) * PPT + own_pix;
                        ob_lat[ob * a.Nt * PPT + ol] = (uint8_t)(g.T - __popc(bits));
                        if (PSTAR && bits == 0) ob_ps[ob * a.Nt * PPT + ol] = 0.0f;  // never fired
                    }
                }
            }
            if (!released) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0 && !(SPK_EXP & 8192)) mbar_arrive(acce0 + 8 * buf);
            }
            const long long ec3 = rc.on ? clock64() : 0;
            if (threadIdx.x == kProdWarps * 32) TRACE(2, ep_it);
            ++ep_it;
            if (EPI != SPK_EPI_POTENTIAL) {  // hand the staged tile to the flusher warp
                __syncwarp();
                if (lane == 0) mbar_arrive(stg0 + 8 * ob);
            }
            if (++buf == a.NB) buf = 0, acc_ph ^= 1u;
            if (++ob == kNOB) ob = 0, ob_ph ^= 1u;
            if (rc.on) {
                const long long ec4 = clock64();
                if (threadIdx.x == kProdWarps * 32) {
                    ep_t[0] += ec1 - ec0, ep_t[1] += ec2 - ec1, ep_t[2] += ec3 - ec2, ep_t[3] += ec4 - ec3;
                } else if (threadIdx.x == (kProdWarps + 5) * 32) {
                    ep_t[4] += ec2 - ec0, ep_t[5] += ec3 - ec2;
                }
            }
        }
        if (rc.on && blockIdx.x < 1024) {
            if (threadIdx.x == kProdWarps * 32)
                for (int q = 0; q < 4; ++q) g_conv_prof[blockIdx.x][17 + q][0] = ep_t[q];
            if (threadIdx.x == (kProdWarps + 5) * 32)
                for (int q = 4; q < 6; ++q) g_conv_prof[blockIdx.x][17 + q][0] = ep_t[q];
            if (threadIdx.x == kProdWarps * 32) g_conv_prof[blockIdx.x][23][0] = ep_w;
            if (threadIdx.x == (kProdWarps + 5) * 32) g_conv_prof[blockIdx.x][24][0] = ep_w;
        }
        if (threadIdx.x == kProdWarps * 32) rc.store(1);
    } else if (warp == kMmaWarp) {
        // ======================= MMA issuer =======================
        RoleClock rc(a.prof != 0);
        {  // the whole warp runs the loop (uniform control flow); elected lanes issue
            auto mk_idesc = [](int n) {  // s32 D, u8 A/B, K-major, M = 128
                return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            };
            const uint32_t idesc = mk_idesc(a.Nt);  // one plane per MMA (stack == 0)
            // live digit planes (written by the pack kernel earlier on the stream)
            uint32_t pA, nA, pB, nB;
            plane_plan(a, pA, nA, pB, nB);
            const uint32_t idA = mk_idesc((int)nA * a.Nt), idB = mk_idesc(a.Nt);
            const uint32_t b_base = smem_u32(Bs);
            const uint32_t bstage = 3u * a.Nt * KS, bchunk = 3u * a.Nt * 16;  // chunk stride (LBO)
            const uint64_t d0 = smem_desc(b_base, bchunk, 128);                // descriptor template
            const uint64_t inck = (2u * bchunk) >> 4;                          // next k-step (2 chunks)
            const uint64_t incd = ((uint32_t)a.Nt * 16u) >> 4;                 // next digit plane (Nt rows)
            if (a.bres) rc.wait_warp(bresb, 0u);
            long long f_fence = 0, f_issue = 0, f_commit = 0;
            TileIter ti;
            ti.init(a);
            int mma_it = 0, mma_st = 0;
            int as_cur = 0, bs = 0, buf = 0;  // A ring (TMEM, NA slots), B ring (smem, NS slots), accumulators
            uint32_t aph_cur = 0, b_ph = 0, acc_ph = 0;
            for (; ti.valid(); ti.next(a)) {
                // a retained A is produced at the first N tile and released after the last one
                const bool newA = !a.retain || ti.nt == 0, lastA = !a.retain || ti.nt == a.n_ntiles - 1;
                const bool wacc = !(SPK_EXP & 8192);
                if (lane == 0) TRACE(3, mma_it);
                tc_fence_after();
                const uint32_t dbase = tmem + (uint32_t)(buf * 3 * a.Nt);
                int kb_next = 0;
                int s = as_cur;  // slot group (G slots per hand-off)
                uint32_t aph = aph_cur;
                const int ngrp = a.NA / a.G;
#if SPK_MMA_FAST
                // retained A already in TMEM and this tile's weights in one hand-off: every K stage
                // of the tile is issued back to back after one wait (no per-stage fence or probes)
                if (a.retain && !newA && (a.bres || a.GB == a.nks) && !(SPK_EXP & 32)) {
                    rc.wait3(bfull0 + 8 * bs, b_ph, !a.bres && !(SPK_EXP & 4096), acce0 + 8 * buf, acc_ph ^ 1u, wacc);
                    tc_fence_after();
                    const uint64_t dst0 = d0 + (((a.bres ? 0u : (uint32_t)(bs * a.GB)) * bstage) >> 4);
                    const uint32_t eA = dbase + pA * a.Nt, eB = dbase + pB * a.Nt;
                    const uint32_t two = nB ? 1u : 0u;
                    for (int ks = 0; ks < a.nks; ks += a.G) {
                        if (ks) {
                            if (++s == ngrp) s = 0, aph ^= 1u;
                        }
                        const uint64_t dst = dst0 + (((uint32_t)ks * bstage) >> 4);
                        const uint32_t at = tmem + (uint32_t)(a.aCol0 + s * a.G * kACols);
                        const int nk = min(a.G * (KS / 32), (a.K - ks * KS + 31) / 32);
                        const uint32_t acc0 = ks ? 1u : 0u;
                        const uint64_t xA = dst + incd * pA, xB = dst + incd * pB;
                        if (nk == 4) {
                            tc_stage_gen<4>(eA, eB, at, xA, xB, inck, idA, idB, acc0, two);
                        } else if (nk == 8) {
                            tc_stage_gen<8>(eA, eB, at, xA, xB, inck, idA, idB, acc0, two);
                        } else {
#pragma unroll 1
                            for (int kk = 0; kk < nk; ++kk)
                                tc_stage_gen<1>(eA, eB, at + 8u * kk, xA + inck * kk, xB + inck * kk, inck, idA, idB,
                                                kk ? 1u : acc0, two);
                        }
                        if (lastA && !(SPK_EXP & 16384)) tc_commit_elect(empty0 + 8 * s);
                    }
                    if (!a.bres && !(SPK_EXP & 4096)) {
                        tc_commit_elect(bempty0 + 8 * bs);
                        if (++bs == a.NS) bs = 0, b_ph ^= 1u;
                    }
                } else
#endif
                for (int ks = 0; ks < a.nks; ks += a.G) {
                    if (ks) {
                        if (++s == ngrp) s = 0, aph ^= 1u;
                    }
                    if (lane == 0) TRACE(9, mma_st);
                    // all lanes probe (no divergence); the tile's accumulator wait joins the first hand-off's
                    const int kb = kb_next;  // slot offset inside the current B hand-off
                    kb_next = kb + a.G >= a.GB ? 0 : kb + a.G;
                    rc.wait3(full0 + 8 * s, aph, newA && !(SPK_EXP & 16384), bfull0 + 8 * bs, b_ph,
                             !a.bres && !(SPK_EXP & 4096) && kb == 0, acce0 + 8 * buf, acc_ph ^ 1u, wacc && ks == 0);
                    if (lane == 0) TRACE(7, mma_st);
                    ++mma_st;
                    const long long c0 = rc.on ? clock64() : 0;
                    tc_fence_after();
                    const long long c1 = rc.on ? clock64() : 0;
                    // the group's slots and B blocks are contiguous: k-step kk at + 8 kk, dst + kk inck
                    const uint64_t dst = d0 + (((a.bres ? (uint32_t)ks : (uint32_t)(bs * a.GB + kb)) * bstage) >> 4);
                    const uint32_t at = tmem + (uint32_t)(a.aCol0 + s * a.G * kACols);
                    // k-steps of 32 synapses this hand-off holds (the last one may be partial)
                    const int nk = min(a.G * (KS / 32), (a.K - ks * KS + 31) / 32);
                    const uint32_t acc0 = ks ? 1u : 0u;
// full hand-offs take one straight-line block; a partial last one issues single
// k-steps in a loop (no jump table: an indirect branch costs a constant-bank load and
// an instruction fetch at a far target on every hand-off)
#define SPK_NK_DISPATCH(CALL)                                                 \
    {                                                                         \
        uint32_t f8 = nk == 8, f4 = nk == 4;                                  \
        asm volatile("" : "+r"(f8), "+r"(f4));                                \
        if (f8) {                                                             \
            CALL(8, 0);                                                       \
        } else if (f4) {                                                      \
            CALL(4, 0);                                                       \
        } else {                                                              \
            _Pragma("unroll 1") for (int kk = 0; kk < nk; ++kk) CALL(1, kk);  \
        }                                                                     \
    }
                    if (SPK_EXP & 32) {
                    } else if (a.stack != 0) {
                        const uint32_t eA = dbase + pA * a.Nt, eB = dbase + pB * a.Nt;
                        const uint64_t xA = dst + incd * pA, xB = dst + incd * pB;
                        const uint32_t two = nB ? 1u : 0u;
#define SPK_GEN(n, kk) \
    tc_stage_gen<n>(eA, eB, at + 8u * (kk), xA + inck * (kk), xB + inck * (kk), inck, idA, idB, (kk) ? 1u : acc0, two)
                        SPK_NK_DISPATCH(SPK_GEN)
#undef SPK_GEN
                    } else {
                        const uint32_t e1 = dbase + a.Nt, e2 = dbase + 2 * a.Nt;
#define SPK_SEP(n, kk) \
    tc_stage_sep<n>(dbase, e1, e2, at + 8u * (kk), dst + inck * (kk), inck, incd, idesc, (kk) ? 1u : acc0)
                        SPK_NK_DISPATCH(SPK_SEP)
#undef SPK_SEP
                    }
#undef SPK_NK_DISPATCH
                    if (lane == 0) TRACE(10, mma_st - 1);
                    const long long c2 = rc.on ? clock64() : 0;
                    if (!a.bres && !(SPK_EXP & 4096) && (kb_next == 0 || ks + a.G >= a.nks)) {
                        tc_commit_elect(bempty0 + 8 * bs);
                        if (++bs == a.NS) bs = 0, b_ph ^= 1u;
                    }
                    if (lastA && !(SPK_EXP & 16384)) tc_commit_elect(empty0 + 8 * s);
                    if (lane == 0) TRACE(11, mma_st - 1);
                    if (rc.on) {
                        const long long c3 = clock64();
                        f_fence += c1 - c0;
                        f_issue += c2 - c1;
                        f_commit += c3 - c2;
                    }
                }
                if (lane == 0) TRACE(0, mma_it);
                if (!(SPK_EXP & 8192)) tc_commit_elect(accf0 + 8 * buf);
                ++mma_it;
                if (lastA) {  // the next M tile starts after this tile's slot groups
                    as_cur = s + 1 == ngrp ? 0 : s + 1;
                    if (s + 1 == ngrp) aph ^= 1u;
                    aph_cur = aph;
                }
                if (++buf == a.NB) buf = 0, acc_ph ^= 1u;
            }
            if (lane == 0) rc.store(2);
            if (rc.on && lane == 0 && blockIdx.x < 1024) {
                g_conv_prof[blockIdx.x][5][0] = f_fence;
                g_conv_prof[blockIdx.x][6][0] = f_issue;
                g_conv_prof[blockIdx.x][7][0] = f_commit;
            }
        }
        __syncwarp();
    } else if (warp == kMmaWarp + 1) {
        // ======================= B loader =======================
        RoleClock rc(a.prof != 0);
        if (lane == 0) {
            const uint32_t bstage = 3u * a.Nt * KS;
            const uint32_t b_base = smem_u32(Bs);
            if (SPK_EXP & 4096) {
            } else if (a.bres) {
                // whole packed B of the (single) N tile, resident for the kernel
                for (int ks = 0; ks < a.nks; ++ks) {
                    mbar_arrive_tx(bresb, bstage);
                    bulk_g2s(b_base + ks * bstage, a.wpk + (size_t)ks * bstage, bstage, bresb);
                }
            } else {
                TileIter ti;
                ti.init(a);
                int s = 0, bl_st = 0;
                uint32_t ph = 0;
                for (; ti.valid(); ti.next(a)) {
                    for (int ks = 0; ks < a.nks; ks += a.GB) {  // one copy per B hand-off
                        const uint32_t bytes = (uint32_t)min(a.GB, a.nks - ks) * bstage;
                        rc.wait_idle(bempty0 + 8 * s, ph ^ 1u);
                        TRACE(8, bl_st);
                        ++bl_st;
#if (SPK_EXP & 256)  // timing experiment: no B traffic (stale smem operands)
                        mbar_arrive(bfull0 + 8 * s);
#else
                        mbar_arrive_tx(bfull0 + 8 * s, bytes);
                        bulk_g2s(b_base + s * a.GB * bstage, a.wpk + ((size_t)ti.nt * a.nks + ks) * bstage, bytes,
                                 bfull0 + 8 * s);
#endif
                        if (++s == a.NS) s = 0, ph ^= 1u;
                    }
                }
            }
            rc.store(3);
        }
        __syncwarp();
    } else if (warp < kFlushWarp && (SPK_EXP & 32768)) {  // no band loaders either
    } else if (warp < kFlushWarp) {
        // ======================= input band loaders =======================
        RoleClock rc(a.prof != 0);
        const int lt = threadIdx.x - (kMmaWarp + 2) * 32;  // 0..kLoaders-1
        const size_t plane = (size_t)g.Hi * g.Wi;
        TileIter ti;
        ti.init(a);
        int rb = 0;
        uint32_t rph = 0;
        bool need_region = true;
        for (; ti.valid(); ti.next(a)) {
            const bool load = need_region;
            need_region = ti.template region_ends<PPT>(a);
            if (!load) continue;  // same staged region as the previous tile
            uint8_t* dst = RG + rb * a.rb_stride;
            rc.template group_wait<kBarBand, kLoaders>(rge0 + 8 * rb, rph ^ 1u, lt == 0);
            // region[c][r][x] = min(lat[b][c][pr0 + r - Ph][x - Pw], 0x7F), 0x7F (never) in the halo
            const uint8_t* src = a.lat_in + (size_t)ti.b * g.Ci * plane;
            const int total = g.Ci * a.band;
            if (SPK_EXP & 2048) {  // timing experiment: no input staging (stale region)
            } else if (a.NR == a.HiP) {
                // whole padded sample: the halo was filled once at kernel start; copy the interior
                // rows, one input row (c, iy) per lane per pass — four rows' loads in flight, 4-byte
                // loads when the sample is 4-byte aligned (Wi % 4 == 0 keeps every row aligned)
                const int nrows = g.Ci * g.Hi;
                const bool al4 = (g.Wi & 3) == 0 && (reinterpret_cast<uintptr_t>(src) & 3) == 0;
                for (int r0 = lt; r0 < nrows; r0 += kLoaders) {
                    const int c = r0 / g.Hi, iy = r0 - c * g.Hi;
                    const uint8_t* sr = src + (size_t)r0 * g.Wi;
                    uint8_t* d = dst + c * a.band + (iy + g.Ph) * a.WiP + g.Pw;
                    if (al4) {
                        const uint32_t* s4 = reinterpret_cast<const uint32_t*>(sr);
                        int x4 = 0;
                        for (; x4 + 4 <= (g.Wi >> 2); x4 += 4) {
                            uint32_t v[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) v[u] = __ldg(s4 + x4 + u);
#pragma unroll
                            for (int u = 0; u < 4; ++u)
#pragma unroll
                                for (int e = 0; e < 4; ++e) d[4 * (x4 + u) + e] = (uint8_t)min((v[u] >> (8 * e)) & 0xFFu, 0x7Fu);
                        }
                        for (; x4 < (g.Wi >> 2); ++x4) {
                            const uint32_t v = __ldg(s4 + x4);
#pragma unroll
                            for (int e = 0; e < 4; ++e) d[4 * x4 + e] = (uint8_t)min((v >> (8 * e)) & 0xFFu, 0x7Fu);
                        }
                    } else {
                        for (int x = 0; x < g.Wi; ++x) d[x] = min(__ldg(sr + x), (uint8_t)0x7F);
                    }
                }
            } else {
                // band of NR padded rows: one padded row (c, r) per thread per pass
                const int pr0 = ti.r0<PPT>(a);
                for (int row = lt; row < g.Ci * a.NR; row += kLoaders) {
                    const int c = row / a.NR, r = row - c * a.NR;
                    const int iy = pr0 + r - g.Ph;
                    uint8_t* d = dst + c * a.band + r * a.WiP;
                    if ((unsigned)iy >= (unsigned)g.Hi) {
                        for (int x = 0; x < a.WiP; ++x) d[x] = 0x7F;
                        continue;
                    }
                    const uint8_t* sr = src + (size_t)c * plane + (size_t)iy * g.Wi;
                    for (int x = 0; x < g.Pw; ++x) d[x] = 0x7F;
                    for (int x = 0; x < g.Pw; ++x) d[g.Pw + g.Wi + x] = 0x7F;
                    int x = 0;
                    for (; x + 4 <= g.Wi; x += 4) {
                        const uint8_t v0 = __ldg(sr + x), v1 = __ldg(sr + x + 1), v2 = __ldg(sr + x + 2),
                                      v3 = __ldg(sr + x + 3);
                        d[g.Pw + x] = min(v0, (uint8_t)0x7F);
                        d[g.Pw + x + 1] = min(v1, (uint8_t)0x7F);
                        d[g.Pw + x + 2] = min(v2, (uint8_t)0x7F);
                        d[g.Pw + x + 3] = min(v3, (uint8_t)0x7F);
                    }
                    for (; x < g.Wi; ++x) d[g.Pw + x] = min(__ldg(sr + x), (uint8_t)0x7F);
                }
            }
            if (lt < 16) dst[total + lt] = 0x7F;  // sentinel block for padding synapses
            __syncwarp();
            if (lane == 0) mbar_arrive(rgf0 + 8 * rb);
            if (++rb == a.nrb) rb = 0, rph ^= 1u;
        }
        if (lt == 0) rc.store(4);
    }

    if (warp == kFlushWarp && EPI != SPK_EPI_POTENTIAL && !(SPK_EXP & 65536)) {
        // ======================= flusher: staged tile -> one run of PPT pixels per output map
        const uint8_t* ob_lat = smem + a.ob_off;
        const float* ob_ps = reinterpret_cast<const float*>(smem + a.ob_off + kNOB * a.Nt * PPT);
        TileIter ti;
        ti.init(a);
        int ob = 0, fl_it = 0;
        uint32_t ph = 0;
        for (; ti.valid(); ti.next(a)) {
            if (lane == 0) mbar_wait_idle(stg0 + 8 * ob, ph);
            if (lane == 0) TRACE(4, fl_it);
            __syncwarp();
            const int b = ti.b, nt = ti.nt, p0 = ti.j * PPT;
            const uint8_t* sl = ob_lat + ob * a.Nt * PPT;
            const float* sp = ob_ps + ob * a.Nt * PPT;
            const int npix = min(PPT, a.HWo - p0);
            if (TP == 1) {
                const int nmap = min(a.Nt, g.Co - nt * a.Nt);
                for (int ol = 0; ol < nmap; ++ol) {
                    const size_t oi = ((size_t)b * g.Co + nt * a.Nt + ol) * a.HWo + p0;
                    uint8_t* dl = static_cast<uint8_t*>(a.out0) + oi;
                    if (npix == PPT && (reinterpret_cast<uintptr_t>(dl) & 3) == 0) {
                        reinterpret_cast<uint32_t*>(dl)[lane] = reinterpret_cast<const uint32_t*>(sl + ol * PPT)[lane];
                    } else {
                        for (int q = lane; q < npix; q += 32) dl[q] = sl[ol * PPT + q];
                    }
                    if (PSTAR)
                        for (int q = lane; q < npix; q += 32) a.out1[oi + q] = sp[ol * PPT + q];
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(fls0 + 8 * ob);
                ++fl_it;
                if (++ob == kNOB) ob = 0, ph ^= 1u;
                continue;
            }
            for (int ol = lane; ol < a.Nt; ol += 32) {
                const int o = nt * a.Nt + ol;
                if (o >= g.Co || (SPK_EXP & 8)) continue;
                const size_t oi = ((size_t)b * g.Co + o) * a.HWo + p0;
                uint8_t* dl = static_cast<uint8_t*>(a.out0) + oi;
                // widest aligned stores (a map's run starts at (b Co + o) HWo + p0: with HWo = 196,
                // half the runs are only 4-byte aligned)
                const uintptr_t al = reinterpret_cast<uintptr_t>(dl);
                if (npix == PPT && PPT == 8 && (al & 7) == 0) {
                    *reinterpret_cast<uint2*>(dl) = *reinterpret_cast<const uint2*>(sl + ol * PPT);
                } else if (npix == PPT && (PPT == 4 || PPT == 8) && (al & 3) == 0) {
                    const uint32_t* s4 = reinterpret_cast<const uint32_t*>(sl + ol * PPT);
                    reinterpret_cast<uint32_t*>(dl)[0] = s4[0];
                    if (PPT == 8) reinterpret_cast<uint32_t*>(dl)[1] = s4[1];
                } else if (npix == PPT && (PPT == 4 || PPT == 8) && (al & 1) == 0) {
                    const uint16_t* s2 = reinterpret_cast<const uint16_t*>(sl + ol * PPT);
#pragma unroll
                    for (int q = 0; q < PPT / 2; ++q) reinterpret_cast<uint16_t*>(dl)[q] = s2[q];
                } else {
                    for (int q = 0; q < npix; ++q) dl[q] = sl[ol * PPT + q];
                }
                if (PSTAR) {
                    float* dp = a.out1 + oi;
                    if (npix == PPT && (PPT == 4 || PPT == 8) && (oi & 3) == 0) {
#pragma unroll
                        for (int q = 0; q < PPT; q += 4)
                            *reinterpret_cast<float4*>(dp + q) = *reinterpret_cast<const float4*>(sp + ol * PPT + q);
                    } else if (npix == PPT && (PPT == 4 || PPT == 8) && (oi & 1) == 0) {
#pragma unroll
                        for (int q = 0; q < PPT; q += 2)
                            *reinterpret_cast<float2*>(dp + q) = *reinterpret_cast<const float2*>(sp + ol * PPT + q);
                    } else {
                        for (int q = 0; q < npix; ++q) dp[q] = sp[ol * PPT + q];
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(fls0 + 8 * ob);
            if (lane == 0) TRACE(5, fl_it);
            ++fl_it;
            if (++ob == kNOB) ob = 0, ph ^= 1u;
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// ------------------------------------------------------------------ weight packing
// Digit planes in the exact smem image of each (n-tile, K-stage) block, digit-stacked
// along N:  block (nt, ks): [chunk 0..KS/16-1][3*Nt/8 row groups][8 rows][16 bytes],
// row d*Nt + n holding digit d of output map nt*Nt + n.
__global__ void pack_weights_kernel(const float* __restrict__ w, int Co, int K, int Nt, int n_ntiles, int nks,
                                    float inv_scale23, uint8_t* __restrict__ wpk, int* __restrict__ flag) {
    spk_pdl_wait();
    // one thread per (nt, ks, c, n, 4 consecutive synapses e0..e0+3): one 4-byte store per digit
    // plane instead of four byte stores
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // over (nt, ks, c, n, e4)
    const size_t per_plane4 = (size_t)Nt * (KS / 4);
    if (q >= (size_t)n_ntiles * nks * per_plane4) return;
    const size_t blk = q / per_plane4, r = q % per_plane4;
    const int nt = (int)(blk / nks), ks = (int)(blk % nks);
    const int c = (int)(r / ((size_t)Nt * 4)), r2 = (int)(r % ((size_t)Nt * 4));
    const int n = r2 / 4, e0 = (r2 % 4) * 4;
    const int k0 = ks * KS + c * 16 + e0, o = nt * Nt + n;
    uint32_t pk[3] = {0u, 0u, 0u};
    uint32_t live = 0;  // bit 1 + d: digit d non-zero
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float v = 0.0f;
        if (o < Co && k0 + i < K) v = w[(size_t)o * K + k0 + i];
        float x = __fmul_rn(v, inv_scale23);  // exact: inv_scale23 is a power of two
        if (!(x >= 0.0f) || x > 8388608.0f) {  // negative, NaN or above the scale: clamp and flag
            atomicOr(flag, 1);
            x = (x > 8388608.0f) ? 8388608.0f : 0.0f;
        }
        const uint32_t qv = (uint32_t)__float2int_rn(x);  // 0 .. 2^23
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const uint32_t digit = (qv >> (8 * d)) & 255u;
            pk[d] |= digit << (8 * i);
            live |= digit ? 2u << d : 0u;
        }
    }
    uint8_t* base = wpk + blk * 3 * ((size_t)Nt * KS) + (size_t)c * 3 * Nt * 16;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const int row = d * Nt + n;
        *reinterpret_cast<uint32_t*>(base + (size_t)(row >> 3) * 128 + (row & 7) * 16 + e0) = pk[d];
    }
    live = __reduce_or_sync(__activemask(), live);
    // one atomic per warp, and only while it still adds a bit (the flag fills up at once)
    if ((threadIdx.x & 31) == 0 && (live & ~(uint32_t)__ldcg(flag))) atomicOr(flag, (int)live);
}

template <int EPI, bool PSTAR, int TP>
void launch(const TcArgs& a, unsigned grid, size_t smem, cudaStream_t s) {
    static std::atomic<uint64_t> done{0};
    if (spk::first_on_device(done)) {
        cudaFuncSetAttribute(conv_tc_kernel<EPI, PSTAR, TP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    }
    spk::launch(conv_tc_kernel<EPI, PSTAR, TP>, grid, kThreads, smem, s, a);
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
    // rows of an M tile: (pixel, t) with t padded to 16 or 32; one time step (T = 1): pixels only
    p.TP = g.T == 1 ? 1 : g.T <= 16 ? 16 : 32;
    p.PPT = 128 / p.TP;
    if ((long long)g.B * ((p.Ho * p.Wo + p.PPT - 1) / p.PPT) * 4 >= (1ll << 31))
        return false;  // tile indices are 32-bit
    p.KS = KS;
    p.nks = (p.K + KS - 1) / KS;
    // N tiling: accumulators (3 digit planes) + the TMEM A ring share 512 columns; at least
    // 4 A slots, at most 2 accumulator buffers, every remaining column to the A ring
    const int acc_cols = 512 - 4 * kACols;  // 384
    // a reduction that fits the TMEM A ring is produced once per M tile and kept for every
    // N tile; N tiles of 64 then give two accumulator buffers (epilogue overlaps the MMAs)
    static const int retain_ok = [] {
        const char* e = std::getenv("SPK_CONV_RETAIN");  // tuning knob: 0 disables A retention
        return e ? std::atoi(e) : 1;
    }();
    p.retain = (retain_ok && p.nks <= 4 && g.Co > 64) ? 1 : 0;
    static const int nt_force = [] {
        const char* e = std::getenv("SPK_CONV_NT");  // tuning knob: force the N tile (multiple of 16)
        return e ? std::atoi(e) : 0;
    }();
    if (nt_force >= 16 && nt_force % 16 == 0 && nt_force <= 128) {
        p.Nt = nt_force;
    } else if (p.TP == 1) {
        p.Nt = std::min(32, ((g.Co + 15) / 16) * 16);  // output staging of 128-pixel rows: 32 maps per tile
        p.retain = p.retain && g.Co > 32;
    } else if (p.retain) {
        p.Nt = 64;
    } else if (g.Co <= 64) {
        p.Nt = ((g.Co + 15) / 16) * 16;
    } else {
        const int nn = (g.Co + 127) / 128;
        const int per = (g.Co + nn - 1) / nn;
        p.Nt = ((per + 15) / 16) * 16;
    }
    static const int nb_cap = [] {
        const char* e = std::getenv("SPK_CONV_NB");  // tuning knob: accumulator buffers cap (1..4)
        return e ? std::max(1, std::min(4, std::atoi(e))) : 2;
    }();
    p.NB = std::min(nb_cap, acc_cols / (3 * p.Nt));  // TMEM accumulator buffers (MMA/epilogue overlap)
    if (p.NB < 1 || 3 * p.Nt * p.NB > acc_cols) return false;
    p.NA = std::min(kMaxA, (512 - 3 * p.Nt * p.NB) / kACols);
    p.aCol0 = 512 - p.NA * kACols;
    // digit planes per MMA: all three (N = 3 Nt), planes 0-1 + plane 2, or one each
    p.stack = (3 * p.Nt <= 256) ? 1 : (2 * p.Nt <= 256) ? 2 : 0;
    p.n_ntiles = (g.Co + p.Nt - 1) / p.Nt;
    const int HWo = p.Ho * p.Wo;
    p.tps = (HWo + p.PPT - 1) / p.PPT;
    // input rows one tile needs: (rows its pixels span) * Sh + Kh - Sh, at most Hi
    int span = 0;
    for (int j = 0; j < p.tps; ++j) {
        const int y0 = (j * p.PPT) / p.Wo, y1 = (std::min(j * p.PPT + p.PPT, HWo) - 1) / p.Wo;
        span = std::max(span, (y1 - y0) * g.Sh + g.Kh);
    }
    // staged region: padded rows (zero-padding halo included, as "never") of every channel
    p.WiP = g.Wi + 2 * g.Pw;
    p.HiP = g.Hi + 2 * g.Ph;
    p.NR = std::min(p.HiP, span);
    // stage whole (padded) sample maps when two fit comfortably: one load serves every tile of the sample
    if ((size_t)g.Ci * p.HiP * p.WiP <= 24 * 1024) p.NR = p.HiP;
    p.band = p.NR * p.WiP;
    p.NP = (long long)g.B * HWo;
    p.n_mtiles = (long long)g.B * p.tps;
    p.total_tiles = p.n_mtiles * p.n_ntiles;
    p.packed_bytes = (size_t)p.n_ntiles * p.nks * 3 * p.Nt * KS;
    p.ws_bytes = 256 + p.packed_bytes;
    p.kt16 = (size_t)g.Ci * p.band + 16 < 65536 ? 1 : 0;
    const size_t bstage = (size_t)3 * p.Nt * KS, lc = 8 * 4 * (KS / 2),
                 kt = (p.kt16 ? 2 : 4) * (size_t)p.nks * KS;
    const size_t ob = (size_t)kNOB * p.Nt * p.PPT * 5;  // output staging ring (lat + P*)
    const size_t region = ((size_t)g.Ci * p.band + 16 + 15) & ~(size_t)15;  // + sentinel block
    const size_t cap = 227 * 1024;
    if ((size_t)g.Ci * p.band >= (1u << 24)) return false;
    const size_t other = lc + kt + ob + 1024;
    // resident B when there is one N tile and all its K stages fit next to two band buffers
    const size_t bres_bytes = (size_t)p.nks * bstage;
    p.bres = (p.n_ntiles == 1 && bres_bytes + other + 2 * region <= cap) ? 1 : 0;
    // hand-offs of G = 2 slots (half the mbarrier round trips) when the ring keeps >= 2
    // groups and at least two streamed B groups fit; a retained A keeps G = 1
    static const int g_cap = [] {
        const char* e = std::getenv("SPK_CONV_G");  // tuning knob: 1 or 2
        return e ? std::max(1, std::min(2, std::atoi(e))) : 2;
    }();
    p.G = 1;
    {
        // a retained A needs room for two M tiles' groups, a streamed one for two groups
        const int need = p.retain ? 2 * ((p.nks + 1) / 2) : 2;
        if (g_cap == 2 && p.nks >= 2 && p.NA / 2 >= need && (p.bres || 2 * 2 * bstage + other + region <= cap))
            p.G = 2;
    }
    // streamed B: one hand-off per tile when two whole-tile B stages fit (retained A: the
    // MMA warp then probes once per N tile), else per slot group
    p.GB = p.G;
    if (!p.bres && p.retain && (size_t)2 * p.nks * bstage + other + region <= cap) p.GB = p.nks;
    const size_t gstage = (size_t)p.GB * bstage;
    p.NS = S;
    while (!p.bres && p.NS > 2 && (size_t)p.NS * gstage + other + region > cap) --p.NS;
    const size_t b = p.bres ? bres_bytes : (size_t)p.NS * gstage;
    const size_t fixed = b + other;
    if (fixed + region > cap) return false;
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

    int* flag = static_cast<int*>(ws);
    uint8_t* wpk = static_cast<uint8_t*>(ws) + 256;
    if (w) {  // w == nullptr: the workspace already holds this layer's packed weights (spk_conv_prepack)
        if (cudaMemsetAsync(flag, 0, sizeof(int), s) != cudaSuccess) return spk::launched("memset(flag)");
        const size_t nthreads = (size_t)p.n_ntiles * p.nks * p.Nt * (KS / 4);
        spk::launch(pack_weights_kernel, spk::ceil_div(nthreads, 256), 256, 0, s, w, g.Co, p.K, p.Nt, p.n_ntiles, p.nks,
                                                                        inv_scale23, wpk, flag);
        spk_status st = spk::launched("pack_weights_kernel");
        if (st != SPK_OK) return st;
    }
    if (!lat_in) return SPK_OK;  // pack only (spk_conv_prepack)

    TcArgs a{};
    a.lat_in = lat_in;
    a.wpk = wpk;
    a.wflag = flag;
    a.out0 = out0;
    a.out1 = static_cast<float*>(out1);
    a.g = g;
    a.Ho = p.Ho;
    a.Wo = p.Wo;
    a.HWo = p.Ho * p.Wo;
    a.K = p.K;
    a.nks = p.nks;
    a.Nt = p.Nt;
    a.n_ntiles = p.n_ntiles;
    a.NB = p.NB;
    a.tps = p.tps;
    a.NR = p.NR;
    a.band = p.band;
    a.WiP = p.WiP;
    a.HiP = p.HiP;
    a.nrb = p.nrb;
    a.rb_stride = (int)p.rb_stride;
    a.bres = p.bres;
    a.stack = p.stack;
    a.NS = p.NS;
    a.NA = p.NA;
    a.aCol0 = p.aCol0;
    a.G = p.G;
    a.GB = p.GB;
    a.retain = p.retain;
    a.total_tiles = p.total_tiles;
    // fire iff X * s 2^-23 > theta  <=>  X > floor(theta 2^23 / s)   (X integer, scaling exact)
    // spikes enter the MMA as 128: X is in units of s 2^-30
    a.theta_q = (long long)std::floor((double)theta * (1073741824.0 / scale));
    // digit sums are at most 128 * 255 * K: the 32-bit test needs them below 2^24
    // (and d1*256 + d0 + thC below 2^32)
    a.small_x = ((double)p.K * 32640.0 * 257.0 + 65536.0 < 4294967296.0 && a.theta_q < (1ll << 46)) ? 1 : 0;
    a.thH = (int)(a.theta_q >> 16);
    a.thC = 65535u - (uint32_t)(a.theta_q & 65535);
    a.out_scale = (float)(scale / 1073741824.0);
    static const int prof_env = [] {
        const char* e = std::getenv("SPK_CONV_PROF");
        return e && e[0] == '1' ? 1 : 0;
    }();
    a.prof = prof_env;
    const size_t bstage = (size_t)3 * p.Nt * KS;
    a.b_off = 0;
    a.lc_off = (uint32_t)(p.bres ? p.nks * bstage : p.NS * p.GB * bstage);
    a.kt_off = a.lc_off + 8u * 4u * (KS / 2);
    a.rg_off = (a.kt_off + (uint32_t)((p.kt16 ? 2 : 4) * p.nks * KS) + 15u) & ~15u;
    a.kt16 = p.kt16;
    a.ob_off = (a.rg_off + (uint32_t)(p.nrb * p.rb_stride) + 15u) & ~15u;
    a.bar_off = (a.ob_off + (uint32_t)(kNOB * p.Nt * p.PPT * 5) + 15u) & ~15u;
    const long long grid = p.total_tiles < spk::sm_count() ? p.total_tiles : spk::sm_count();
    if (p.TP == 1) launch_tp<1>(a, epi, out1 != nullptr, (unsigned)grid, p.smem_bytes, s);
    else if (p.TP == 16) launch_tp<16>(a, epi, out1 != nullptr, (unsigned)grid, p.smem_bytes, s);
    else launch_tp<32>(a, epi, out1 != nullptr, (unsigned)grid, p.smem_bytes, s);
    return spk::launched("conv_tc_kernel");
}

// Debug: copy the per-role cycle counters of the last profiled conv (SPK_CONV_PROF=1)
// into host memory [1024][17][2] (u64).  Not part of the public ABI.
extern "C" __attribute__((visibility("default"))) int spk_debug_conv_trace(void* host) {
#ifdef SPK_CONV_TRACE
    return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace));
#else
    (void)host;
    return -1;
#endif
}
extern "C" __attribute__((visibility("default"))) int spk_debug_conv_prof(void* host) {
    return (int)cudaMemcpyFromSymbol(host, g_conv_prof, sizeof(g_conv_prof));
}
