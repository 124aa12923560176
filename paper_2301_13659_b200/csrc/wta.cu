// wta.cu — a7: convolutional k-winners-take-all (convwta(array, radius, count)).
//
// Every live neuron (lat < T) carries the unique 64-bit key
//   lat (8 bits) | ~order(P*) (32 bits) | flat (c,y,x) index (24 bits)
// so "earliest, then higher potential, then lower index" is a plain unsigned
// minimum.  Greedy rounds pick the least key that no earlier winner suppresses
// (its whole channel + the |dy|,|dx| <= radius square in every channel,
// R-WTA-FOOTPRINT).
//
// One thread-block CLUSTER per sample (1..8 CTAs, grid = CS x B).  CTA r of the
// cluster owns the pixel slice [r HW/CS, (r+1) HW/CS) of every channel:
//  phase 1 (one HBM pass over the records): its slice's candidate keys are
//    compacted into shared memory.  When the slice is too large to keep every
//    live key, each pixel keeps only its min(k, C) least keys — EXACT: a winner
//    at pixel (y,x) suppresses that pixel in every channel, so before it is picked
//    every smaller key at (y,x) must be dead by CHANNEL suppression, and at most
//    k-1 channels are dead; hence every winner is among the k least keys of its
//    pixel, and the greedy minimum over the reduced set equals the one over all
//    live neurons at every round.
//  phase 2 (k rounds, on chip): each CTA takes the least unsuppressed key of its
//    slice (warp shuffles + smem), the cluster's minimum is read through
//    distributed shared memory (one cluster barrier per round, parity-buffered
//    slots), and every CTA appends the same winner.
// A slice whose candidates overflow the shared buffer re-reads its records from
// HBM each round (exact, slow; not hit by C1-C4).
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 256;
constexpr int kMaxK = 64;
constexpr int kMaxCS = 8;
constexpr int kCapKeys = 12288;  // 96 KB of keys per CTA

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) {
    return a < b ? a : b;
}

__device__ __forceinline__ unsigned long long wta_key(const uint8_t* L, const float* P, int i, int T) {
    const int l = __ldg(L + i);
    if (l >= T) return ~0ull;
    const unsigned int po = ~spk_float_order_u32(__ldg(P + i));  // higher potential first
    return ((unsigned long long)l << 56) | ((unsigned long long)po << 24) | (unsigned long long)i;
}

struct WtaArgs {
    const uint8_t* lat;
    const float* pstar;
    int C, H, W, T, k, radius, cs;
    int mode;  // 0: emit every live key of the slice, 1: per-pixel top-KK, 2: overflow (re-read)
    unsigned cap;  // keys the shared buffer holds
    spk_winner* win;
    int32_t* nwin;
};

// KK = per-pixel keep count (>= min(k, C)) for mode 1
template <int KK>
__global__ void __launch_bounds__(kThreads) wta_cluster_kernel(const WtaArgs a) {
    spk_pdl_wait();
    constexpr int kChan = KK >= 4 ? 16 : 8;  // channels read per batch in the per-pixel pre-reduction
    extern __shared__ unsigned long long keys[];  // [kCapKeys]
    __shared__ unsigned long long red[kThreads / 32];
    __shared__ unsigned long long cmin[2];
    __shared__ int pc[kMaxK], py[kMaxK], px[kMaxK];
    __shared__ unsigned int nkeys;
    __shared__ int overflow;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int b = blockIdx.y;
    const int HW = a.H * a.W, N = a.C * HW, T = a.T;
    const int lane = threadIdx.x & 31;
    const uint8_t* L = a.lat + (size_t)b * N;
    const float* P = a.pstar + (size_t)b * N;
    int p_lo = (int)((long long)HW * rank / a.cs), p_hi = (int)((long long)HW * (rank + 1) / a.cs);
    if (a.mode == 4) {  // 4-pixel aligned slices (HW % 4 == 0)
        p_lo = (int)((long long)(HW >> 2) * rank / a.cs) * 4;
        p_hi = (int)((long long)(HW >> 2) * (rank + 1) / a.cs) * 4;
    }
    const int np_slice = p_hi - p_lo;
    if (threadIdx.x == 0) {
        nkeys = 0;
        overflow = a.mode == 2;
    }
    __syncthreads();

    auto emit = [&](unsigned long long key, bool valid) {
        const unsigned m = __ballot_sync(0xffffffffu, valid);
        unsigned base = 0;
        if (lane == 0 && m) base = atomicAdd(&nkeys, (unsigned)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        const unsigned pos = base + __popc(m & ((1u << lane) - 1u));
        if (valid) {
            if (pos < a.cap) keys[pos] = key;
            else overflow = 1;
        }
    };

    if (a.mode == 0) {
        const int n = a.C * np_slice;
        for (int q0 = 0; q0 < n; q0 += kThreads) {
            const int q = q0 + threadIdx.x;
            unsigned long long key = ~0ull;
            if (q < n) {
                const int c = q / np_slice, p = p_lo + (q - c * np_slice);
                key = wta_key(L, P, c * HW + p, T);
            }
            emit(key, key != ~0ull);
        }
    } else if (a.mode == 4) {
        // fused inhibition on a large slice, 4 pixels per thread: the latencies of 4 neighbouring
        // pixels of a channel are one 4-byte load (8 channels in flight), P* is read as one float4
        // only when one of them fired; the per-pixel minimum key is the inhibition survivor
        const int q_lo = p_lo >> 2, q_hi = p_hi >> 2;  // slices are 4-pixel aligned in this mode
        constexpr int kC4 = 8;
        const int iters = (q_hi - q_lo + kThreads - 1) / kThreads;  // the same count in every thread (emit)
        for (int it = 0; it < iters; ++it) {
            const int q = q_lo + it * kThreads + (int)threadIdx.x;
            unsigned long long best[4] = {~0ull, ~0ull, ~0ull, ~0ull};
            const bool qv = q < q_hi;
            if (qv) {
                int c = 0;
                for (; c < a.C; c += kC4) {
                    uint32_t w[kC4];
#pragma unroll
                    for (int u = 0; u < kC4; ++u)
                        w[u] = (c + u < a.C) ? __ldg(reinterpret_cast<const uint32_t*>(L + (size_t)(c + u) * HW) + q)
                                             : 0xFFFFFFFFu;
#pragma unroll
                    for (int u = 0; u < kC4; ++u) {
                        const uint32_t lw = w[u];
                        const bool any = ((lw & 0xFFu) < (uint32_t)T) || (((lw >> 8) & 0xFFu) < (uint32_t)T) ||
                                         (((lw >> 16) & 0xFFu) < (uint32_t)T) || ((lw >> 24) < (uint32_t)T);
                        if (!any) continue;
                        const int i0 = (c + u) * HW + 4 * q;
                        const float4 pv = __ldg(reinterpret_cast<const float4*>(P + i0));
                        const float pe[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const uint32_t l = (lw >> (8 * e)) & 0xFFu;
                            if (l < (uint32_t)T) {
                                const unsigned long long key = ((unsigned long long)l << 56) |
                                                               ((unsigned long long)(~spk_float_order_u32(pe[e])) << 24) |
                                                               (unsigned long long)(i0 + e);
                                best[e] = umin64(best[e], key);
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) emit(best[e], best[e] != ~0ull);
        }
    } else if (a.mode == 3) {
        // fused inhibition on a small slice (C2 layer 3: 16 pixels x 200 maps): the per-pixel
        // minimum key (the inhibition survivor) with channel groups in parallel — thread q takes
        // pixel q % np and channels q / np, q / np + ng, ... — combined by a shared 64-bit atomicMin
        for (int q = threadIdx.x; q < np_slice; q += kThreads) keys[q] = ~0ull;
        __syncthreads();
        const int ng = kThreads / np_slice;
        const int pp = threadIdx.x % np_slice, gq = threadIdx.x / np_slice;
        if (gq < ng) {
            // four channels per trip: their latency loads, then the P* loads of those that fired,
            // are in flight together instead of two dependent loads per channel
            unsigned long long m = ~0ull;
            const int i0 = p_lo + pp;
            for (int c0 = gq; c0 < a.C; c0 += 4 * ng) {
                int l[4];
                float pv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int c = c0 + u * ng;
                    l[u] = c < a.C ? (int)__ldg(L + c * HW + i0) : T;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) pv[u] = l[u] < T ? __ldg(P + (c0 + u * ng) * HW + i0) : 0.0f;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (l[u] >= T) continue;
                    const unsigned int po = ~spk_float_order_u32(pv[u]);  // higher potential first
                    m = umin64(m, ((unsigned long long)l[u] << 56) | ((unsigned long long)po << 24) |
                                      (unsigned long long)((c0 + u * ng) * HW + i0));
                }
            }
            if (m != ~0ull) atomicMin(&keys[pp], m);
        }
        __syncthreads();
        const unsigned long long key = threadIdx.x < np_slice ? keys[threadIdx.x] : ~0ull;
        __syncthreads();
        emit(key, key != ~0ull);  // np_slice <= kThreads / 2: one pass compacts every survivor
    } else if (a.mode == 1) {
        for (int q0 = 0; q0 < np_slice; q0 += kThreads) {
            const int p = p_lo + q0 + threadIdx.x;
            unsigned long long top[KK];
#pragma unroll
            for (int j = 0; j < KK; ++j) top[j] = ~0ull;
            if (p < p_hi) {
                int c = 0;
                for (; c + kChan <= a.C; c += kChan) {  // kChan independent loads in flight
                    int l[kChan];
#pragma unroll
                    for (int u = 0; u < kChan; ++u) l[u] = __ldg(L + (size_t)(c + u) * HW + p);
#pragma unroll
                    for (int u = 0; u < kChan; ++u) {
                        if (l[u] < T) {
                            const int i = (c + u) * HW + p;
                            unsigned long long key = ((unsigned long long)l[u] << 56) |
                                                     ((unsigned long long)(~spk_float_order_u32(__ldg(P + i))) << 24) |
                                                     (unsigned long long)i;
#pragma unroll
                            for (int j = 0; j < KK; ++j) {  // sorted insertion, registers only
                                const unsigned long long lo = umin64(top[j], key);
                                key = top[j] < key ? key : top[j];
                                top[j] = lo;
                            }
                        }
                    }
                }
                for (; c < a.C; ++c) {
                    unsigned long long key = wta_key(L, P, c * HW + p, T);
                    if (key != ~0ull) {
#pragma unroll
                        for (int j = 0; j < KK; ++j) {
                            const unsigned long long lo = umin64(top[j], key);
                            key = top[j] < key ? key : top[j];
                            top[j] = lo;
                        }
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < KK; ++j) emit(top[j], top[j] != ~0ull);
        }
    }
    __syncthreads();
    const bool cached = !overflow;
    const int nl = cached ? (int)nkeys : 0;

    if (a.cs == 1 && cached && nl <= 32) {
        // few candidates (C2 layer 3 after inhibition: <= 16 per sample): one warp runs every
        // round with shuffles — each lane holds one key and drops it when a pick suppresses it
        if (threadIdx.x >= 32) return;
        const unsigned long long key = lane < nl ? keys[lane] : ~0ull;
        const int i = (int)(key & 0xffffffull);
        const int c = i / HW, r = i - c * HW, y = r / a.W, x = r - y * a.W;
        bool alive = key != ~0ull;
        int np = 0;
        for (int round = 0; round < a.k; ++round) {
            unsigned long long best = alive ? key : ~0ull;
            for (int o = 16; o; o >>= 1) best = umin64(best, __shfl_xor_sync(0xffffffffu, best, o));
            if (best == ~0ull) break;
            const int wi = (int)(best & 0xffffffull);
            const int wc = wi / HW, wr = wi - wc * HW, wy = wr / a.W, wx = wr - wy * a.W;
            if (lane == 0) a.win[(size_t)b * a.k + round] = spk_winner{b, (int)(best >> 56), wc, wy, wx, 0};
            if (c == wc || (abs(y - wy) <= a.radius && abs(x - wx) <= a.radius)) alive = false;
            ++np;
        }
        if (lane == 0) {
            for (int q = np; q < a.k; ++q) a.win[(size_t)b * a.k + q] = spk_winner{-1, -1, -1, -1, -1, -1};
            a.nwin[b] = np;
        }
        return;
    }
    int npicked = 0;
    for (int round = 0; round < a.k; ++round) {
        unsigned long long best = ~0ull;
        auto consider = [&](unsigned long long key) {
            const int i = (int)(key & 0xffffffull);
            const int c = i / HW, r = i - c * HW, y = r / a.W, x = r - y * a.W;
            for (int t = 0; t < npicked; ++t)
                if (pc[t] == c || (abs(py[t] - y) <= a.radius && abs(px[t] - x) <= a.radius)) return;
            best = umin64(best, key);
        };
        if (cached) {
            for (int q = threadIdx.x; q < nl; q += kThreads) consider(keys[q]);
        } else {
            const int n = a.C * np_slice;
            for (int q = threadIdx.x; q < n; q += kThreads) {
                const int c = q / np_slice, p = p_lo + (q - c * np_slice);
                const unsigned long long key = wta_key(L, P, c * HW + p, T);
                if (key != ~0ull) consider(key);
            }
        }
        for (int o = 16; o; o >>= 1) best = umin64(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) red[threadIdx.x >> 5] = best;
        __syncthreads();
        if (threadIdx.x < 32) {
            best = lane < kThreads / 32 ? red[lane] : ~0ull;
            for (int o = 16; o; o >>= 1) best = umin64(best, __shfl_xor_sync(0xffffffffu, best, o));
            if (lane == 0) cmin[round & 1] = best;
        }
        cluster.sync();  // every CTA's slice minimum of this round is visible
        if (threadIdx.x == 0) {
            unsigned long long g = ~0ull;
            for (int r = 0; r < a.cs; ++r) g = umin64(g, *cluster.map_shared_rank(&cmin[round & 1], r));
            red[0] = g;
        }
        __syncthreads();
        const unsigned long long g = red[0];
        if (g == ~0ull) break;  // nothing live and unsuppressed anywhere in the sample
        const int i = (int)(g & 0xffffffull);
        const int c = i / HW, r = i - c * HW, y = r / a.W, x = r - y * a.W;
        if (threadIdx.x == 0) {
            pc[npicked] = c;
            py[npicked] = y;
            px[npicked] = x;
            if (rank == 0) a.win[(size_t)b * a.k + round] = spk_winner{b, (int)(g >> 56), c, y, x, 0};
        }
        ++npicked;
        __syncthreads();
    }
    if (rank == 0 && threadIdx.x == 0) {
        for (int r = npicked; r < a.k; ++r) a.win[(size_t)b * a.k + r] = spk_winner{-1, -1, -1, -1, -1, -1};
        a.nwin[b] = npicked;
    }
    // no CTA may exit while a peer can still read its cmin slot
    cluster.sync();
}

template <int KK>
spk_status launch_wta(const WtaArgs& a, int B, size_t cap, cudaStream_t s) {
    auto kern = wta_cluster_kernel<KK>;
    const size_t smem = cap * 8;  // shared key buffer sized to the slice's candidate bound
    static std::atomic<uint64_t> attr{0};
    if (spk::first_on_device(attr)) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kCapKeys * 8) != cudaSuccess)
            return spk::launched("wta_cluster_kernel(attr)");
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)a.cs, (unsigned)B, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)a.cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see spk::launch
    at[1].val.programmaticStreamSerializationAllowed = spk::pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, kern, a);
    return spk::launched("wta_cluster_kernel");
}

}  // namespace

static spk_status wta_impl(const uint8_t* lat, const float* pstar, int B, int C, int H, int W, int T, int k,
                           int radius, spk_winner* win, int32_t* nwin, spk_stream stream, bool inhibit);

extern "C" spk_status spk_wta(const uint8_t* lat, const float* pstar, int B, int C, int H, int W, int T,
                              int k, int radius, spk_winner* win, int32_t* nwin, spk_stream stream) {
    return wta_impl(lat, pstar, B, C, H, W, T, k, radius, win, nwin, stream, false);
}

// Lateral inhibition fused into the k-WTA (Listing 3 inhibit -> convwta on the trained layer):
// the inhibition survivor of a pixel is its least (lat, P*, c) key (R-INHIBIT-TIE), which is
// also its least WTA key, so keeping exactly the per-pixel minimum in phase 1 and running the
// rounds on those keys gives the winners of spk_wta(spk_inhibit(records)) — in one read of the
// records, without writing the inhibited map.
extern "C" spk_status spk_inhibit_wta(const uint8_t* lat, const float* pstar, int B, int C, int H, int W, int T,
                                      int k, int radius, spk_winner* win, int32_t* nwin, spk_stream stream) {
    return wta_impl(lat, pstar, B, C, H, W, T, k, radius, win, nwin, stream, true);
}

static spk_status wta_impl(const uint8_t* lat, const float* pstar, int B, int C, int H, int W, int T, int k,
                           int radius, spk_winner* win, int32_t* nwin, spk_stream stream, bool inhibit) {
    spk::clear_error();
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(pstar);
    SPK_CHECK_PTR(win);
    SPK_CHECK_PTR(nwin);
    SPK_CHECK(B >= 1 && C >= 1 && H >= 1 && W >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK((long long)C * H * W <= (1 << 24), SPK_ERR_UNSUPPORTED, "C*H*W > 2^24 per sample");
    SPK_CHECK(B <= 65535, SPK_ERR_UNSUPPORTED, "B=%d > 65535", B);
    SPK_CHECK(T >= 1 && T <= 254, SPK_ERR_UNSUPPORTED, "T=%d outside 1..254", T);
    SPK_CHECK(k >= 1 && k <= kMaxK, SPK_ERR_ARG, "k=%d outside 1..%d", k, kMaxK);
    SPK_CHECK(radius >= 0, SPK_ERR_ARG, "radius < 0");
    WtaArgs a{lat, pstar, C, H, W, T, k, radius, 1, 0, 0u, win, nwin};
    const long long N = (long long)C * H * W, HW = (long long)H * W;
    // cluster size: about 16K neurons per CTA, at most 8 CTAs and at most one pixel... per CTA
    long long cs = std::min<long long>(kMaxCS, (N + 16383) / 16384);
    // a few samples (C1: one) leave the GPU idle: widen the cluster so phase 1's HBM pass is
    // spread over up to 8 SMs (about 2K neurons per CTA)
    if ((long long)B * cs < 148) cs = std::max(cs, std::min<long long>(kMaxCS, (N + 2047) / 2048));
    a.cs = (int)std::min<long long>(cs, HW);
    if (a.cs < 1) a.cs = 1;
    const long long slice_n = C * ((HW + a.cs - 1) / a.cs);
    const int keep = std::min(k, C);
    int KK = 1;
    while (KK < keep) KK <<= 1;
    const long long slice_p = (HW + a.cs - 1) / a.cs;
    long long cap = 1;
    if (inhibit) {  // per-pixel minimum only (the inhibition survivor)
        SPK_CHECK(slice_p <= kCapKeys, SPK_ERR_UNSUPPORTED,
                  "fused inhibit+WTA needs <= %d pixels per CTA slice (H*W=%lld); call spk_inhibit + spk_wta",
                  kCapKeys, HW);
        const bool vec4 = (HW & 3) == 0 && (reinterpret_cast<uintptr_t>(lat) & 3) == 0 &&
                          (reinterpret_cast<uintptr_t>(pstar) & 15) == 0;
        // small slices: channel groups in parallel; large ones: 4 pixels per thread when aligned
        const long long q_slice = ((HW >> 2) + a.cs - 1) / a.cs;
        a.mode = slice_p * 2 <= kThreads ? 3 : (vec4 && q_slice * 4 <= kCapKeys) ? 4 : 1;
        if (a.mode == 4) {
            a.cap = (unsigned)(q_slice * 4);
            return launch_wta<1>(a, B, (size_t)(q_slice * 4), spk::as_cuda(stream));
        }
        a.cap = (unsigned)slice_p;
        return launch_wta<1>(a, B, (size_t)slice_p, spk::as_cuda(stream));
    }
    if (slice_n <= kCapKeys) a.mode = 0, cap = slice_n;
    else if (KK <= 16 && slice_p * KK <= kCapKeys) a.mode = 1, cap = slice_p * KK;
    else a.mode = 2;
    a.cap = (unsigned)cap;
    const cudaStream_t s = spk::as_cuda(stream);
    if (a.mode != 1) return launch_wta<1>(a, B, (size_t)cap, s);
    switch (KK) {
        case 1: return launch_wta<1>(a, B, (size_t)cap, s);
        case 2: return launch_wta<2>(a, B, (size_t)cap, s);
        case 4: return launch_wta<4>(a, B, (size_t)cap, s);
        case 8: return launch_wta<8>(a, B, (size_t)cap, s);
        default: return launch_wta<16>(a, B, (size_t)cap, s);
    }
}
