// rank_code.cu — a2: threshold + rank-order coding into T cumulative bins
// (Listing 1 `threshold(data, .01)`, `code(data, T)`).
//
// One CTA per sample.  The exact rank bins are found WITHOUT sorting: every
// positive value gets the unique 64-bit key  (float bits << 32) | ~index , so
// "larger key" == "earlier in (value desc, index asc)" (R-TIE).  A value of
// rank r (number of larger keys) lands in bin floor(r*T/n) (R-BINS), i.e. its
// bin is the number of bin boundaries t = 1..T-1 with r >= R_t = ceil(t*n/T).
// The boundary keys K_t (the key with exactly R_t larger keys) are found by a
// multi-target MSB radix select over the 8 key bytes (histograms in shared
// memory), after which  lat = #{t : key <= K_t}.  Deterministic, exact, one
// read of the sample per radix pass (values staged in shared memory when they
// fit).
#include <cstdlib>

#include "common.cuh"

namespace {

#ifndef SPK_RANK_SMALL_SHIFT
#define SPK_RANK_SMALL_SHIFT 20  // small samples: 2048 buckets (exponent + 3 mantissa bits)
#endif
#ifndef SPK_RANK_SMALL_THREADS
#define SPK_RANK_SMALL_THREADS 512  // C2 front end: 49 -> 31 us against 4096 buckets x 256 threads (profiles/r02_ab_rank_small.txt)
#endif
#ifndef SPK_RANK_RUNS
#define SPK_RANK_RUNS 0  // 1: pass-1 histogram atomics aggregated over runs of equal buckets
#endif
constexpr int kGroup = 16;                    // boundary targets resolved per sweep
constexpr int kStageMax = 40 * 1024;          // values staged in smem up to this many

struct RankSmem {
    unsigned int hist[kGroup][256];
    unsigned long long prefix[kGroup];
    unsigned long long kt[256];               // resolved boundary keys K_t, t = 1..T-1
    unsigned int rem[kGroup];
    int slot[kGroup];
    unsigned long long dpre[kGroup];
    int ndist;
    unsigned int red[32];
    unsigned int n, umin, umax;
};

__device__ __forceinline__ unsigned int thr_bits(float v, float thresh) {
    // threshold (strict, R-STRICT) then keep positives; 0 marks "never fires"
    if (!(v > thresh)) v = 0.0f;
    return v > 0.0f ? __float_as_uint(v) : 0u;
}

__device__ __forceinline__ unsigned int block_sum(unsigned int v, unsigned int* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = (l < (int)(blockDim.x >> 5)) ? red[l] : 0u;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (l == 0) red[0] = v;
    }
    __syncthreads();
    v = red[0];
    __syncthreads();
    return v;
}

template <bool STAGED, int kThreads>
__device__ __forceinline__ void rank_code_body(const float* __restrict__ ys, int N, int T, float thresh, int sort,
                                               uint8_t* __restrict__ out, RankSmem& sm, unsigned int* vals) {

    auto U = [&](int i) -> unsigned int { return STAGED ? vals[i] : thr_bits(__ldg(ys + i), thresh); };

    // pass 0: threshold, count positives, min/max (positive floats order like their bits)
    unsigned int cnt = 0, mn = 0xffffffffu, mx = 0u;
    for (int i = threadIdx.x; i < N; i += kThreads) {
        const unsigned int u = thr_bits(__ldg(ys + i), thresh);
        if (STAGED) vals[i] = u;
        if (u) {
            ++cnt;
            mn = min(mn, u);
            mx = max(mx, u);
        }
    }
    for (int o = 16; o; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (threadIdx.x == 0) {
        sm.umin = 0xffffffffu;
        sm.umax = 0u;
    }
    const unsigned int n = block_sum(cnt, sm.red);  // contains __syncthreads
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&sm.umin, mn);
        atomicMax(&sm.umax, mx);
    }
    __syncthreads();

    if (n == 0) {
        for (int i = threadIdx.x; i < N; i += kThreads) out[i] = (uint8_t)T;
        return;
    }

    if (!sort) {
        // R-SORTOFF: lat = min(T-1, floor(T*(vmax - v)/((vmax - vmin) + ulp(vmax)))), fp32 in this order
        const float vmax = __uint_as_float(sm.umax), vmin = __uint_as_float(sm.umin);
        const float ulp = __fsub_rn(__uint_as_float(sm.umax + 1u), vmax);
        const float den = __fadd_rn(__fsub_rn(vmax, vmin), ulp);
        for (int i = threadIdx.x; i < N; i += kThreads) {
            const unsigned int u = U(i);
            int l = T;
            if (u) {
                const float num = __fmul_rn((float)T, __fsub_rn(vmax, __uint_as_float(u)));
                l = (int)floorf(__fdiv_rn(num, den));
                if (l > T - 1) l = T - 1;
            }
            out[i] = (uint8_t)l;
        }
        return;
    }

    // boundary targets t = 1..T-1 with R_t = ceil(t n / T) < n
    const int ntgt = T - 1;
    for (int g0 = 0; g0 < ntgt; g0 += kGroup) {
        const int gn = min(kGroup, ntgt - g0);
        if (threadIdx.x < gn) {
            const int t = g0 + threadIdx.x + 1;
            const unsigned long long R = ((unsigned long long)t * n + T - 1) / T;
            sm.rem[threadIdx.x] = (unsigned int)R;  // >= n means "no such key"
            sm.prefix[threadIdx.x] = 0ull;
        }
        for (int p = 0; p < 8; ++p) {
            const int shift = 56 - 8 * p;
            __syncthreads();
            if (threadIdx.x == 0) {
                // distinct prefixes of the live targets (targets are in key-descending order)
                int nd = 0;
                for (int q = 0; q < gn; ++q) {
                    if (sm.rem[q] >= n) { sm.slot[q] = -1; continue; }
                    const unsigned long long pre = sm.prefix[q];
                    if (nd == 0 || sm.dpre[nd - 1] != pre) sm.dpre[nd++] = pre;
                    sm.slot[q] = nd - 1;
                }
                sm.ndist = nd;
            }
            __syncthreads();
            const int nd = sm.ndist;
            if (nd == 0) break;
            for (int q = threadIdx.x; q < nd * 256; q += kThreads) (&sm.hist[0][0])[q] = 0u;
            __syncthreads();
            for (int i0 = 0; i0 < N; i0 += kThreads) {
                const int i = i0 + threadIdx.x;
                int s = -1;
                unsigned int dig = 0;
                if (i < N) {
                    const unsigned int u = U(i);
                    if (u) {
                        const unsigned long long key = ((unsigned long long)u << 32) | (0xffffffffu - (unsigned)i);
                        const unsigned long long pre = p ? (key >> (shift + 8)) : 0ull;
                        for (int q = 0; q < nd; ++q)
                            if (sm.dpre[q] == pre) { s = q; break; }
                        dig = (unsigned int)(key >> shift) & 255u;
                    }
                }
                // warp-aggregated shared-memory histogram update
                const unsigned int code = (s < 0) ? 0xffffffffu : ((unsigned)s << 8 | dig);
                const unsigned int peers = __match_any_sync(0xffffffffu, code);
                if (s >= 0 && (__ffs(peers) - 1) == (int)(threadIdx.x & 31))
                    atomicAdd(&sm.hist[s][dig], (unsigned)__popc(peers));
            }
            __syncthreads();
            if (threadIdx.x < gn && sm.slot[threadIdx.x] >= 0) {
                const unsigned int* h = sm.hist[sm.slot[threadIdx.x]];
                unsigned int rem = sm.rem[threadIdx.x], cum = 0;
                int d = 255;
                for (; d > 0; --d) {
                    if (cum + h[d] > rem) break;
                    cum += h[d];
                }
                sm.rem[threadIdx.x] = rem - cum;
                sm.prefix[threadIdx.x] = (sm.prefix[threadIdx.x] << 8) | (unsigned)d;
            }
        }
        __syncthreads();
        if (threadIdx.x < gn) {
            const int t = g0 + threadIdx.x + 1;
            const unsigned long long R = ((unsigned long long)t * n + T - 1) / T;
            sm.kt[t] = (R < n) ? sm.prefix[threadIdx.x] : 0ull;  // key 0 never matches a positive
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += kThreads) {
        const unsigned int u = U(i);
        int l = T;
        if (u) {
            const unsigned long long key = ((unsigned long long)u << 32) | (0xffffffffu - (unsigned)i);
            l = 0;
            for (int t = 1; t < T; ++t) {
                if (key <= sm.kt[t]) l = t;
                else break;  // K_t is non-increasing in t
            }
        }
        out[i] = (uint8_t)l;
    }
}

template <bool STAGED, int kThreads>
__global__ void __launch_bounds__(kThreads) rank_code_kernel(const float* __restrict__ y, int N, int T,
                                                            float thresh, int sort,
                                                            uint8_t* __restrict__ lat) {
    spk_pdl_wait();
    extern __shared__ __align__(16) unsigned char dyn[];
    __shared__ RankSmem sm;
    rank_code_body<STAGED, kThreads>(y + (size_t)blockIdx.x * N, N, T, thresh, sort, lat + (size_t)blockIdx.x * N, sm,
                                     reinterpret_cast<unsigned int*>(dyn));
}

// Small samples (N <= kSortMax), sort mode: the unique keys of the positive values
// are compacted into shared memory and bitonic-sorted descending; the value at
// sorted position r gets bin floor(r T / n) (R-BINS) — the same ranks as the
// radix select, with far fewer passes over shared memory.
constexpr int kSortMax = 8192, kSortThreads = 512;

__global__ void __launch_bounds__(kSortThreads) rank_code_sort_kernel(const float* __restrict__ y, int N, int T,
                                                                      float thresh, uint8_t* __restrict__ lat) {
    spk_pdl_wait();
    extern __shared__ unsigned long long keys[];  // capacity: next power of two >= N
    __shared__ unsigned int s_n;
    const float* ys = y + (size_t)blockIdx.x * N;
    uint8_t* out = lat + (size_t)blockIdx.x * N;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    // compaction (order irrelevant: keys are unique); non-positive values never fire
    for (int i0 = 0; i0 < N; i0 += kSortThreads) {
        const int i = i0 + threadIdx.x;
        const unsigned int u = i < N ? thr_bits(__ldg(ys + i), thresh) : 0u;
        const unsigned int m = __ballot_sync(0xffffffffu, u != 0u);
        unsigned int base = 0;
        if (lane == 0 && m) base = atomicAdd(&s_n, (unsigned)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (u) keys[base + __popc(m & ((1u << lane) - 1u))] = ((unsigned long long)u << 32) | (0xffffffffu - (unsigned)i);
        else if (i < N) out[i] = (uint8_t)T;
    }
    __syncthreads();
    const int n = (int)s_n;
    if (n == 0) return;
    int P = 1;
    while (P < n) P <<= 1;
    for (int q = n + threadIdx.x; q < P; q += kSortThreads) keys[q] = 0ull;  // sorts last
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = threadIdx.x; t < (P >> 1); t += kSortThreads) {
                const int a = ((t & ~(j - 1)) << 1) | (t & (j - 1)), b = a + j;
                const unsigned long long ka = keys[a], kb = keys[b];
                const bool desc = (a & k) == 0;
                if ((ka < kb) == desc) {
                    keys[a] = kb;
                    keys[b] = ka;
                }
            }
            __syncthreads();
        }
    }
    for (int r = threadIdx.x; r < n; r += kSortThreads) {
        const unsigned int idx = 0xffffffffu - (unsigned int)(keys[r] & 0xffffffffull);
        out[idx] = (uint8_t)(((long long)r * T) / n);
    }
}


// Large samples, sort mode (C4, C5: N = 160,000 / 301,056 values per sample): one
// CTA per sample, TWO reads of the sample and no radix passes.
//  pass 1: histogram of the positive values over 32768 buckets = the top 15 bits of
//          the float (exponent + 7 mantissa bits; positive floats order like their
//          bits, so buckets are ordered key ranges of width <= 2^-7 relative).
//  scan:   for every bucket, above = #values in higher buckets, so its values hold
//          ranks [above, above + cnt); when floor(r T / n) is the same at both ends
//          every value of the bucket gets that bin (R-BINS) — all but the <= T-1
//          buckets that straddle a bin boundary.
//  pass 2: values of ordinary buckets are written at once; values of boundary
//          buckets are compacted as unique keys (value bits << 32 | ~index, R-TIE),
//          grouped by bucket, and get rank = above + (number of larger keys in their
//          bucket).  Exactly the ranks of the full sort.
// More boundary-bucket values than fit shared memory (massive exact ties) -> the
// sample falls back to the multi-target radix select above (exact, slower).
constexpr int kMaxBnd = 256, kUnroll = 4;
// Two instantiations: C4/C5 samples (32768 buckets = exponent + 7 mantissa bits, 1024
// threads, values read twice from global memory) and C1-C3 samples (<= 8192 values:
// 2048 buckets = exponent + 3 mantissa bits, 512 threads, values staged in smem).
template <int SHIFT, int kHT, int kCand, bool STAGE>
struct HistCfg {
    static constexpr int kBkt = 1 << (31 - SHIFT);
    static size_t smem(int N) { return (size_t)kBkt * 4 + (size_t)kCand * 8 + (STAGE ? (size_t)N * 4 : 0); }
};

template <int SHIFT, int kHT, int kCand, bool STAGE>
__global__ void __launch_bounds__(kHT) rank_code_hist_kernel(const float* __restrict__ y, int N, int T, float thresh,
                                                            uint8_t* __restrict__ lat) {
    spk_pdl_wait();
    constexpr int kBkt = HistCfg<SHIFT, kHT, kCand, STAGE>::kBkt, kNW = kHT / 32;
    static_assert(kBkt / 2 >= kCand, "the bucket table is reused for the grouped candidates");
    extern __shared__ __align__(16) unsigned char dyn[];
    unsigned int* tab = reinterpret_cast<unsigned int*>(dyn);                         // [kBkt]
    unsigned long long* cand = reinterpret_cast<unsigned long long*>(dyn + (size_t)kBkt * 4);  // [kCand]
    unsigned int* vals = reinterpret_cast<unsigned int*>(dyn + (size_t)kBkt * 4 + (size_t)kCand * 8);  // STAGE: [N]
    __shared__ unsigned int red[32];
    __shared__ unsigned int bnd_b[kMaxBnd], bnd_c[kMaxBnd];
    __shared__ unsigned int s_nbnd, s_ncand, s_n;
    const float* ys = y + (size_t)blockIdx.x * N;
    uint8_t* out = lat + (size_t)blockIdx.x * N;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const bool vec = (N & 3) == 0;  // float4 / uchar4 access (sample bases stay aligned)

    for (int q = tid; q < kBkt; q += kHT) tab[q] = 0u;
    if (tid == 0) {
        s_nbnd = 0;
        s_ncand = 0;
    }
    __syncthreads();
    // pass 1: bucket histogram
    if (vec) {
        const float4* y4 = reinterpret_cast<const float4*>(ys);
        const int n4 = N >> 2;
        for (int q0 = tid; q0 < n4; q0 += kUnroll * kHT) {  // kUnroll 16-byte loads in flight per thread
            float4 v[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const int q = q0 + u * kHT;
                v[u] = q < n4 ? __ldg(y4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                if (q0 + u * kHT >= n4) break;
                const unsigned int u0 = thr_bits(v[u].x, thresh), u1 = thr_bits(v[u].y, thresh),
                                   u2 = thr_bits(v[u].z, thresh), u3 = thr_bits(v[u].w, thresh);
                if (STAGE) reinterpret_cast<uint4*>(vals)[q0 + u * kHT] = make_uint4(u0, u1, u2, u3);
#if SPK_RANK_RUNS
                // neighbouring values usually share a bucket: one atomic per run of equal buckets
                {
                    const unsigned int b0 = u0 ? (u0 >> SHIFT) : 0xFFFFFFFFu, b1 = u1 ? (u1 >> SHIFT) : 0xFFFFFFFFu,
                                       b2 = u2 ? (u2 >> SHIFT) : 0xFFFFFFFFu, b3 = u3 ? (u3 >> SHIFT) : 0xFFFFFFFFu;
                    unsigned int cur = b0, n = u0 ? 1u : 0u;
                    auto push = [&](unsigned int b, bool live) {
                        if (b == cur) {
                            n += live;
                        } else {
                            if (n) atomicAdd(&tab[cur], n);
                            cur = b;
                            n = live;
                        }
                    };
                    push(b1, u1 != 0);
                    push(b2, u2 != 0);
                    push(b3, u3 != 0);
                    if (n) atomicAdd(&tab[cur], n);
                }
#else
                if (u0) atomicAdd(&tab[u0 >> SHIFT], 1u);
                if (u1) atomicAdd(&tab[u1 >> SHIFT], 1u);
                if (u2) atomicAdd(&tab[u2 >> SHIFT], 1u);
                if (u3) atomicAdd(&tab[u3 >> SHIFT], 1u);
#endif
            }
        }
    } else {
        for (int i = tid; i < N; i += kHT) {
            const unsigned int u = thr_bits(__ldg(ys + i), thresh);
            if (STAGE) vals[i] = u;
            if (u) atomicAdd(&tab[u >> SHIFT], 1u);
        }
    }
    __syncthreads();
    // scan from the top bucket down: thread tid owns buckets [kPer tid, kPer tid + kPer)
    constexpr int kPer = kBkt / kHT;
    unsigned int loc = 0;
#pragma unroll 8
    for (int j = 0; j < kPer; ++j) loc += tab[tid * kPer + j];
    // exclusive scan over threads in DEScending tid order: above_start(tid) = sum_{tid' > tid}
    unsigned int incl = loc;  // inclusive suffix within the warp (lanes > lane)
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int v = __shfl_down_sync(0xffffffffu, incl, o);
        if (lane + o < 32) incl += v;
    }
    if (lane == 0) red[wid] = incl;  // warp total
    __syncthreads();
    if (wid == 0) {
        const unsigned int wt = lane < kNW ? red[lane] : 0u;
        unsigned int ws = wt;  // inclusive suffix over warps
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int v = __shfl_down_sync(0xffffffffu, ws, o);
            if (lane + o < 32) ws += v;
        }
        if (lane == 0) s_n = ws;
        __syncwarp();
        red[lane] = ws - wt;  // sum over warps above this one
    }
    __syncthreads();
    const unsigned int n = s_n;
    if (n == 0) {
        for (int i = tid; i < N; i += kHT) out[i] = (uint8_t)T;
        return;
    }
    unsigned int run = red[wid] + (incl - loc);  // values in buckets above this thread's range
    for (int j = kPer - 1; j >= 0; --j) {
        const int B = tid * kPer + j;
        const unsigned int c = tab[B];
        unsigned int tag = 0;
        if (c) {
            const unsigned int lo = (unsigned int)(((unsigned long long)run * T) / n),
                               hi = (unsigned int)(((unsigned long long)(run + c - 1) * T) / n);
            if (lo == hi) {
                tag = lo;
            } else {
                tag = 255;
                const unsigned int slot = atomicAdd(&s_nbnd, 1u);  // <= T-1 < kMaxBnd boundary buckets
                bnd_b[slot] = (unsigned int)B;
                bnd_c[slot] = c;
            }
        }
        tab[B] = run | (tag << 24);
        run += c;
    }
    __syncthreads();
    // pass 2: ordinary buckets are final; boundary-bucket values become candidates
    auto one = [&](unsigned int u, int i) -> unsigned int {
        if (!u) return (unsigned int)T;
        const unsigned int tag = tab[u >> SHIFT] >> 24;
        if (tag != 255u) return tag;
        const unsigned int pos = atomicAdd(&s_ncand, 1u);
        if (pos < (unsigned)kCand) cand[pos] = ((unsigned long long)u << 32) | (0xffffffffu - (unsigned)i);
        return 0u;  // placeholder, rewritten below
    };
    if (STAGE && vec) {
        const uint4* v4 = reinterpret_cast<const uint4*>(vals);
        uchar4* o4 = reinterpret_cast<uchar4*>(out);
        for (int q = tid; q < (N >> 2); q += kHT) {
            const uint4 w = v4[q];
            o4[q] = make_uchar4((uint8_t)one(w.x, 4 * q), (uint8_t)one(w.y, 4 * q + 1), (uint8_t)one(w.z, 4 * q + 2),
                                (uint8_t)one(w.w, 4 * q + 3));
        }
    } else if (STAGE) {
        for (int i = tid; i < N; i += kHT) out[i] = (uint8_t)one(vals[i], i);
    } else if (vec) {
        const float4* y4 = reinterpret_cast<const float4*>(ys);
        uchar4* o4 = reinterpret_cast<uchar4*>(out);
        const int n4 = N >> 2;
        for (int q0 = tid; q0 < n4; q0 += kUnroll * kHT) {
            float4 v[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const int q = q0 + u * kHT;
                v[u] = q < n4 ? __ldg(y4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const int q = q0 + u * kHT;
                if (q < n4) {
                    uchar4 r;
                    r.x = (uint8_t)one(thr_bits(v[u].x, thresh), 4 * q);
                    r.y = (uint8_t)one(thr_bits(v[u].y, thresh), 4 * q + 1);
                    r.z = (uint8_t)one(thr_bits(v[u].z, thresh), 4 * q + 2);
                    r.w = (uint8_t)one(thr_bits(v[u].w, thresh), 4 * q + 3);
                    o4[q] = r;
                }
            }
        }
    } else {
        for (int i = tid; i < N; i += kHT) out[i] = (uint8_t)one(thr_bits(__ldg(ys + i), thresh), i);
    }
    __syncthreads();
    const int nc = (int)s_ncand;
    if (nc > kCand) {  // massive exact ties: exact radix select over the sample (global reads)
        RankSmem& sm = *reinterpret_cast<RankSmem*>(dyn);
        rank_code_body<false, kHT>(ys, N, T, thresh, 1, out, sm, nullptr);
        return;
    }
    // group the candidates by boundary bucket (segments sized by the histogram), then rank
    // each one inside its own bucket by counting the larger keys there — no sort
    __shared__ unsigned int seg_start[kMaxBnd], seg_cur[kMaxBnd], seg_above[kMaxBnd];
    const int nb = (int)s_nbnd;
    if (tid == 0) {
        unsigned int acc = 0;
        for (int q = 0; q < nb; ++q) {
            seg_start[q] = acc;
            seg_cur[q] = 0;
            seg_above[q] = tab[bnd_b[q]] & 0xffffffu;  // values in higher buckets
            acc += bnd_c[q];
        }
    }
    __syncthreads();
    // the bucket table is no longer read: its space holds the grouped keys
    unsigned long long* grp = reinterpret_cast<unsigned long long*>(tab);
    for (int j = tid; j < nc; j += kHT) {
        const unsigned long long key = cand[j];
        const unsigned int B = (unsigned int)(key >> 32) >> SHIFT;
        int q = 0;
        while (bnd_b[q] != B) ++q;  // its boundary bucket (one of <= T-1)
        grp[seg_start[q] + atomicAdd(&seg_cur[q], 1u)] = key;
    }
    __syncthreads();
    for (int j = tid; j < nc; j += kHT) {
        const unsigned long long key = grp[j];
        const unsigned int B = (unsigned int)(key >> 32) >> SHIFT;
        int q = 0;
        while (bnd_b[q] != B) ++q;
        const unsigned int s0 = seg_start[q], s1 = s0 + bnd_c[q];
        unsigned int larger = 0;
        for (unsigned int e = s0; e < s1; ++e) larger += grp[e] > key;
        const unsigned int idx = 0xffffffffu - (unsigned int)(key & 0xffffffffull);
        const unsigned int rank = seg_above[q] + larger;
        out[idx] = (uint8_t)(((unsigned long long)rank * T) / n);
    }
}

}  // namespace

extern "C" size_t spk_rank_code_workspace(int, int, int, int) { return 0; }

extern "C" spk_status spk_rank_code(const float* y, int B, int N, int T, float thresh, int sort,
                                    uint8_t* lat, void* ws, size_t ws_bytes, spk_stream stream) {
    spk::clear_error();
    (void)ws;
    (void)ws_bytes;
    SPK_CHECK_PTR(y);
    SPK_CHECK_PTR(lat);
    SPK_CHECK(B >= 1 && N >= 1, SPK_ERR_SHAPE, "B=%d N=%d", B, N);
    SPK_CHECK(N <= (1 << 24), SPK_ERR_UNSUPPORTED, "N=%d > 2^24", N);
    SPK_CHECK(T >= 1, SPK_ERR_ARG, "T=%d < 1", T);
    SPK_CHECK(T <= 254, SPK_ERR_UNSUPPORTED, "T=%d > 254 (u8 latency)", T);
    SPK_CHECK(B <= 0x7fffffff, SPK_ERR_SHAPE, "B too large");
    cudaStream_t s = spk::as_cuda(stream);
    static const int old_sort = [] {
        const char* e = std::getenv("SPK_RANK_SORT");  // A/B knob: 1 = bitonic sort kernel for small samples
        return e ? std::atoi(e) : 0;
    }();
    if (sort && N <= kSortMax && !old_sort) {  // small samples: staged values, 2048-bucket histogram
        constexpr int SH = SPK_RANK_SMALL_SHIFT, TH = SPK_RANK_SMALL_THREADS;
        using Cfg = HistCfg<SH, TH, 1024, true>;
        static std::atomic<uint64_t> attr{0};
        if (spk::first_on_device(attr)) {
            cudaFuncSetAttribute(rank_code_hist_kernel<SH, TH, 1024, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::smem(kSortMax));
        }
        spk::launch(rank_code_hist_kernel<SH, TH, 1024, true>, B, TH, Cfg::smem(N), s, y, N, T, thresh, lat);
        return spk::launched("rank_code_hist_kernel<small>");
    }
    if (sort && N <= kSortMax) {
        int cap = 1;
        while (cap < N) cap <<= 1;
        const size_t smem = sizeof(unsigned long long) * (size_t)cap;
        static std::atomic<uint64_t> attr{0};
        if (spk::first_on_device(attr)) {
            cudaFuncSetAttribute(rank_code_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sizeof(unsigned long long) * kSortMax));
        }
        spk::launch(rank_code_sort_kernel, B, kSortThreads, smem, s, y, N, T, thresh, lat);
        return spk::launched("rank_code_sort_kernel");
    }
    if (sort) {  // larger samples: bucket histogram + boundary-bucket sort
        // 16384 buckets (exponent + 6 mantissa bits) and 4096 candidates: 96 KB, two CTAs per
        // SM (C5 samples have 2-3K boundary-bucket values; more falls back to the radix select)
        using Cfg = HistCfg<17, 1024, 4096, false>;
        static std::atomic<uint64_t> attr{0};
        if (spk::first_on_device(attr)) {
            cudaFuncSetAttribute(rank_code_hist_kernel<17, 1024, 4096, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::smem(0));
        }
        spk::launch(rank_code_hist_kernel<17, 1024, 4096, false>, B, 1024, Cfg::smem(0), s, y, N, T, thresh, lat);
        return spk::launched("rank_code_hist_kernel");
    }
    if (N <= 8192) {  // small samples: 256-thread CTAs, several resident per SM
        const size_t smem = sizeof(unsigned int) * (size_t)N;
        static std::atomic<uint64_t> attr{0};  // up to 32 KB of staged values next to the static RankSmem
        if (spk::first_on_device(attr)) {
            cudaFuncSetAttribute(rank_code_kernel<true, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sizeof(unsigned int) * 8192));
        }
        spk::launch(rank_code_kernel<true, 256>, B, 256, smem, s, y, N, T, thresh, sort, lat);
        return spk::launched("rank_code_kernel<staged,256>");
    }
    if (N <= kStageMax) {
        const size_t smem = sizeof(unsigned int) * (size_t)N;
        static std::atomic<uint64_t> attr{0};
        if (spk::first_on_device(attr)) {
            cudaFuncSetAttribute(rank_code_kernel<true, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sizeof(unsigned int) * kStageMax));
        }
        spk::launch(rank_code_kernel<true, 1024>, B, 1024, smem, s, y, N, T, thresh, sort, lat);
        return spk::launched("rank_code_kernel<staged,1024>");
    }
    spk::launch(rank_code_kernel<false, 1024>, B, 1024, 0, s, y, N, T, thresh, sort, lat);
    return spk::launched("rank_code_kernel<global,1024>");
}
