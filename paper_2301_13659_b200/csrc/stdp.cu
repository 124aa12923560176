// stdp.cu — a8: STDP / R-STDP weight update of a conv layer (Eq. 4-6).
//
// Winners are applied in (sample asc, pick order) (R-BATCH: "the batch update
// rule does not differ from single-sample processing").  A weight
// W[o][c][i][j] is touched only by winners of map o, and its update depends
// only on itself, so the sequential semantics are kept exactly by
//   (1) bucketing winners per output map with a stable block compaction
//       (one CTA per map), then
//   (2) one thread per weight element walking its map's winners in order.
// The per-weight arithmetic is fp32 in the order of Eq. 4-6 with explicit
// round-to-nearest intrinsics (no contraction): bit-identical to the oracle.
#include <cstdlib>

#include "common.cuh"

namespace {

constexpr int kMaxCfg = 8;
struct Cfgs {
    spk_stdp_config c[kMaxCfg];
};

// Bucketing: slotmap[s] = map of winner slot s (b*k + q) if it is a valid winner,
// else -1; then one CTA per map collects its slots in slot order with a single
// block-wide exclusive scan per pass (each thread owns a contiguous run of slots).
__device__ __forceinline__ bool winner_valid(const spk_winner& w, int B, int ncfg, int Ho, int Wo, int Co) {
    return w.c >= 0 && w.c < Co && w.cfg >= 0 && w.cfg < ncfg && w.y >= 0 && w.y < Ho && w.x >= 0 && w.x < Wo &&
           w.b >= 0 && w.b < B;
}

__global__ void stdp_slotmap_kernel(const spk_winner* __restrict__ win, const int32_t* __restrict__ nwin, int B,
                                    int k, int ncfg, int Ho, int Wo, int Co, int32_t* __restrict__ slotmap,
                                    int32_t* __restrict__ invalid) {
    spk_pdl_wait();
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= B * k) return;
    const int b = s / k, q = s - b * k;
    int m = -1;
    if (q < min(nwin[b], k)) {
        const spk_winner w = win[s];
        if (winner_valid(w, B, ncfg, Ho, Wo, Co)) m = w.c;
        else atomicAdd(invalid, 1);  // out-of-range coordinate or config: skipped, counted
    }
    slotmap[s] = m;
}

constexpr int kBucketThreads = 1024, kBucketRun = 16;  // slots per thread per pass

__global__ void __launch_bounds__(kBucketThreads) stdp_bucket_kernel(const int32_t* __restrict__ slotmap, int S,
                                                                    int cap, int32_t* __restrict__ list,
                                                                    int32_t* __restrict__ start,
                                                                    int32_t* __restrict__ cnt) {
    spk_pdl_wait();
    constexpr int kWarps = kBucketThreads / 32;
    __shared__ int wsum[kWarps];
    const int o = blockIdx.x;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    int total = 0;
    for (int p0 = 0; p0 < S; p0 += kBucketThreads * kBucketRun) {
        const int s0 = p0 + threadIdx.x * kBucketRun;
        int v[kBucketRun];
        int mine = 0;
#pragma unroll
        for (int u = 0; u < kBucketRun; ++u) {
            v[u] = (s0 + u < S) ? slotmap[s0 + u] : -1;
            mine += (v[u] == o);
        }
        // block exclusive scan of `mine`
        int incl = mine;
        for (int d = 1; d < 32; d <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += t;
        }
        if (lane == 31) wsum[wp] = incl;
        __syncthreads();
        int before = 0, chunk = 0;
        for (int q = 0; q < kWarps; ++q) {
            const int x = wsum[q];
            before += (q < wp) ? x : 0;
            chunk += x;
        }
        int pos = total + before + incl - mine;
#pragma unroll
        for (int u = 0; u < kBucketRun; ++u)
            if (v[u] == o) {
                if (pos < cap) list[(size_t)o * cap + pos] = s0 + u;
                ++pos;
            }
        total += chunk;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        cnt[o] = min(total, cap);
        start[o] = o * cap;
    }
}

// Grid (K chunks of kUpdW weights, Co).  Per chunk of up to kWinChunk winners of
// map o (in order): phase 1 — all threads, one (winner, weight) pair each —
// gathers the pre-synaptic latency and stores the Eq. 4 case (t_j <= t_i) as a
// byte; phase 2 — one thread per weight — runs the sequential fp32 chain of
// Eq. 4-6 from shared memory only.  The gathers are thus fully parallel and the
// order-dependent part is a few dependent flops per winner.
// kUpdW weights per CTA: 32 when maps collect many winners (C2 layer 3: ~41 per map, the ordered
// chain dominates), 128 when they collect few (C3 decision layer: the gathers dominate) —
// profiles/r02_ab_stdp_width.txt
constexpr int kWinChunk = 256;
#ifndef SPK_STDP_T32
#define SPK_STDP_T32 256  // threads per CTA of the 32-weight tile
#endif

template <int kUpdW, int kUpdThreads>
__global__ void __launch_bounds__(kUpdThreads) stdp_update_kernel(float* __restrict__ w, spk_conv_geom g,
                                                                  const uint8_t* __restrict__ lat_in,
                                                                  const spk_winner* __restrict__ win,
                                                                  const int32_t* __restrict__ list,
                                                                  const int32_t* __restrict__ start,
                                                                  const int32_t* __restrict__ cnt,
                                                                  const Cfgs cfgs, int ncfg) {
    spk_pdl_wait();
    __shared__ long long s_ofs[kWinChunk];  // lat_in offset of (b, channel 0, y0, x0)
    __shared__ int s_y0[kWinChunk], s_x0[kWinChunk], s_t[kWinChunk];
    __shared__ float s_ap[kWinChunk], s_am[kWinChunk], s_lo[kWinChunk], s_hi[kWinChunk];  // winner's config
    __shared__ uint8_t s_st[kWinChunk];
    __shared__ uint8_t s_le[kWinChunk][kUpdW];  // [winner][weight]: t_j <= t_i
    __shared__ spk_stdp_config s_cf[kMaxCfg];
    const int o = blockIdx.y;
    const int n = cnt[o];
    if (n == 0) return;
    const int K = g.Ci * g.Kh * g.Kw;
    const int KhKw = g.Kh * g.Kw;
    const long long HW = (long long)g.Hi * g.Wi;
    const int k0 = blockIdx.x * kUpdW;
    // phase-1 role: weight lane wl of this CTA's chunk (fixed per thread)
    const int wl = threadIdx.x & (kUpdW - 1), e_lane = threadIdx.x / kUpdW;
    const int kk1 = k0 + wl;
    const bool valid1 = kk1 < K;
    const int c1 = kk1 / KhKw, r1 = kk1 - c1 * KhKw, i1 = r1 / g.Kw, j1 = r1 - i1 * g.Kw;
    const long long own1 = c1 * HW + (long long)i1 * g.Wi + j1;
#pragma unroll
    for (int q = 0; q < kMaxCfg; ++q)  // static indices: the parameter block stays in constant space
        if (threadIdx.x == q && q < ncfg) s_cf[q] = cfgs.c[q];
    // phase-2 role (threads < kUpdW): the weight kk2 = k0 + threadIdx.x
    const int kk2 = k0 + threadIdx.x;
    const bool valid2 = threadIdx.x < kUpdW && kk2 < K;
    float W = valid2 ? w[(size_t)o * K + kk2] : 0.0f;
    for (int e0 = 0; e0 < n; e0 += kWinChunk) {
        const int m = min(kWinChunk, n - e0);
        __syncthreads();
        for (int q = threadIdx.x; q < m; q += kUpdThreads) {
            const spk_winner wn = win[list[(size_t)start[o] + e0 + q]];
            const int y0 = wn.y * g.Sh - g.Ph, x0 = wn.x * g.Sw - g.Pw;
            s_ofs[q] = (long long)wn.b * g.Ci * HW + (long long)y0 * g.Wi + x0;
            s_y0[q] = y0;
            s_x0[q] = x0;
            s_t[q] = wn.t;
            const spk_stdp_config cf = s_cf[wn.cfg];
            s_ap[q] = cf.a_plus;
            s_am[q] = cf.a_minus;
            s_lo[q] = cf.lower;
            s_hi[q] = cf.upper;
            s_st[q] = cf.stabilize != 0;
        }
        __syncthreads();
        // phase 1: gathers, kUpdThreads / kUpdW winners per pass, several passes in flight
        if (valid1) {
            constexpr int kStep = kUpdThreads / kUpdW, kBatch = 32;  // kBatch independent loads in flight
            for (int e0b = e_lane; e0b < m; e0b += kStep * kBatch) {
                int tj[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int e = e0b + u * kStep;
                    tj[u] = 0x7fffffff;  // padded input: never fires (R-NEVER)
                    if (e < m) {
                        const int iy = s_y0[e] + i1, ix = s_x0[e] + j1;
                        if ((unsigned)iy < (unsigned)g.Hi && (unsigned)ix < (unsigned)g.Wi)
                            tj[u] = __ldg(lat_in + s_ofs[e] + own1);  // == T: never
                    }
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int e = e0b + u * kStep;
                    if (e < m) s_le[e][wl] = (uint8_t)(tj[u] <= s_t[e]);  // R-EQ4-TIE
                }
            }
        }
        __syncthreads();
        // phase 2: the ordered chain
        if (valid2) {
#pragma unroll 8
            for (int e = 0; e < m; ++e) {
                const float A = s_le[e][threadIdx.x] ? s_ap[e] : s_am[e];
                const float lo = s_lo[e], hi = s_hi[e];
                // (W-L)(U-W) soft bound, Eq. 4; plain A, Eq. 5
                const float d = s_st[e] ? __fmul_rn(A, __fmul_rn(__fsub_rn(W, lo), __fsub_rn(hi, W))) : A;
                float nw = __fadd_rn(W, d);
                if (nw > hi) nw = hi;  // Eq. 6 on W + dW (R-EQ6-CLAMP)
                if (nw < lo) nw = lo;
                W = nw;
            }
        }
    }
    if (valid2) w[(size_t)o * K + kk2] = W;
}

// Per-weight form: one thread per weight runs ITS gathers and ITS ordered chain together — no
// shared [winner][weight] table and no phase barrier, so a CTA covers 256 weights with 256 chains
// (the 32-weight tile leaves 7 of 8 warps idle during the chain) and the gathers of the next
// winners are issued while the chain of the current ones runs.  Same fp32 chain, same order.
template <int kThr>
__global__ void __launch_bounds__(kThr) stdp_update_pw_kernel(float* __restrict__ w, spk_conv_geom g,
                                                              const uint8_t* __restrict__ lat_in,
                                                              const spk_winner* __restrict__ win,
                                                              const int32_t* __restrict__ list,
                                                              const int32_t* __restrict__ start,
                                                              const int32_t* __restrict__ cnt, const Cfgs cfgs,
                                                              int ncfg) {
    spk_pdl_wait();
    __shared__ long long s_ofs[kWinChunk];  // lat_in offset of (b, channel 0, y0, x0)
    __shared__ int s_y0[kWinChunk], s_x0[kWinChunk], s_t[kWinChunk];
    __shared__ float s_ap[kWinChunk], s_am[kWinChunk], s_lo[kWinChunk], s_hi[kWinChunk];  // winner's config
    __shared__ uint8_t s_st[kWinChunk];
    __shared__ spk_stdp_config s_cf[kMaxCfg];
    const int o = blockIdx.y;
    const int n = cnt[o];
    if (n == 0) return;
    const int K = g.Ci * g.Kh * g.Kw;
    const int KhKw = g.Kh * g.Kw;
    const long long HW = (long long)g.Hi * g.Wi;
    const int kk = blockIdx.x * kThr + threadIdx.x;
    const bool valid = kk < K;
    const int c1 = kk / KhKw, r1 = kk - c1 * KhKw, i1 = r1 / g.Kw, j1 = r1 - i1 * g.Kw;
    const long long own = c1 * HW + (long long)i1 * g.Wi + j1;
#pragma unroll
    for (int q = 0; q < kMaxCfg; ++q)  // static indices: the parameter block stays in constant space
        if (threadIdx.x == q && q < ncfg) s_cf[q] = cfgs.c[q];
    float W = valid ? w[(size_t)o * K + kk] : 0.0f;
    for (int e0 = 0; e0 < n; e0 += kWinChunk) {
        const int m = min(kWinChunk, n - e0);
        __syncthreads();
        for (int q = threadIdx.x; q < m; q += kThr) {
            const spk_winner wn = win[list[(size_t)start[o] + e0 + q]];
            const int y0 = wn.y * g.Sh - g.Ph, x0 = wn.x * g.Sw - g.Pw;
            s_ofs[q] = (long long)wn.b * g.Ci * HW + (long long)y0 * g.Wi + x0;
            s_y0[q] = y0;
            s_x0[q] = x0;
            s_t[q] = wn.t;
            const spk_stdp_config cf = s_cf[wn.cfg];
            s_ap[q] = cf.a_plus;
            s_am[q] = cf.a_minus;
            s_lo[q] = cf.lower;
            s_hi[q] = cf.upper;
            s_st[q] = cf.stabilize != 0;
        }
        __syncthreads();
        if (valid) {
            constexpr int kB = 8;  // gathers issued ahead of the chain
            for (int eb = 0; eb < m; eb += kB) {
                int tj[kB];
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                    const int e = eb + u;
                    tj[u] = 0x7fffffff;  // padded input: never fires (R-NEVER)
                    if (e < m) {
                        const int iy = s_y0[e] + i1, ix = s_x0[e] + j1;
                        if ((unsigned)iy < (unsigned)g.Hi && (unsigned)ix < (unsigned)g.Wi)
                            tj[u] = __ldg(lat_in + s_ofs[e] + own);  // == T: never
                    }
                }
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                    const int e = eb + u;
                    if (e >= m) break;
                    const float A = tj[u] <= s_t[e] ? s_ap[e] : s_am[e];  // R-EQ4-TIE
                    const float lo = s_lo[e], hi = s_hi[e];
                    // (W-L)(U-W) soft bound, Eq. 4; plain A, Eq. 5
                    const float d = s_st[e] ? __fmul_rn(A, __fmul_rn(__fsub_rn(W, lo), __fsub_rn(hi, W))) : A;
                    float nw = __fadd_rn(W, d);
                    if (nw > hi) nw = hi;  // Eq. 6 on W + dW (R-EQ6-CLAMP)
                    if (nw < lo) nw = lo;
                    W = nw;
                }
            }
        }
    }
    if (valid) w[(size_t)o * K + kk] = W;
}

}  // namespace

extern "C" size_t spk_stdp_workspace(const spk_conv_geom* g, int k) {
    if (!g || g->Co < 1 || g->B < 1 || k < 1) return 0;
    const size_t cap = (size_t)g->B * (size_t)k;
    return sizeof(int32_t) * ((size_t)g->Co * cap + 2 * (size_t)g->Co + cap) + 256;
}

extern "C" spk_status spk_stdp(float* w, const spk_conv_geom* g, const uint8_t* lat_in, const spk_winner* win,
                               const int32_t* nwin, int k, const spk_stdp_config* cfgs, int ncfg, void* ws,
                               size_t ws_bytes, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(w);
    SPK_CHECK_PTR(g);
    SPK_CHECK_PTR(lat_in);
    SPK_CHECK_PTR(win);
    SPK_CHECK_PTR(nwin);
    SPK_CHECK_PTR(cfgs);
    SPK_CHECK(ncfg >= 1 && ncfg <= kMaxCfg, SPK_ERR_ARG, "ncfg=%d outside 1..%d", ncfg, kMaxCfg);
    SPK_CHECK(k >= 1, SPK_ERR_ARG, "k < 1");
    SPK_CHECK(g->B >= 1 && g->Ci >= 1 && g->Hi >= 1 && g->Wi >= 1 && g->Co >= 1 && g->Kh >= 1 && g->Kw >= 1 &&
                  g->Sh >= 1 && g->Sw >= 1 && g->Ph >= 0 && g->Pw >= 0,
              SPK_ERR_SHAPE, "bad conv geometry");
    SPK_CHECK(g->Hi + 2 * g->Ph >= g->Kh && g->Wi + 2 * g->Pw >= g->Kw, SPK_ERR_SHAPE, "kernel larger than padded input");
    Cfgs cc{};
    for (int q = 0; q < ncfg; ++q) {
        SPK_CHECK(cfgs[q].lower < cfgs[q].upper, SPK_ERR_ARG, "config %d: lower >= upper", q);
        cc.c[q] = cfgs[q];
    }
    const size_t need = spk_stdp_workspace(g, k);
    SPK_CHECK(ws != nullptr && ws_bytes >= need, SPK_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
    const int Ho = (g->Hi + 2 * g->Ph - g->Kh) / g->Sh + 1, Wo = (g->Wi + 2 * g->Pw - g->Kw) / g->Sw + 1;
    const int cap = g->B * k;
    int32_t* list = static_cast<int32_t*>(ws);
    int32_t* start = list + (size_t)g->Co * cap;
    int32_t* cnt = start + g->Co;
    int32_t* slotmap = cnt + g->Co;
    cudaStream_t s = spk::as_cuda(stream);
    int32_t* invalid = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + need - 256);  // spk_stdp_status
    if (cudaMemsetAsync(invalid, 0, sizeof(int32_t), s) != cudaSuccess) return spk::launched("memset(invalid)");
    spk::launch(stdp_slotmap_kernel, spk::ceil_div((size_t)cap, 256), 256, 0, s, win, nwin, g->B, k, ncfg, Ho, Wo, g->Co,
                                                                      slotmap, invalid);
    spk_status st = spk::launched("stdp_slotmap_kernel");
    if (st != SPK_OK) return st;
    spk::launch(stdp_bucket_kernel, g->Co, kBucketThreads, 0, s, slotmap, cap, cap, list, start, cnt);
    st = spk::launched("stdp_bucket_kernel");
    if (st != SPK_OK) return st;
    const size_t K = (size_t)g->Ci * g->Kh * g->Kw;
    SPK_CHECK(g->Co <= 65535, SPK_ERR_SHAPE, "Co=%d > 65535", g->Co);
    static const int pw = [] {  // A/B knob: SPK_STDP_PW=0 keeps the two-phase tiles, 2 forces the per-weight form
        const char* e = std::getenv("SPK_STDP_PW");
        return e ? std::atoi(e) : 1;
    }();
    // per-weight form for few winners per map on short rows (C1: K 50, FC: K 3200; FC 57 -> 24 us);
    // maps with many winners (C2 layer 3: ~41, the chain dominates) keep the 32-weight tiles and
    // few winners on long rows (C3 decision layer, K 6250) the 128-weight ones —
    // profiles/r02_ab_stdp_pw.txt
    if (pw == 2 || (pw == 1 && (long long)g->B * k < 16ll * g->Co && K < 4096)) {
        const dim3 grid(spk::ceil_div(K, 256), (unsigned)g->Co);
        spk::launch(stdp_update_pw_kernel<256>, grid, 256, 0, s, w, *g, lat_in, win, list, start, cnt, cc, ncfg);
        return spk::launched("stdp_update_pw_kernel");
    }
    // average winners per map (upper bound: every slot a winner) picks the tile width
    if ((long long)g->B * k >= 16ll * g->Co) {
        const dim3 grid(spk::ceil_div(K, 32), (unsigned)g->Co);
        spk::launch(stdp_update_kernel<32, SPK_STDP_T32>, grid, SPK_STDP_T32, 0, s, w, *g, lat_in, win, list, start, cnt, cc, ncfg);
    } else {
        const dim3 grid(spk::ceil_div(K, 128), (unsigned)g->Co);
        spk::launch(stdp_update_kernel<128, 256>, grid, 256, 0, s, w, *g, lat_in, win, list, start, cnt, cc, ncfg);
    }
    return spk::launched("stdp_update_kernel");
}

extern "C" spk_status spk_stdp_status(const void* ws, const spk_conv_geom* g, int k, int32_t* invalid_out,
                                      spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(ws);
    SPK_CHECK_PTR(g);
    SPK_CHECK_PTR(invalid_out);
    const size_t need = spk_stdp_workspace(g, k);
    SPK_CHECK(need > 0, SPK_ERR_ARG, "bad geometry or k");
    cudaStream_t s = spk::as_cuda(stream);
    int32_t v = 0;
    if (cudaMemcpyAsync(&v, static_cast<const char*>(ws) + need - 256, sizeof(int32_t), cudaMemcpyDeviceToHost, s) !=
            cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return spk::launched("spk_stdp_status");
    *invalid_out = v;
    return SPK_OK;
}
