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
#include "common.cuh"

namespace {

constexpr int kMaxCfg = 8;
struct Cfgs {
    spk_stdp_config c[kMaxCfg];
};

constexpr int kBucketThreads = 256;

// list[o][0..cnt[o]) = winner slot indices (b*k + q) of map o, in slot order.
__global__ void __launch_bounds__(kBucketThreads) stdp_bucket_kernel(const spk_winner* __restrict__ win,
                                                                    const int32_t* __restrict__ nwin,
                                                                    int B, int k, int ncfg, int Ho,
                                                                    int Wo, int cap,
                                                                    int32_t* __restrict__ list,
                                                                    int32_t* __restrict__ cnt) {
    __shared__ int scan[kBucketThreads];
    const int o = blockIdx.x;
    const int S = B * k;
    const int chunk = (S + kBucketThreads - 1) / kBucketThreads;
    const int s0 = threadIdx.x * chunk, s1 = min(S, s0 + chunk);
    auto take = [&](int s) -> bool {
        const int b = s / k, q = s % k;
        if (q >= nwin[b]) return false;
        const spk_winner w = win[s];
        return w.c == o && w.cfg >= 0 && w.cfg < ncfg && w.y >= 0 && w.y < Ho && w.x >= 0 && w.x < Wo &&
               w.b >= 0 && w.b < B;
    };
    int mine = 0;
    for (int s = s0; s < s1; ++s) mine += take(s);
    scan[threadIdx.x] = mine;
    __syncthreads();
    for (int off = 1; off < kBucketThreads; off <<= 1) {  // inclusive Hillis-Steele scan
        const int v = threadIdx.x >= off ? scan[threadIdx.x - off] : 0;
        __syncthreads();
        scan[threadIdx.x] += v;
        __syncthreads();
    }
    int pos = scan[threadIdx.x] - mine;
    for (int s = s0; s < s1; ++s)
        if (take(s) && pos < cap) list[(size_t)o * cap + pos++] = s;
    if (threadIdx.x == kBucketThreads - 1) cnt[o] = min(scan[kBucketThreads - 1], cap);
}

// Grid (K chunks of kUpdThreads, Co): the winners of map o are staged in shared
// memory (decoded once per CTA), then each thread walks them in order for its
// weight, with the pre-synaptic latencies of a group of winners loaded ahead.
constexpr int kUpdThreads = 256, kWinChunk = 256, kAhead = 4;

__global__ void __launch_bounds__(kUpdThreads) stdp_update_kernel(float* __restrict__ w, spk_conv_geom g,
                                                                  const uint8_t* __restrict__ lat_in,
                                                                  const spk_winner* __restrict__ win,
                                                                  const int32_t* __restrict__ list,
                                                                  const int32_t* __restrict__ cnt, int cap,
                                                                  const Cfgs cfgs) {
    __shared__ long long s_base[kWinChunk];  // lat_in offset of channel 0 of the winner's sample
    __shared__ int s_y0[kWinChunk], s_x0[kWinChunk], s_t[kWinChunk], s_cfg[kWinChunk];
    const int K = g.Ci * g.Kh * g.Kw;
    const int o = blockIdx.y;
    const int kk = blockIdx.x * kUpdThreads + threadIdx.x;
    const bool valid = kk < K;
    const int KhKw = g.Kh * g.Kw;
    const int c = kk / KhKw, r = kk - c * KhKw, i = r / g.Kw, j = r - i * g.Kw;
    const long long HW = (long long)g.Hi * g.Wi;
    float W = valid ? w[(size_t)o * K + kk] : 0.0f;
    const int n = cnt[o];
    for (int e0 = 0; e0 < n; e0 += kWinChunk) {
        const int m = min(kWinChunk, n - e0);
        __syncthreads();
        if (threadIdx.x < m) {
            const spk_winner wn = win[list[(size_t)o * cap + e0 + threadIdx.x]];
            s_base[threadIdx.x] = (long long)wn.b * g.Ci * HW;
            s_y0[threadIdx.x] = wn.y * g.Sh - g.Ph;
            s_x0[threadIdx.x] = wn.x * g.Sw - g.Pw;
            s_t[threadIdx.x] = wn.t;
            s_cfg[threadIdx.x] = wn.cfg;
        }
        __syncthreads();
        if (!valid) continue;
        for (int e = 0; e < m; e += kAhead) {
            int tj[kAhead];
#pragma unroll
            for (int u = 0; u < kAhead; ++u) {  // loads first: independent of W
                tj[u] = 0x7fffffff;               // padded input: never fires (R-NEVER)
                if (e + u < m) {
                    const int iy = s_y0[e + u] + i, ix = s_x0[e + u] + j;
                    if (iy >= 0 && iy < g.Hi && ix >= 0 && ix < g.Wi)
                        tj[u] = __ldg(lat_in + s_base[e + u] + c * HW + (long long)iy * g.Wi + ix);  // T: never
                }
            }
#pragma unroll
            for (int u = 0; u < kAhead; ++u) {
                if (e + u >= m) break;
                const spk_stdp_config cf = cfgs.c[s_cfg[e + u]];
                const float A = (tj[u] <= s_t[e + u]) ? cf.a_plus : cf.a_minus;  // R-EQ4-TIE
                float d;
                if (cf.stabilize) {
                    const float sw = __fmul_rn(__fsub_rn(W, cf.lower), __fsub_rn(cf.upper, W));  // (W-L)(U-W), Eq. 4
                    d = __fmul_rn(A, sw);
                } else {
                    d = A;  // Eq. 5
                }
                float nw = __fadd_rn(W, d);
                if (nw > cf.upper) nw = cf.upper;  // Eq. 6 on W + dW (R-EQ6-CLAMP)
                if (nw < cf.lower) nw = cf.lower;
                W = nw;
            }
        }
    }
    if (valid) w[(size_t)o * K + kk] = W;
}

}  // namespace

extern "C" size_t spk_stdp_workspace(const spk_conv_geom* g, int k) {
    if (!g || g->Co < 1 || g->B < 1 || k < 1) return 0;
    const size_t cap = (size_t)g->B * (size_t)k;
    return sizeof(int32_t) * ((size_t)g->Co * cap + (size_t)g->Co) + 256;
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
    int32_t* cnt = list + (size_t)g->Co * cap;
    cudaStream_t s = spk::as_cuda(stream);
    stdp_bucket_kernel<<<g->Co, kBucketThreads, 0, s>>>(win, nwin, g->B, k, ncfg, Ho, Wo, cap, list, cnt);
    spk_status st = spk::launched("stdp_bucket_kernel");
    if (st != SPK_OK) return st;
    const size_t K = (size_t)g->Ci * g->Kh * g->Kw;
    SPK_CHECK(g->Co <= 65535, SPK_ERR_SHAPE, "Co=%d > 65535", g->Co);
    const dim3 grid(spk::ceil_div(K, kUpdThreads), (unsigned)g->Co);
    stdp_update_kernel<<<grid, kUpdThreads, 0, s>>>(w, *g, lat_in, win, list, cnt, cap, cc);
    return spk::launched("stdp_update_kernel");
}
