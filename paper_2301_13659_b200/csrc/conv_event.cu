// conv_event.cu — a3 + a4, event (latency-histogram) form of the spiking conv on CUDA
// cores: SURVEY §8(f) NEXT-1, "a GPU form of the sparse interface the paper lists as
// future work".
//
// Each input fires at most once (rank-order coding), so the potential of
// Eq. 2 at step t is a prefix sum over latencies:
//   P[t] = sum_{k : lat_k <= t} W_k = sum_{t' <= t} H[t'],   H[t'] = sum_{k : lat_k = t'} W_k.
// Only active synapses (lat < T) are touched, once each — instead of the T-binned
// GEMM's T passes over every synapse.  The arithmetic is the EXACT_I8 path's:
// the same 23-bit fixed-point weights q = round(w 2^23 / s) summed exactly in
// integers, the same fire test (128 S > floor(theta 2^30 / s)) and the same single
// rounding of the potential — so the outputs are bit-identical to the tensor path.
//
// Grid (pixel chunks, blocks of 32 maps, B); small samples are staged whole in shared
// memory and one CTA covers all their pixels.  16 warps, each owns every 16th pixel of
// the chunk; a lane owns one output map.  Per pixel the warp
// (1) compacts the active synapses of the receptive field into a shared list
// (ballot), (2) adds each one's weight column into per-lane latency bins H[t][lane]
// in shared memory, (3) prefix-sums the bins: first crossing -> lat, P* (FIRE), or
// every P[t] (POTENTIAL).  Weights of the map block live in shared memory,
// transposed [k][map] so a warp's 32 lanes read one 128-byte row.
#include <cmath>

#include "conv.cuh"

namespace {

constexpr int kMB = 32;  // maps per CTA (one per lane); warps per CTA NW = 16, or 8 for large footprints
constexpr int kStageMax = 48 * 1024;  // input samples up to this many bytes are staged in smem
constexpr int kPchMax = 4096;         // output pixels per CTA (a whole sample when it fits)

struct EvArgs {
    const uint8_t* lat_in;
    const uint32_t* qT;  // [K][Co_pad] fixed-point weights (Co_pad = 32 * map blocks)
    void* out0;
    float* out1;
    spk_conv_geom g;
    int Ho, Wo, HWo, K, Co_pad, pch, stage, nw;
    int pool, Hp, Wp;   // fused pooling (Eq. 3) of the latency map in the write-out: out0 = pooled lat
    spk_pool_geom pg;
    uint32_t th;          // fire iff S > th  (S = sum of q; th = floor(theta 2^30 / s) >> 7)
    float out_scale;      // P = (128 S) * out_scale  (identical to the tensor path's rounding)
};

__global__ void ev_pack_kernel(const float* __restrict__ w, int Co, int K, int Co_pad, float inv_scale23,
                               uint32_t* __restrict__ qT, int* __restrict__ flag) {
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (size_t)K * Co_pad) return;
    const int k = (int)(q / Co_pad), o = (int)(q % Co_pad);
    float x = 0.0f;
    if (o < Co) {
        x = __fmul_rn(w[(size_t)o * K + k], inv_scale23);  // exact: a power of two
        if (!(x >= 0.0f) || x > 8388608.0f) {                // negative, NaN or above the scale
            atomicOr(flag, 1);
            x = (x > 8388608.0f) ? 8388608.0f : 0.0f;
        }
    }
    qT[q] = (uint32_t)__float2int_rn(x);
}

// shared-memory carve-up (bytes), 16-byte aligned pieces
struct EvSmem {
    size_t sq, koff, kij, in, lists, H, olat, ops, total;
};
__host__ __device__ inline size_t ev_al(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ inline EvSmem ev_smem(int K, int T, int accb, int pch, size_t in_bytes, bool pstar, int nw) {
    EvSmem m;
    m.sq = 0;
    m.koff = ev_al(m.sq + (size_t)K * kMB * 4);
    m.kij = ev_al(m.koff + (size_t)K * 4);
    m.in = ev_al(m.kij + (size_t)K * 2);
    m.lists = ev_al(m.in + in_bytes);
    m.H = ev_al(m.lists + (size_t)nw * ((K + 3) & ~3) * 4);
    m.olat = ev_al(m.H + (size_t)nw * T * 32 * accb);
    m.ops = ev_al(m.olat + (size_t)kMB * pch);
    m.total = ev_al(m.ops + (pstar ? (size_t)kMB * pch * 4 : 0));
    return m;
}

// ACC = uint32_t when K * 2^23 < 2^32, else unsigned long long
template <typename ACC, int EPI, bool PSTAR, bool SMALLK, int NW>
__global__ void __launch_bounds__(NW * 32) conv_event_kernel(const EvArgs a) {
    constexpr int kEvThreads = NW * 32, kEvWarps = NW;
    extern __shared__ __align__(16) unsigned char sm[];
    const spk_conv_geom& g = a.g;
    const int K = a.K, T = g.T;
    const size_t HWi = (size_t)g.Hi * g.Wi;
    const EvSmem ms = ev_smem(K, T, (int)sizeof(ACC), a.pch, a.stage ? (size_t)g.Ci * HWi : 0, PSTAR, NW);
    uint32_t* sq = reinterpret_cast<uint32_t*>(sm + ms.sq);        // [K][32] weight columns
    int* koff = reinterpret_cast<int*>(sm + ms.koff);              // [K] c*Hi*Wi + i*Wi + j
    uint16_t* kij = reinterpret_cast<uint16_t*>(sm + ms.kij);      // [K] (i << 8) | j
    uint8_t* sin = sm + ms.in;                                     // staged input sample (a.stage)
    uint32_t* lists = reinterpret_cast<uint32_t*>(sm + ms.lists);  // [warps][K] (k << 8) | lat
    ACC* H = reinterpret_cast<ACC*>(sm + ms.H);                    // [warps][T][32] latency bins
    uint8_t* olat = sm + ms.olat;                                  // [32][pch]
    float* ops = reinterpret_cast<float*>(sm + ms.ops);            // [32][pch] (P*)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.z, m0 = blockIdx.y * kMB, p0 = blockIdx.x * a.pch;
    const int npix = min(a.pch, a.HWo - p0);
    const uint8_t* L = a.lat_in + (size_t)b * g.Ci * HWi;

    // stage this map block's weight columns, the synapse table and (small samples) the input
    for (int q = threadIdx.x; q < K * kMB; q += kEvThreads) sq[q] = a.qT[(size_t)(q >> 5) * a.Co_pad + m0 + (q & 31)];
    const int KhKw = g.Kh * g.Kw;
    for (int k = threadIdx.x; k < K; k += kEvThreads) {
        const int c = k / KhKw, r = k - c * KhKw, i = r / g.Kw, j = r - i * g.Kw;
        koff[k] = (int)(c * HWi) + i * g.Wi + j;
        kij[k] = (uint16_t)((i << 8) | j);
    }
    if (a.stage) {
        const int n = g.Ci * (int)HWi;
        if (((reinterpret_cast<uintptr_t>(L) | (uintptr_t)n) & 15) == 0) {
            const uint4* s4 = reinterpret_cast<const uint4*>(L);
            uint4* d4 = reinterpret_cast<uint4*>(sin);
            for (int q = threadIdx.x; q < n / 16; q += kEvThreads) d4[q] = __ldg(s4 + q);
        } else {
            for (int q = threadIdx.x; q < n; q += kEvThreads) sin[q] = __ldg(L + q);
        }
    }
    __syncthreads();
    const uint8_t* src = a.stage ? sin : L;

    const int o = m0 + lane;  // this lane's output map
    uint32_t* list = lists + (size_t)warp * ((K + 3) & ~3);  // 16-byte aligned per warp
    ACC* h = H + (size_t)warp * T * 32;
    for (int t = 0; t < T; ++t) h[t * 32 + lane] = 0;
    const uint32_t* wcol = sq + lane;
    // small receptive fields: this lane's synapse offsets stay in registers
    constexpr int kRegChunks = 8;  // K <= 256
    int rko[kRegChunks], rij[kRegChunks];
    if (SMALLK) {
#pragma unroll
        for (int c = 0; c < kRegChunks; ++c) {
            const int k = c * 32 + lane;
            rko[c] = k < K ? koff[k] : 0;
            rij[c] = k < K ? kij[k] : 0xFFFF;  // out of the window: never active
        }
    }
    const unsigned lanemask_lt = (1u << lane) - 1u;
    const int pstep = kEvWarps;
    int pl = warp;
    int y = (p0 + pl) / a.Wo, x = (p0 + pl) - y * a.Wo;  // advanced incrementally
    for (; pl < npix; pl += pstep) {
        const int p = p0 + pl;
        const int y0 = y * g.Sh - g.Ph, x0 = x * g.Sw - g.Pw;
        const ptrdiff_t org = (ptrdiff_t)y0 * g.Wi + x0;
        // (1) compact the active synapses of the receptive field; list entry =
        //     (byte offset of the weight row k * 128) << 8 | latency
        const bool interior = y0 >= 0 && x0 >= 0 && y0 + g.Kh <= g.Hi && x0 + g.Kw <= g.Wi;  // warp-uniform
        int n = 0;
        auto take = [&](int k, int lat) {
            const bool act = lat < T;
            const unsigned m = __ballot_sync(0xffffffffu, act);
            if (act) list[n + __popc(m & lanemask_lt)] = ((uint32_t)k << 15) | (uint32_t)lat;
            n += __popc(m);
        };
        if (SMALLK) {
#pragma unroll
            for (int c = 0; c < kRegChunks; ++c) {
                if (c * 32 >= K) break;
                int lat = T;
                if (interior) {
                    if (c * 32 + lane < K) lat = src[org + rko[c]];
                } else {
                    const int iy = y0 + (rij[c] >> 8), ix = x0 + (rij[c] & 255);
                    if (c * 32 + lane < K && (unsigned)iy < (unsigned)g.Hi && (unsigned)ix < (unsigned)g.Wi)
                        lat = src[org + rko[c]];  // padded taps never fire
                }
                take(c * 32 + lane, lat);
            }
        } else {
            for (int k0 = 0; k0 < K; k0 += 32) {
                const int k = k0 + lane;
                int lat = T;
                if (k < K) {
                    const int ij = kij[k], iy = y0 + (ij >> 8), ix = x0 + (ij & 255);
                    if ((unsigned)iy < (unsigned)g.Hi && (unsigned)ix < (unsigned)g.Wi)
                        lat = src[org + koff[k]];  // padded taps never fire
                }
                take(k, lat);
            }
        }
        x += pstep;
        while (x >= a.Wo) x -= a.Wo, ++y;
        __syncwarp();
        // (2) latency bins: H[lat] += W_k (exact integer sums); the bins were zeroed by
        //     the previous pixel's prefix pass (or at start)
        const unsigned char* wrow = reinterpret_cast<const unsigned char*>(wcol);
        int e = 0;
        for (; e + 4 <= n; e += 4) {
            const uint4 v = *reinterpret_cast<const uint4*>(list + e);  // 16-byte aligned: e % 4 == 0
            const ACC w0 = *reinterpret_cast<const uint32_t*>(wrow + (v.x >> 8)),
                      w1 = *reinterpret_cast<const uint32_t*>(wrow + (v.y >> 8)),
                      w2 = *reinterpret_cast<const uint32_t*>(wrow + (v.z >> 8)),
                      w3 = *reinterpret_cast<const uint32_t*>(wrow + (v.w >> 8));
            h[(v.x & 255) * 32 + lane] += w0;
            h[(v.y & 255) * 32 + lane] += w1;
            h[(v.z & 255) * 32 + lane] += w2;
            h[(v.w & 255) * 32 + lane] += w3;
        }
        for (; e < n; ++e) {
            const uint32_t v = list[e];
            h[(v & 255) * 32 + lane] += (ACC)*reinterpret_cast<const uint32_t*>(wrow + (v >> 8));
        }
        // (3) prefix over latencies
        ACC S = 0;
        if (EPI == SPK_EPI_POTENTIAL) {
            for (int t = 0; t < T; ++t) {
                S += h[t * 32 + lane];
                h[t * 32 + lane] = 0;
                if (o < g.Co)
                    static_cast<float*>(a.out0)[(((size_t)b * T + t) * g.Co + o) * a.HWo + p] =
                        __fmul_rn(__ll2float_rn((long long)S * 128ll), a.out_scale);
            }
        } else if (!PSTAR) {
            // potentials are non-decreasing in t (W >= 0), so the steps at or below the
            // threshold are exactly t < lat: lat = their count
            int lat = 0;
            for (int t = 0; t < T; ++t) {
                S += h[t * 32 + lane];
                h[t * 32 + lane] = 0;
                lat += (S <= (ACC)a.th);
            }
            olat[lane * a.pch + pl] = (uint8_t)lat;
        } else {
            int lat = T;
            ACC Sf = 0;
            for (int t = 0; t < T; ++t) {
                S += h[t * 32 + lane];
                h[t * 32 + lane] = 0;
                if (lat == T && S > (ACC)a.th) {
                    lat = t;
                    Sf = S;
                }
            }
            olat[lane * a.pch + pl] = (uint8_t)lat;
            if (PSTAR) ops[lane * a.pch + pl] = lat < T ? __fmul_rn(__ll2float_rn((long long)Sf * 128ll), a.out_scale) : 0.0f;
        }
        __syncwarp();
    }
    if (EPI == SPK_EPI_POTENTIAL) return;
    __syncthreads();
    if (a.pool) {  // whole sample staged: window minimum of latencies (Eq. 3), padding never fires
        const int HWp = a.Hp * a.Wp;
        for (int r = warp; r < kMB; r += kEvWarps) {
            const int om = m0 + r;
            if (om >= g.Co) continue;
            uint8_t* dl = static_cast<uint8_t*>(a.out0) + ((size_t)b * g.Co + om) * HWp;
            const uint8_t* ml = olat + r * a.pch;
            for (int q = lane; q < HWp; q += 32) {
                const int py = q / a.Wp, px = q - py * a.Wp;
                const int y0 = py * a.pg.Sh - a.pg.Ph, x0 = px * a.pg.Sw - a.pg.Pw;
                int m = T;
                for (int i = max(0, -y0); i < a.pg.Lh && y0 + i < a.Ho; ++i)
                    for (int j = max(0, -x0); j < a.pg.Lw && x0 + j < a.Wo; ++j)
                        m = min(m, (int)ml[(y0 + i) * a.Wo + x0 + j]);
                dl[q] = (uint8_t)m;
            }
        }
        return;
    }
    // coalesced write-out: one run of npix latencies (and P*) per map
    for (int r = warp; r < kMB; r += kEvWarps) {
        const int om = m0 + r;
        if (om >= g.Co) continue;
        const size_t base = ((size_t)b * g.Co + om) * a.HWo + p0;
        uint8_t* dl = static_cast<uint8_t*>(a.out0) + base;
        for (int q = lane; q < npix; q += 32) dl[q] = olat[r * a.pch + q];
        if (PSTAR)
            for (int q = lane; q < npix; q += 32) a.out1[base + q] = ops[r * a.pch + q];
    }
}

template <typename ACC, int EPI, bool PSTAR>
spk_status launch_ev(const EvArgs& a, dim3 grid, size_t smem, cudaStream_t s) {
    auto k = a.nw == 16 ? (a.K <= 256 ? conv_event_kernel<ACC, EPI, PSTAR, true, 16> : conv_event_kernel<ACC, EPI, PSTAR, false, 16>)
                        : (a.K <= 256 ? conv_event_kernel<ACC, EPI, PSTAR, true, 8> : conv_event_kernel<ACC, EPI, PSTAR, false, 8>);
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return spk::launched("conv_event_kernel(attr)");
    k<<<grid, a.nw * 32, smem, s>>>(a);
    return spk::launched("conv_event_kernel");
}

}  // namespace

bool ev_plan(const spk_conv_geom& g, EvPlan& p) {
    p.Ho = (g.Hi + 2 * g.Ph - g.Kh) / g.Sh + 1;
    p.Wo = (g.Wi + 2 * g.Pw - g.Kw) / g.Sw + 1;
    p.K = g.Ci * g.Kh * g.Kw;
    if (g.Kh > 255 || g.Kw > 255 || g.T > 254 || p.K >= (1 << 17)) return false;  // list entry k << 15
    if ((double)g.Ci * g.Hi * g.Wi >= 2147483647.0) return false;
    p.acc64 = (double)p.K * 8388608.0 >= 4294967296.0 ? 1 : 0;
    const int HWo = p.Ho * p.Wo;
    const size_t in_bytes = (size_t)g.Ci * g.Hi * g.Wi;
    p.stage = in_bytes <= (size_t)kStageMax ? 1 : 0;
    p.pch = std::min(HWo, p.stage ? kPchMax : 256);
    // smem with P* staging (the larger of the two epilogue variants); 16 warps when it fits
    p.nw = 16;
    p.smem_bytes = ev_smem(p.K, g.T, p.acc64 ? 8 : 4, p.pch, p.stage ? in_bytes : 0, true, 16).total;
    if (p.smem_bytes > 200 * 1024) {
        p.nw = 8;
        p.smem_bytes = ev_smem(p.K, g.T, p.acc64 ? 8 : 4, p.pch, p.stage ? in_bytes : 0, true, 8).total;
    }
    if (p.smem_bytes > 200 * 1024) return false;
    p.n_mb = (g.Co + kMB - 1) / kMB;
    p.Co_pad = p.n_mb * kMB;
    p.MB = kMB;
    p.ws_bytes = 256 + (size_t)p.K * p.Co_pad * 4;
    return true;
}

spk_status spk_conv_event(const uint8_t* lat_in, const float* w, const spk_conv_geom& g, const EvPlan& p,
                          spk_epilogue epi, float theta, float w_max, void* out0, void* out1, void* ws,
                          cudaStream_t s, const spk_pool_geom* pool) {
    // same scale and fixed point as the tensor path: s = smallest power of two >= w_max
    int ex = 0;
    std::frexp((double)w_max, &ex);
    double scale = std::ldexp(1.0, ex);
    if (std::ldexp(1.0, ex - 1) >= (double)w_max) scale = std::ldexp(1.0, ex - 1);
    const float inv_scale23 = (float)(8388608.0 / scale);
    int* flag = static_cast<int*>(ws);
    uint32_t* qT = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ws) + 256);
    if (cudaMemsetAsync(flag, 0, sizeof(int), s) != cudaSuccess) return spk::launched("memset(flag)");
    const size_t n = (size_t)p.K * p.Co_pad;
    ev_pack_kernel<<<spk::ceil_div(n, 256), 256, 0, s>>>(w, g.Co, p.K, p.Co_pad, inv_scale23, qT, flag);
    spk_status st = spk::launched("ev_pack_kernel");
    if (st != SPK_OK) return st;

    EvArgs a{};
    a.lat_in = lat_in;
    a.qT = qT;
    a.out0 = out0;
    a.out1 = static_cast<float*>(out1);
    a.g = g;
    a.Ho = p.Ho;
    a.Wo = p.Wo;
    a.HWo = p.Ho * p.Wo;
    a.K = p.K;
    a.Co_pad = p.Co_pad;
    a.pch = p.pch;
    a.stage = p.stage;
    if (pool) {  // caller checked: FIRE, whole sample in one CTA
        a.pool = 1;
        a.pg = *pool;
        a.Hp = (p.Ho + 2 * pool->Ph - pool->Lh) / pool->Sh + 1;
        a.Wp = (p.Wo + 2 * pool->Pw - pool->Lw) / pool->Sw + 1;
    }
    const long long theta_q = (long long)std::floor((double)theta * (1073741824.0 / scale));  // tensor path's
    a.th = (uint32_t)std::min<long long>(theta_q >> 7, 0xffffffffll);
    a.out_scale = (float)(scale / 1073741824.0);
    const dim3 grid((unsigned)((a.HWo + p.pch - 1) / p.pch), (unsigned)p.n_mb, (unsigned)g.B);
    const bool ps = out1 != nullptr && epi == SPK_EPI_FIRE;
    const size_t in_bytes = p.stage ? (size_t)g.Ci * g.Hi * g.Wi : 0;
    a.nw = p.nw;
    const size_t smem = ev_smem(p.K, g.T, p.acc64 ? 8 : 4, p.pch, in_bytes, ps, p.nw).total;
    if (epi == SPK_EPI_POTENTIAL)
        return p.acc64 ? launch_ev<unsigned long long, SPK_EPI_POTENTIAL, false>(a, grid, smem, s)
                       : launch_ev<uint32_t, SPK_EPI_POTENTIAL, false>(a, grid, smem, s);
    if (p.acc64)
        return ps ? launch_ev<unsigned long long, SPK_EPI_FIRE, true>(a, grid, smem, s)
                  : launch_ev<unsigned long long, SPK_EPI_FIRE, false>(a, grid, smem, s);
    return ps ? launch_ev<uint32_t, SPK_EPI_FIRE, true>(a, grid, smem, s)
              : launch_ev<uint32_t, SPK_EPI_FIRE, false>(a, grid, smem, s);
}
