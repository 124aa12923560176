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
// Grid (chunks of whole output rows, blocks of 32 maps, B); the chunk's input band is
// staged in shared memory with its zero-padding halo written as "never fires", and a
// small sample is one chunk.  16 warps, each owns every 16th pixel of the chunk; a lane
// owns one output map.  Per pixel the warp (1) counting-sorts the receptive field's
// active synapses by latency into a shared list, (2) walks the list once keeping the
// running potential in a register: the first element that lifts it above the
// threshold gives lat, the end of that latency group gives P* (FIRE), or every P[t]
// is written (POTENTIAL).  Weights of the map block live in shared memory, transposed
// [k][map] so a warp's 32 lanes read one 128-byte row.
#include <cmath>
#include <cstdlib>

#include "conv.cuh"

namespace {

constexpr int kMB = 32;  // maps per CTA per map-per-lane (MB = 32 MPL); warps per CTA NW = 16, or 8 for large footprints
constexpr int kStageMax = 48 * 1024;  // input samples up to this many bytes are staged in smem
constexpr int kPchMax = 4096;         // output pixels per CTA (a whole sample when it fits)

struct EvArgs {
    const uint8_t* lat_in;
    const uint32_t* qT;  // [K][Co_pad] fixed-point weights (Co_pad = 32 * map blocks)
    void* out0;
    float* out1;
    spk_conv_geom g;
    int Ho, Wo, HWo, K, Co_pad, pch, nw;
    int rpc, Wq, band;  // output rows per CTA, staged row length, staged band bytes
    int mpl;            // output maps per lane (1 or 2): a CTA covers MB = 32 mpl maps
    int pool, Hp, Wp;   // fused pooling (Eq. 3) of the latency map in the write-out: out0 = pooled lat
    spk_pool_geom pg;
    uint32_t th;          // fire iff S > th  (S = sum of q; th = floor(theta 2^30 / s) >> 7)
    float out_scale;      // P = (128 S) * out_scale  (identical to the tensor path's rounding)
};

__global__ void ev_pack_kernel(const float* __restrict__ w, int Co, int K, int Co_pad, float inv_scale23,
                               uint32_t* __restrict__ qT, int* __restrict__ flag) {
    spk_pdl_wait();
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
    size_t sq, koff, in, lists, cnt, olat, ops, total;
};
__host__ __device__ inline size_t ev_al(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ inline int ev_list_len(int K) { return (K + 3) & ~3; }   // padded to whole uint4 batches
__host__ __device__ inline int ev_cnt_len(int T) { return (T + 32) & ~31; }  // T bins, 32-lane chunks
__host__ __device__ inline EvSmem ev_smem(int K, int T, int pch, size_t in_bytes, bool pstar, int nw, int mb) {
    EvSmem m;
    m.sq = 0;
    m.koff = ev_al(m.sq + (size_t)(K + 1) * mb * 4);  // + one zero row for list padding
    m.in = ev_al(m.koff + (size_t)K * 4);
    m.lists = ev_al(m.in + in_bytes);
    m.cnt = ev_al(m.lists + (size_t)nw * ev_list_len(K) * 4);
    m.olat = ev_al(m.cnt + (size_t)nw * ev_cnt_len(T) * 4);
    m.ops = ev_al(m.olat + (size_t)mb * pch);
    m.total = ev_al(m.ops + (pstar ? (size_t)mb * pch * 4 : 0));
    return m;
}

// ACC = uint32_t when K * 2^23 < 2^32, else unsigned long long.
// Per output pixel, one warp (lane = output map):
//  (1) counting sort of the receptive field's ACTIVE synapses by latency: shared
//      counters per latency, a warp scan, and placement through the running
//      cursors — the list holds (weight-row byte offset << 8 | lat), latency-ascending;
//  (2) one pass over the sorted list in uint4 batches: acc += W_k (exact integer
//      sums, registers only).  Potentials are non-decreasing (R-NONNEG), so the
//      first element whose running sum exceeds the threshold has the output latency;
//      P* = the running sum at the end of that latency group (its end is the
//      group's final cursor).  Zero-weight padding entries complete the last batch.
__device__ __forceinline__ int lds_u8(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));  // the band is read-only after staging
    return (int)v;
}

// NCH = ceil(K / 32) synapse chunks held in registers (1..8), or 0 for large receptive fields
template <typename ACC, int EPI, bool PSTAR, int NCH, int NW, int MPL>
__global__ void __launch_bounds__(NW * 32) conv_event_kernel(const EvArgs a) {
    spk_pdl_wait();
    constexpr bool SMALLK = NCH > 0;
    constexpr int MB = 32 * MPL, LOGM = MPL == 4 ? 2 : MPL == 2 ? 1 : 0;  // maps per CTA; entry = k << (15 + LOGM) | lat
    constexpr int kEvThreads = NW * 32, kEvWarps = NW;
    extern __shared__ __align__(16) unsigned char sm[];
    const spk_conv_geom& g = a.g;
    const int K = a.K, T = g.T;
    const size_t HWi = (size_t)g.Hi * g.Wi;
    const EvSmem ms = ev_smem(K, T, a.pch, (size_t)a.band, PSTAR, NW, MB);
    uint32_t* sq = reinterpret_cast<uint32_t*>(sm + ms.sq);        // [K+1][32] weight rows (row K = 0)
    int* koff = reinterpret_cast<int*>(sm + ms.koff);              // [K] c*Hi*Wi + i*Wi + j
    uint8_t* sin = sm + ms.in;                                     // staged input band [Ci][rows][Wq]
    uint32_t* lists = reinterpret_cast<uint32_t*>(sm + ms.lists);  // [warps][K pad 4] (k << 15) | lat
    uint32_t* cnts = reinterpret_cast<uint32_t*>(sm + ms.cnt);     // [warps][T pad] counters / cursors
    uint8_t* olat = sm + ms.olat;                                  // [32][pch]
    float* ops = reinterpret_cast<float*>(sm + ms.ops);            // [32][pch] (P*)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.z, m0 = blockIdx.y * MB;
    const int ya = blockIdx.x * a.rpc;                 // first output row of this CTA's chunk
    const int p0 = ya * a.Wo;
    const int npix = min(a.rpc, a.Ho - ya) * a.Wo;
    const int nrows = (min(a.rpc, a.Ho - ya) - 1) * g.Sh + g.Kh;  // staged input rows (halo incl.)
    const int Wq = a.Wq;                                // staged row length (Wi + 2 Pw)
    const uint8_t* L = a.lat_in + (size_t)b * g.Ci * HWi;

    // stage this map block's weight rows, the synapse table and the input band with its
    // zero-padding halo written as "never fires", so synapse reads need no bounds test
    for (int q = threadIdx.x; q < K * MB; q += kEvThreads) sq[q] = a.qT[(size_t)(q / MB) * a.Co_pad + m0 + (q % MB)];
    if (threadIdx.x < MB) sq[K * MB + threadIdx.x] = 0u;
    const int KhKw = g.Kh * g.Kw;
    for (int k = threadIdx.x; k < K; k += kEvThreads) {
        const int c = k / KhKw, r = k - c * KhKw, i = r / g.Kw, j = r - i * g.Kw;
        koff[k] = (c * nrows + i) * Wq + j;
    }
    {
        const int per_c = nrows * Wq, n = g.Ci * per_c;
        const int iy0 = ya * g.Sh - g.Ph;
        for (int q = threadIdx.x; q < n; q += kEvThreads) {
            const int c = q / per_c, r = q - c * per_c, rr = r / Wq, xx = r - rr * Wq;
            const int iy = iy0 + rr, ix = xx - g.Pw;
            sin[q] = ((unsigned)iy < (unsigned)g.Hi && (unsigned)ix < (unsigned)g.Wi)
                         ? __ldg(L + (size_t)c * HWi + (size_t)iy * g.Wi + ix)
                         : (uint8_t)T;
        }
    }
    const int ncnt = ev_cnt_len(T);
    for (int q = threadIdx.x; q < kEvWarps * ncnt; q += kEvThreads) cnts[q] = 0u;
    __syncthreads();

    const int o0 = m0 + lane * MPL;  // this lane's first output map
    uint32_t* list = lists + (size_t)warp * ev_list_len(K);  // 16-byte aligned per warp
    uint32_t* cnt = cnts + (size_t)warp * ncnt;
    const unsigned char* wrow = reinterpret_cast<const unsigned char*>(sq + lane * MPL);
    const uint32_t pad_entry = ((uint32_t)K << (15 + LOGM)) | (uint32_t)T;  // zero weight row, never a crossing
    // this lane's MPL weights of the synapse whose list entry is v (row byte offset = v >> 8)
    auto ldw = [&](uint32_t v, ACC (&w)[MPL]) {
        if (MPL == 4) {
            const uint4 q = *reinterpret_cast<const uint4*>(wrow + (v >> 8));
            w[0] = (ACC)q.x;
            w[1 % MPL] = (ACC)q.y;
            w[2 % MPL] = (ACC)q.z;
            w[3 % MPL] = (ACC)q.w;
        } else if (MPL == 2) {
            const uint2 q = *reinterpret_cast<const uint2*>(wrow + (v >> 8));
            w[0] = (ACC)q.x;
            w[MPL - 1] = (ACC)q.y;
        } else {
            w[0] = (ACC)*reinterpret_cast<const uint32_t*>(wrow + (v >> 8));
        }
    };
    // small receptive fields: this lane's synapse offsets stay in registers
    constexpr int kRegChunks = SMALLK ? NCH : 1;
    int rko[kRegChunks];
    const bool last_ok = (kRegChunks - 1) * 32 + lane < K;  // lanes of the last chunk inside K
    if (SMALLK) {
#pragma unroll
        for (int c = 0; c < kRegChunks; ++c) {
            const int k = c * 32 + lane;
            rko[c] = k < K ? koff[k] : 0;
        }
    }
    const uint32_t sin_s = (uint32_t)__cvta_generic_to_shared(sin);
    const int pstep = kEvWarps;
    int pl = warp;
    int y = pl / a.Wo, x = pl - y * a.Wo;  // chunk-relative, advanced incrementally
    for (; pl < npix; pl += pstep) {
        const int p = p0 + pl;
        const uint32_t bs = sin_s + (uint32_t)(y * g.Sh * Wq + x * g.Sw);  // receptive field origin in the band
        x += pstep;
        while (x >= a.Wo) x -= a.Wo, ++y;
        auto lat_of = [&](int k, int c) -> int {  // input latency of synapse k (T: padded / never)
            if (SMALLK) {
                const int l = lds_u8(bs + (uint32_t)rko[c]);
                return (c < kRegChunks - 1 || last_ok) ? l : T;
            }
            return k < K ? lds_u8(bs + (uint32_t)koff[k]) : T;
        };
        // (1a) count active synapses per latency
        int lr[kRegChunks];
        if (SMALLK) {
#pragma unroll
            for (int c = 0; c < kRegChunks; ++c) {
                lr[c] = lat_of(c * 32 + lane, c);
                if (lr[c] < T) atomicAdd(cnt + lr[c], 1u);
            }
        } else {
            for (int k0 = 0; k0 < K; k0 += 32) {
                const int l = lat_of(k0 + lane, 0);
                if (l < T) atomicAdd(cnt + l, 1u);
            }
        }
        __syncwarp();
        // (1b) exclusive scan of the counts -> group starts (cursors)
        uint32_t carry = 0;
        if (T <= 32) {  // one 32-lane chunk (every config)
            const uint32_t c = lane < T ? cnt[lane] : 0u;
            uint32_t incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            if (lane < T) cnt[lane] = incl - c;
            carry = __shfl_sync(0xffffffffu, incl, 31);
        } else
        for (int t0 = 0; t0 < T; t0 += 32) {
            const int t = t0 + lane;
            const uint32_t c = t < T ? cnt[t] : 0u;
            uint32_t incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            if (t < T) cnt[t] = carry + incl - c;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        const int n = (int)carry;
        const int n4 = (n + 3) & ~3;
        if (lane < n4 - n) list[n + lane] = pad_entry;
        __syncwarp();
        // (1c) place: after this, cnt[t] = end of latency group t
        if (SMALLK) {
#pragma unroll
            for (int c = 0; c < kRegChunks; ++c)
                if (lr[c] < T)
                    list[atomicAdd(cnt + lr[c], 1u)] = ((uint32_t)(c * 32 + lane) << (15 + LOGM)) | (uint32_t)lr[c];
        } else {
            for (int k0 = 0; k0 < K; k0 += 32) {
                const int l = lat_of(k0 + lane, 0);
                if (l < T) list[atomicAdd(cnt + l, 1u)] = ((uint32_t)(k0 + lane) << (15 + LOGM)) | (uint32_t)l;
            }
        }
        __syncwarp();
        // (2) running sums over the latency-sorted list (MPL maps per lane)
        if (EPI == SPK_EPI_POTENTIAL) {
            ACC S[MPL] = {};
            int e = 0;
            for (int t = 0; t < T; ++t) {
                const int end = (int)cnt[t];
                for (; e < end; ++e) {
                    ACC w[MPL];
                    ldw(list[e], w);
#pragma unroll
                    for (int m = 0; m < MPL; ++m) S[m] += w[m];
                }
#pragma unroll
                for (int m = 0; m < MPL; ++m)
                    if (o0 + m < g.Co)
                        static_cast<float*>(a.out0)[(((size_t)b * T + t) * g.Co + o0 + m) * a.HWo + p] =
                            __fmul_rn(__ll2float_rn((long long)S[m] * 128ll), a.out_scale);
            }
        } else {
            const ACC th = (ACC)a.th;
            ACC S[MPL] = {}, Sps[MPL] = {};
            int lo[MPL], pe[MPL];  // output latency (first crossing); PSTAR: end index of its latency group
#pragma unroll
            for (int m = 0; m < MPL; ++m) lo[m] = T, pe[m] = 0x7fffffff;
            for (int e = 0; e < n4; e += 4) {
                const uint4 v = *reinterpret_cast<const uint4*>(list + e);
                ACC w0[MPL], w1[MPL], w2[MPL], w3[MPL];
                ldw(v.x, w0);
                ldw(v.y, w1);
                ldw(v.z, w2);
                ldw(v.w, w3);
#pragma unroll
                for (int m = 0; m < MPL; ++m) {
                    const ACC s0 = S[m] + w0[m], s1 = s0 + w1[m], s2 = s1 + w2[m], s3 = s2 + w3[m];
                    if (lo[m] == T && s3 > th) {  // this map crosses inside the batch (once)
                        lo[m] = (int)((s0 > th ? v.x : s1 > th ? v.y : s2 > th ? v.z : v.w) & 255u);
                        if (PSTAR) pe[m] = (int)cnt[lo[m]];
                    }
                    if (PSTAR && pe[m] <= e + 4) {  // the crossing's group ends inside this batch
                        const int j = pe[m] - e;     // 1..4 (pe > e: groups end after their crossing)
                        Sps[m] = j == 1 ? s0 : j == 2 ? s1 : j == 3 ? s2 : s3;
                        pe[m] = 0x7fffffff;
                    }
                    S[m] = s3;
                }
            }
#pragma unroll
            for (int m = 0; m < MPL; ++m) {
                olat[(lane * MPL + m) * a.pch + pl] = (uint8_t)lo[m];
                if (PSTAR)
                    ops[(lane * MPL + m) * a.pch + pl] =
                        lo[m] < T ? __fmul_rn(__ll2float_rn((long long)Sps[m] * 128ll), a.out_scale) : 0.0f;
            }
        }
        __syncwarp();
        if (T <= 32) {  // counters for the next pixel
            if (lane < T) cnt[lane] = 0u;
        } else {
            for (int t = lane; t < T; t += 32) cnt[t] = 0u;
        }
        __syncwarp();
    }
    if (EPI == SPK_EPI_POTENTIAL) return;
    __syncthreads();
    if (a.pool) {  // window minimum of latencies (Eq. 3), padding never fires; this CTA's output
                   // rows [ya, ya + rows) hold whole windows (whole sample, or Ph = 0, Lh = Sh | rpc)
        const int rows = npix / a.Wo;
        const int py0 = a.rpc >= a.Ho ? 0 : ya / a.pg.Sh;
        const int py1 = a.rpc >= a.Ho ? a.Hp : min(a.Hp, (ya + rows) / a.pg.Sh);
        const bool p2 = a.pg.Lh == 2 && a.pg.Lw == 2 && a.pg.Sh == 2 && a.pg.Sw == 2 && a.pg.Ph == 0 && a.pg.Pw == 0 &&
                        (a.Wo & 1) == 0 && (a.pch & 1) == 0;
        if (p2 && a.Wp < 32) {  // short rows (C2): lanes over the map's pooled outputs
            const int nq = (py1 - py0) * a.Wp;
            for (int r = warp; r < MB; r += kEvWarps) {
                const int om = m0 + r;
                if (om >= g.Co) continue;
                uint8_t* dl = static_cast<uint8_t*>(a.out0) + (((size_t)b * g.Co + om) * a.Hp + py0) * a.Wp;
                const uint8_t* ml = olat + r * a.pch;
                for (int q = lane; q < nq; q += 32) {
                    const int pr = q / a.Wp, px = q - pr * a.Wp;
                    const uint8_t* r0 = ml + (2 * (py0 + pr) - ya) * a.Wo + 2 * px;
                    const uint32_t m = __vminu4(*reinterpret_cast<const uint16_t*>(r0),
                                                *reinterpret_cast<const uint16_t*>(r0 + a.Wo));
                    dl[q] = (uint8_t)min(m & 0xffu, m >> 8);
                }
            }
            return;
        }
        // one (map, pooled row) per warp iteration: lanes run along the row (no divisions)
        for (int item = warp; item < MB * (py1 - py0); item += kEvWarps) {
            const int r = item / (py1 - py0), py = py0 + item % (py1 - py0);
            const int om = m0 + r;
            if (om >= g.Co) continue;
            uint8_t* dl = static_cast<uint8_t*>(a.out0) + (((size_t)b * g.Co + om) * a.Hp + py) * a.Wp;
            const uint8_t* ml = olat + r * a.pch;
            const int y0 = py * a.pg.Sh - a.pg.Ph;
            if (p2) {  // 2x2/2: two 2-byte reads, byte-SIMD minimum
                const uint8_t* r0 = ml + (y0 - ya) * a.Wo;
                for (int px = lane; px < a.Wp; px += 32) {
                    const uint32_t m = __vminu4(*reinterpret_cast<const uint16_t*>(r0 + 2 * px),
                                                *reinterpret_cast<const uint16_t*>(r0 + a.Wo + 2 * px));
                    dl[px] = (uint8_t)min(m & 0xffu, m >> 8);
                }
                continue;
            }
            const int i0 = max(0, -y0), i1 = min(a.pg.Lh, a.Ho - y0);
            for (int px = lane; px < a.Wp; px += 32) {
                const int x0 = px * a.pg.Sw - a.pg.Pw;
                int m = T;
                for (int i = i0; i < i1; ++i)
                    for (int j = max(0, -x0); j < a.pg.Lw && x0 + j < a.Wo; ++j)
                        m = min(m, (int)ml[(y0 + i - ya) * a.Wo + x0 + j]);
                dl[px] = (uint8_t)m;
            }
        }
        return;
    }
    // coalesced write-out: one run of npix latencies (and P*) per map
    for (int r = warp; r < MB; r += kEvWarps) {
        const int om = m0 + r;
        if (om >= g.Co) continue;
        const size_t base = ((size_t)b * g.Co + om) * a.HWo + p0;
        uint8_t* dl = static_cast<uint8_t*>(a.out0) + base;
        for (int q = lane; q < npix; q += 32) dl[q] = olat[r * a.pch + q];
        if (PSTAR)
            for (int q = lane; q < npix; q += 32) a.out1[base + q] = ops[r * a.pch + q];
    }
}

template <typename ACC, int EPI, bool PSTAR, int NCH, int NW, int MPL>
spk_status launch_ev1(const EvArgs& a, dim3 grid, size_t smem, cudaStream_t s) {
    auto k = conv_event_kernel<ACC, EPI, PSTAR, NCH, NW, MPL>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return spk::launched("conv_event_kernel(attr)");
    spk::launch(k, grid, NW * 32, smem, s, a);
    return spk::launched("conv_event_kernel");
}

template <typename ACC, int EPI, bool PSTAR, int MPL>
spk_status launch_ev_m(const EvArgs& a, dim3 grid, size_t smem, cudaStream_t s) {
    if (a.nw == 8) return launch_ev1<ACC, EPI, PSTAR, 0, 8, MPL>(a, grid, smem, s);
    if constexpr (sizeof(ACC) == 4) {  // K <= 256 always sums in 32 bits
        switch ((a.K + 31) / 32) {
            case 1: return launch_ev1<ACC, EPI, PSTAR, 1, 16, MPL>(a, grid, smem, s);
            case 2: return launch_ev1<ACC, EPI, PSTAR, 2, 16, MPL>(a, grid, smem, s);
            case 3: return launch_ev1<ACC, EPI, PSTAR, 3, 16, MPL>(a, grid, smem, s);
            case 4: return launch_ev1<ACC, EPI, PSTAR, 4, 16, MPL>(a, grid, smem, s);
            case 5: return launch_ev1<ACC, EPI, PSTAR, 5, 16, MPL>(a, grid, smem, s);
            case 6: return launch_ev1<ACC, EPI, PSTAR, 6, 16, MPL>(a, grid, smem, s);
            case 7: return launch_ev1<ACC, EPI, PSTAR, 7, 16, MPL>(a, grid, smem, s);
            case 8: return launch_ev1<ACC, EPI, PSTAR, 8, 16, MPL>(a, grid, smem, s);
            default: break;
        }
    }
    return launch_ev1<ACC, EPI, PSTAR, 0, 16, MPL>(a, grid, smem, s);
}

template <typename ACC, int EPI, bool PSTAR>
spk_status launch_ev(const EvArgs& a, dim3 grid, size_t smem, cudaStream_t s) {
    if (a.mpl == 4) return launch_ev_m<ACC, EPI, PSTAR, 4>(a, grid, smem, s);
    return a.mpl == 2 ? launch_ev_m<ACC, EPI, PSTAR, 2>(a, grid, smem, s) : launch_ev_m<ACC, EPI, PSTAR, 1>(a, grid, smem, s);
}

}  // namespace

bool ev_plan(const spk_conv_geom& g, EvPlan& p, bool fill) {
    p.Ho = (g.Hi + 2 * g.Ph - g.Kh) / g.Sh + 1;
    p.Wo = (g.Wi + 2 * g.Pw - g.Kw) / g.Sw + 1;
    p.K = g.Ci * g.Kh * g.Kw;
    if (g.Kh > 255 || g.Kw > 255 || g.T > 254) return false;
    // several output maps per lane (64 or 128 per CTA) divide the per-pixel sort and list
    // work per map for wide layers; one for narrow ones (Co <= 32)
    static const int mpl_env = [] {
        const char* e = std::getenv("SPK_EV_MPL");  // tuning knob: 1, 2 or 4
        return e ? std::atoi(e) : 0;
    }();
    // (measured: two maps per lane win on every wide layer — C4 conv0 5.26 -> 3.51 ms, C5 conv0
    // 304 -> 236 ms; four lose: the 128-map output staging shrinks the row chunks)
    p.mpl = (mpl_env == 1 || mpl_env == 2 || mpl_env == 4) ? mpl_env : g.Co > 32 ? 2 : 1;
    // the weight rows of a CTA's map block must leave room for the rest (at most 128 KB)
    while (p.mpl > 1 && (size_t)(p.K + 1) * kMB * p.mpl * 4 > 128 * 1024 && mpl_env == 0) p.mpl >>= 1;
    if ((long long)p.K << (15 + (p.mpl == 4 ? 2 : p.mpl == 2 ? 1 : 0)) >= (1ll << 32)) return false;  // list entry
    const int mb = kMB * p.mpl;
    if ((double)g.Ci * g.Hi * g.Wi >= 2147483647.0) return false;
    p.acc64 = (double)p.K * 8388608.0 >= 4294967296.0 ? 1 : 0;
    p.Wq = g.Wi + 2 * g.Pw;
    // whole output rows per CTA: the staged band (with halo) and the output staging must fit;
    // a whole sample per CTA when possible (enables the fused pooling write-out)
    auto band = [&](int r) { return (size_t)g.Ci * (size_t)((r - 1) * g.Sh + g.Kh) * p.Wq; };
    auto smem = [&](int r, int nw) { return ev_smem(p.K, g.T, r * p.Wo, band(r), true, nw, mb).total; };
    int r = std::max(1, std::min(p.Ho, kPchMax / std::max(1, p.Wo)));
    while (r > 1 && (band(r) > (size_t)kStageMax || smem(r, 16) > 200 * 1024)) --r;
    // small batches (C1: one image) would leave most SMs idle with a whole sample per CTA:
    // split the rows until the grid covers ~two CTAs per SM (unfused launches only — the
    // fused pooling write-out keeps its chunking)
    const long long blocks = (long long)g.B * ((g.Co + mb - 1) / mb);
    if (fill && blocks * ((p.Ho + r - 1) / r) < 148) {
        const long long want = (296 + blocks - 1) / blocks;  // row chunks per (sample, map block)
        r = std::max(1, std::min(r, (int)((p.Ho + want - 1) / want)));
    }
    p.nw = 16;
    if (smem(r, 16) > 200 * 1024) p.nw = 8;
    if (band(r) > (size_t)kStageMax * 2 || smem(r, p.nw) > 200 * 1024 || r * p.Wo > 65535) return false;
    p.rpc = r;
    p.pch = r * p.Wo;
    p.band = band(r);
    p.stage = r >= p.Ho ? 1 : 0;  // whole sample in one CTA
    p.smem_bytes = smem(r, p.nw);
    p.n_mb = (g.Co + mb - 1) / mb;
    p.Co_pad = p.n_mb * mb;
    p.MB = mb;
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
    if (w) {  // w == nullptr: the workspace already holds this layer's packed weights (spk_conv_prepack)
        if (cudaMemsetAsync(flag, 0, sizeof(int), s) != cudaSuccess) return spk::launched("memset(flag)");
        const size_t n = (size_t)p.K * p.Co_pad;
        spk::launch(ev_pack_kernel, spk::ceil_div(n, 256), 256, 0, s, w, g.Co, p.K, p.Co_pad, inv_scale23, qT, flag);
        spk_status st = spk::launched("ev_pack_kernel");
        if (st != SPK_OK) return st;
    }
    if (!lat_in) return SPK_OK;  // pack only (spk_conv_prepack)

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
    a.rpc = p.rpc;
    a.Wq = p.Wq;
    a.band = (int)p.band;
    a.mpl = p.mpl;
    if (pool) {  // caller checked: FIRE, whole sample in one CTA
        a.pool = 1;
        a.pg = *pool;
        a.Hp = (p.Ho + 2 * pool->Ph - pool->Lh) / pool->Sh + 1;
        a.Wp = (p.Wo + 2 * pool->Pw - pool->Lw) / pool->Sw + 1;
    }
    const long long theta_q = (long long)std::floor((double)theta * (1073741824.0 / scale));  // tensor path's
    a.th = (uint32_t)std::min<long long>(theta_q >> 7, 0xffffffffll);
    a.out_scale = (float)(scale / 1073741824.0);
    const bool ps = out1 != nullptr && epi == SPK_EPI_FIRE;
    a.nw = p.nw;
    const size_t smem = ev_smem(p.K, g.T, p.pch, p.band, ps, p.nw, p.MB).total;
    // samples go on grid z (<= 65535 per launch): larger batches (rate-coded steps, B' = B T)
    // run as consecutive launches over sample chunks
    const size_t in_b = (size_t)g.Ci * g.Hi * g.Wi;
    const size_t out_b = epi == SPK_EPI_POTENTIAL ? (size_t)g.T * g.Co * a.HWo * sizeof(float)
                                                  : (size_t)g.Co * (a.pool ? (size_t)a.Hp * a.Wp : (size_t)a.HWo);
    const size_t ps_b = (size_t)g.Co * a.HWo;
    spk_status st2 = SPK_OK;
    for (int b0 = 0; b0 < g.B && st2 == SPK_OK; b0 += 65535) {
        EvArgs c = a;
        c.g.B = std::min(65535, g.B - b0);
        c.lat_in = lat_in + (size_t)b0 * in_b;
        c.out0 = static_cast<uint8_t*>(out0) + (size_t)b0 * out_b;
        c.out1 = a.out1 ? a.out1 + (size_t)b0 * ps_b : nullptr;
        const dim3 grid((unsigned)((p.Ho + p.rpc - 1) / p.rpc), (unsigned)p.n_mb, (unsigned)c.g.B);
        if (epi == SPK_EPI_POTENTIAL)
            st2 = p.acc64 ? launch_ev<unsigned long long, SPK_EPI_POTENTIAL, false>(c, grid, smem, s)
                          : launch_ev<uint32_t, SPK_EPI_POTENTIAL, false>(c, grid, smem, s);
        else if (p.acc64)
            st2 = ps ? launch_ev<unsigned long long, SPK_EPI_FIRE, true>(c, grid, smem, s)
                     : launch_ev<unsigned long long, SPK_EPI_FIRE, false>(c, grid, smem, s);
        else
            st2 = ps ? launch_ev<uint32_t, SPK_EPI_FIRE, true>(c, grid, smem, s)
                     : launch_ev<uint32_t, SPK_EPI_FIRE, false>(c, grid, smem, s);
    }
    return st2;
}
