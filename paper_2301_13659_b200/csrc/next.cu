// next.cu — the SURVEY §8(f) NEXT-3 / NEXT-4 steps around the hot path:
//   spk_rate_code     rate coding ("Spyker supports rank order and
//                     rate coding"): per-step Bernoulli spikes from a counter-based stream
//   spk_pool_rates    rate-based max pooling (P:L149 `pool(array, kernel, stride, pad, rates)`)
//   spk_rate_gather   firing rate of a rate-coded train (count / T, P:L269 + P:L281)
//   spk_quantize      Listing 4 `spyker.quantize(kernel, 0, 0.5, 1)`
//   spk_fcwta         fully connected winner-take-all (P:L198 `spyker.fcwta`)
// Rate-coded trains are carried as STEP MAPS: u8 [B][T][C][H][W] with 0 where the neuron
// spikes at that step and 1 where it does not — i.e. a one-step latency map (T' = 1) per time
// step, so spk_conv / spk_pool / the fire epilogue run on them unchanged with B' = B*T, T' = 1.
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace {

constexpr int kT = 256;

// ------------------------------------------------------------ rate coding
// pass 1: per-sample maximum of the thresholded values (positive floats order like their
// bits, so an integer atomicMax on the bit pattern is exact and order-independent)
__global__ void __launch_bounds__(kT) rate_max_kernel(const float* __restrict__ y, int N, float thresh,
                                                      unsigned* __restrict__ vmax_bits) {
    spk_pdl_wait();
    const int b = blockIdx.y;
    const float* v = y + (size_t)b * N;
    unsigned m = 0u;
    for (int i = blockIdx.x * kT + threadIdx.x; i < N; i += gridDim.x * kT) {
        const float x = __ldg(v + i);
        if (x > thresh) m = max(m, __float_as_uint(x));  // x > thresh >= 0: positive
    }
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ unsigned red[kT / 32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < kT / 32 ? red[threadIdx.x] : 0u;
        for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0 && m) atomicMax(vmax_bits + b, m);
    }
}

// pass 2: step map out[b][t][i] = 0 if u24(b, t, i) * 2^-24 < p_i else 1, p_i = min(1, v_i / vmax)
// (fp32 IEEE division, as the oracle).  A thread owns 4 consecutive neurons of one sample and walks
// the T steps: p is divided once per neuron, and the generator state of step t+1 is that of step t
// plus N golden increments (the counter advances by N per step), so a draw costs the two
// multiply-xorshift rounds of the mix only.  One 4-byte coalesced store per step.
__device__ __forceinline__ uint64_t mix_state(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void __launch_bounds__(kT) rate_emit_kernel(const float* __restrict__ y, int N, int T, float thresh,
                                                       uint64_t seed, uint64_t b0, const unsigned* __restrict__ vmax_bits,
                                                       uint8_t* __restrict__ out) {
    spk_pdl_wait();
    const int b = blockIdx.y;
    const int i0 = (blockIdx.x * kT + threadIdx.x) * 4;
    if (i0 >= N) return;
    const float vmax = __uint_as_float(vmax_bits[b]);
    const float* v = y + (size_t)b * N;
    const int n = min(4, N - i0);
    float p[4];
    uint64_t z[4];  // splitmix64 state of step 0: seed + (counter + 1) * golden
    const uint64_t c0 = (b0 + (uint64_t)b) * (uint64_t)T * (uint64_t)N;  // counter of (global sample, t = 0, i = 0)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        p[e] = 0.0f;
        if (e < n) {
            const float x = __ldg(v + i0 + e);
            if (vmax > 0.0f && x > thresh) p[e] = fminf(__fdiv_rn(x, vmax), 1.0f);
        }
        z[e] = seed + (c0 + (uint64_t)(i0 + e) + 1ull) * 0x9E3779B97F4A7C15ull;
    }
    const uint64_t step = (uint64_t)N * 0x9E3779B97F4A7C15ull;
    uint8_t* o = out + (size_t)b * T * N + i0;
    const bool vec = n == 4 && ((reinterpret_cast<uintptr_t>(o) & 3) == 0) && (N & 3) == 0;
    for (int t = 0; t < T; ++t) {
        uint32_t word = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t u24 = (uint32_t)(mix_state(z[e]) >> 40);
            const float u = __fmul_rn((float)u24, 5.9604644775390625e-8f);  // exact: 24-bit integer * 2^-24
            word |= ((u < p[e]) ? 0u : 1u) << (8 * e);
            z[e] += step;
        }
        uint8_t* ot = o + (size_t)t * N;
        if (vec) {
            *reinterpret_cast<uint32_t*>(ot) = word;
        } else {
            for (int e = 0; e < n; ++e) ot[e] = (uint8_t)((word >> (8 * e)) & 0xFFu);
        }
    }
}

// ------------------------------------------------------------ rate gather
// rate[b][i] = (#t with step[b][t][i] == 0) / T (R-GATHER on a non-cumulative train)
__global__ void __launch_bounds__(kT) rate_gather_kernel(const uint8_t* __restrict__ step, int B, int T, size_t N,
                                                         float* __restrict__ rate) {
    spk_pdl_wait();
    const size_t q = (size_t)blockIdx.x * kT + threadIdx.x;
    if (q >= (size_t)B * N) return;
    const size_t b = q / N, i = q % N;
    const uint8_t* s = step + b * (size_t)T * N + i;
    int cnt = 0;
    for (int t = 0; t < T; ++t) cnt += (__ldg(s + (size_t)t * N) == 0) ? 1 : 0;
    rate[q] = (float)cnt / (float)T;
}

// ------------------------------------------------------------ rate pooling
// One thread per output cell (b, c, y, x): the window's in-image cell of largest rate (ties:
// lowest flat index iy*W+ix, R-RATE-POOL-TIE) is copied for every step t.
__global__ void __launch_bounds__(kT) pool_rates_kernel(const uint8_t* __restrict__ step, const float* __restrict__ rate,
                                                        int B, int T, int C, int H, int W, spk_pool_geom g, int Ho,
                                                        int Wo, uint8_t* __restrict__ out) {
    spk_pdl_wait();
    const size_t q = (size_t)blockIdx.x * kT + threadIdx.x;
    const size_t plane = (size_t)Ho * Wo;
    if (q >= (size_t)B * C * plane) return;
    const size_t bc = q / plane;
    const int r = (int)(q % plane), y = r / Wo, x = r - y * Wo;
    const int b = (int)(bc / C), c = (int)(bc % C);
    const float* rp = rate + bc * (size_t)H * W;
    int by = -1, bx = -1;
    float br = 0.0f;
    for (int i = 0; i < g.Lh; ++i) {
        const int iy = y * g.Sh - g.Ph + i;
        if (iy < 0 || iy >= H) continue;
        for (int j = 0; j < g.Lw; ++j) {
            const int ix = x * g.Sw - g.Pw + j;
            if (ix < 0 || ix >= W) continue;
            const float v = __ldg(rp + (size_t)iy * W + ix);
            // row-major scan visits flat indices in increasing order: strict > keeps the lowest on ties
            if (by < 0 || v > br) {
                by = iy;
                bx = ix;
                br = v;
            }
        }
    }
    const size_t in_plane = (size_t)H * W, in_t = (size_t)C * in_plane, out_t = (size_t)C * plane;
    const uint8_t* src = step + (size_t)b * T * in_t + (size_t)c * in_plane + (size_t)max(by, 0) * W + max(bx, 0);
    uint8_t* dst = out + (size_t)b * T * out_t + (size_t)c * plane + r;
    for (int t = 0; t < T; ++t) dst[(size_t)t * out_t] = by < 0 ? (uint8_t)1 : __ldg(src + (size_t)t * in_t);
}

// ------------------------------------------------------------ quantize
__global__ void __launch_bounds__(kT) quantize_kernel(float* __restrict__ w, size_t n, float lower, float mid,
                                                      float upper) {
    spk_pdl_wait();
    for (size_t i = (size_t)blockIdx.x * kT + threadIdx.x; i < n; i += (size_t)gridDim.x * kT)
        w[i] = (w[i] < mid) ? lower : upper;
}

// ------------------------------------------------------------ fcwta
// One CTA per sample.  Key of a live neuron o: (lat << 56) | (~order(P*) << 24) | o — the
// least key is the earliest, then the highest potential, then the lowest index (R-FCWTA);
// dead / silent neurons hold ~0.  k rounds of a block-wide minimum; a pick kills |o' - o| <= r.
__device__ __forceinline__ uint64_t fc_key(const uint8_t* lat, const float* ps, int o, int T) {
    const int l = lat[o];
    if (l >= T) return ~0ull;
    const uint32_t ord = spk_float_order_u32(ps[o]);
    return ((uint64_t)l << 56) | ((uint64_t)(~ord) << 24) | (uint64_t)o;
}

__device__ __forceinline__ uint64_t block_min_u64(uint64_t v, uint64_t* red) {
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    v = ~0ull;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = min(v, red[w]);
    __syncthreads();
    return v;
}

__global__ void __launch_bounds__(kT) fcwta_kernel(const uint8_t* __restrict__ lat, const float* __restrict__ pstar,
                                                   int O, int T, int k, int radius, int use_smem,
                                                   spk_winner* __restrict__ win, int32_t* __restrict__ nwin) {
    spk_pdl_wait();
    extern __shared__ uint64_t keys[];  // [O] when use_smem
    __shared__ uint64_t red[kT / 32];
    const int b = blockIdx.x;
    const uint8_t* l = lat + (size_t)b * O;
    const float* p = pstar + (size_t)b * O;
    // dead marks live in the key array (smem) or, for very wide layers, are recomputed each
    // round against the already-picked winners (at most k)
    if (use_smem)
        for (int o = threadIdx.x; o < O; o += kT) keys[o] = fc_key(l, p, o, T);
    __syncthreads();
    __shared__ int picked[64];
    int got = 0;
    for (int q = 0; q < k; ++q) {
        uint64_t m = ~0ull;
        for (int o = threadIdx.x; o < O; o += kT) {
            uint64_t key;
            if (use_smem) {
                key = keys[o];
            } else {
                key = fc_key(l, p, o, T);
                for (int j = 0; j < got && key != ~0ull; ++j)
                    if (abs(o - picked[j]) <= radius) key = ~0ull;
            }
            m = min(m, key);
        }
        m = block_min_u64(m, red);
        if (m == ~0ull) break;
        const int o = (int)(m & 0xFFFFFFull);
        if (threadIdx.x == 0) {
            spk_winner w;
            w.b = b;
            w.t = (int)(m >> 56);
            w.c = o;
            w.y = 0;
            w.x = 0;
            w.cfg = 0;
            win[(size_t)b * k + q] = w;
            if (q < 64) picked[q] = o;
        }
        if (use_smem)
            for (int d = (int)threadIdx.x - radius; d <= radius; d += kT) {
                const int oo = o + d;
                if (oo >= 0 && oo < O) keys[oo] = ~0ull;
            }
        ++got;
        __syncthreads();
    }
    if (threadIdx.x == 0) nwin[b] = got;
    for (int q = got + (int)threadIdx.x; q < k; q += kT) {
        spk_winner w;
        w.b = w.t = w.c = w.y = w.x = w.cfg = -1;
        win[(size_t)b * k + q] = w;
    }
}

}  // namespace

// ============================================================ C ABI
extern "C" size_t spk_rate_code_workspace(int B, int N, int T) {
    (void)N;
    (void)T;
    return B > 0 ? (size_t)B * sizeof(unsigned) : 0;
}

extern "C" spk_status spk_rate_code(const float* y, int B, int N, int T, float thresh, uint64_t seed, uint64_t b0,
                                    uint8_t* step, void* ws, size_t ws_bytes, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(y);
    SPK_CHECK_PTR(step);
    SPK_CHECK(B >= 1 && N >= 1 && T >= 1, SPK_ERR_SHAPE, "B, N, T must be >= 1");
    SPK_CHECK(std::isfinite(thresh) && thresh >= 0.0f, SPK_ERR_ARG, "thresh must be finite and >= 0");
    SPK_CHECK((double)B * T * N < 9.0e18, SPK_ERR_SHAPE, "output too large");
    SPK_CHECK(T <= 65535 && B <= 65535, SPK_ERR_UNSUPPORTED, "T and B <= 65535 (grid dimensions)");
    SPK_CHECK(ws != nullptr && ws_bytes >= spk_rate_code_workspace(B, N, T), SPK_ERR_WORKSPACE,
              "workspace %zu < %zu bytes", ws_bytes, spk_rate_code_workspace(B, N, T));
    cudaStream_t s = spk::as_cuda(stream);
    unsigned* vmax = static_cast<unsigned*>(ws);
    if (cudaMemsetAsync(vmax, 0, (size_t)B * sizeof(unsigned), s) != cudaSuccess) return spk::launched("memset(vmax)");
    const int chunks = std::min(64, (N + kT - 1) / kT);
    spk::launch(rate_max_kernel, dim3(chunks, B), kT, 0, s, y, N, thresh, vmax);
    spk_status st = spk::launched("rate_max_kernel");
    if (st != SPK_OK) return st;
    const unsigned gx = spk::ceil_div((size_t)(N + 3) / 4, kT);
    spk::launch(rate_emit_kernel, dim3(gx, B), kT, 0, s, y, N, T, thresh, seed, b0, vmax, step);
    return spk::launched("rate_emit_kernel");
}

extern "C" spk_status spk_rate_gather(const uint8_t* step, int B, int T, size_t N, float* rate, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(step);
    SPK_CHECK_PTR(rate);
    SPK_CHECK(B >= 1 && T >= 1 && N >= 1, SPK_ERR_SHAPE, "B, T, N must be >= 1");
    spk::launch(rate_gather_kernel, spk::ceil_div((size_t)B * N, kT), kT, 0, spk::as_cuda(stream), step, B, T, N, rate);
    return spk::launched("rate_gather_kernel");
}

extern "C" spk_status spk_pool_rates(const uint8_t* step, const float* rate, int B, int T, int C, int H, int W,
                                     const spk_pool_geom* p, uint8_t* out, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(step);
    SPK_CHECK_PTR(rate);
    SPK_CHECK_PTR(p);
    SPK_CHECK_PTR(out);
    SPK_CHECK(B >= 1 && T >= 1 && C >= 1 && H >= 1 && W >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK(p->Lh >= 1 && p->Lw >= 1 && p->Sh >= 1 && p->Sw >= 1 && p->Ph >= 0 && p->Pw >= 0, SPK_ERR_ARG,
              "bad pooling window/stride/padding");
    SPK_CHECK(H + 2 * p->Ph >= p->Lh && W + 2 * p->Pw >= p->Lw, SPK_ERR_SHAPE, "window larger than padded input (Eq. 3)");
    const int Ho = (H + 2 * p->Ph - p->Lh) / p->Sh + 1, Wo = (W + 2 * p->Pw - p->Lw) / p->Sw + 1;
    const size_t n = (size_t)B * C * Ho * Wo;
    spk::launch(pool_rates_kernel, spk::ceil_div(n, kT), kT, 0, spk::as_cuda(stream), step, rate, B, T, C, H, W, *p, Ho, Wo,
                                                                              out);
    return spk::launched("pool_rates_kernel");
}

extern "C" spk_status spk_quantize(float* w, size_t n, float lower, float mid, float upper, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(w);
    SPK_CHECK(std::isfinite(lower) && std::isfinite(mid) && std::isfinite(upper), SPK_ERR_ARG,
              "quantize levels must be finite");
    SPK_CHECK(lower <= mid && mid <= upper, SPK_ERR_ARG, "quantize needs lower <= mid <= upper");
    if (n == 0) return SPK_OK;
    const unsigned grid = std::min<size_t>(spk::ceil_div(n, kT), 148u * 16u);
    spk::launch(quantize_kernel, grid, kT, 0, spk::as_cuda(stream), w, n, lower, mid, upper);
    return spk::launched("quantize_kernel");
}

extern "C" spk_status spk_fcwta(const uint8_t* lat, const float* pstar, int B, int O, int T, int k, int radius,
                                spk_winner* win, int32_t* nwin, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(pstar);
    SPK_CHECK_PTR(win);
    SPK_CHECK_PTR(nwin);
    SPK_CHECK(B >= 1 && O >= 1 && T >= 1, SPK_ERR_SHAPE, "B, O, T must be >= 1");
    SPK_CHECK(O < (1 << 24), SPK_ERR_UNSUPPORTED, "O < 2^24");
    SPK_CHECK(T <= 254, SPK_ERR_UNSUPPORTED, "T=%d > 254 (u8 latency)", T);
    SPK_CHECK(k >= 1 && radius >= 0, SPK_ERR_ARG, "k >= 1 and radius >= 0");
    const size_t smem = (size_t)O * sizeof(uint64_t);
    const int use_smem = smem <= 200 * 1024 ? 1 : 0;
    SPK_CHECK(use_smem || k <= 64, SPK_ERR_UNSUPPORTED, "fcwta with O > 25600 supports k <= 64");
    cudaStream_t s = spk::as_cuda(stream);
    if (use_smem && smem > 48 * 1024)
        cudaFuncSetAttribute(fcwta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    spk::launch(fcwta_kernel, B, kT, use_smem ? smem : 0, s, lat, pstar, O, T, k, radius, use_smem, win, nwin);
    return spk::launched("fcwta_kernel");
}
