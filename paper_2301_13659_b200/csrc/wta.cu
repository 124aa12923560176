// wta.cu — a7: convolutional k-winners-take-all (convwta(array, radius, count)).
//
// One CTA per sample; the live neurons' keys are compacted into shared memory
// once (when they fit).  Each live neuron carries the unique 64-bit key
//   lat (8 bits) | ~order(P*) (32 bits) | flat (c,y,x) index (24 bits)
// so "earliest, then higher potential, then lower index" is a plain unsigned
// minimum.  Each of the k greedy rounds is one pass over the sample's records
// with a warp-shuffle + shared-memory min reduction; suppression (whole
// channel + |dy|,|dx| <= radius square in every channel, R-WTA-FOOTPRINT) is
// evaluated against the winners picked so far.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kMaxK = 64;
constexpr int kCap = 2048;  // live neurons kept in shared memory (else re-read each round)

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) {
    return a < b ? a : b;
}

__device__ __forceinline__ unsigned long long wta_key(const uint8_t* L, const float* P, int i, int T) {
    const int l = __ldg(L + i);
    if (l >= T) return ~0ull;
    const unsigned int po = ~spk_float_order_u32(__ldg(P + i));  // higher potential first
    return ((unsigned long long)l << 56) | ((unsigned long long)po << 24) | (unsigned long long)i;
}

__global__ void __launch_bounds__(kThreads) wta_kernel(const uint8_t* __restrict__ lat,
                                                      const float* __restrict__ pstar, int C, int H,
                                                      int W, int T, int k, int radius,
                                                      spk_winner* __restrict__ win,
                                                      int32_t* __restrict__ nwin) {
    __shared__ unsigned long long keys[kCap];
    __shared__ int pc[kMaxK], py[kMaxK], px[kMaxK];
    __shared__ unsigned long long red[kThreads / 32];
    __shared__ int npicked;
    __shared__ unsigned int nlive;
    const int b = blockIdx.x;
    const int HW = H * W;
    const int N = C * HW;
    const int lane = threadIdx.x & 31;
    const uint8_t* L = lat + (size_t)b * N;
    const float* P = pstar + (size_t)b * N;
    if (threadIdx.x == 0) {
        npicked = 0;
        nlive = 0;
    }
    __syncthreads();
    // compact the live neurons' keys (order irrelevant: keys are unique)
    for (int i0 = 0; i0 < N; i0 += kThreads) {
        const int i = i0 + threadIdx.x;
        const unsigned long long key = i < N ? wta_key(L, P, i, T) : ~0ull;
        const unsigned m = __ballot_sync(0xffffffffu, key != ~0ull);
        unsigned base = 0;
        if (lane == 0 && m) base = atomicAdd(&nlive, (unsigned)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        const unsigned pos = base + __popc(m & ((1u << lane) - 1u));
        if (key != ~0ull && pos < kCap) keys[pos] = key;
    }
    __syncthreads();
    const int nl = (int)nlive;
    const bool cached = nl <= kCap;
    for (int round = 0; round < k; ++round) {
        const int np = npicked;
        unsigned long long best = ~0ull;
        const int n = cached ? nl : N;
        for (int q = threadIdx.x; q < n; q += kThreads) {
            const unsigned long long key = cached ? keys[q] : wta_key(L, P, q, T);
            if (key == ~0ull) continue;
            const int i = (int)(key & 0xffffffull);
            const int c = i / HW, r = i - c * HW, y = r / W, x = r - y * W;
            bool dead = false;
            for (int t = 0; t < np; ++t)
                if (pc[t] == c || (abs(py[t] - y) <= radius && abs(px[t] - x) <= radius)) {
                    dead = true;
                    break;
                }
            if (!dead) best = umin64(best, key);
        }
        for (int o = 16; o; o >>= 1) best = umin64(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) red[threadIdx.x >> 5] = best;
        __syncthreads();
        if (threadIdx.x < 32) {
            best = lane < kThreads / 32 ? red[lane] : ~0ull;
            for (int o = 16; o; o >>= 1) best = umin64(best, __shfl_xor_sync(0xffffffffu, best, o));
            if (threadIdx.x == 0) {
                spk_winner w;
                if (best != ~0ull) {
                    const int i = (int)(best & 0xffffffull);
                    const int c = i / HW, r = i - c * HW, y = r / W, x = r - y * W;
                    w = {b, (int)(best >> 56), c, y, x, 0};
                    pc[np] = c;
                    py[np] = y;
                    px[np] = x;
                    npicked = np + 1;
                } else {
                    w = {-1, -1, -1, -1, -1, -1};
                }
                win[(size_t)b * k + round] = w;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) nwin[b] = npicked;
}

}  // namespace

extern "C" spk_status spk_wta(const uint8_t* lat, const float* pstar, int B, int C, int H, int W, int T,
                              int k, int radius, spk_winner* win, int32_t* nwin, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(pstar);
    SPK_CHECK_PTR(win);
    SPK_CHECK_PTR(nwin);
    SPK_CHECK(B >= 1 && C >= 1 && H >= 1 && W >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK((long long)C * H * W <= (1 << 24), SPK_ERR_UNSUPPORTED, "C*H*W > 2^24 per sample");
    SPK_CHECK(T >= 1 && T <= 254, SPK_ERR_UNSUPPORTED, "T=%d outside 1..254", T);
    SPK_CHECK(k >= 1 && k <= kMaxK, SPK_ERR_ARG, "k=%d outside 1..%d", k, kMaxK);
    SPK_CHECK(radius >= 0, SPK_ERR_ARG, "radius < 0");
    wta_kernel<<<B, kThreads, 0, spk::as_cuda(stream)>>>(lat, pstar, C, H, W, T, k, radius, win, nwin);
    return spk::launched("wta_kernel");
}
