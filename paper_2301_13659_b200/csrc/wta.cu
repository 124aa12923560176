// wta.cu — a7: convolutional k-winners-take-all (convwta(array, radius, count)).
//
// One CTA per sample.  Each live neuron carries the unique 64-bit key
//   lat (8 bits) | ~order(P*) (32 bits) | flat (c,y,x) index (24 bits)
// so "earliest, then higher potential, then lower index" is a plain unsigned
// minimum.  Each of the k greedy rounds is one pass over the sample's records
// with a warp-shuffle + shared-memory min reduction; suppression (whole
// channel + |dy|,|dx| <= radius square in every channel, R-WTA-FOOTPRINT) is
// evaluated against the winners picked so far.
#include "common.cuh"

namespace {

constexpr int kThreads = 1024;
constexpr int kMaxK = 64;

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) {
    return a < b ? a : b;
}

__global__ void __launch_bounds__(kThreads) wta_kernel(const uint8_t* __restrict__ lat,
                                                      const float* __restrict__ pstar, int C, int H,
                                                      int W, int T, int k, int radius,
                                                      spk_winner* __restrict__ win,
                                                      int32_t* __restrict__ nwin) {
    __shared__ int pc[kMaxK], py[kMaxK], px[kMaxK];
    __shared__ unsigned long long red[32];
    __shared__ int npicked;
    const int b = blockIdx.x;
    const int HW = H * W;
    const int N = C * HW;
    const uint8_t* L = lat + (size_t)b * N;
    const float* P = pstar + (size_t)b * N;
    if (threadIdx.x == 0) npicked = 0;
    __syncthreads();
    for (int round = 0; round < k; ++round) {
        const int np = npicked;
        unsigned long long best = ~0ull;
        for (int i = threadIdx.x; i < N; i += kThreads) {
            const int l = __ldg(L + i);
            if (l >= T) continue;
            const int c = i / HW, r = i - c * HW, y = r / W, x = r - y * W;
            bool dead = false;
            for (int q = 0; q < np; ++q)
                if (pc[q] == c || (abs(py[q] - y) <= radius && abs(px[q] - x) <= radius)) {
                    dead = true;
                    break;
                }
            if (dead) continue;
            const unsigned int po = ~spk_float_order_u32(__ldg(P + i));  // higher potential first
            const unsigned long long key =
                ((unsigned long long)l << 56) | ((unsigned long long)po << 24) | (unsigned long long)i;
            best = umin64(best, key);
        }
        for (int o = 16; o; o >>= 1) best = umin64(best, __shfl_xor_sync(0xffffffffu, best, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
        __syncthreads();
        if (threadIdx.x < 32) {
            best = red[threadIdx.x];
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
