// neuron.cu — bandwidth-bound per-neuron stages on latency maps:
//   a4 spk_fire (IF on materialised potentials), a5 spk_pool (Eq. 3,
//   P:L140-149), a6 spk_inhibit, a8 spk_rstdp_route (Eq. 7),
//   a9 spk_gather and the dense <-> latency boundary conversions.
#include <algorithm>

#include "common.cuh"

namespace {

constexpr int kT = 256;

// ---------------------------------------------------------------- fire
// One thread per neuron; the T potentials of a neuron are a stride-N column of
// BTCHW, so a warp reads 32 consecutive floats per step (coalesced).
__global__ void fire_kernel(const float* __restrict__ pot, int B, int T, size_t N, float theta,
                            uint8_t* __restrict__ lat, float* __restrict__ pstar) {
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (size_t)B * N) return;
    const size_t b = q / N, i = q % N;
    const float* p = pot + b * (size_t)T * N + i;
    int l = T;
    float ps = 0.0f;
    for (int t = 0; t < T; ++t) {
        const float v = __ldg(p + (size_t)t * N);
        if (v > theta) {  // strict "higher than" (R-STRICT)
            l = t;
            ps = v;
            break;
        }
    }
    lat[q] = (uint8_t)l;
    if (pstar) pstar[q] = ps;
}

// ---------------------------------------------------------------- pool
// Per-step window max of cumulative trains == window min of latencies; padded
// cells never fire.  Grid: x = chunks of one output plane, (y, z) = plane index
// (32-bit index math inside a plane).
__global__ void __launch_bounds__(kT) pool_kernel(const uint8_t* __restrict__ lat, long long BC, int ppy, int H, int W,
                                                  int T, spk_pool_geom g, int Ho, int Wo, uint8_t* __restrict__ out) {
    // blockIdx.y selects a slice of ppy planes; inside it all index math is 32-bit
    const int plane_out = Ho * Wo;
    const int q = blockIdx.x * kT + threadIdx.x;  // < ppy * plane_out <= 2^30
    const long long bc = (long long)blockIdx.y * ppy + q / plane_out;
    if (bc >= BC || q >= ppy * plane_out) return;
    const int r = q % plane_out, y = r / Wo, x = r - y * Wo;
    const int y0 = y * g.Sh - g.Ph, x0 = x * g.Sw - g.Pw;
    const int i0 = max(0, -y0), i1 = min(g.Lh, H - y0), j0 = max(0, -x0), j1 = min(g.Lw, W - x0);
    const uint8_t* p = lat + (size_t)bc * H * W + (long long)y0 * W + x0;
    int m = T;
    for (int i = i0; i < i1; ++i)
        for (int j = j0; j < j1; ++j) m = min(m, (int)__ldg(p + (size_t)i * W + j));
    out[(size_t)bc * plane_out + r] = (uint8_t)min(m, T);
}

// ---------------------------------------------------------------- inhibit
// One CTA per (sample, chunk of <= kInhPix pixels); threads stride over the
// chunk's (channel, pixel) cells so that a sample with few pixels and many maps
// still fills the CTA.  Pass 1: per pixel, shared-memory atomicMin of the unique
// key (lat asc, P* desc, c asc) over firing cells; pass 2: every other firing
// cell of the pixel is set to never.
constexpr int kInhPix = 256;

__global__ void __launch_bounds__(kT) inhibit_kernel(uint8_t* __restrict__ lat, float* __restrict__ pstar, int C,
                                                     int HW, int T) {
    __shared__ unsigned long long best[kInhPix];
    const int b = blockIdx.y, p0 = blockIdx.x * kInhPix;
    const int np = min(kInhPix, HW - p0);
    uint8_t* L = lat + (size_t)b * C * HW + p0;
    float* P = pstar + (size_t)b * C * HW + p0;
    for (int q = threadIdx.x; q < np; q += kT) best[q] = ~0ull;
    __syncthreads();
    const int n = C * np;
    for (int e = threadIdx.x; e < n; e += kT) {
        const int c = e / np, pl = e - c * np;
        const int l = L[(size_t)c * HW + pl];
        if (l >= T) continue;
        const float ps = P[(size_t)c * HW + pl] + 0.0f;  // -0 -> +0: equal potentials tie on c
        const uint32_t pd = ~spk_float_order_u32(ps);        // larger P* -> smaller key
        atomicMin(&best[pl], ((unsigned long long)l << 56) | ((unsigned long long)pd << 24) | (unsigned)c);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += kT) {
        const int c = e / np, pl = e - c * np;
        const size_t o = (size_t)c * HW + pl;
        if (L[o] < T && (unsigned)c != (unsigned)(best[pl] & 0xFFFFFFu)) {
            L[o] = (uint8_t)T;
            P[o] = 0.0f;
        }
    }
}

// ---------------------------------------------------------------- gather
__global__ void gather_kernel(const uint8_t* __restrict__ lat, size_t n, int T, float* __restrict__ f) {
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int l = min((int)lat[q], T);
    f[q] = __fdiv_rn((float)(T - l), (float)T);
}

// ---------------------------------------------------------------- boundary conversions
__global__ void lat_to_dense_kernel(const uint8_t* __restrict__ lat, int B, int T, size_t N,
                                    uint8_t* __restrict__ dense) {
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t total = (size_t)B * T * N;
    if (q >= total) return;
    const size_t i = q % N, t = (q / N) % T, b = q / ((size_t)N * T);
    dense[q] = (uint8_t)(lat[b * N + i] <= t);
}

__global__ void dense_to_lat_kernel(const uint8_t* __restrict__ dense, int B, int T, size_t N,
                                    uint8_t* __restrict__ lat, unsigned int* __restrict__ bad) {
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (size_t)B * N) return;
    const size_t b = q / N, i = q % N;
    int l = T;
    bool ok = true;
    for (int t = 0; t < T; ++t) {
        const uint8_t v = dense[(b * T + t) * N + i];
        if (v > 1) ok = false;
        if (v && l == T) l = t;
        if (!v && l < T) ok = false;  // a 1 followed by a 0: not cumulative
    }
    lat[q] = (uint8_t)l;
    if (!ok) atomicMin(bad, (unsigned int)q);
}

// ---------------------------------------------------------------- R-STDP routing
__global__ void rstdp_route_kernel(spk_winner* __restrict__ win, const int32_t* __restrict__ nwin, int B,
                                   int k, const int32_t* __restrict__ labels, int mpc) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= B * k) return;
    const int b = q / k, s = q % k;
    if (s >= nwin[b]) return;
    spk_winner& w = win[q];
    w.cfg = (w.c / mpc == labels[w.b]) ? 0 : 1;  // reward : punish (R-CLASSMAP)
}

}  // namespace

extern "C" spk_status spk_fire(const float* pot, int B, int T, int C, int H, int W, float theta,
                               uint8_t* lat, float* pstar, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(pot);
    SPK_CHECK_PTR(lat);
    SPK_CHECK(B >= 1 && T >= 1 && C >= 1 && H >= 1 && W >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK(T <= 254, SPK_ERR_UNSUPPORTED, "T > 254");
    const size_t N = (size_t)C * H * W;
    fire_kernel<<<spk::ceil_div((size_t)B * N, kT), kT, 0, spk::as_cuda(stream)>>>(pot, B, T, N, theta, lat,
                                                                                 pstar);
    return spk::launched("fire_kernel");
}

extern "C" spk_status spk_pool(const uint8_t* lat, int B, int C, int H, int W, int T,
                               const spk_pool_geom* p, uint8_t* out, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(p);
    SPK_CHECK_PTR(out);
    SPK_CHECK(B >= 1 && C >= 1 && H >= 1 && W >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK(T >= 1 && T <= 254, SPK_ERR_UNSUPPORTED, "T=%d outside 1..254", T);
    SPK_CHECK(p->Lh >= 1 && p->Lw >= 1 && p->Sh >= 1 && p->Sw >= 1 && p->Ph >= 0 && p->Pw >= 0, SPK_ERR_ARG,
              "bad pool geometry");
    const int Ho = (H + 2 * p->Ph - p->Lh) / p->Sh + 1, Wo = (W + 2 * p->Pw - p->Lw) / p->Sw + 1;
    SPK_CHECK(H + 2 * p->Ph >= p->Lh && W + 2 * p->Pw >= p->Lw && Ho >= 1 && Wo >= 1, SPK_ERR_SHAPE,
              "pool window larger than padded input (Eq. 3)");
    SPK_CHECK((long long)H * W < (1ll << 31), SPK_ERR_SHAPE, "input plane too large");
    SPK_CHECK((long long)Ho * Wo <= (1 << 30), SPK_ERR_SHAPE, "output plane too large");
    const long long BC = (long long)B * C;
    const int plane_out = Ho * Wo;
    const long long ppy = std::min<long long>(BC, std::max(1, (1 << 30) / plane_out));
    const long long gy = (BC + ppy - 1) / ppy;
    SPK_CHECK(gy <= 65535, SPK_ERR_SHAPE, "B*C too large");
    const dim3 grid(spk::ceil_div((size_t)ppy * plane_out, kT), (unsigned)gy);
    pool_kernel<<<grid, kT, 0, spk::as_cuda(stream)>>>(lat, BC, (int)ppy, H, W, T, *p, Ho, Wo, out);
    return spk::launched("pool_kernel");
}

extern "C" spk_status spk_inhibit(uint8_t* lat, float* pstar, int B, int C, int H, int W, int T,
                                  spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(pstar);
    SPK_CHECK(B >= 1 && C >= 1 && H >= 1 && W >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK(T >= 1 && T <= 254, SPK_ERR_UNSUPPORTED, "T=%d outside 1..254", T);
    SPK_CHECK(C < (1 << 24), SPK_ERR_UNSUPPORTED, "C=%d >= 2^24", C);
    SPK_CHECK((long long)H * W < (1ll << 31) && (long long)C * kInhPix < (1ll << 31), SPK_ERR_SHAPE, "map too large");
    SPK_CHECK(B <= 65535, SPK_ERR_SHAPE, "B=%d > 65535", B);
    const int HW = H * W;
    const dim3 grid(spk::ceil_div((size_t)HW, kInhPix), (unsigned)B);
    inhibit_kernel<<<grid, kT, 0, spk::as_cuda(stream)>>>(lat, pstar, C, HW, T);
    return spk::launched("inhibit_kernel");
}

extern "C" spk_status spk_gather(const uint8_t* lat, size_t n, int T, float* feat, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(feat);
    SPK_CHECK(T >= 1 && T <= 254, SPK_ERR_UNSUPPORTED, "T=%d outside 1..254", T);
    if (n == 0) return SPK_OK;
    gather_kernel<<<spk::ceil_div(n, kT), kT, 0, spk::as_cuda(stream)>>>(lat, n, T, feat);
    return spk::launched("gather_kernel");
}

extern "C" spk_status spk_lat_to_dense(const uint8_t* lat, int B, int T, size_t N, uint8_t* dense,
                                       spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(dense);
    SPK_CHECK(B >= 1 && N >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK(T >= 1 && T <= 254, SPK_ERR_UNSUPPORTED, "T=%d outside 1..254", T);
    const size_t n = (size_t)B * T * N;
    lat_to_dense_kernel<<<spk::ceil_div(n, kT), kT, 0, spk::as_cuda(stream)>>>(lat, B, T, N, dense);
    return spk::launched("lat_to_dense_kernel");
}

extern "C" spk_status spk_dense_to_lat(const uint8_t* dense, int B, int T, size_t N, uint8_t* lat,
                                       int32_t* bad_index, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(dense);
    SPK_CHECK_PTR(lat);
    SPK_CHECK_PTR(bad_index);
    SPK_CHECK(B >= 1 && N >= 1, SPK_ERR_SHAPE, "non-positive size");
    SPK_CHECK(T >= 1 && T <= 254, SPK_ERR_UNSUPPORTED, "T=%d outside 1..254", T);
    SPK_CHECK((size_t)B * N < 0x7fffffffull, SPK_ERR_SHAPE, "B*N too large for the i32 bad_index");
    cudaStream_t s = spk::as_cuda(stream);
    if (cudaMemsetAsync(bad_index, 0xff, sizeof(int32_t), s) != cudaSuccess)
        return spk::launched("memset(bad_index)");
    const size_t n = (size_t)B * N;
    dense_to_lat_kernel<<<spk::ceil_div(n, kT), kT, 0, s>>>(dense, B, T, N, lat,
                                                            reinterpret_cast<unsigned int*>(bad_index));
    return spk::launched("dense_to_lat_kernel");
}

extern "C" spk_status spk_rstdp_route(spk_winner* win, const int32_t* nwin, int B, int k,
                                      const int32_t* labels, int maps_per_class, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(win);
    SPK_CHECK_PTR(nwin);
    SPK_CHECK_PTR(labels);
    SPK_CHECK(B >= 1 && k >= 1, SPK_ERR_ARG, "B=%d k=%d", B, k);
    SPK_CHECK(maps_per_class >= 1, SPK_ERR_ARG, "maps_per_class < 1");
    rstdp_route_kernel<<<spk::ceil_div((size_t)B * k, kT), kT, 0, spk::as_cuda(stream)>>>(win, nwin, B, k, labels,
                                                                                        maps_per_class);
    return spk::launched("rstdp_route_kernel");
}
