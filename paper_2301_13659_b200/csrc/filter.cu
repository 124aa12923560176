// filter.cu — a1: DoG / Gabor (LoG = DoG pairs) feature-enhancement filter banks
// (Eq. 1).  Kernel coefficients are built on the host in double from
// the filter descriptions (tiny, per call) and passed by value; the filtering
// runs on the GPU.
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace {

constexpr int kMaxCoef = 2048;  // K * (2r+1)^2 floats passed by value (8 KB of params)

struct FilterCoef {
    float c[kMaxCoef];
};

// Unit-sum isotropic Gaussian on the integer grid [-r, r]^2 (R-DOG-NORM).
void unit_gaussian(double sigma, int r, std::vector<double>& g) {
    const int e = 2 * r + 1;
    g.assign((size_t)e * e, 0.0);
    double sum = 0.0;
    for (int i = 0; i < e; ++i)
        for (int j = 0; j < e; ++j) {
            const double dy = i - r, dx = j - r;
            const double v = std::exp(-(dx * dx + dy * dy) / (2.0 * sigma * sigma));
            g[(size_t)i * e + j] = v;
            sum += v;
        }
    for (double& v : g) v /= sum;
}

// Filter tile: 32 x 8 outputs of one (b, ci) plane, all K kernels per output pixel.
// The (2R+1)^2 window of a pixel is read from the staged tile into registers once
// and reused by every kernel.  Taps outside the image read a staged 0: the oracle
// skips them, and fmaf(k, 0, acc) == acc exactly because acc starts at +0 and can
// never become -0 (R-FILTER-ORDER), so the fmaf chain — same tap order — is
// bit-identical.
constexpr int TX = 32, TY = 8;

// KC > 0: the kernel count is a compile-time constant (every config: 2, 4 or 6), so each
// coefficient is an immediate constant-bank operand of its FFMA and the KC independent
// fmaf chains of a pixel interleave; KC = 0: runtime kernel count.
// PAIR: kernel 2m+1 is exactly the negation of kernel 2m (on/off DoG and LoG pairs):
// one fmaf chain per pair, the second output is 0 - acc — bit-identical to the negated
// chain (round-to-nearest is symmetric, and an exactly-zero sum is +0 on both sides).
template <int R, int KC, bool PAIR = false>
__global__ void __launch_bounds__(TX* TY) filter_kernel(const uint8_t* __restrict__ img, int C, int H, int W,
                                                       int Kr, int pad, int Ho, int Wo, float* __restrict__ out,
                                                       const FilterCoef coef) {
    spk_pdl_wait();
    constexpr int E = 2 * R + 1, TW = TX + 2 * R, TH = TY + 2 * R;
    __shared__ float tile[TH][TW];
    __shared__ float lut[256];  // u8 / 255 in fp32 (R-SCALE), one IEEE division per value
    const int K = KC > 0 ? (PAIR ? 2 * KC : KC) : Kr;
    const int tid = threadIdx.y * TX + threadIdx.x;
    lut[tid] = __fdiv_rn((float)tid, 255.0f);  // TX * TY == 256
    const int bc = blockIdx.z;  // b * C + ci
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const uint8_t* plane = img + (size_t)bc * H * W;
    __syncthreads();
    // stage the input tile: pixel value u8 / 255 (R-SCALE), outside the image -> 0
    for (int q = tid; q < TH * TW; q += TX * TY) {
        const int ty = q / TW, tx = q - ty * TW;
        const int iy = y0 - pad + ty, ix = x0 - pad + tx;
        float v = 0.0f;
        if (iy >= 0 && iy < H && ix >= 0 && ix < W) v = lut[__ldg(plane + (size_t)iy * W + ix)];
        tile[ty][tx] = v;
    }
    __syncthreads();
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    if (x >= Wo || y >= Ho) return;
    const int b = bc / C, ci = bc - b * C;
    float* o = out + (((size_t)b * C + ci) * K * Ho + y) * Wo + x;
    if constexpr (KC > 0) {
        constexpr int KS = PAIR ? 2 : 1;  // kernel stride between chains
        float acc[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) acc[k] = 0.0f;
#pragma unroll
        for (int i = 0; i < E; ++i)
#pragma unroll
            for (int j = 0; j < E; ++j) {
                const float v = tile[threadIdx.y + i][threadIdx.x + j];
#pragma unroll
                for (int k = 0; k < KC; ++k) acc[k] = __fmaf_rn(coef.c[KS * k * E * E + i * E + j], v, acc[k]);
            }
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            o[(size_t)KS * k * Ho * Wo] = acc[k];
            if (PAIR) o[(size_t)(KS * k + 1) * Ho * Wo] = __fsub_rn(0.0f, acc[k]);
        }
    } else if constexpr (E * E <= 81) {  // window in registers, reused by all K kernels
        float v[E * E];
#pragma unroll
        for (int i = 0; i < E; ++i)
#pragma unroll
            for (int j = 0; j < E; ++j) v[i * E + j] = tile[threadIdx.y + i][threadIdx.x + j];
        for (int k = 0; k < K; ++k) {
            const float* kc = coef.c + k * E * E;
            float acc = 0.0f;
#pragma unroll
            for (int q = 0; q < E * E; ++q) acc = __fmaf_rn(kc[q], v[q], acc);
            o[(size_t)k * Ho * Wo] = acc;
        }
    } else {  // large windows: read the tile per kernel
        for (int k = 0; k < K; ++k) {
            const float* kc = coef.c + k * E * E;
            float acc = 0.0f;
            for (int i = 0; i < E; ++i)
#pragma unroll
                for (int j = 0; j < E; ++j) acc = __fmaf_rn(kc[i * E + j], tile[threadIdx.y + i][threadIdx.x + j], acc);
            o[(size_t)k * Ho * Wo] = acc;
        }
    }
}

// Compile-time kernel count (every config's front end: R = 3, K = 2, 4 or 6): a CTA
// covers 32 x 32 outputs, each thread RY = 4 vertically adjacent pixels.  Every input
// row of the thread's (RY + 2R) x E window is read from shared memory once and feeds
// the RY outputs it overlaps; per output the taps still run i = 0..E-1, j = 0..E-1
// (R-FILTER-ORDER), so the K fmaf chains are the oracle's, bit for bit.
constexpr int RY = 4;

template <int R, int KC, bool PAIR = false>
__global__ void __launch_bounds__(TX* TY) filter_rb_kernel(const uint8_t* __restrict__ img, int C, int H, int W,
                                                          int pad, int Ho, int Wo, float* __restrict__ out,
                                                          const FilterCoef coef) {
    spk_pdl_wait();
    constexpr int E = 2 * R + 1, OY = TY * RY, TW = TX + 2 * R, TH = OY + 2 * R;
    __shared__ float tile[TH][TW];
    __shared__ float lut[256];  // u8 / 255 in fp32 (R-SCALE)
    const int tid = threadIdx.y * TX + threadIdx.x;
    lut[tid] = __fdiv_rn((float)tid, 255.0f);
    const int bc = blockIdx.z;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * OY;
    const uint8_t* plane = img + (size_t)bc * H * W;
    __syncthreads();
    for (int ty = threadIdx.y; ty < TH; ty += TY) {
        const int iy = y0 - pad + ty;
        const bool rowin = iy >= 0 && iy < H;
        for (int tx = threadIdx.x; tx < TW; tx += TX) {
            const int ix = x0 - pad + tx;
            tile[ty][tx] = (rowin && ix >= 0 && ix < W) ? lut[__ldg(plane + (size_t)iy * W + ix)] : 0.0f;
        }
    }
    __syncthreads();
    const int x = x0 + threadIdx.x, yb = y0 + threadIdx.y * RY;
    if (x >= Wo || yb >= Ho) return;
    float acc[RY][KC];
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
        for (int k = 0; k < KC; ++k) acc[r][k] = 0.0f;
#pragma unroll
    for (int iy = 0; iy < RY + 2 * R; ++iy) {
        float v[E];
#pragma unroll
        for (int j = 0; j < E; ++j) v[j] = tile[threadIdx.y * RY + iy][threadIdx.x + j];
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            const int i = iy - r;  // kernel row of this input row for output row r
            if (i < 0 || i >= E) continue;
#pragma unroll
            for (int j = 0; j < E; ++j)
#pragma unroll
                for (int k = 0; k < KC; ++k)
                    acc[r][k] = __fmaf_rn(coef.c[(PAIR ? 2 : 1) * k * E * E + i * E + j], v[j], acc[r][k]);
        }
    }
    const int b = bc / C, ci = bc - b * C;
    constexpr int KO = PAIR ? 2 * KC : KC;  // output kernels
    float* o = out + (((size_t)b * C + ci) * KO * Ho + yb) * Wo + x;
#pragma unroll
    for (int r = 0; r < RY; ++r)
        if (yb + r < Ho)
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                o[(size_t)(PAIR ? 2 * k : k) * Ho * Wo + (size_t)r * Wo] = acc[r][k];
                if (PAIR) o[(size_t)(2 * k + 1) * Ho * Wo + (size_t)r * Wo] = __fsub_rn(0.0f, acc[r][k]);
            }
}

spk_status run_filter(const uint8_t* img, int B, int C, int H, int W, const std::vector<float>& coef,
                      int K, int radius, int pad, float* y, spk_stream stream) {
    const int e = 2 * radius + 1;
    const int Ho = H + 2 * pad - e + 1, Wo = W + 2 * pad - e + 1;
    SPK_CHECK(Ho >= 1 && Wo >= 1, SPK_ERR_SHAPE, "filter output %dx%d (Eq. 1) is empty", Ho, Wo);
    SPK_CHECK((size_t)B * C * K * Ho * Wo < (1ull << 40), SPK_ERR_SHAPE, "output too large");
    FilterCoef fc;
    for (size_t q = 0; q < coef.size(); ++q) fc.c[q] = coef[q];
    dim3 grid(spk::ceil_div(Wo, TX), spk::ceil_div(Ho, TY), (unsigned)(B * C));
    SPK_CHECK(grid.z <= 65535u, SPK_ERR_SHAPE, "B*C=%d > 65535", B * C);
    cudaStream_t s = spk::as_cuda(stream);
    const dim3 blk(TX, TY);
    // exact negation pairs (on/off DoG, LoG): kernel 2m+1 == -kernel 2m for every coefficient
    const int E2 = (2 * radius + 1) * (2 * radius + 1);
    bool pairs = K % 2 == 0;
    for (int k = 0; pairs && k < K; k += 2)
        for (int q = 0; q < E2; ++q)
            if (!(coef[(size_t)(k + 1) * E2 + q] == -coef[(size_t)k * E2 + q])) {
                pairs = false;
                break;
            }
    if (radius == 3 && pairs && (K == 2 || K == 4 || K == 6)) {  // every DoG / LoG front end
        // small maps of few planes (C1: one image) keep one output row per thread, which spreads them
        // over more CTAs; with many planes (C2: 1024 images) the 4-row kernel is faster
        // (21.8 -> 19.8 us, profiles/r02_ab_filter_small.txt)
        const bool small = Ho * Wo < 64 * 64 && (long long)B * C < 2 * 148;
        const dim3 g4(spk::ceil_div(Wo, TX), spk::ceil_div(Ho, TY * RY), (unsigned)(B * C));
        switch (K / 2 + (small ? 0 : 8)) {
            case 1: spk::launch(filter_kernel<3, 1, true>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
            case 2: spk::launch(filter_kernel<3, 2, true>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
            case 3: spk::launch(filter_kernel<3, 3, true>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
            case 9: spk::launch(filter_rb_kernel<3, 1, true>, g4, blk, 0, s, img, C, H, W, pad, Ho, Wo, y, fc); break;
            case 10: spk::launch(filter_rb_kernel<3, 2, true>, g4, blk, 0, s, img, C, H, W, pad, Ho, Wo, y, fc); break;
            default: spk::launch(filter_rb_kernel<3, 3, true>, g4, blk, 0, s, img, C, H, W, pad, Ho, Wo, y, fc); break;
        }
        return spk::launched("filter_kernel<pairs>");
    }
    if (radius == 3 && (K == 1 || K == 2 || K == 4 || K == 6) && Ho * Wo < 64 * 64) {  // small maps (C1-C3)
        switch (K) {
            case 1: spk::launch(filter_kernel<3, 1>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
            case 2: spk::launch(filter_kernel<3, 2>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
            case 4: spk::launch(filter_kernel<3, 4>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
            default: spk::launch(filter_kernel<3, 6>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
        }
        return spk::launched("filter_kernel");
    }
    if (radius == 3 && (K == 1 || K == 2 || K == 4 || K == 6)) {  // large maps (C4, C5)
        const dim3 g4(spk::ceil_div(Wo, TX), spk::ceil_div(Ho, TY * RY), (unsigned)(B * C));
        switch (K) {
            case 1: spk::launch(filter_rb_kernel<3, 1>, g4, blk, 0, s, img, C, H, W, pad, Ho, Wo, y, fc); break;
            case 2: spk::launch(filter_rb_kernel<3, 2>, g4, blk, 0, s, img, C, H, W, pad, Ho, Wo, y, fc); break;
            case 4: spk::launch(filter_rb_kernel<3, 4>, g4, blk, 0, s, img, C, H, W, pad, Ho, Wo, y, fc); break;
            default: spk::launch(filter_rb_kernel<3, 6>, g4, blk, 0, s, img, C, H, W, pad, Ho, Wo, y, fc); break;
        }
        return spk::launched("filter_rb_kernel");
    }
    switch (radius) {
        case 0: spk::launch(filter_kernel<0, 0>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
        case 1: spk::launch(filter_kernel<1, 0>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
        case 2: spk::launch(filter_kernel<2, 0>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
        case 3: spk::launch(filter_kernel<3, 0>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
        case 4: spk::launch(filter_kernel<4, 0>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
        case 5: spk::launch(filter_kernel<5, 0>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
        case 6: spk::launch(filter_kernel<6, 0>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
        default: spk::launch(filter_kernel<7, 0>, grid, blk, 0, s, img, C, H, W, K, pad, Ho, Wo, y, fc); break;
    }
    return spk::launched("filter_kernel");
}

spk_status check_common(const uint8_t* img, int B, int C, int H, int W, const double* p, int K,
                        int radius, int pad, float* y) {
    SPK_CHECK_PTR(img);
    SPK_CHECK_PTR(p);
    SPK_CHECK_PTR(y);
    SPK_CHECK(B >= 1 && C >= 1 && H >= 1 && W >= 1, SPK_ERR_SHAPE, "non-positive image size");
    SPK_CHECK(K >= 1, SPK_ERR_ARG, "K=%d < 1", K);
    SPK_CHECK(radius >= 0 && radius <= 7, SPK_ERR_UNSUPPORTED, "radius %d outside 0..7", radius);
    SPK_CHECK(pad >= 0, SPK_ERR_ARG, "pad < 0");
    SPK_CHECK(K * (2 * radius + 1) * (2 * radius + 1) <= kMaxCoef, SPK_ERR_UNSUPPORTED,
              "K*(2r+1)^2 > %d coefficients", kMaxCoef);
    return SPK_OK;
}

}  // namespace

extern "C" spk_status spk_dog(const uint8_t* img, int B, int C, int H, int W, const double* sigmas,
                              int K, int radius, int pad, float* y, spk_stream stream) {
    spk::clear_error();
    spk_status st = check_common(img, B, C, H, W, sigmas, K, radius, pad, y);
    if (st != SPK_OK) return st;
    const int e = 2 * radius + 1;
    std::vector<float> coef((size_t)K * e * e);
    std::vector<double> g1, g2;
    for (int k = 0; k < K; ++k) {
        const double s1 = sigmas[2 * k], s2 = sigmas[2 * k + 1];
        SPK_CHECK(s1 > 0 && s2 > 0 && std::isfinite(s1) && std::isfinite(s2), SPK_ERR_ARG,
                  "DoG sigmas must be positive");
        unit_gaussian(s1, radius, g1);
        unit_gaussian(s2, radius, g2);
        for (int q = 0; q < e * e; ++q) coef[(size_t)k * e * e + q] = (float)(g1[q] - g2[q]);
    }
    return run_filter(img, B, C, H, W, coef, K, radius, pad, y, stream);
}

// LoG(sigma) ~ {DoG(sigma*sqrt2, sigma/sqrt2), DoG(sigma/sqrt2, sigma*sqrt2)}: the
// pair expansion of `spyker.LoG(size, stds, pad)` is part of the definition, so it lives here,
// behind the ABI, in the std-list order of R-CHORDER.
extern "C" spk_status spk_log(const uint8_t* img, int B, int C, int H, int W, const double* stds, int n,
                              int radius, int pad, float* y, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(stds);
    SPK_CHECK(n >= 1 && n <= 1024, SPK_ERR_ARG, "need 1..1024 LoG standard deviations");
    std::vector<double> pairs((size_t)4 * n);
    const double r2 = std::sqrt(2.0);
    for (int q = 0; q < n; ++q) {
        SPK_CHECK(stds[q] > 0 && std::isfinite(stds[q]), SPK_ERR_ARG, "LoG std %d must be positive", q);
        pairs[4 * q + 0] = stds[q] * r2;
        pairs[4 * q + 1] = stds[q] / r2;
        pairs[4 * q + 2] = stds[q] / r2;
        pairs[4 * q + 3] = stds[q] * r2;
    }
    return spk_dog(img, B, C, H, W, pairs.data(), 2 * n, radius, pad, y, stream);
}

extern "C" spk_status spk_gabor(const uint8_t* img, int B, int C, int H, int W, const double* params,
                                int K, int radius, int pad, float* y, spk_stream stream) {
    spk::clear_error();
    spk_status st = check_common(img, B, C, H, W, params, K, radius, pad, y);
    if (st != SPK_OK) return st;
    const int e = 2 * radius + 1;
    std::vector<float> coef((size_t)K * e * e);
    for (int k = 0; k < K; ++k) {
        const double* p = params + 5 * k;
        const double sigma = p[0], theta = p[1], gamma = p[2], lambda = p[3], psi = p[4];
        SPK_CHECK(sigma > 0 && gamma > 0 && lambda > 0, SPK_ERR_ARG, "Gabor sigma/gamma/lambda must be > 0");
        for (int i = 0; i < e; ++i)
            for (int j = 0; j < e; ++j) {
                const double yy = i - radius, xx = j - radius;
                const double xr = xx * std::cos(theta) + yy * std::sin(theta);
                const double yr = -xx * std::sin(theta) + yy * std::cos(theta);
                const double env = std::exp(-(xr * xr + gamma * gamma * yr * yr) / (2.0 * sigma * sigma));
                coef[(size_t)k * e * e + i * e + j] = (float)(env * std::cos(2.0 * M_PI * xr / lambda + psi));
            }
    }
    return run_filter(img, B, C, H, W, coef, K, radius, pad, y, stream);
}
