// zca.cu — ZCA whitening front end:
//   "Spyker implements an efficient version of ZCA whitening by taking advantage of routines
//    from highly optimized linear algebra libraries (BLAS and LAPACK) that operate on symmetric
//    matrices ... a fit(array, epsilon) and a call function."
// fit:   mean and the symmetric covariance C = Xc^T Xc / (B-1) on the GPU in fp64 (a SYRK: only
//        the upper triangle's tiles are computed and mirrored), then the symmetric
//        eigendecomposition C = E diag(lam) E^T on the host in fp64 (Householder tridiagonal
//        reduction + implicit-shift QL, the LAPACK SYEV route), Wz = E diag((lam+eps)^-1/2) E^T.
// apply: y = (x - mu) Wz — one tiled fp32 GEMM with the centering fused into the operand load.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace {

constexpr int kT = 256;

__global__ void __launch_bounds__(kT) zca_mean_kernel(const float* __restrict__ x, int B, int F,
                                                      double* __restrict__ mean) {
    const int f = blockIdx.x * kT + threadIdx.x;
    if (f >= F) return;
    double s = 0.0;
    for (int b = 0; b < B; ++b) s += (double)__ldg(x + (size_t)b * F + f);
    mean[f] = s / (double)B;
}

// C[i][j] for the 32x32 tile (bi, bj), bj >= bi (upper triangle), mirrored into (bj, bi).
constexpr int CT = 32;
__global__ void __launch_bounds__(CT * 8) zca_cov_kernel(const float* __restrict__ x, int B, int F,
                                                         const double* __restrict__ mean, double* __restrict__ C) {
    const int bi = blockIdx.y, bj = blockIdx.x;
    if (bj < bi) return;
    __shared__ double xa[CT][CT + 1], xb[CT][CT + 1];
    const int tx = threadIdx.x & (CT - 1), ty = threadIdx.x / CT;  // 32 x 8 threads, 4 rows each
    const int i0 = bi * CT, j0 = bj * CT;
    double acc[4] = {0, 0, 0, 0};
    for (int b0 = 0; b0 < B; b0 += CT) {
        for (int r = ty; r < CT; r += 8) {
            const int b = b0 + r;
            const int fi = i0 + tx, fj = j0 + tx;
            xa[r][tx] = (b < B && fi < F) ? (double)__ldg(x + (size_t)b * F + fi) - mean[fi] : 0.0;
            xb[r][tx] = (b < B && fj < F) ? (double)__ldg(x + (size_t)b * F + fj) - mean[fj] : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int r = 0; r < CT; ++r) {
            const double vb = xb[r][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(xa[r][ty + 8 * q], vb, acc[q]);
        }
        __syncthreads();
    }
    const double inv = 1.0 / (double)(B - 1);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = i0 + ty + 8 * q, j = j0 + tx;
        if (i < F && j < F) {
            C[(size_t)i * F + j] = acc[q] * inv;
            C[(size_t)j * F + i] = acc[q] * inv;
        }
    }
}

// y = (x - mu) W: 64 x 64 output tile per CTA, 256 threads x (4 x 4) outputs, K tiles of 16.
constexpr int GT = 64, GK = 16;
__global__ void __launch_bounds__(256) zca_apply_kernel(const float* __restrict__ x, int B, int F,
                                                        const float* __restrict__ mu, const float* __restrict__ W,
                                                        float* __restrict__ y) {
    __shared__ float As[GK][GT + 4];  // As[k][row]
    __shared__ float Bs[GK][GT + 4];  // Bs[k][col]
    const int row0 = blockIdx.y * GT, col0 = blockIdx.x * GT;
    const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < F; k0 += GK) {
        for (int e = threadIdx.x; e < GT * GK; e += 256) {
            const int r = e / GK, k = e % GK;  // x tile: row r, column k0 + k
            const int b = row0 + r, f = k0 + k;
            As[k][r] = (b < B && f < F) ? __fsub_rn(__ldg(x + (size_t)b * F + f), __ldg(mu + f)) : 0.0f;
            const int kk = e / GT, c = e % GT;  // W tile: row k0 + kk, column c
            Bs[kk][c] = (k0 + kk < F && col0 + c < F) ? __ldg(W + (size_t)(k0 + kk) * F + col0 + c) : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < GK; ++k) {
            float a[4], bv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                a[q] = As[k][tr * 4 + q];
                bv[q] = Bs[k][tc * 4 + q];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int b = row0 + tr * 4 + i;
        if (b >= B) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = col0 + tc * 4 + j;
            if (c < F) y[(size_t)b * F + c] = acc[i][j];
        }
    }
}

// ---------------------------------------------------------------- host symmetric eigensolver
// Householder reduction of the symmetric V (row-major n x n) to tridiagonal form, accumulating
// the orthogonal transform in V (d = diagonal, e = sub-diagonal), then implicit-shift QL on the
// tridiagonal matrix, rotating V's columns: on return d holds the eigenvalues and column j of V
// the j-th eigenvector (the EISPACK tred2 / tql2 pair behind LAPACK's symmetric routines).
void tred2(int n, double* V, double* d, double* e) {
    auto v = [&](int i, int j) -> double& { return V[(size_t)i * n + j]; };
    for (int j = 0; j < n; ++j) d[j] = v(n - 1, j);
    for (int i = n - 1; i > 0; --i) {
        double scale = 0.0, h = 0.0;
        for (int k = 0; k < i; ++k) scale += std::fabs(d[k]);
        if (scale == 0.0) {
            e[i] = d[i - 1];
            for (int j = 0; j < i; ++j) {
                d[j] = v(i - 1, j);
                v(i, j) = 0.0;
                v(j, i) = 0.0;
            }
        } else {
            for (int k = 0; k < i; ++k) {
                d[k] /= scale;
                h += d[k] * d[k];
            }
            double f = d[i - 1];
            double g = std::sqrt(h);
            if (f > 0) g = -g;
            e[i] = scale * g;
            h -= f * g;
            d[i - 1] = f - g;
            for (int j = 0; j < i; ++j) e[j] = 0.0;
            for (int j = 0; j < i; ++j) {
                f = d[j];
                v(j, i) = f;
                g = e[j] + v(j, j) * f;
                for (int k = j + 1; k <= i - 1; ++k) {
                    g += v(k, j) * d[k];
                    e[k] += v(k, j) * f;
                }
                e[j] = g;
            }
            f = 0.0;
            for (int j = 0; j < i; ++j) {
                e[j] /= h;
                f += e[j] * d[j];
            }
            const double hh = f / (h + h);
            for (int j = 0; j < i; ++j) e[j] -= hh * d[j];
            for (int j = 0; j < i; ++j) {
                f = d[j];
                g = e[j];
                for (int k = j; k <= i - 1; ++k) v(k, j) -= (f * e[k] + g * d[k]);
                d[j] = v(i - 1, j);
                v(i, j) = 0.0;
            }
        }
        d[i] = h;
    }
    for (int i = 0; i < n - 1; ++i) {
        v(n - 1, i) = v(i, i);
        v(i, i) = 1.0;
        const double h = d[i + 1];
        if (h != 0.0) {
            for (int k = 0; k <= i; ++k) d[k] = v(k, i + 1) / h;
            for (int j = 0; j <= i; ++j) {
                double g = 0.0;
                for (int k = 0; k <= i; ++k) g += v(k, i + 1) * v(k, j);
                for (int k = 0; k <= i; ++k) v(k, j) -= g * d[k];
            }
        }
        for (int k = 0; k <= i; ++k) v(k, i + 1) = 0.0;
    }
    for (int j = 0; j < n; ++j) {
        d[j] = v(n - 1, j);
        v(n - 1, j) = 0.0;
    }
    v(n - 1, n - 1) = 1.0;
    e[0] = 0.0;
}

bool tql2(int n, double* V, double* d, double* e) {
    auto v = [&](int i, int j) -> double& { return V[(size_t)i * n + j]; };
    for (int i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    double f = 0.0, tst1 = 0.0;
    const double eps = std::ldexp(1.0, -52);
    for (int l = 0; l < n; ++l) {
        tst1 = std::max(tst1, std::fabs(d[l]) + std::fabs(e[l]));
        int m = l;
        while (m < n && std::fabs(e[m]) > eps * tst1) ++m;
        if (m == n) m = n - 1;
        if (m > l) {
            int iter = 0;
            do {
                if (++iter > 60) return false;
                double g = d[l];
                double p = (d[l + 1] - g) / (2.0 * e[l]);
                double r = std::hypot(p, 1.0);
                if (p < 0) r = -r;
                d[l] = e[l] / (p + r);
                d[l + 1] = e[l] * (p + r);
                const double dl1 = d[l + 1];
                double h = g - d[l];
                for (int i = l + 2; i < n; ++i) d[i] -= h;
                f += h;
                p = d[m];
                double c = 1.0, c2 = c, c3 = c;
                const double el1 = e[l + 1];
                double s = 0.0, s2 = 0.0;
                for (int i = m - 1; i >= l; --i) {
                    c3 = c2;
                    c2 = c;
                    s2 = s;
                    g = c * e[i];
                    h = c * p;
                    r = std::hypot(p, e[i]);
                    e[i + 1] = s * r;
                    s = e[i] / r;
                    c = p / r;
                    p = c * d[i] - s * g;
                    d[i + 1] = h + s * (c * g + s * d[i]);
                    for (int k = 0; k < n; ++k) {
                        h = v(k, i + 1);
                        v(k, i + 1) = s * v(k, i) + c * h;
                        v(k, i) = c * v(k, i) - s * h;
                    }
                }
                p = -s * s2 * c3 * el1 * e[l] / dl1;
                e[l] = s * p;
                d[l] = c * p;
            } while (std::fabs(e[l]) > eps * tst1);
        }
        d[l] += f;
        e[l] = 0.0;
    }
    return true;
}

}  // namespace

extern "C" size_t spk_zca_fit_workspace(int B, int F) {
    (void)B;
    return F > 0 ? ((size_t)F * F + F) * sizeof(double) : 0;
}

extern "C" spk_status spk_zca_fit(const float* x, int B, int F, double eps, float* mean, float* wz, void* ws,
                                  size_t ws_bytes, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(x);
    SPK_CHECK_PTR(mean);
    SPK_CHECK_PTR(wz);
    SPK_CHECK(B >= 2 && F >= 1, SPK_ERR_SHAPE, "ZCA fit needs B >= 2 rows and F >= 1 features");
    SPK_CHECK(std::isfinite(eps) && eps >= 0.0, SPK_ERR_ARG, "eps must be finite and >= 0");
    SPK_CHECK(F <= 8192, SPK_ERR_UNSUPPORTED, "F <= 8192 (host eigendecomposition)");
    SPK_CHECK(ws != nullptr && ws_bytes >= spk_zca_fit_workspace(B, F), SPK_ERR_WORKSPACE, "workspace %zu < %zu",
              ws_bytes, spk_zca_fit_workspace(B, F));
    cudaStream_t s = spk::as_cuda(stream);
    double* C = static_cast<double*>(ws);
    double* mu = C + (size_t)F * F;
    zca_mean_kernel<<<spk::ceil_div(F, kT), kT, 0, s>>>(x, B, F, mu);
    spk_status st = spk::launched("zca_mean_kernel");
    if (st != SPK_OK) return st;
    const int nt = (F + CT - 1) / CT;
    zca_cov_kernel<<<dim3(nt, nt), CT * 8, 0, s>>>(x, B, F, mu, C);
    st = spk::launched("zca_cov_kernel");
    if (st != SPK_OK) return st;
    // symmetric eigendecomposition on the host (fp64), as the paper's LAPACK route
    std::vector<double> V((size_t)F * F), d(F), e(F), hmu(F);
    if (cudaMemcpyAsync(V.data(), C, V.size() * sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(hmu.data(), mu, F * sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return spk::launched("zca_fit(copy C)");
    tred2(F, V.data(), d.data(), e.data());
    SPK_CHECK(tql2(F, V.data(), d.data(), e.data()), SPK_ERR_ARG, "eigendecomposition did not converge");
    double lmin = d[0];
    for (int j = 1; j < F; ++j) lmin = std::min(lmin, d[j]);
    SPK_CHECK(!(eps == 0.0 && lmin <= 0.0), SPK_ERR_ARG, "singular covariance with eps = 0 (numerical rank < F)");
    // Wz = E diag((lam + eps)^-1/2) E^T
    std::vector<double> sc(F);
    for (int j = 0; j < F; ++j) sc[j] = 1.0 / std::sqrt(std::max(d[j] + eps, 1e-300));
    std::vector<float> W((size_t)F * F), m32(F);
    std::vector<double> row(F);
    for (int i = 0; i < F; ++i) {
        for (int j = 0; j < F; ++j) row[j] = V[(size_t)i * F + j] * sc[j];
        for (int k = i; k < F; ++k) {
            double acc = 0.0;
            const double* vk = &V[(size_t)k * F];
            for (int j = 0; j < F; ++j) acc += row[j] * vk[j];
            W[(size_t)i * F + k] = W[(size_t)k * F + i] = (float)acc;
        }
        m32[i] = (float)hmu[i];
    }
    if (cudaMemcpyAsync(wz, W.data(), W.size() * sizeof(float), cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(mean, m32.data(), F * sizeof(float), cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return spk::launched("zca_fit(copy W)");
    return SPK_OK;
}

extern "C" spk_status spk_zca_apply(const float* x, int B, int F, const float* mean, const float* wz, float* y,
                                    spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(x);
    SPK_CHECK_PTR(mean);
    SPK_CHECK_PTR(wz);
    SPK_CHECK_PTR(y);
    SPK_CHECK(B >= 1 && F >= 1, SPK_ERR_SHAPE, "B, F must be >= 1");
    SPK_CHECK(x != y, SPK_ERR_ARG, "apply is not in place (y must not alias x)");
    const dim3 grid(spk::ceil_div(F, GT), spk::ceil_div(B, GT));
    SPK_CHECK(grid.y <= 65535, SPK_ERR_UNSUPPORTED, "B <= 4194240");
    zca_apply_kernel<<<grid, 256, 0, spk::as_cuda(stream)>>>(x, B, F, mean, wz, y);
    return spk::launched("zca_apply_kernel");
}
