/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of what the Spyker SDNN
 * hot path computes (arXiv 2301.13659, /root/reference/PAPER.md, cited as
 * P:Lnn), written from the paper's definitions on dense BTCHW arrays
 * ("five-dimensional arrays with BTCHW order").  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this file.  It shares no code, header, table or constant generator
 * with the CUDA path (paper_2301_13659_b200/csrc); the two meet only through
 * the seeded input generators in synth/.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (no FMA
 * contraction, so every float expression rounds exactly as written).
 *
 * Precision (DESIGN.md "Readings" R-PREC): the paper fixes four-byte floats
 * for values and 8-bit integers for spikes.  The oracle
 * therefore keeps weights and filter responses in fp32 exactly as the paper's
 * library stores them, and computes convolution potentials in fp64 (sums of
 * fp32 weights accumulated in double, i.e. the exact real sum up to 2^-53).
 * Where a float decides an integer (rank order of filter responses, sort-off
 * binning, the STDP branch) the decision is taken on the fp32 values
 * (task rule: "both sides take that decision in the same precision").
 *
 * Every function below names the passage it follows.  Parity pins live in
 * tests/test_oracle_*.py.  Functions without an independent pin say so
 * ("parity unpinned") — currently none.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------- */
/* O2  Filter kernels (§Feature Enhancement)                        */
/* ------------------------------------------------------------------------- */

/* Isotropic Gaussian sampled at integer offsets on [-r, r]^2 and normalised
 * to unit discrete sum (reading R-DOG-NORM; the paper gives no formula).
 * out[(i)*(2r+1)+j] for offset (i-r, j-r).  Computed in double. */
static void gauss_unit(double sigma, int r, double* out) {
    int e = 2 * r + 1;
    double s = 0.0;
    for (int i = 0; i < e; ++i)
        for (int j = 0; j < e; ++j) {
            double y = (double)(i - r), x = (double)(j - r);
            double g = exp(-(x * x + y * y) / (2.0 * sigma * sigma));
            out[i * e + j] = g;
            s += g;
        }
    for (int i = 0; i < e * e; ++i) out[i] /= s;
}

/* DoG(sigma1, sigma2) = G_sigma1 - G_sigma2  ("Difference of Gaussian",
 * "each description takes in two standard deviations").  `size` of the paper's
 * DoG(size, ...) is the radius r (reading R-RADIUS: P:L302 LoG(3, pad=3) keeps
 * 28x28, "window sizes of the filters are 7").  Rounded to fp32. */
ORC_API void oracle_dog_kernel(double sigma1, double sigma2, int r, float* out) {
    int e = 2 * r + 1;
    double* a = (double*)malloc(sizeof(double) * e * e);
    double* b = (double*)malloc(sizeof(double) * e * e);
    gauss_unit(sigma1, r, a);
    gauss_unit(sigma2, r, b);
    for (int i = 0; i < e * e; ++i) out[i] = (float)(a[i] - b[i]);
    free(a);
    free(b);
}

/* Gabor ("sigma, theta, gamma, lambda, and psi"): the standard formula
 * g = exp(-(x'^2 + gamma^2 y'^2)/(2 sigma^2)) cos(2 pi x'/lambda + psi),
 * x' = x cos(theta) + y sin(theta), y' = -x sin(theta) + y cos(theta),
 * x along columns, y along rows (pointing down).  Unnormalised (R-GABOR). */
ORC_API void oracle_gabor_kernel(double sigma, double theta, double gamma, double lambda,
                                 double psi, int r, float* out) {
    int e = 2 * r + 1;
    for (int i = 0; i < e; ++i)
        for (int j = 0; j < e; ++j) {
            double y = (double)(i - r), x = (double)(j - r);
            double xp = x * cos(theta) + y * sin(theta);
            double yp = -x * sin(theta) + y * cos(theta);
            double g = exp(-(xp * xp + gamma * gamma * yp * yp) / (2.0 * sigma * sigma)) *
                       cos(2.0 * M_PI * xp / lambda + psi);
            out[i * e + j] = (float)g;
        }
}

/* LoG(sigma) ~ {DoG(sigma*sqrt2, sigma/sqrt2), DoG(sigma/sqrt2, sigma*sqrt2)}
 * (P:L80).  out holds 2*n kernels in std-list order. */
ORC_API void oracle_log_kernels(const double* stds, int n, int r, float* out) {
    int e2 = (2 * r + 1) * (2 * r + 1);
    for (int q = 0; q < n; ++q) {
        double s = stds[q];
        oracle_dog_kernel(s * sqrt(2.0), s / sqrt(2.0), r, out + (2 * q) * e2);
        oracle_dog_kernel(s / sqrt(2.0), s * sqrt(2.0), r, out + (2 * q + 1) * e2);
    }
}

/* ------------------------------------------------------------------------- */
/* O1 + O3  Filter application (Eq. 1)                              */
/* ------------------------------------------------------------------------- */

/* Pixel scale: x = (float)u8 / 255.0f (reading R-SCALE).  Each of the K
 * kernels is applied to each input channel separately ("The K_c filters are
 * applied to each channel separately"); output channel ci*K + kc
 * (reading R-CHORDER); Ho = H + 2P - (2r+1) + 1 (Eq. 1, with P_w for the width,
 * reading R-EQ1-TYPO).  Cross-correlation, zero padding.  Accumulation in
 * fp32 with one fused multiply-add per tap in (i, j) row-major order, skipping
 * taps outside the image (reading R-FILTER-ORDER: rank coding is decided by
 * these fp32 values, so the order of rounding is part of the definition). */
ORC_API void oracle_filter(const uint8_t* img, int B, int C, int H, int W, const float* kern,
                           int K, int r, int pad, float* out) {
    int e = 2 * r + 1;
    int Ho = H + 2 * pad - e + 1, Wo = W + 2 * pad - e + 1;
    for (int b = 0; b < B; ++b)
        for (int c = 0; c < C; ++c)
            for (int k = 0; k < K; ++k)
                for (int y = 0; y < Ho; ++y)
                    for (int x = 0; x < Wo; ++x) {
                        float acc = 0.0f;
                        for (int i = 0; i < e; ++i)
                            for (int j = 0; j < e; ++j) {
                                int iy = y - pad + i, ix = x - pad + j;
                                if (iy < 0 || iy >= H || ix < 0 || ix >= W) continue;
                                float v = (float)img[((size_t)(b * C + c) * H + iy) * W + ix] / 255.0f;
                                acc = fmaf(kern[(size_t)k * e * e + i * e + j], v, acc);
                            }
                        out[(((size_t)b * C * K + (size_t)c * K + k) * Ho + y) * Wo + x] = acc;
                    }
}

/* ------------------------------------------------------------------------- */
/* O4  threshold (Listing 1 `spyker.threshold(data, 0.01)`)    */
/* ------------------------------------------------------------------------- */

/* x <- x if x > theta else 0 (strict, reading R-STRICT after P:L125 "higher
 * than a specified threshold"). */
ORC_API void oracle_threshold_f32(float* x, size_t n, float theta) {
    for (size_t i = 0; i < n; ++i)
        if (!(x[i] > theta)) x[i] = 0.0f;
}
ORC_API void oracle_threshold_f64(double* x, size_t n, double theta) {
    for (size_t i = 0; i < n; ++i)
        if (!(x[i] > theta)) x[i] = 0.0;
}

/* ------------------------------------------------------------------------- */
/* O5  Rank-order coding (§Coding in Spyker)                      */
/* ------------------------------------------------------------------------- */

typedef struct { float v; int32_t i; } vi_t;

static int cmp_desc(const void* pa, const void* pb) {
    const vi_t* a = (const vi_t*)pa;
    const vi_t* b = (const vi_t*)pb;
    if (a->v > b->v) return -1;
    if (a->v < b->v) return 1;
    return (a->i < b->i) ? -1 : (a->i > b->i);
}

/* Input y[b][n] is one sample's flat C*H*W response (BTCHW flat order with
 * T=1).  Step 1: threshold (strict) at `thresh`.  Step 2, sort on
 * (default, "Spyker sorts the intensity values by default"): rank the
 * positive values by (value desc, flat index asc) (reading R-TIE), rank r in
 * 0..n-1; "the spikes will be distributed among time steps evenly": first
 * spike step lat = floor(r*T/n) (reading R-BINS); non-positive values never
 * fire (lat = T).  Step 2, sort off ("optionally, it can be disabled", P:L117;
 * reading R-SORTOFF): per sample over the positives,
 * lat = min(T-1, floor(T*(vmax - v)/(vmax - vmin + ulp(vmax)))) with every
 * operation in fp32 in that order.  The cumulative spike train of P:L117 is
 * S[b][t][n] = [lat[b][n] <= t]; oracle_lat_to_dense writes it. */
ORC_API void oracle_rank_code(const float* y, int B, int N, int T, float thresh, int sort,
                              uint8_t* lat) {
    vi_t* buf = (vi_t*)malloc(sizeof(vi_t) * (size_t)(N > 0 ? N : 1));
    for (int b = 0; b < B; ++b) {
        const float* s = y + (size_t)b * N;
        uint8_t* o = lat + (size_t)b * N;
        int n = 0;
        for (int i = 0; i < N; ++i) {
            float v = s[i];
            if (!(v > thresh)) v = 0.0f;
            o[i] = (uint8_t)T;
            if (v > 0.0f) { buf[n].v = v; buf[n].i = i; ++n; }
        }
        if (n == 0) continue;
        if (sort) {
            qsort(buf, (size_t)n, sizeof(vi_t), cmp_desc);
            for (int r = 0; r < n; ++r)
                o[buf[r].i] = (uint8_t)(((long long)r * T) / n);
        } else {
            float vmax = buf[0].v, vmin = buf[0].v;
            for (int q = 1; q < n; ++q) {
                if (buf[q].v > vmax) vmax = buf[q].v;
                if (buf[q].v < vmin) vmin = buf[q].v;
            }
            float ulp = nextafterf(vmax, INFINITY) - vmax;
            float den = (vmax - vmin) + ulp;
            for (int q = 0; q < n; ++q) {
                float num = (float)T * (vmax - buf[q].v);
                float f = floorf(num / den);
                int l = (int)f;
                if (l > T - 1) l = T - 1;
                o[buf[q].i] = (uint8_t)l;
            }
        }
    }
    free(buf);
}

/* Cumulative train from first-spike latencies: S[b][t][n] = [lat[b][n] <= t]
 * ("when a neuron fires in time step t_i, it will also fire at time steps
 * t_{i+1} ... t_n"). */
ORC_API void oracle_lat_to_dense(const uint8_t* lat, int B, int T, size_t N, uint8_t* S) {
    for (int b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
            for (size_t n = 0; n < N; ++n)
                S[((size_t)b * T + t) * N + n] = (uint8_t)(lat[(size_t)b * N + n] <= t);
}

/* First spike time of a dense train (T if it never spikes). */
ORC_API void oracle_dense_to_lat(const uint8_t* S, int B, int T, size_t N, uint8_t* lat) {
    for (int b = 0; b < B; ++b)
        for (size_t n = 0; n < N; ++n) {
            int l = T;
            for (int t = 0; t < T; ++t)
                if (S[((size_t)b * T + t) * N + n]) { l = t; break; }
            lat[(size_t)b * N + n] = (uint8_t)l;
        }
}

/* ------------------------------------------------------------------------- */
/* O6  Spiking convolution (Eq. 2)                                */
/* ------------------------------------------------------------------------- */

/* Direct definition: for every b, t, o, y, x
 *   P[b][t][o][y][x] = sum_{c,i,j} W[o][c][i][j] * S[b][t][c][y*Sh-Ph+i][x*Sw-Pw+j]
 * with zero padding, Ho = floor((Hi + 2Ph - Kh)/Sh) + 1 (Eq. 2).  Each time
 * step is convolved independently ("Spyker processes all the time steps at
 * once", P:L117 — the all-at-once form is exactly this per-t convolution of
 * the cumulative input).  Accumulated in double in (c, i, j) order. */
ORC_API void oracle_conv(const uint8_t* S, int B, int T, int Ci, int Hi, int Wi, const float* Wt,
                         int Co, int Kh, int Kw, int Sh, int Sw, int Ph, int Pw, double* P) {
    int Ho = (Hi + 2 * Ph - Kh) / Sh + 1, Wo = (Wi + 2 * Pw - Kw) / Sw + 1;
    for (int b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
            for (int o = 0; o < Co; ++o)
                for (int y = 0; y < Ho; ++y)
                    for (int x = 0; x < Wo; ++x) {
                        double acc = 0.0;
                        for (int c = 0; c < Ci; ++c)
                            for (int i = 0; i < Kh; ++i)
                                for (int j = 0; j < Kw; ++j) {
                                    int iy = y * Sh - Ph + i, ix = x * Sw - Pw + j;
                                    if (iy < 0 || iy >= Hi || ix < 0 || ix >= Wi) continue;
                                    if (S[((((size_t)b * T + t) * Ci + c) * Hi + iy) * Wi + ix])
                                        acc += (double)Wt[(((size_t)o * Ci + c) * Kh + i) * Kw + j];
                                }
                        P[((((size_t)b * T + t) * Co + o) * Ho + y) * Wo + x] = acc;
                    }
}

/* Event form, an independent derivation used as a cross-check and for large
 * parity samples: since each input fires at most once ("neurons fire at
 * most once when using rank order coding") and the train is cumulative
 * (P:L117), S[t] = sum_{tau<=t} [lat == tau], so
 *   P[t] = sum_{tau <= t} H[tau],  H[tau] = sum_{synapses with lat == tau} W.
 * Input is the latency map lat[b][c][y][x] (T = never).  Double. */
ORC_API void oracle_conv_event(const uint8_t* lat, int B, int T, int Ci, int Hi, int Wi,
                               const float* Wt, int Co, int Kh, int Kw, int Sh, int Sw, int Ph,
                               int Pw, double* P) {
    int Ho = (Hi + 2 * Ph - Kh) / Sh + 1, Wo = (Wi + 2 * Pw - Kw) / Sw + 1;
    double* H = (double*)malloc(sizeof(double) * (size_t)(T > 0 ? T : 1));
    for (int b = 0; b < B; ++b)
        for (int o = 0; o < Co; ++o)
            for (int y = 0; y < Ho; ++y)
                for (int x = 0; x < Wo; ++x) {
                    for (int t = 0; t < T; ++t) H[t] = 0.0;
                    for (int c = 0; c < Ci; ++c)
                        for (int i = 0; i < Kh; ++i)
                            for (int j = 0; j < Kw; ++j) {
                                int iy = y * Sh - Ph + i, ix = x * Sw - Pw + j;
                                if (iy < 0 || iy >= Hi || ix < 0 || ix >= Wi) continue;
                                int l = lat[(((size_t)b * Ci + c) * Hi + iy) * Wi + ix];
                                if (l < T) H[l] += (double)Wt[(((size_t)o * Ci + c) * Kh + i) * Kw + j];
                            }
                    double run = 0.0;
                    for (int t = 0; t < T; ++t) {
                        run += H[t];
                        P[((((size_t)b * T + t) * Co + o) * Ho + y) * Wo + x] = run;
                    }
                }
    free(H);
}

/* ------------------------------------------------------------------------- */
/* O7  IF activation: fire (Listing 3/5 `spyker.fire`)                */
/* ------------------------------------------------------------------------- */

/* "produces spikes where neurons have a potential higher than a specified
 * threshold": S = [P > theta] elementwise (strict, R-STRICT). */
ORC_API void oracle_fire(const double* P, size_t n, double theta, uint8_t* S) {
    for (size_t i = 0; i < n; ++i) S[i] = (uint8_t)(P[i] > theta);
}

/* ------------------------------------------------------------------------- */
/* O8  Max pooling (Eq. 3)                                        */
/* ------------------------------------------------------------------------- */

/* Two-dimensional max pooling of each time step of the spike train with
 * window Lh x Lw, stride, zero padding; Ho = floor((Hi + 2Ph - Lh)/Sh) + 1
 * (Eq. 3).  On cumulative trains it "selects neurons that fire earlier". */
ORC_API void oracle_pool(const uint8_t* S, int B, int T, int C, int H, int W, int Lh, int Lw,
                         int Sh, int Sw, int Ph, int Pw, uint8_t* out) {
    int Ho = (H + 2 * Ph - Lh) / Sh + 1, Wo = (W + 2 * Pw - Lw) / Sw + 1;
    for (int b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
            for (int c = 0; c < C; ++c)
                for (int y = 0; y < Ho; ++y)
                    for (int x = 0; x < Wo; ++x) {
                        uint8_t m = 0;
                        for (int i = 0; i < Lh; ++i)
                            for (int j = 0; j < Lw; ++j) {
                                int iy = y * Sh - Ph + i, ix = x * Sw - Pw + j;
                                if (iy < 0 || iy >= H || ix < 0 || ix >= W) continue;
                                uint8_t v = S[((((size_t)b * T + t) * C + c) * H + iy) * W + ix];
                                if (v > m) m = v;
                            }
                        out[((((size_t)b * T + t) * C + c) * Ho + y) * Wo + x] = m;
                    }
}

/* ------------------------------------------------------------------------- */
/* Neuron keys shared by inhibition and WTA                          */
/* ------------------------------------------------------------------------- */

/* On thresholded potentials Q (Listing 3: `threshold(output, th)` leaves
 * potentials above threshold, zero elsewhere): a neuron's firing time is the
 * first t with Q[t] > 0 (T if none) and its potential "internal potential" at
 * that firing time is Q[lat] (reading R-WTA-POT). */
static void neuron_key(const double* Q, int T, size_t stride_t, int* lat, double* pstar) {
    *lat = T;
    *pstar = 0.0;
    for (int t = 0; t < T; ++t)
        if (Q[(size_t)t * stride_t] > 0.0) { *lat = t; *pstar = Q[(size_t)t * stride_t]; return; }
}

/* a precedes b: earlier, then higher potential, then lower index. */
static int key_less(int la, double pa, long long ia, int lb, double pb, long long ib) {
    if (la != lb) return la < lb;
    if (pa != pb) return pa > pb;
    return ia < ib;
}

/* ------------------------------------------------------------------------- */
/* O9  Lateral inhibition                                        */
/* ------------------------------------------------------------------------- */

/* "When a neuron fires at a specific location, lateral inhibition operation
 * inhibits other neurons belonging to other neural maps from firing in that
 * location".  For every (b, y, x): among channels that fire, keep the
 * one that fires first (ties: higher potential at its firing step, then lower
 * channel — the WTA order of P:L198, reading R-INHIBIT-TIE) and zero every
 * time step of every other channel.  Q is BTCHW thresholded potentials,
 * modified in place. */
ORC_API void oracle_inhibit(double* Q, int B, int T, int C, int H, int W) {
    size_t HW = (size_t)H * W, st = (size_t)C * HW;
    for (int b = 0; b < B; ++b)
        for (size_t p = 0; p < HW; ++p) {
            int best = -1, bl = T;
            double bp = 0.0;
            for (int c = 0; c < C; ++c) {
                int l;
                double ps;
                neuron_key(Q + (size_t)b * T * st + (size_t)c * HW + p, T, st, &l, &ps);
                if (l >= T) continue;
                if (best < 0 || key_less(l, ps, c, bl, bp, best)) { best = c; bl = l; bp = ps; }
            }
            if (best < 0) continue;
            for (int c = 0; c < C; ++c) {
                if (c == best) continue;
                for (int t = 0; t < T; ++t) Q[(size_t)b * T * st + (size_t)t * st + (size_t)c * HW + p] = 0.0;
            }
        }
}

/* ------------------------------------------------------------------------- */
/* O10  Convolutional winner-take-all (`convwta(array, radius, count)`)*/
/* ------------------------------------------------------------------------- */

/* "WTA selects neurons that fire earlier, and if the firing time of neurons
 * is the same, then the one that has a higher internal potential will be
 * selected".  Per sample, up to `count` times: among live neurons
 * (fired, not suppressed) pick the minimum of (lat asc, potential desc, flat
 * (c,y,x) asc); emit winner {b, t=lat, c, y, x, cfg=0}; then suppress the
 * winner's whole channel and every neuron of any channel with |dy| <= radius
 * and |dx| <= radius (reading R-WTA-FOOTPRINT).  Stops early when nothing is
 * live.  win is [B][count][6] int32; nwin[B]. */
ORC_API void oracle_wta(const double* Q, int B, int T, int C, int H, int W, int count, int radius,
                        int32_t* win, int32_t* nwin) {
    size_t HW = (size_t)H * W, N = (size_t)C * HW;
    uint8_t* dead = (uint8_t*)malloc(N ? N : 1);
    int* lat = (int*)malloc(sizeof(int) * (N ? N : 1));
    double* ps = (double*)malloc(sizeof(double) * (N ? N : 1));
    for (int b = 0; b < B; ++b) {
        for (size_t n = 0; n < N; ++n) {
            neuron_key(Q + (size_t)b * T * N + n, T, N, &lat[n], &ps[n]);
            dead[n] = (uint8_t)(lat[n] >= T);
        }
        int got = 0;
        for (int q = 0; q < count; ++q) {
            long long best = -1;
            for (size_t n = 0; n < N; ++n) {
                if (dead[n]) continue;
                if (best < 0 || key_less(lat[n], ps[n], (long long)n, lat[best], ps[best], best))
                    best = (long long)n;
            }
            if (best < 0) break;
            int c = (int)(best / HW), y = (int)((best % HW) / W), x = (int)(best % W);
            int32_t* w = win + ((size_t)b * count + q) * 6;
            w[0] = b; w[1] = lat[best]; w[2] = c; w[3] = y; w[4] = x; w[5] = 0;
            ++got;
            for (size_t n = 0; n < HW; ++n) dead[(size_t)c * HW + n] = 1;
            for (int cc = 0; cc < C; ++cc)
                for (int yy = y - radius; yy <= y + radius; ++yy)
                    for (int xx = x - radius; xx <= x + radius; ++xx)
                        if (yy >= 0 && yy < H && xx >= 0 && xx < W) dead[(size_t)cc * HW + (size_t)yy * W + xx] = 1;
        }
        nwin[b] = got;
    }
    free(dead);
    free(lat);
    free(ps);
}

/* ------------------------------------------------------------------------- */
/* O11  STDP (Eq. 4-6)                                            */
/* ------------------------------------------------------------------------- */

/* cfg[k] = {A+, A-, L, U} as float, stab[k] in {0,1}.  For every winner in
 * (b asc, pick order) — "the batch update rule does not differ from
 * single-sample processing" (reading R-BATCH) — with configuration
 * k = winner.cfg, and every synapse (c, i, j) of its receptive field:
 *   t_j = first spike time of input (b, c, y*Sh-Ph+i, x*Sw-Pw+j) (never if
 *         padded or silent, reading R-NEVER), t_i = winner time (R-TI);
 *   A   = A+ if t_j <= t_i else A-   (Eq. 4 first case, reading R-EQ4-TIE);
 *   dW  = A * (W - L) * (U - W) if stabilised (Eq. 4) else A (Eq. 5);
 *   W   = max(L, min(U, W + dW))    (Eq. 6, reading R-EQ6-CLAMP).
 * fp32 arithmetic in exactly that order (weights are fp32).  S_in is
 * the dense BTCHW input train of the layer (Listing 3 `stdp(data, ...)`).
 * Winners with cfg outside [0, ncfg) are skipped. */
ORC_API void oracle_stdp(float* Wt, int Co, int Ci, int Kh, int Kw, int Sh, int Sw, int Ph, int Pw,
                         const uint8_t* S_in, int B, int T, int Hi, int Wi, const int32_t* win,
                         const int32_t* nwin, int count, const float* cfg, const int32_t* stab,
                         int ncfg) {
    size_t HW = (size_t)Hi * Wi;
    for (int b = 0; b < B; ++b)
        for (int q = 0; q < nwin[b]; ++q) {
            const int32_t* w = win + ((size_t)b * count + q) * 6;
            int wb = w[0], ti = w[1], o = w[2], y = w[3], x = w[4], k = w[5];
            if (k < 0 || k >= ncfg) continue;
            float Ap = cfg[4 * k + 0], Am = cfg[4 * k + 1], L = cfg[4 * k + 2], U = cfg[4 * k + 3];
            for (int c = 0; c < Ci; ++c)
                for (int i = 0; i < Kh; ++i)
                    for (int j = 0; j < Kw; ++j) {
                        int iy = y * Sh - Ph + i, ix = x * Sw - Pw + j;
                        int tj = T + 1; /* never */
                        if (iy >= 0 && iy < Hi && ix >= 0 && ix < Wi) {
                            for (int t = 0; t < T; ++t)
                                if (S_in[(((size_t)wb * T + t) * Ci + c) * HW + (size_t)iy * Wi + ix]) { tj = t; break; }
                        }
                        float A = (tj <= ti) ? Ap : Am;
                        float* pw = &Wt[(((size_t)o * Ci + c) * Kh + i) * Kw + j];
                        float W = *pw;
                        float d;
                        if (stab[k]) {
                            float s = (W - L) * (U - W);
                            d = A * s;
                        } else {
                            d = A;
                        }
                        float nw = W + d;
                        if (nw > U) nw = U;
                        if (nw < L) nw = L;
                        *pw = nw;
                    }
        }
}

/* ------------------------------------------------------------------------- */
/* O12  R-STDP routing (Eq. 7)                                    */
/* ------------------------------------------------------------------------- */

/* "R-STDP can be implemented by passing two configurations to a layer (one
 * for rewarding and one for punishing), and mapping each winner neuron to a
 * configuration based on data labels".  A winner of map c belongs to
 * class c / maps_per_class (reading R-CLASSMAP); cfg = 0 (reward) if that
 * class equals the sample's label, else 1 (punish). */
ORC_API void oracle_rstdp_route(int32_t* win, const int32_t* nwin, int B, int count,
                                const int32_t* labels, int maps_per_class) {
    for (int b = 0; b < B; ++b)
        for (int q = 0; q < nwin[b]; ++q) {
            int32_t* w = win + ((size_t)b * count + q) * 6;
            int cls = w[2] / maps_per_class;
            w[5] = (cls == labels[w[0]]) ? 0 : 1;
        }
}

/* ------------------------------------------------------------------------- */
/* O13  gather ("Firing times (divided by number of time steps)",     */
/*      Listing 5 `spyker.gather(data)`)                                      */
/* ------------------------------------------------------------------------- */

/* Feature = number of steps with a spike / T (reading R-GATHER): for a
 * cumulative train that is (T - first spike time) / T. */
ORC_API void oracle_gather(const uint8_t* S, int B, int T, size_t N, float* f) {
    for (int b = 0; b < B; ++b)
        for (size_t n = 0; n < N; ++n) {
            int cnt = 0;
            for (int t = 0; t < T; ++t) cnt += S[((size_t)b * T + t) * N + n] ? 1 : 0;
            f[(size_t)b * N + n] = (float)cnt / (float)T;
        }
}

/* ========================================================================= */
/* NEXT-3 / NEXT-4: rate coding, rate pooling, quantisation,   */
/* fully connected layer and fcwta.  Same conventions as above.               */
/* ========================================================================= */

/* ------------------------------------------------------------------------- */
/* O14  Counter-based generator for rate coding                               */
/* ------------------------------------------------------------------------- */

/* The random numbers the method draws are an input stream both sides generate
 * from the same counter-based definition (task rule: "each side implements the
 * same counter-based generator"): the 64-bit value number `counter` of stream
 * `seed` is splitmix64's output for the state seed + (counter + 1) *
 * 0x9E3779B97F4A7C15 (so seed 0, counter 0 is splitmix64's first output from
 * state 0).  Pinned against splitmix64's published first outputs. */
ORC_API uint64_t oracle_splitmix64(uint64_t seed, uint64_t counter) {
    uint64_t z = seed + (counter + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* ------------------------------------------------------------------------- */
/* O15  Rate coding ("the rate of firing is dependent on the       */
/*      intensity of the input value ... may be modeled with a Poisson        */
/*      distribution"; "Spyker supports rank order and rate coding")   */
/* ------------------------------------------------------------------------- */

/* Per sample b of y[B][N] (already thresholded, Listing 1): vmax = largest
 * positive value; p_i = clamp(v_i / vmax, 0, 1) in fp32 (reading R-RATE-P); at
 * every step t an independent Bernoulli(p_i) spike (R-RATE-BERNOULLI: discrete
 * steps, the Poisson process of P:L109 in its per-step form): spike iff
 * u24 * 2^-24 < p_i with u24 = the top 24 bits of value (g*T + t)*N + i of
 * stream `seed` (O14), g = b0 + b the GLOBAL sample index (so a shard of a batch
 * draws exactly the numbers of the same rows of the whole batch).  Spikes are NOT cumulative.  Output: the dense BTCHW
 * train S[B][T][N] in {0,1}.  A sample without positives never fires. */
ORC_API void oracle_rate_code(const float* y, int B, int N, int T, uint64_t seed, uint64_t b0, uint8_t* S) {
    for (int b = 0; b < B; ++b) {
        const float* v = y + (size_t)b * N;
        float vmax = 0.0f;
        for (int i = 0; i < N; ++i)
            if (v[i] > vmax) vmax = v[i];
        for (int t = 0; t < T; ++t)
            for (int i = 0; i < N; ++i) {
                float p = 0.0f;
                if (vmax > 0.0f && v[i] > 0.0f) {
                    p = v[i] / vmax;
                    if (p > 1.0f) p = 1.0f;
                }
                uint64_t c = ((b0 + (uint64_t)b) * (uint64_t)T + (uint64_t)t) * (uint64_t)N + (uint64_t)i;
                uint32_t u24 = (uint32_t)(oracle_splitmix64(seed, c) >> 40);
                float u = (float)u24 * 5.9604644775390625e-8f; /* 2^-24, exact */
                S[((size_t)b * T + t) * N + i] = (uint8_t)(u < p);
            }
    }
}

/* ------------------------------------------------------------------------- */
/* O16  Rate-based max pooling ("selects neurons that have a higher    */
/*      firing rate when rate coding is used", `pool(array, k, s, p, rates)`) */
/* ------------------------------------------------------------------------- */

/* For every output cell (b, c, y, x) of Eq. 3's geometry: among the in-image
 * cells of its window, the one with the largest rate[b][c][iy][ix] wins (ties:
 * the lowest flat index iy*W + ix, reading R-RATE-POOL-TIE) and its whole
 * spike train S[b][:][c][iy][ix] is copied to the output; a window with no
 * in-image cell outputs no spikes (zero padding). */
ORC_API void oracle_pool_rates(const uint8_t* S, const float* rate, int B, int T, int C, int H, int W, int Lh,
                               int Lw, int Sh, int Sw, int Ph, int Pw, uint8_t* out) {
    int Ho = (H + 2 * Ph - Lh) / Sh + 1, Wo = (W + 2 * Pw - Lw) / Sw + 1;
    for (int b = 0; b < B; ++b)
        for (int c = 0; c < C; ++c)
            for (int y = 0; y < Ho; ++y)
                for (int x = 0; x < Wo; ++x) {
                    int by = -1, bx = -1;
                    float br = 0.0f;
                    for (int i = 0; i < Lh; ++i)
                        for (int j = 0; j < Lw; ++j) {
                            int iy = y * Sh - Ph + i, ix = x * Sw - Pw + j;
                            if (iy < 0 || iy >= H || ix < 0 || ix >= W) continue;
                            float r = rate[(((size_t)b * C + c) * H + iy) * W + ix];
                            if (by < 0 || r > br || (r == br && iy * W + ix < by * W + bx)) {
                                by = iy; bx = ix; br = r;
                            }
                        }
                    for (int t = 0; t < T; ++t) {
                        uint8_t s = 0;
                        if (by >= 0) s = S[((((size_t)b * T + t) * C + c) * H + by) * W + bx];
                        out[((((size_t)b * T + t) * C + c) * Ho + y) * Wo + x] = s;
                    }
                }
}

/* ------------------------------------------------------------------------- */
/* O17  Weight quantisation (Listing 4                            */
/*      `spyker.quantize(network.conv1.kernel, 0, 0.5, 1)`)                   */
/* ------------------------------------------------------------------------- */

/* In place: w <- lower if w < mid else upper (reading R-QUANT: the value mid
 * itself maps to upper). */
ORC_API void oracle_quantize(float* w, size_t n, float lower, float mid, float upper) {
    for (size_t i = 0; i < n; ++i) w[i] = (w[i] < mid) ? lower : upper;
}

/* ------------------------------------------------------------------------- */
/* O18  Fully connected layer ("kernel with I x O shape ... The   */
/*      input has B x T x I ... The output has B x T x O shape")              */
/* ------------------------------------------------------------------------- */

/* P[b][t][o] = sum_i S[b][t][i] * W[i][o], W in the paper's I x O layout,
 * accumulated in double in i order (as O6). */
ORC_API void oracle_fc(const uint8_t* S, int B, int T, int I, const float* W, int O, double* P) {
    for (int b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
            for (int o = 0; o < O; ++o) {
                double acc = 0.0;
                for (int i = 0; i < I; ++i)
                    if (S[((size_t)b * T + t) * I + i]) acc += (double)W[(size_t)i * O + o];
                P[((size_t)b * T + t) * O + o] = acc;
            }
}

/* STDP of a fully connected layer (Eq. 4-6; "a function belonging to fully
 * connected or convolution layers"): as O11 with the receptive field
 * of output neuron o = every input i, weight W[i][o] (I x O layout). */
ORC_API void oracle_fc_stdp(float* Wt, int I, int O, const uint8_t* S_in, int B, int T, const int32_t* win,
                            const int32_t* nwin, int count, const float* cfg, const int32_t* stab, int ncfg) {
    for (int b = 0; b < B; ++b)
        for (int q = 0; q < nwin[b]; ++q) {
            const int32_t* w = win + ((size_t)b * count + q) * 6;
            int wb = w[0], ti = w[1], o = w[2], k = w[5];
            if (k < 0 || k >= ncfg) continue;
            float Ap = cfg[4 * k + 0], Am = cfg[4 * k + 1], L = cfg[4 * k + 2], U = cfg[4 * k + 3];
            for (int i = 0; i < I; ++i) {
                int tj = T + 1;
                for (int t = 0; t < T; ++t)
                    if (S_in[((size_t)wb * T + t) * I + i]) { tj = t; break; }
                float A = (tj <= ti) ? Ap : Am;
                float* pw = &Wt[(size_t)i * O + o];
                float W = *pw;
                float d;
                if (stab[k]) {
                    float s = (W - L) * (U - W);
                    d = A * s;
                } else {
                    d = A;
                }
                float nw = W + d;
                if (nw > U) nw = U;
                if (nw < L) nw = L;
                *pw = nw;
            }
        }
}

/* ------------------------------------------------------------------------- */
/* O19  Fully connected winner-take-all (P:L198 `spyker.fcwta(array, radius,   */
/*      count, threshold)`)                                                    */
/* ------------------------------------------------------------------------- */

/* As O10 over the output index o of thresholded FC potentials Q[B][T][O]:
 * up to `count` greedy picks of (lat asc, potential at lat desc, o asc) among
 * live neurons; a pick suppresses every o' with |o' - o| <= radius (reading
 * R-FCWTA: "radius" spans output indices).  Winner {b, t, o, 0, 0, cfg=0}. */
ORC_API void oracle_fcwta(const double* Q, int B, int T, int O, int count, int radius, int32_t* win,
                          int32_t* nwin) {
    uint8_t* dead = (uint8_t*)malloc(O ? O : 1);
    int* lat = (int*)malloc(sizeof(int) * (O ? O : 1));
    double* ps = (double*)malloc(sizeof(double) * (O ? O : 1));
    for (int b = 0; b < B; ++b) {
        for (int o = 0; o < O; ++o) {
            neuron_key(Q + (size_t)b * T * O + o, T, (size_t)O, &lat[o], &ps[o]);
            dead[o] = (uint8_t)(lat[o] >= T);
        }
        int got = 0;
        for (int q = 0; q < count; ++q) {
            int best = -1;
            for (int o = 0; o < O; ++o) {
                if (dead[o]) continue;
                if (best < 0 || key_less(lat[o], ps[o], o, lat[best], ps[best], best)) best = o;
            }
            if (best < 0) break;
            int32_t* w = win + ((size_t)b * count + q) * 6;
            w[0] = b; w[1] = lat[best]; w[2] = best; w[3] = 0; w[4] = 0; w[5] = 0;
            ++got;
            for (int o = best - radius; o <= best + radius; ++o)
                if (o >= 0 && o < O) dead[o] = 1;
        }
        nwin[b] = got;
    }
    free(dead);
    free(lat);
    free(ps);
}
