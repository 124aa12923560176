/*
 * spk.h — C ABI of the B200-native Spyker SDNN hot path (libspk.so).
 *
 * Paper: "Spyker: High-performance Library for Spiking Deep Neural Networks"
 * (arXiv 2301.13659).  P:Lnn cites line nn of the paper text
 * (/root/reference/PAPER.md); DESIGN.md lists every reading taken where the
 * paper is silent (R-*).
 *
 * Conventions for every call
 *  - Pointers marked [dev] are CUDA device pointers on the current device;
 *    [host] pointers are read during the call only.  The caller owns and
 *    allocates every buffer (outputs and workspace); the library allocates
 *    nothing and keeps no per-call state.
 *  - Arrays are dense, contiguous, row-major, batch first.  Spike trains are
 *    carried as first-spike LATENCY MAPS: u8 lat[B][C][H][W], lat = first time
 *    step the neuron is on, lat = T for "never".  This is lossless for the
 *    paper's cumulative trains ("when a neuron fires in time step t_i,
 *    it will also fire at time steps t_{i+1} ... t_n") and T times smaller than
 *    the dense BTCHW u8 array of P:L60; spk_lat_to_dense / spk_dense_to_lat
 *    convert.  T <= 254.
 *  - Calls are asynchronous on `stream` (NULL = legacy default stream) and
 *    capture into CUDA graphs.  Arguments and shapes are validated on the host
 *    BEFORE any launch; a failed validation launches nothing and writes
 *    nothing.  Calls never abort: they return a status and set a thread-local
 *    message readable with spk_last_error().  Data-dependent faults found on
 *    the device are reported through device-side outputs (noted per call).
 *  - Every output is bit-reproducible run to run (no floating-point atomics).
 */
#ifndef SPK_H
#define SPK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* spk_stream; /* == cudaStream_t */

#if defined(__GNUC__)
#define SPK_API __attribute__((visibility("default")))
#else
#define SPK_API
#endif

typedef enum {
    SPK_OK = 0,
    SPK_ERR_ARG = 1,         /* null / misaligned pointer, bad scalar argument */
    SPK_ERR_SHAPE = 2,       /* geometry violates Eq. 1-3, non-positive size, channel mismatch */
    SPK_ERR_UNSUPPORTED = 3, /* valid request this build does not implement (e.g. T > 254) */
    SPK_ERR_WORKSPACE = 4,   /* workspace smaller than the matching *_workspace() query */
    SPK_ERR_CUDA = 5         /* launch failed; spk_last_error() has cudaGetErrorString */
} spk_status;

/* Thread-local text of the last non-OK status of this thread ("" if none). */
SPK_API const char* spk_last_error(void);
/* ABI version of this header (bumped on any signature change). */
SPK_API int spk_abi_version(void);
#define SPK_ABI_VERSION 3
/* Name of the last kernel launched by this thread (diagnostics). */
SPK_API const char* spk_last_kernel(void);
/* Number of kernels this process launched through the library. */
SPK_API uint64_t spk_launch_count(void);

/* ========================================================================
 * a1  Feature enhancement filters (Eq. 1)
 * ======================================================================== */

/* spk_dog — Difference-of-Gaussian filter bank, DoG(size, filters, pad)
 * (P:L70-72); LoG(sigma) is the pair DoG(sigma*sqrt2, sigma/sqrt2),
 * DoG(sigma/sqrt2, sigma*sqrt2) and is requested through this call.
 *   img    [dev]  u8  [B][C][H][W] image; pixel value x = u8 / 255 (R-SCALE).
 *   sigmas [host] double [K][2] = (sigma1, sigma2) per filter, both > 0.
 *   radius        kernel edge 2*radius+1 (the paper's `size`, R-RADIUS), 0..7.
 *   pad           zero padding (P_h = P_w, Eq. 1).
 *   y      [dev]  f32 [B][C*K][Ho][Wo], channel ci*K + k (R-CHORDER),
 *                 Ho = H + 2 pad - 2 radius (Eq. 1).
 * Each Gaussian is normalised to unit discrete sum on [-r, r]^2 (R-DOG-NORM).
 * Each output is an fp32 fused-multiply-add chain over the taps in row-major
 * order skipping taps outside the image (R-FILTER-ORDER).
 * Errors: SPK_ERR_ARG (null, K < 1, sigma <= 0), SPK_ERR_SHAPE (Ho/Wo < 1). */
SPK_API spk_status spk_dog(const uint8_t* img, int B, int C, int H, int W, const double* sigmas, int K,
                   int radius, int pad, float* y, spk_stream stream);

/* spk_log — Laplacian-of-Gaussian bank `spyker.LoG(size, stds, pad)`: each
 * std sigma contributes the pair DoG(sigma*sqrt2, sigma/sqrt2), DoG(sigma/sqrt2, sigma*sqrt2),
 * in std-list order (R-CHORDER), so K = 2n output channels per input channel.
 *   stds [host] double [n], each > 0, 1 <= n <= 1024.  Other arguments, layout and
 * errors as spk_dog. */
SPK_API spk_status spk_log(const uint8_t* img, int B, int C, int H, int W, const double* stds, int n,
                           int radius, int pad, float* y, spk_stream stream);

/* spk_gabor — Gabor filter bank: params [host] double [K][5] =
 * (sigma, theta, gamma, lambda, psi); g = exp(-(x'^2 + gamma^2 y'^2)/(2 sigma^2))
 * * cos(2 pi x'/lambda + psi), x' = x cos theta + y sin theta,
 * y' = -x sin theta + y cos theta (R-GABOR, unnormalised).  Other arguments,
 * layout and errors as spk_dog (sigma, gamma, lambda > 0). */
SPK_API spk_status spk_gabor(const uint8_t* img, int B, int C, int H, int W, const double* params, int K,
                     int radius, int pad, float* y, spk_stream stream);

/* ========================================================================
 * a2  Threshold + rank-order coding (Listing 1)
 * ======================================================================== */

/* Bytes of workspace spk_rank_code needs (0 today; query it anyway). */
SPK_API size_t spk_rank_code_workspace(int B, int N, int T, int sort);

/* spk_rank_code — per sample b: values v = y[b][0..N) (one sample's C*H*W
 * response in BTCHW flat order) are thresholded (v <= thresh -> 0, strict,
 * R-STRICT, `threshold(data, 0.01)` P:L307) and the positives coded into T
 * cumulative bins.
 *   sort = 1 (the paper's default, "Spyker sorts the intensity values"): the
 *     n positives are ranked by (value desc, flat index asc) (R-TIE) and
 *     lat = floor(rank * T / n) ("distributed among time steps evenly",
 *     R-BINS); ranking is per sample.
 *   sort = 0 ("it can be disabled", R-SORTOFF): lat = min(T-1,
 *     floor(T*(vmax - v)/((vmax - vmin) + ulp(vmax)))) in fp32, per sample.
 *   non-positives: lat = T (never).
 *   y   [dev] f32 [B][N];  lat [dev] u8 [B][N].  N <= 2^24.  T in 1..254.
 * Errors: SPK_ERR_ARG, SPK_ERR_SHAPE (N < 1), SPK_ERR_UNSUPPORTED (T > 254),
 * SPK_ERR_WORKSPACE. */
SPK_API spk_status spk_rank_code(const float* y, int B, int N, int T, float thresh, int sort, uint8_t* lat,
                         void* ws, size_t ws_bytes, spk_stream stream);

/* ========================================================================
 * a3  Spiking convolution (Eq. 2) + a4 IF epilogues
 * ======================================================================== */

typedef struct {
    int B, T;            /* batch, time steps */
    int Ci, Hi, Wi;      /* input latency map [B][Ci][Hi][Wi] */
    int Co, Kh, Kw;      /* kernel [Co][Ci][Kh][Kw] */
    int Sh, Sw, Ph, Pw;  /* stride, zero padding (Eq. 2) */
} spk_conv_geom;

typedef struct {
    int Lh, Lw, Sh, Sw, Ph, Pw; /* window, stride, zero padding (Eq. 3) */
} spk_pool_geom;

typedef enum {
    /* fp32 CUDA-core reference variant: potentials accumulated in fp32. */
    SPK_PREC_FP32 = 0,
    /* tcgen05 tensor-core path, exact: weights as 23-bit fixed point
     * w = s * sum_d q_d 2^(8d-23) (three u8 digit planes, s = smallest power of
     * two >= w_max), spikes as u8 {0,1}, kind::i8 MMAs with s32 accumulators;
     * potentials are the exact integer sums rounded once to fp32 (error
     * <= n_active * s * 2^-24 against the fp32-weight sum). */
    SPK_PREC_EXACT_I8 = 1,
    /* event (latency-histogram) form on CUDA cores (the paper's
     * sparse interface): every input fires at most once, so
     * P[t] = sum_{t' <= t} H[t'] with H[t'] the weight sum of the synapses of
     * latency t'; only active synapses are touched.  Same fixed-point weights,
     * integer sums, fire test and rounding as EXACT_I8: outputs are
     * bit-identical to it.  Faster when inputs are sparse and Co is small. */
    SPK_PREC_EVENT = 2
} spk_precision;

typedef enum {
    /* out0 = f32 potentials P[B][T][Co][Ho][Wo] ("internal potentials"). */
    SPK_EPI_POTENTIAL = 0,
    /* IF fire: out0 = u8 lat[B][Co][Ho][Wo] = first t with P[t] > theta
     * (strict, R-STRICT), T if none; out1 (nullable) = f32 P*[B][Co][Ho][Wo] =
     * potential at that step (0 if never) — the record inhibition and WTA need
     * (Listing 3 threshold -> inhibit -> convwta). */
    SPK_EPI_FIRE = 1
} spk_epilogue;

/* Bytes of workspace spk_conv needs for this geometry and precision. */
SPK_API size_t spk_conv_workspace(const spk_conv_geom* g, spk_precision prec);

/* spk_conv — potentials of every time step of the cumulative input train
 *   P[b][t][o][y][x] = sum_{c,i,j} W[o][c][i][j] * [lat_in[b][c][y*Sh-Ph+i][x*Sw-Pw+j] <= t]
 * (Eq. 2; padded taps never fire), Ho = floor((Hi + 2Ph - Kh)/Sh) + 1.
 *   lat_in [dev] u8 [B][Ci][Hi][Wi] (values 0..T; > T treated as never).
 *   w      [dev] f32 [Co][Ci][Kh][Kw], or NULL when `ws` holds the weights packed by
 *          spk_conv_prepack (EXACT_I8 / EVENT); PRECONDITION 0 <= w <= w_max (weights are
 *          non-negative in the paper's bounded STDP, L = 0 — required for the
 *          latency map to be lossless, R-NONNEG).  EXACT_I8 clamps out-of-range
 *          weights into [0, s] and raises the device flag in the workspace
 *          (spk_conv_status reads it).
 *   theta  IF threshold for SPK_EPI_FIRE, >= 0.
 *   ws     workspace of spk_conv_workspace(g, prec) bytes (weight digit planes).
 * Errors: SPK_ERR_ARG (null, theta < 0 or not finite, w_max <= 0),
 * SPK_ERR_SHAPE (Eq. 2 violated, sizes < 1), SPK_ERR_UNSUPPORTED (T > 254, or
 * EXACT_I8 with T > 32, Ci*Kh*Kw > 8192 or Kh,Kw > 16, or EVENT whose weight
 * block does not fit shared memory), SPK_ERR_WORKSPACE, SPK_ERR_CUDA. */
SPK_API spk_status spk_conv(const uint8_t* lat_in, const float* w, const spk_conv_geom* g,
                    spk_precision prec, spk_epilogue epi, float theta, float w_max, void* out0,
                    void* out1, void* ws, size_t ws_bytes, spk_stream stream);

/* spk_conv_prepack — pack a layer's weights into `ws` once (the fixed-point digit
 * planes of EXACT_I8 / the weight block of EVENT, as spk_conv does on every call):
 * a later spk_conv / spk_conv_fire_pool with w == NULL, the same geometry,
 * precision and w_max runs on the packed copy without re-packing (layers whose
 * weights do not change between steps — every layer but the trained one).
 * Errors: as spk_conv (SPK_ERR_ARG for FP32). */
SPK_API spk_status spk_conv_prepack(const float* w, const spk_conv_geom* g, spk_precision prec, float w_max,
                                    void* ws, size_t ws_bytes, spk_stream stream);

/* spk_conv_fire_pool — spk_conv(FIRE) followed by spk_pool (Eq. 3) on its latency
 * map, fused (Listing 5 `fire` then `pool`): out [dev] u8 pooled lat
 * [B][Co][Hp][Wp], Hp = floor((Ho + 2Ph - Lh)/Sh) + 1; the unpooled map is never
 * written and no P* is produced (layers that are not trained need neither).
 * Supported for prec = SPK_PREC_EVENT when a whole output map of a sample fits one
 * CTA — query spk_conv_fire_pool_supported (1 = yes).  ws as spk_conv(EVENT).
 * Errors: as spk_conv; SPK_ERR_UNSUPPORTED when not supported. */
SPK_API int spk_conv_fire_pool_supported(const spk_conv_geom* g, spk_precision prec, const spk_pool_geom* pool);
SPK_API spk_status spk_conv_fire_pool(const uint8_t* lat_in, const float* w, const spk_conv_geom* g,
                                      spk_precision prec, float theta, float w_max, const spk_pool_geom* pool,
                                      uint8_t* out, void* ws, size_t ws_bytes, spk_stream stream);

/* spk_fire — IF activation on materialised potentials (Listing 3
 * `spyker.fire(data, th)`): lat[b][c][y][x] = first t with pot[b][t][c][y][x] >
 * theta (T if none), pstar (nullable) = pot at that step (0 if never).
 *   pot [dev] f32 [B][T][C][H][W] (BTCHW).  Errors: SPK_ERR_ARG, SPK_ERR_SHAPE. */
SPK_API spk_status spk_fire(const float* pot, int B, int T, int C, int H, int W, float theta, uint8_t* lat,
                    float* pstar, spk_stream stream);

/* ========================================================================
 * a5  Max pooling (Eq. 3)
 * ======================================================================== */

/* spk_pool — per-step window max of the cumulative trains == window MIN of
 * latencies ("selects neurons that fire earlier"); zero padding never
 * fires.  lat [dev] u8 [B][C][H][W] -> out [dev] u8 [B][C][Ho][Wo],
 * Ho = floor((H + 2Ph - Lh)/Sh) + 1.  Errors: SPK_ERR_ARG, SPK_ERR_SHAPE. */
SPK_API spk_status spk_pool(const uint8_t* lat, int B, int C, int H, int W, int T, const spk_pool_geom* p,
                    uint8_t* out, spk_stream stream);

/* ========================================================================
 * a6  Lateral inhibition
 * ======================================================================== */

/* spk_inhibit — in place on the (lat, P*) record of spk_conv(FIRE): for every
 * (b, y, x) keep the channel with the least key (lat asc, P* desc, channel
 * asc) among channels that fire (R-INHIBIT-TIE) and set every other channel to
 * never (lat = T, P* = 0).  Locations where nothing fires are untouched.
 *   lat [dev] u8 [B][C][H][W], pstar [dev] f32 [B][C][H][W].
 * Errors: SPK_ERR_ARG, SPK_ERR_SHAPE. */
SPK_API spk_status spk_inhibit(uint8_t* lat, float* pstar, int B, int C, int H, int W, int T,
                       spk_stream stream);

/* ========================================================================
 * a7  k-winners-take-all (convwta(array, radius, count))
 * ======================================================================== */

typedef struct {
    int32_t b, t, c, y, x, cfg; /* sample, firing step t_i, map, row, col, STDP config */
} spk_winner;

/* spk_wta — per sample, up to k greedy picks of the least key (lat asc, P*
 * desc, flat (c, y, x) asc) among live neurons (lat < T, not suppressed); after
 * each pick its whole channel and the square |dy|,|dx| <= radius in every
 * channel are suppressed (R-WTA-FOOTPRINT).  ("WTA selects neurons that fire
 * earlier, and if the firing time of neurons is the same, then the one that
 * has a higher internal potential will be selected".)
 *   win  [dev] spk_winner [B][k] (slots >= nwin[b] are written with -1),
 *   nwin [dev] i32 [B].  cfg of every winner = 0.
 * Errors: SPK_ERR_ARG (k < 1, radius < 0), SPK_ERR_SHAPE. */
SPK_API spk_status spk_wta(const uint8_t* lat, const float* pstar, int B, int C, int H, int W, int T, int k,
                   int radius, spk_winner* win, int32_t* nwin, spk_stream stream);

/* spk_inhibit_wta — spk_inhibit then spk_wta, fused (the trained layer's
 * Listing 3 `inhibit(output)` -> `convwta(output, r, k)`): the
 * winners are exactly spk_wta's on the inhibited records, computed in ONE read
 * of the (lat, P*) record without writing the inhibited map (nothing downstream
 * of the WTA reads it: STDP uses the winners and the layer's INPUT).  The
 * inhibition survivor of a pixel is its least (lat, P* desc, c) key, which is
 * also its least WTA key, so keeping the per-pixel minimum and running the
 * greedy rounds on those keys is exact.  Arguments as spk_wta (lat, pstar are
 * read only).  Errors: as spk_wta; SPK_ERR_UNSUPPORTED when a cluster slice
 * holds more than 12288 pixels (H*W > 98304): use the unfused pair. */
SPK_API spk_status spk_inhibit_wta(const uint8_t* lat, const float* pstar, int B, int C, int H, int W, int T,
                                   int k, int radius, spk_winner* win, int32_t* nwin, spk_stream stream);

/* ========================================================================
 * a8  STDP / R-STDP (Eq. 4-7)
 * ======================================================================== */

typedef struct {
    float a_plus, a_minus; /* A+_k (t_j <= t_i), A-_k (t_j > t_i) */
    float lower, upper;    /* L_k < U_k */
    int32_t stabilize;     /* 1: dW = A (W-L)(U-W) (Eq. 4); 0: dW = A (Eq. 5) */
} spk_stdp_config;         /* spyker.STDPConfig(positive, negative, stabilize, lower, upper) */

/* Bytes of workspace spk_stdp needs. */
SPK_API size_t spk_stdp_workspace(const spk_conv_geom* g, int k);

/* spk_stdp — in-place weight update of a conv layer from its winners
 * (Listing 3 `conv.stdp(data, winners, spikes)`): for winners in (b asc, pick
 * order) (R-BATCH) with config k = winner.cfg, for every synapse
 * (c, i, j): t_j = lat_in[b][c][y*Sh-Ph+i][x*Sw-Pw+j] (never if padded),
 * A = t_j <= t_i ? A+ : A- (R-EQ4-TIE), dW = A*((W-L)*(U-W)) or A,
 * W = min(U, max(L, W + dW)) (R-EQ6-CLAMP) — fp32, this operation order, no
 * contraction: bit-identical to the oracle.
 *   w [dev] f32 [Co][Ci][Kh][Kw] updated in place (exclusive access);
 *   g: geometry of the conv layer whose input is lat_in [dev] u8 [B][Ci][Hi][Wi];
 *   win/nwin [dev] as spk_wta (winner.t = t_i, winner.(y,x) = output position);
 *   cfgs [host] spk_stdp_config [ncfg], 1 <= ncfg <= 8.
 * Winners with cfg outside [0, ncfg) or coordinates outside the output (S:L422 errors)
 * are skipped and COUNTED in the workspace: spk_stdp_status reads the count.
 * Errors: SPK_ERR_ARG (L >= U, ncfg out of range), SPK_ERR_SHAPE, SPK_ERR_WORKSPACE. */
SPK_API spk_status spk_stdp(float* w, const spk_conv_geom* g, const uint8_t* lat_in, const spk_winner* win,
                    const int32_t* nwin, int k, const spk_stdp_config* cfgs, int ncfg, void* ws,
                    size_t ws_bytes, spk_stream stream);

/* spk_stdp_status — number of winners the last spk_stdp on `ws` (same g, k) skipped
 * because a coordinate or its cfg was out of range (a data-dependent fault, e.g. a
 * mis-rebased data-parallel winner).  Synchronises `stream`. */
SPK_API spk_status spk_stdp_status(const void* ws, const spk_conv_geom* g, int k, int32_t* invalid_out,
                                   spk_stream stream);

/* spk_rstdp_route — R-STDP configuration routing (Eq. 7: "passing
 * two configurations ... and mapping each winner neuron to a configuration
 * based on data labels"): winner.cfg = 0 (reward) if winner.c / maps_per_class
 * == labels[winner.b], else 1 (punish) (R-CLASSMAP).  labels [dev] i32 [B].
 * Errors: SPK_ERR_ARG. */
SPK_API spk_status spk_rstdp_route(spk_winner* win, const int32_t* nwin, int B, int k,
                           const int32_t* labels, int maps_per_class, spk_stream stream);

/* spk_winners_rebase — data-parallel mini-batch STDP:
 * a rank that forwarded the samples [b0, b0 + B) of a global mini-batch adds b0 to
 * the sample index of each of its valid winners (slots < nwin[b]; empty slots stay
 * -1), so that after an all-gather every replica applies the same winners, in the
 * same (global sample, pick) order, to the global batch's input latency maps (R-BATCH).
 *   win [dev] spk_winner [B][k] (in place), nwin [dev] i32 [B].
 * Errors: SPK_ERR_ARG (B < 1, k < 1, b0 < 0). */
SPK_API spk_status spk_winners_rebase(spk_winner* win, const int32_t* nwin, int B, int k, int b0,
                              spk_stream stream);

/* ========================================================================
 * a9  gather + boundary conversions
 * ======================================================================== */

/* spk_gather — "Firing times (divided by number of time steps)" (P:L269,
 * Listing 5 `spyker.gather`): feat[i] = (T - min(lat[i], T)) / T (R-GATHER).
 * lat [dev] u8 [n], feat [dev] f32 [n]. */
SPK_API spk_status spk_gather(const uint8_t* lat, size_t n, int T, float* feat, spk_stream stream);

/* spk_lat_to_dense — dense cumulative train dense[b][t][i] = (lat[b][i] <= t)
 * (P:L117), BTCHW when N = C*H*W.  lat [dev] u8 [B][N], dense [dev] u8 [B][T][N]. */
SPK_API spk_status spk_lat_to_dense(const uint8_t* lat, int B, int T, size_t N, uint8_t* dense,
                            spk_stream stream);

/* spk_dense_to_lat — first spike of a dense train; bad_index [dev] i32 (one
 * value) receives the smallest flat index b*N + i whose train is not cumulative
 * (a 1 followed by a 0) or holds a value other than 0/1, or -1. */
SPK_API spk_status spk_dense_to_lat(const uint8_t* dense, int B, int T, size_t N, uint8_t* lat,
                            int32_t* bad_index, spk_stream stream);

/* Device-side status of the last EXACT_I8 spk_conv that used `ws`:
 * *flag_out (host) = 1 if a weight was outside [0, s] and was clamped.
 * Synchronises `stream`. */
SPK_API spk_status spk_conv_status(const void* ws, int* flag_out, spk_stream stream);

/* ========================================================================
 * NEXT-3  Rate coding, rate pooling, T = 300 inference (
 *         P:L107-109)
 * ========================================================================
 * Rate-coded trains are NOT cumulative, so they are carried as STEP MAPS:
 * u8 step[B][T][C][H][W] (BTCHW) with 0 where the neuron spikes at
 * step t and 1 where it does not — one one-step latency map (T' = 1) per time
 * step.  spk_conv / spk_conv(FIRE) / spk_pool therefore run on them unchanged
 * with geometry B' = B*T, T' = 1: the potential of step t is the convolution
 * of the spikes of step t (Eq. 2 "time steps independent"), fire gives the
 * next layer's step map, and spk_pool gives the per-step window max ("no
 * rates" pooling).  The dense spike array of P:L60 is S = 1 - step. */

/* Bytes of workspace spk_rate_code needs (4 per sample). */
SPK_API size_t spk_rate_code_workspace(int B, int N, int T);

/* spk_rate_code — per sample b of y[b][0..N): v = y if y > thresh else 0
 * (Listing 1 threshold, strict), vmax = max v; each step t independently
 * spikes with probability p = min(1, v / vmax) (fp32 IEEE division; "the rate
 * of firing is dependent on the intensity", "modeled with a Poisson
 * distribution", P:L109 — per-step Bernoulli form, R-RATE-BERNOULLI):
 * spike iff u24 * 2^-24 < p, u24 = top 24 bits of value ((b0+b)*T + t)*N + i of
 * the counter-based stream `seed` (splitmix64 of seed + (counter+1)*0x9E3779B97F4A7C15,
 * R-RATE-RNG); b0 = global index of sample 0, so a shard draws exactly the numbers
 * of the same rows of the whole batch.  A sample with no value above thresh never spikes.
 *   y [dev] f32 [B][N]; step [dev] u8 [B][T][N] (0 = spike); ws >= spk_rate_code_workspace.
 * Errors: SPK_ERR_ARG, SPK_ERR_SHAPE, SPK_ERR_UNSUPPORTED (B or T > 65535), SPK_ERR_WORKSPACE. */
SPK_API spk_status spk_rate_code(const float* y, int B, int N, int T, float thresh, uint64_t seed, uint64_t b0,
                                 uint8_t* step, void* ws, size_t ws_bytes, spk_stream stream);

/* spk_rate_gather — firing rate of a step map ("firing times divided
 * by the number of time steps" in its rate form; "firing rates as
 * output features"): rate[b][i] = #{t : step[b][t][i] == 0} / T (fp32 of the
 * integer count / T).  step [dev] u8 [B][T][N], rate [dev] f32 [B][N]. */
SPK_API spk_status spk_rate_gather(const uint8_t* step, int B, int T, size_t N, float* rate, spk_stream stream);

/* spk_pool_rates — `spyker.pool(array, kernel, stride, pad, rates)` (P:L149:
 * "selects neurons that have a higher firing rate when rate coding is used"):
 * for every output cell of Eq. 3's geometry the in-image window cell with the
 * largest rate (ties: lowest flat index y*W + x, R-RATE-POOL-TIE) is selected
 * and its whole train copied; a window without in-image cells never spikes.
 *   step [dev] u8 [B][T][C][H][W], rate [dev] f32 [B][C][H][W] (spk_rate_gather),
 *   out [dev] u8 [B][T][C][Ho][Wo].  Errors: SPK_ERR_ARG, SPK_ERR_SHAPE. */
SPK_API spk_status spk_pool_rates(const uint8_t* step, const float* rate, int B, int T, int C, int H, int W,
                                  const spk_pool_geom* p, uint8_t* out, spk_stream stream);

/* ========================================================================
 * NEXT-4  Quantisation, fully connected layer + fcwta, ZCA (
 *         P:L356-366)
 * ======================================================================== */

/* spk_quantize — Listing 4 `spyker.quantize(kernel, lower, mid, upper)`
 * (P:L361): in place w = (w < mid) ? lower : upper (mid maps to upper,
 * R-QUANT).  Binary {0, 1} weights make every potential an integer, so the
 * EXACT_I8 conv then issues one int8 MMA per MAC (only the top digit plane is
 * non-zero; spk_conv skips all-zero planes).  w [dev] f32 [n].
 * Errors: SPK_ERR_ARG (null, non-finite, not lower <= mid <= upper). */
SPK_API spk_status spk_quantize(float* w, size_t n, float lower, float mid, float upper, spk_stream stream);

/* spk_fc — fully connected IF layer ("kernel with I x O shape ...
 * input B x T x I ... output B x T x O"): the 1x1 convolution of a 1x1 map,
 * i.e. spk_conv with geometry {B, T, Ci = I, 1, 1, Co = O, 1, 1, 1, 1, 0, 0}.
 *   lat_in [dev] u8 [B][I] latencies; w [dev] f32 [O][I] — the paper's I x O
 *   kernel stored output-major (its transpose, R-FC-LAYOUT) so each output
 *   neuron's synapses are contiguous, as a conv kernel's are;
 *   POTENTIAL: out0 f32 [B][T][O]; FIRE: out0 u8 lat [B][O], out1 f32 P* [B][O].
 * Workspace, precisions, errors: as spk_conv.  STDP of an FC layer is spk_stdp
 * with the same 1x1 geometry and winners {b, t, o, 0, 0, cfg} (spk_fcwta). */
SPK_API size_t spk_fc_workspace(int B, int T, int I, int O, spk_precision prec);
SPK_API spk_status spk_fc(const uint8_t* lat_in, const float* w, int B, int T, int I, int O, spk_precision prec,
                          spk_epilogue epi, float theta, float w_max, void* out0, void* out1, void* ws,
                          size_t ws_bytes, spk_stream stream);

/* spk_fcwta — `spyker.fcwta(array, radius, count)`: per sample up
 * to k greedy picks of the least key (lat asc, P* desc, o asc) among live
 * neurons (lat < T); a pick suppresses every o' with |o' - o| <= radius
 * (R-FCWTA).  lat [dev] u8 [B][O], pstar [dev] f32 [B][O] (spk_fc FIRE);
 * win [dev] spk_winner [B][k] = {b, t, o, 0, 0, 0} (slots >= nwin[b]: -1),
 * nwin [dev] i32 [B].  Errors: SPK_ERR_ARG, SPK_ERR_SHAPE,
 * SPK_ERR_UNSUPPORTED (O >= 2^24, T > 254, O > 25600 with k > 64). */
SPK_API spk_status spk_fcwta(const uint8_t* lat, const float* pstar, int B, int O, int T, int k, int radius,
                             spk_winner* win, int32_t* nwin, spk_stream stream);

/* spk_zca_fit — ZCA whitening fit ("fit(array, epsilon)", R-ZCA):
 * mu = column means of x[B][F]; C = (x - mu)^T (x - mu) / (B - 1) in fp64 on
 * the device; C = E diag(lam) E^T by a host fp64 symmetric eigensolver
 * (Householder tridiagonalisation + implicit QL — the LAPACK symmetric route
 * the paper names); Wz = E diag((lam + eps)^-1/2) E^T.
 *   x [dev] f32 [B][F]; mean [dev] f32 [F]; wz [dev] f32 [F][F] (symmetric);
 *   ws [dev] >= spk_zca_fit_workspace(B, F) bytes.
 * SYNCHRONOUS: waits for `stream` and uses host scratch (a fit is a one-off).
 * Errors: SPK_ERR_SHAPE (B < 2), SPK_ERR_ARG (eps < 0; eps = 0 with a singular
 * covariance; no convergence), SPK_ERR_UNSUPPORTED (F > 8192), SPK_ERR_WORKSPACE. */
SPK_API size_t spk_zca_fit_workspace(int B, int F);
SPK_API spk_status spk_zca_fit(const float* x, int B, int F, double eps, float* mean, float* wz, void* ws,
                               size_t ws_bytes, spk_stream stream);

/* spk_zca_apply — the ZCA "call": y = (x - mu) Wz in fp32 (one tiled
 * GEMM, centering fused into the operand load).  x, y [dev] f32 [B][F]
 * (y must not alias x), mean [F], wz [F][F].  Errors: SPK_ERR_ARG, SPK_ERR_SHAPE. */
SPK_API spk_status spk_zca_apply(const float* x, int B, int F, const float* mean, const float* wz, float* y,
                                 spk_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* SPK_H */
