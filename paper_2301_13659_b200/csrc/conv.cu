// conv.cu — spk_conv entry point: validation (Eq. 2) and dispatch to the
// tcgen05 exact engine (conv_tc.cu) or the fp32 CUDA-core engine (conv_fp32.cu).
#include <cmath>

#include "conv.cuh"

namespace {

spk_status check_geom(const spk_conv_geom* g, int& Ho, int& Wo) {
    SPK_CHECK_PTR(g);
    SPK_CHECK(g->B >= 1 && g->T >= 1 && g->Ci >= 1 && g->Hi >= 1 && g->Wi >= 1 && g->Co >= 1 && g->Kh >= 1 &&
                  g->Kw >= 1,
              SPK_ERR_SHAPE, "non-positive size in conv geometry");
    SPK_CHECK(g->Sh >= 1 && g->Sw >= 1 && g->Ph >= 0 && g->Pw >= 0, SPK_ERR_ARG, "bad stride/padding");
    SPK_CHECK(g->Hi + 2 * g->Ph >= g->Kh && g->Wi + 2 * g->Pw >= g->Kw, SPK_ERR_SHAPE,
              "kernel %dx%d larger than padded input %dx%d (Eq. 2)", g->Kh, g->Kw, g->Hi + 2 * g->Ph,
              g->Wi + 2 * g->Pw);
    SPK_CHECK(g->T <= 254, SPK_ERR_UNSUPPORTED, "T=%d > 254 (u8 latency)", g->T);
    Ho = (g->Hi + 2 * g->Ph - g->Kh) / g->Sh + 1;
    Wo = (g->Wi + 2 * g->Pw - g->Kw) / g->Sw + 1;
    SPK_CHECK((double)g->B * g->Co * Ho * Wo * g->T < 9.0e18, SPK_ERR_SHAPE, "output too large");
    return SPK_OK;
}

}  // namespace

extern "C" size_t spk_conv_workspace(const spk_conv_geom* g, spk_precision prec) {
    if (!g) return 0;
    if (prec == SPK_PREC_EVENT) {
        EvPlan e;
        return ev_plan(*g, e) ? e.ws_bytes : 0;
    }
    if (prec != SPK_PREC_EXACT_I8) return 0;
    TcPlan p;
    if (!tc_plan(*g, p)) return 0;
    return p.ws_bytes;
}

extern "C" spk_status spk_conv(const uint8_t* lat_in, const float* w, const spk_conv_geom* g,
                               spk_precision prec, spk_epilogue epi, float theta, float w_max, void* out0,
                               void* out1, void* ws, size_t ws_bytes, spk_stream stream) {
    spk::clear_error();
    int Ho = 0, Wo = 0;
    spk_status st = check_geom(g, Ho, Wo);
    if (st != SPK_OK) return st;
    SPK_CHECK_PTR(lat_in);
    SPK_CHECK(w != nullptr || prec != SPK_PREC_FP32, SPK_ERR_ARG, "w is null (prepacked weights need EXACT_I8 or EVENT)");
    SPK_CHECK_PTR(out0);
    SPK_CHECK(epi == SPK_EPI_POTENTIAL || epi == SPK_EPI_FIRE, SPK_ERR_ARG, "unknown epilogue %d", (int)epi);
    SPK_CHECK(std::isfinite(theta) && theta >= 0.0f, SPK_ERR_ARG, "theta must be finite and >= 0");
    cudaStream_t s = spk::as_cuda(stream);
    if (prec == SPK_PREC_FP32) return spk_conv_fp32(lat_in, w, g, Ho, Wo, epi, theta, out0, out1, s);
    SPK_CHECK(prec == SPK_PREC_EXACT_I8 || prec == SPK_PREC_EVENT, SPK_ERR_ARG, "unknown precision %d", (int)prec);
    SPK_CHECK(std::isfinite(w_max) && w_max > 0.0f, SPK_ERR_ARG, "w_max must be finite and > 0");
    if (prec == SPK_PREC_EVENT) {
        EvPlan e;
        SPK_CHECK(ev_plan(*g, e, true), SPK_ERR_UNSUPPORTED, "EVENT: a 32-map weight block of K=%d synapses does not fit shared memory",
                  g->Ci * g->Kh * g->Kw);
        SPK_CHECK(ws != nullptr && ws_bytes >= e.ws_bytes, SPK_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes,
                  e.ws_bytes);
        return spk_conv_event(lat_in, w, *g, e, epi, theta, w_max, out0, out1, ws, s);
    }
    TcPlan p;
    SPK_CHECK(tc_plan(*g, p), SPK_ERR_UNSUPPORTED,
              "EXACT_I8 needs T <= 32, Ci*Kh*Kw <= %d, Kh,Kw <= 16, Ci*Hi*Wi < 2^24", kTcMaxK);
    SPK_CHECK(ws != nullptr && ws_bytes >= p.ws_bytes, SPK_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes,
              p.ws_bytes);
    return spk_conv_tc(lat_in, w, *g, p, epi, theta, w_max, out0, out1, ws, s);
}

extern "C" spk_status spk_conv_prepack(const float* w, const spk_conv_geom* g, spk_precision prec, float w_max,
                                       void* ws, size_t ws_bytes, spk_stream stream) {
    spk::clear_error();
    int Ho = 0, Wo = 0;
    spk_status st = check_geom(g, Ho, Wo);
    if (st != SPK_OK) return st;
    SPK_CHECK_PTR(w);
    SPK_CHECK(std::isfinite(w_max) && w_max > 0.0f, SPK_ERR_ARG, "w_max must be finite and > 0");
    cudaStream_t s = spk::as_cuda(stream);
    if (prec == SPK_PREC_EVENT) {
        EvPlan e;
        SPK_CHECK(ev_plan(*g, e, true), SPK_ERR_UNSUPPORTED, "EVENT: weight block does not fit shared memory");
        SPK_CHECK(ws != nullptr && ws_bytes >= e.ws_bytes, SPK_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes,
                  e.ws_bytes);
        return spk_conv_event(nullptr, w, *g, e, SPK_EPI_FIRE, 0.0f, w_max, nullptr, nullptr, ws, s);
    }
    SPK_CHECK(prec == SPK_PREC_EXACT_I8, SPK_ERR_ARG, "prepacking needs EXACT_I8 or EVENT");
    TcPlan p;
    SPK_CHECK(tc_plan(*g, p), SPK_ERR_UNSUPPORTED, "EXACT_I8 geometry not supported");
    SPK_CHECK(ws != nullptr && ws_bytes >= p.ws_bytes, SPK_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes,
              p.ws_bytes);
    return spk_conv_tc(nullptr, w, *g, p, SPK_EPI_FIRE, 0.0f, w_max, nullptr, nullptr, ws, s);
}

extern "C" int spk_conv_fire_pool_supported(const spk_conv_geom* g, spk_precision prec, const spk_pool_geom* pool) {
    if (!g || !pool || prec != SPK_PREC_EVENT) return 0;
    EvPlan e;
    if (!ev_plan(*g, e)) return 0;
    const bool geom_ok = pool->Lh >= 1 && pool->Lw >= 1 && pool->Sh >= 1 && pool->Sw >= 1 && pool->Ph >= 0 &&
                         pool->Pw >= 0 && e.Ho + 2 * pool->Ph >= pool->Lh && e.Wo + 2 * pool->Pw >= pool->Lw;
    // a whole sample per CTA, or chunks of whole output rows that no pooling window straddles
    const bool chunk_ok = e.stage || (pool->Ph == 0 && pool->Lh == pool->Sh && e.rpc % pool->Sh == 0);
    return geom_ok && chunk_ok ? 1 : 0;
}

extern "C" spk_status spk_conv_fire_pool(const uint8_t* lat_in, const float* w, const spk_conv_geom* g,
                                         spk_precision prec, float theta, float w_max, const spk_pool_geom* pool,
                                         uint8_t* out, void* ws, size_t ws_bytes, spk_stream stream) {
    spk::clear_error();
    int Ho = 0, Wo = 0;
    spk_status st = check_geom(g, Ho, Wo);
    if (st != SPK_OK) return st;
    SPK_CHECK_PTR(lat_in);
    SPK_CHECK_PTR(pool);
    SPK_CHECK_PTR(out);
    SPK_CHECK(std::isfinite(theta) && theta >= 0.0f, SPK_ERR_ARG, "theta must be finite and >= 0");
    SPK_CHECK(std::isfinite(w_max) && w_max > 0.0f, SPK_ERR_ARG, "w_max must be finite and > 0");
    SPK_CHECK(spk_conv_fire_pool_supported(g, prec, pool), SPK_ERR_UNSUPPORTED,
              "fused fire+pool needs prec=EVENT, a valid pool geometry (Eq. 3) and CTA row chunks no window straddles");
    EvPlan e;
    ev_plan(*g, e);
    SPK_CHECK(ws != nullptr && ws_bytes >= e.ws_bytes, SPK_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes,
              e.ws_bytes);
    return spk_conv_event(lat_in, w, *g, e, SPK_EPI_FIRE, theta, w_max, out, nullptr, ws, spk::as_cuda(stream), pool);
}

extern "C" spk_status spk_conv_status(const void* ws, int* flag_out, spk_stream stream) {
    spk::clear_error();
    SPK_CHECK_PTR(ws);
    SPK_CHECK_PTR(flag_out);
    // The flag lives in the first 16 bytes of the workspace (see conv_tc.cu).
    int v = 0;
    cudaStream_t s = spk::as_cuda(stream);
    if (cudaMemcpyAsync(&v, ws, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return spk::launched("spk_conv_status");
    *flag_out = v & 1;  // bit 0: clamped weight (bits 1-3: live digit planes, internal)
    return SPK_OK;
}

// ------------------------------------------------------------------ fully connected layer
// "kernel with I x O shape ... input B x T x I ... output B x T x O".  An FC layer
// is the 1x1 convolution of a 1x1 map with Ci = I input and Co = O output channels, so it runs
// on the spk_conv engines with that geometry (weights stored output-major [O][I], R-FC-LAYOUT).
static spk_conv_geom fc_geom(int B, int T, int I, int O) {
    spk_conv_geom g{};
    g.B = B;
    g.T = T;
    g.Ci = I;
    g.Hi = g.Wi = 1;
    g.Co = O;
    g.Kh = g.Kw = 1;
    g.Sh = g.Sw = 1;
    g.Ph = g.Pw = 0;
    return g;
}

// EXACT_I8 with T > 1: the samples become the pixels of ONE image (Bp = B rounded up to 8 pixels,
// laid out as Bp/8 rows of 8), so an M tile holds 8 samples x 16 steps instead of one sample's
// single pixel: the input is transposed to channel-major [I][Bp] ("never" in the padding), the
// 1x1 conv writes [O][Bp], and the records are transposed back to [B][O].
static bool fc_batched(int B, int T, spk_precision prec) { return prec == SPK_PREC_EXACT_I8 && T > 1 && B >= 8; }

static spk_conv_geom fc_geom_batched(int B, int T, int I, int O) {
    spk_conv_geom g = fc_geom(1, T, I, O);
    const int Bp = (B + 7) / 8 * 8;
    g.Hi = Bp / 8;
    g.Wi = 8;
    return g;
}

static size_t fc_conv_ws(const spk_conv_geom& g) { return (spk_conv_workspace(&g, SPK_PREC_EXACT_I8) + 255) / 256 * 256; }

extern "C" size_t spk_fc_workspace(int B, int T, int I, int O, spk_precision prec) {
    if (B < 1 || T < 1 || I < 1 || O < 1) return 0;
    if (fc_batched(B, T, prec)) {
        const spk_conv_geom g = fc_geom_batched(B, T, I, O);
        const size_t cw = fc_conv_ws(g);
        if (cw == 0) return 0;
        const size_t Bp = (size_t)(B + 7) / 8 * 8;
        return cw + (size_t)I * Bp + (size_t)O * Bp * 5 + 256;
    }
    const spk_conv_geom g = fc_geom(B, T, I, O);
    return spk_conv_workspace(&g, prec);
}

namespace {
// out[c * ldo + r] = in[r * ldi + c] for r < R, c < C, `pad` elsewhere; c < Cout, r < Rout
// (32 x 32 tiles through shared memory)
template <typename E>
__global__ void transpose_kernel(const E* __restrict__ in, int R, int C, int ldi, int Cout, int Rout, E pad,
                                 E* __restrict__ out, int ldo) {
    spk_pdl_wait();
    __shared__ E tile[32][33];
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (r < R && c < C) ? in[(size_t)r * ldi + c] : pad;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int c = c0 + i, r = r0 + threadIdx.x;
        if (c < Cout && r < Rout) out[(size_t)c * ldo + r] = tile[threadIdx.x][i];
    }
}

template <typename E>
spk_status transpose(const E* in, int R, int C, int ldi, int Cout, int Rout, E pad, E* out, int ldo, cudaStream_t s) {
    const dim3 grid(spk::ceil_div(Cout, 32), spk::ceil_div(Rout, 32)), block(32, 8);
    spk::launch(transpose_kernel<E>, grid, block, 0, s, in, R, C, ldi, Cout, Rout, pad, out, ldo);
    return spk::launched("transpose_kernel");
}
}  // namespace

extern "C" spk_status spk_fc(const uint8_t* lat_in, const float* w, int B, int T, int I, int O, spk_precision prec,
                             spk_epilogue epi, float theta, float w_max, void* out0, void* out1, void* ws,
                             size_t ws_bytes, spk_stream stream) {
    if (!fc_batched(B, T, prec) || epi != SPK_EPI_FIRE) {
        const spk_conv_geom g = fc_geom(B, T, I, O);
        return spk_conv(lat_in, w, &g, prec, epi, theta, w_max, out0, out1, ws, ws_bytes, stream);
    }
    spk::clear_error();
    SPK_CHECK_PTR(lat_in);
    SPK_CHECK_PTR(out0);
    SPK_CHECK(T <= 254, SPK_ERR_UNSUPPORTED, "T=%d > 254 (u8 latency)", T);
    const spk_conv_geom g = fc_geom_batched(B, T, I, O);
    const size_t cw = fc_conv_ws(g);
    const size_t need = spk_fc_workspace(B, T, I, O, prec);
    SPK_CHECK(cw > 0 && need > 0, SPK_ERR_UNSUPPORTED, "EXACT_I8 FC geometry not supported (I=%d)", I);
    SPK_CHECK(ws != nullptr && ws_bytes >= need, SPK_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
    const int Bp = (B + 7) / 8 * 8;
    uint8_t* base = static_cast<uint8_t*>(ws);
    uint8_t* lat_t = base + cw;                          // [I][Bp]
    uint8_t* lo_t = lat_t + (size_t)I * Bp;              // [O][Bp]
    float* ps_t = reinterpret_cast<float*>(lo_t + (size_t)O * Bp);  // [O][Bp]
    cudaStream_t s = spk::as_cuda(stream);
    // [B][I] -> [I][Bp]; the padding samples never fire
    spk_status st = transpose<uint8_t>(lat_in, B, I, I, I, Bp, (uint8_t)T, lat_t, Bp, s);
    if (st != SPK_OK) return st;
    st = spk_conv(lat_t, w, &g, SPK_PREC_EXACT_I8, SPK_EPI_FIRE, theta, w_max, lo_t, out1 ? ps_t : nullptr, base, cw,
                  stream);
    if (st != SPK_OK) return st;
    st = transpose<uint8_t>(lo_t, O, Bp, Bp, B, O, 0, static_cast<uint8_t*>(out0), O, s);  // [O][Bp] -> [B][O]
    if (st != SPK_OK || !out1) return st;
    return transpose<float>(ps_t, O, Bp, Bp, B, O, 0.0f, static_cast<float*>(out1), O, s);
}
