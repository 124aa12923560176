// conv.cuh — internal interface between the spk_conv dispatcher and its two engines.
#pragma once
#include "common.cuh"

// Geometry of the tcgen05 exact path (see conv_tc.cu).
struct TcPlan {
    int Ho, Wo, K, KS, nks, TP, PPT, Nt, n_ntiles, NB;
    int tps, NR, band, nrb, bres, stack, NS, WiP, HiP, retain, NA, aCol0, G, kt16, GB;  // M tiles per sample, staged input rows per tile, bytes per channel band, band buffers, resident B
    size_t rb_stride;
    long long NP, n_mtiles, total_tiles;
    size_t packed_bytes, ws_bytes, smem_bytes;
};

constexpr int kTcKS = 128;      // K bytes (= synapses) per pipeline stage
constexpr int kTcStages = 4;    // pipeline depth (A stages in TMEM, B stages in smem)
constexpr int kTcMaxK = 8192;   // synapses per neuron supported by the tcgen05 path

bool tc_plan(const spk_conv_geom& g, TcPlan& p);

// Geometry of the event (latency-histogram) path (see conv_event.cu).
struct EvPlan {
    int Ho, Wo, K, MB, n_mb, Co_pad, acc64, stage, pch, nw, rpc, Wq, mpl;  // stage: whole sample per CTA
    size_t band;
    size_t smem_bytes, ws_bytes;
};
bool ev_plan(const spk_conv_geom& g, EvPlan& p, bool fill = false);  // fill: split rows for small grids (spk_conv)
spk_status spk_conv_event(const uint8_t* lat_in, const float* w, const spk_conv_geom& g, const EvPlan& p,
                          spk_epilogue epi, float theta, float w_max, void* out0, void* out1, void* ws,
                          cudaStream_t s, const spk_pool_geom* pool = nullptr);
spk_status spk_conv_tc(const uint8_t* lat_in, const float* w, const spk_conv_geom& g, const TcPlan& p,
                       spk_epilogue epi, float theta, float w_max, void* out0, void* out1, void* ws,
                       cudaStream_t s);
spk_status spk_conv_fp32(const uint8_t* lat_in, const float* w, const spk_conv_geom* g, int Ho, int Wo,
                         spk_epilogue epi, float theta, void* out0, void* out1, cudaStream_t s);
