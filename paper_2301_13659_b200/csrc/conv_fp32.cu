// conv_fp32.cu — a3 reference variant: the spiking convolution (Eq. 2) on CUDA
// cores in fp32, one thread per output neuron, compensated (Kahan) summation
// over the synapses in (c, i, j) order for every time step.  Kept alongside the
// tensor-core path (north_star: "with an fp32 CUDA-core variant kept alongside").
#include "conv.cuh"

namespace {

__global__ void conv_fp32_kernel(const uint8_t* __restrict__ lat_in, const float* __restrict__ w,
                                 spk_conv_geom g, int Ho, int Wo, int epi, float theta,
                                 void* __restrict__ out0, float* __restrict__ out1) {
    spk_pdl_wait();
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t HWo = (size_t)Ho * Wo;
    if (q >= (size_t)g.B * g.Co * HWo) return;
    const int x = (int)(q % Wo), y = (int)((q / Wo) % Ho);
    const int o = (int)((q / HWo) % g.Co);
    const size_t b = q / (HWo * g.Co);
    const size_t HWi = (size_t)g.Hi * g.Wi;
    const uint8_t* L = lat_in + b * g.Ci * HWi;
    const float* Wo_ = w + (size_t)o * g.Ci * g.Kh * g.Kw;
    const int y0 = y * g.Sh - g.Ph, x0 = x * g.Sw - g.Pw;
    int fired = g.T;
    float pstar = 0.0f;
    for (int t = 0; t < g.T; ++t) {
        float s = 0.0f, comp = 0.0f;
        for (int c = 0; c < g.Ci; ++c)
            for (int i = 0; i < g.Kh; ++i) {
                const int iy = y0 + i;
                if (iy < 0 || iy >= g.Hi) continue;
                for (int j = 0; j < g.Kw; ++j) {
                    const int ix = x0 + j;
                    if (ix < 0 || ix >= g.Wi) continue;
                    if (__ldg(L + c * HWi + (size_t)iy * g.Wi + ix) <= t) {
                        const float v = __fsub_rn(__ldg(Wo_ + (c * g.Kh + i) * g.Kw + j), comp);
                        const float nsum = __fadd_rn(s, v);
                        comp = __fsub_rn(__fsub_rn(nsum, s), v);
                        s = nsum;
                    }
                }
            }
        if (epi == SPK_EPI_POTENTIAL) {
            static_cast<float*>(out0)[(((b * g.T + t) * g.Co + o) * HWo) + (size_t)y * Wo + x] = s;
        } else if (s > theta) {
            fired = t;
            pstar = s;
            break;
        }
    }
    if (epi == SPK_EPI_FIRE) {
        const size_t oi = ((b * g.Co + o) * HWo) + (size_t)y * Wo + x;
        static_cast<uint8_t*>(out0)[oi] = (uint8_t)fired;
        if (out1) out1[oi] = pstar;
    }
}

}  // namespace

spk_status spk_conv_fp32(const uint8_t* lat_in, const float* w, const spk_conv_geom* g, int Ho, int Wo,
                         spk_epilogue epi, float theta, void* out0, void* out1, cudaStream_t s) {
    const size_t n = (size_t)g->B * g->Co * Ho * Wo;
    spk::launch(conv_fp32_kernel, spk::ceil_div(n, 128), 128, 0, s, lat_in, w, *g, Ho, Wo, (int)epi, theta, out0,
                                                          static_cast<float*>(out1));
    return spk::launched("conv_fp32_kernel");
}
