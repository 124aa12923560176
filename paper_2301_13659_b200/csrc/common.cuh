// common.cuh — host-side status plumbing shared by the libspk translation units.
// (Product code only; nothing here is shared with oracle/.)
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "spk.h"

namespace spk {

// Record `st` with a printf-style message in the thread-local error slot.
spk_status fail(spk_status st, const char* fmt, ...);
// Clear the error slot (called at the start of every entry point).
void clear_error();
// After a launch: record the kernel name, count it, map a launch error to SPK_ERR_CUDA.
spk_status launched(const char* kernel);

inline cudaStream_t as_cuda(spk_stream s) { return reinterpret_cast<cudaStream_t>(s); }

inline unsigned ceil_div(size_t a, size_t b) { return (unsigned)((a + b - 1) / b); }

// True the first time it is called for the current device with this mask (per-device,
// thread-safe one-time setup such as cudaFuncSetAttribute opt-ins; devices 0..63).
inline bool first_on_device(std::atomic<uint64_t>& mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    return !(mask.fetch_or(bit) & bit);
}

// SM count of the current device (cached per device).
inline int sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    int n = cache[dev & 63].load();
    if (n <= 0) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        cache[dev & 63].store(n);
    }
    return n;
}

// Programmatic dependent launch (PDL): every libspk kernel starts with spk_pdl_wait()
// (griddepcontrol.wait: a no-op without a programmatic dependency), so a launch may be marked
// programmatic-serialization-allowed — the next kernel of a stream (or of a captured graph) is
// then scheduled while the previous one drains and starts its work the moment it completes.
// SPK_PDL=0 switches the attribute off (A/B).
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SPK_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                          Args&&... args) {
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace spk

__device__ __forceinline__ void spk_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

#define SPK_CHECK(cond, status, ...)                          \
    do {                                                      \
        if (!(cond)) return spk::fail((status), __VA_ARGS__); \
    } while (0)

#define SPK_CHECK_PTR(p) SPK_CHECK((p) != nullptr, SPK_ERR_ARG, "%s is null", #p)

// Device-side orderable key helpers (product side).
__device__ __forceinline__ uint32_t spk_float_order_u32(float f) {
    uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // ascending with f
}
