// common.cuh — host-side status plumbing shared by the libspk translation units.
// (Product code only; nothing here is shared with oracle/.)
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>

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

}  // namespace spk

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
