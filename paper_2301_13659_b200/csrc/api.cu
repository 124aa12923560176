// api.cu — status plumbing and ABI metadata of libspk (see include/spk.h).
#include <atomic>
#include <cstring>

#include "common.cuh"

namespace {
thread_local char g_err[512] = "";
thread_local const char* g_last_kernel = "";
std::atomic<uint64_t> g_launches{0};
}  // namespace

namespace spk {

spk_status fail(spk_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return st;
}

void clear_error() { g_err[0] = '\0'; }

spk_status launched(const char* kernel) {
    g_last_kernel = kernel;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SPK_ERR_CUDA, "%s: %s", kernel, cudaGetErrorString(e));
    return SPK_OK;
}

}  // namespace spk

extern "C" {

const char* spk_last_error(void) { return g_err; }
int spk_abi_version(void) { return SPK_ABI_VERSION; }
const char* spk_last_kernel(void) { return g_last_kernel; }
uint64_t spk_launch_count(void) { return g_launches.load(); }

}  // extern "C"
