// Thread-local error text and version string for the C ABI.
#include <stdarg.h>

#include "common.cuh"

namespace rs {
static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
// The library links its own (static) CUDA runtime. Kernels go to the runtime's current device,
// which follows the driver context current on the calling thread; to be independent of how the
// caller selected its device, each launching entry point binds the device that owns its first
// device-pointer argument (a no-op when it already is current).
void bind_device(const void* p) {
    if (!p) return;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return;
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != a.device) cudaSetDevice(a.device);
    cudaGetLastError();
}
}  // namespace rs

extern "C" const char* rs_last_error(void) { return rs::g_err; }

extern "C" const char* rs_version(void) {
    return "rlhfspec_core 0.1 (sm_100a; tcgen05/TMEM/TMA tree attention)";
}
