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
}  // namespace rs

extern "C" const char* rs_last_error(void) { return rs::g_err; }

extern "C" const char* rs_version(void) {
    return "rlhfspec_core 0.1 (sm_100a; tcgen05/TMEM/TMA tree attention)";
}
