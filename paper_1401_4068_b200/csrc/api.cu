// C-ABI glue: error reporting and version string.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace ente {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

}  // namespace ente

extern "C" const char *ente_last_error(void) { return ente::g_err; }

extern "C" const char *ente_version(void) { return "ente_b200 0.1.0 sm_100a"; }
