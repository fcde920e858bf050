// Launch accounting: every kernel launch of the library goes through
// ENTE_LAUNCH, which counts it and -- when profiling is enabled -- brackets
// it with CUDA events on its own stream (so the timing is the kernel's
// on-stream duration, whatever stream the caller used).
#pragma once

#include <cuda_runtime.h>

namespace ente {
void prof_begin(const char *name, cudaStream_t st);
void prof_end(const char *name, cudaStream_t st);
bool ente_profile_enabled();
}  // namespace ente

#define ENTE_LAUNCH(name, st, ...)         \
    do {                                   \
        ::ente::prof_begin(name, st);      \
        __VA_ARGS__;                       \
        ::ente::prof_end(name, st);        \
    } while (0)
