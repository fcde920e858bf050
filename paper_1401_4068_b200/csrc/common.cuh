// Shared helpers for the ente_b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/ente_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "ente_b200 is written for sm_100a (B200) only"
#endif

namespace ente {

constexpr int kMaxDim = 32;     // column bitmasks are uint32
constexpr int kMaxMarg = 8;     // marginals per search call
constexpr int kNT = 128;        // threads per CTA in the sweep kernels
#ifndef ENTE_KRT
#define ENTE_KRT 2
#endif
constexpr int kRT = ENTE_KRT;   // reference points per thread (sweep lanes)
constexpr int kRefTile = kNT * kRT;
constexpr int kTJ = 128;        // candidate points per shared-memory stage
constexpr int kCap = 16;        // band events kept per reference point

// Per-chunk state shared by the sweep kernels.
struct ChunkInfo {
    int64_t row0;   // first row in pts64 / outputs
    int64_t prow0;  // first row in the padded fp32 copy
    int32_t n;      // points
    int32_t npad;   // n rounded up to kTJ (pad rows hold +inf)
    double delta;   // |d32 - d64| bound (set by prep)
    int32_t ok32;   // fp32 filter usable for this chunk
    int32_t tile_lo;  // first sweep tile of this call's reference range (split searches)
    int32_t sbg, sbk;  // float4 offsets of this chunk's block boxes in fbox / fboxk
};

struct TileRef {
    int32_t chunk;
    int32_t r0;
};

void set_error(const char *fmt, ...);

#define ENTE_CUDA(call)                                                                   \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            ::ente::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),     \
                              __FILE__, __LINE__);                                        \
            return ENTE_ERR_CUDA;                                                         \
        }                                                                                 \
    } while (0)

// Bump allocator over the caller's workspace; with base == nullptr it only
// measures, so the same layout code serves *_workspace_size().
struct Arena {
    char *base;
    size_t cap;
    size_t used = 0;
    Arena(void *b, size_t c) : base(static_cast<char *>(b)), cap(c) {}
    template <class T>
    T *take(size_t count) {
        size_t off = (used + 255) & ~size_t(255);
        used = off + count * sizeof(T);
        if (!base) return nullptr;
        return used <= cap ? reinterpret_cast<T *>(base + off) : nullptr;
    }
    bool ok() const { return base == nullptr || used <= cap; }
};

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Order this thread's earlier generic-proxy shared accesses before later
// async-proxy (bulk copy) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Binary search: the chunk owning a given row (chunks sorted by row0).
__device__ __forceinline__ int chunk_of_row(const ChunkInfo *info, int n_chunks, int64_t row) {
    int lo = 0, hi = n_chunks - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (info[mid].row0 <= row) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

}  // namespace ente
