// CTA-wide stable LSD radix sort (8-bit digits) over global-memory ping-pong
// buffers, one CTA per segment.  Used for the per-chunk spatial (Morton)
// order of the sweeps and for numpy's ascending sort in the TE reduction.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ente {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;

struct SortSmem {
    int hist[256];
    int wcnt[kSortWarps][256];
};

// Sorts (keys, vals) of length n by the low `bits` bits of the keys.  The
// result ends in (ka, va) when the function returns 0, in (kb, vb) when it
// returns 1.  vals may be null (keys only).  Passes whose digit is shared by
// every key are skipped.  Must be called by all kSortThreads threads.
template <typename K, typename V>
__device__ int cta_radix_sort(K *ka, K *kb, V *va, V *vb, int n, int bits, SortSmem &sm) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    int parity = 0;
    K *src = ka, *dst = kb;
    V *vsrc = va, *vdst = vb;
    for (int shift = 0; shift < bits; shift += 8) {
        sm.hist[tid] = 0;
        __syncthreads();
        for (int i = tid; i < n; i += kSortThreads) atomicAdd(&sm.hist[(int)((src[i] >> shift) & 255)], 1);
        __syncthreads();
        bool single = false;
        for (int d = 0; d < 256; ++d) single |= sm.hist[d] == n;
        __syncthreads();
        if (single) continue;
        if (tid == 0) {
            int run = 0;
            for (int d = 0; d < 256; ++d) {
                const int h = sm.hist[d];
                sm.hist[d] = run;
                run += h;
            }
        }
        __syncthreads();
        for (int base = 0; base < n; base += kSortThreads) {
            const int i = base + tid;
            const bool valid = i < n;
            const K key = valid ? src[i] : K(0);
            const int dig = valid ? (int)((key >> shift) & 255) : 256 + warp;
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) sm.wcnt[w][tid] = 0;
            __syncthreads();
            const unsigned peers = __match_any_sync(0xffffffffu, dig);
            const int rank = __popc(peers & lt_mask);
            if (valid && rank == 0) sm.wcnt[warp][dig] = __popc(peers);
            __syncthreads();
            if (valid) {
                int pre = 0;
                for (int w = 0; w < warp; ++w) pre += sm.wcnt[w][dig];
                const int pos = sm.hist[dig] + pre + rank;
                dst[pos] = key;
                if (vsrc) vdst[pos] = vsrc[i];
            }
            __syncthreads();
            int add = 0;
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) add += sm.wcnt[w][tid];
            sm.hist[tid] += add;
            __syncthreads();
        }
        K *t = src;
        src = dst;
        dst = t;
        V *tv = vsrc;
        vsrc = vdst;
        vdst = tv;
        parity ^= 1;
        __syncthreads();
    }
    return parity;
}

}  // namespace ente
