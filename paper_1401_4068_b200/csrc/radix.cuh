// CTA-wide stable LSD radix sort (8-bit digits) over global-memory ping-pong
// buffers, one CTA per segment.  Used for the per-chunk spatial orders of the
// sweeps and for numpy's ascending sort in the TE reduction.
//
// Each pass: a digit histogram (per-warp shared counters), then the segment
// is scattered in tiles of kSortThreads * kSortItems keys held in registers.
// Within a tile every warp ranks its 8 x 32 keys step by step with
// __match_any_sync (stable: step-major, lane-minor order), the per-warp digit
// counts are scanned across warps by one thread per digit, and every key goes
// to running_offset[digit] + warp prefix + local rank.  Five CTA barriers per
// tile of 4096 keys.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ente {

constexpr int kSortThreads = 512;      // CTA size for large segments
constexpr int kSortThreadsSmall = 128;  // ... for segments of <= kSortSmallN keys,
constexpr int kSortSmallN = 1024;       // sorted in shared memory (keys + values: 16 KB)
constexpr int kSortItems = 8;  // keys per thread per tile

template <int T>
struct SortSmemT {
    int wcnt[T / 32][256];  // per-warp digit counts, then their exclusive scan
    int off[256];           // running output offset of each digit
    int tile_total[256];
    int single;
};
using SortSmem = SortSmemT<kSortThreads>;

// Sorts (keys, vals) of length n by key bits [shift0, shift0 + bits).  The
// result ends in (ka, va) when the function returns 0, in (kb, vb) when it
// returns 1.  vals may be null (keys only).  Passes whose digit is shared by
// every key are skipped.  Must be called by all kSortThreads threads.
template <int T, typename K, typename V>
__device__ int cta_radix_sort(K *ka, K *kb, V *va, V *vb, int n, int bits, SortSmemT<T> &sm,
                              int shift0 = 0) {
    constexpr int kSortWarps = T / 32, kSortThreads = T, kSortTile = T * kSortItems;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    int parity = 0;
    K *src = ka, *dst = kb;
    V *vsrc = va, *vdst = vb;
    for (int shift = shift0; shift < shift0 + bits; shift += 8) {
        // ---- histogram
        for (int e = tid; e < kSortWarps * 256; e += kSortThreads) (&sm.wcnt[0][0])[e] = 0;
        if (tid == 0) sm.single = 0;
        __syncthreads();
        for (int i = tid; i < n; i += kSortThreads)
            atomicAdd(&sm.wcnt[warp][(int)((src[i] >> shift) & 255)], 1);
        __syncthreads();
        for (int d = tid; d < 256; d += kSortThreads) {
            int t = 0;
            for (int w = 0; w < kSortWarps; ++w) t += sm.wcnt[w][d];
            sm.tile_total[d] = t;
            if (t == n) sm.single = 1;
        }
        __syncthreads();
        const int single = sm.single;
        __syncthreads();
        if (single) continue;  // uniform: every key shares this digit
        if (tid < 32) {  // exclusive scan of the 256 digit totals by one warp
            int v[8], s = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                v[q] = sm.tile_total[lane * 8 + q];
                s += v[q];
            }
            int inc = s;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += u;
            }
            int run = inc - s;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                sm.off[lane * 8 + q] = run;
                run += v[q];
            }
        }
        __syncthreads();
        // ---- tiled scatter
        for (int base = 0; base < n; base += kSortTile) {
            for (int e = tid; e < kSortWarps * 256; e += kSortThreads) (&sm.wcnt[0][0])[e] = 0;
            __syncthreads();
            K key[kSortItems];
            V val[kSortItems];
            int dig[kSortItems], rank[kSortItems];
#pragma unroll
            for (int it = 0; it < kSortItems; ++it) {
                const int i = base + warp * (32 * kSortItems) + it * 32 + lane;
                const bool valid = i < n;
                key[it] = valid ? src[i] : K(0);
                if (vsrc) val[it] = valid ? vsrc[i] : V(0);
                const int d = valid ? (int)((key[it] >> shift) & 255) : 256;
                dig[it] = d;
                const unsigned peers = __match_any_sync(0xffffffffu, d);
                int before = 0;
                if (valid) before = sm.wcnt[warp][d];
                rank[it] = before + __popc(peers & lt_mask);
                __syncwarp();
                if (valid && (peers & lt_mask) == 0) sm.wcnt[warp][d] = before + __popc(peers);
                __syncwarp();
            }
            __syncthreads();
            for (int d = tid; d < 256; d += kSortThreads) {  // scan the warps' counts of digit d
                int run = 0;
#pragma unroll
                for (int w = 0; w < kSortWarps; ++w) {
                    const int c = sm.wcnt[w][d];
                    sm.wcnt[w][d] = run;
                    run += c;
                }
                sm.tile_total[d] = run;
            }
            __syncthreads();
#pragma unroll
            for (int it = 0; it < kSortItems; ++it) {
                const int d = dig[it];
                if (d < 256) {
                    const int pos = sm.off[d] + sm.wcnt[warp][d] + rank[it];
                    dst[pos] = key[it];
                    if (vsrc) vdst[pos] = val[it];
                }
            }
            __syncthreads();
            for (int d = tid; d < 256; d += kSortThreads) sm.off[d] += sm.tile_total[d];
            // (the next tile's zeroing barrier orders this update)
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
