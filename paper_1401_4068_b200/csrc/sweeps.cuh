// Templated fp32 sweeps of the neighbour search (kNN pass, count passes,
// tie rescan) and their per-layout instantiation tables.
//
// Shared by search.cu (host dispatch) and the sweeps_*.cu translation units,
// each of which instantiates a group of (d_y, d_x) TE layouts -- split so the
// sm_100a build compiles the layout groups in parallel.  See search.cu for
// the algorithm (fp32 filter, fp64 certification, box pruning).
#pragma once

#include <cuda_runtime.h>
#include <math.h>

#include <type_traits>

#include "common.cuh"

namespace ente {

#ifndef ENTE_KSUB
#define ENTE_KSUB 32
#endif
constexpr int kSub = ENTE_KSUB;             // candidate rows per sub-tile (one TMA copy); 16 or 32
static_assert(kSub == 16 || kSub == 32, "sub-tiles are half or whole warps of rows");
constexpr int kWarpRefs = 32 * kRT;         // references per sweep CTA (one warp)
constexpr int kGate = 4;                    // gate columns in the Morton key and the boxes
// minimum resident sweep CTAs (one warp each) per SM: caps the registers
#ifndef ENTE_KNN_NSLOT
#define ENTE_KNN_NSLOT 4
#endif
#ifndef ENTE_CNT_NSLOT
#define ENTE_CNT_NSLOT 2
#endif
#ifndef ENTE_CNT_GROUPS
#define ENTE_CNT_GROUPS 2  // grouped count rounds: 0 off, 1 up to 4 groups, 2 up to 8 groups
#endif
#ifndef ENTE_KNNC_NSLOT
#define ENTE_KNNC_NSLOT 2  // ring slots of the compacted kNN pass
#endif
#ifndef ENTE_KNNC_REGREF
#define ENTE_KNNC_REGREF 1  // compacted kNN: walker tests from register copies of the lane's refs
#endif
#define ENTE_PRAGMA(x) _Pragma(#x)
#define ENTE_UNROLL(n) ENTE_PRAGMA(unroll n)
#ifndef ENTE_CNT_UNROLL
#define ENTE_CNT_UNROLL 2    // count pass: row-pair iterations unrolled per loop trip
#endif
#ifndef ENTE_KO_UNROLL
#define ENTE_KO_UNROLL 1     // m3 sweep: row-pair iterations unrolled per loop trip
#endif
#ifndef ENTE_KNNC_UNROLL
#define ENTE_KNNC_UNROLL 2   // compacted kNN pass: row-pair iterations per loop trip
#endif
#ifndef ENTE_KO_RT
#define ENTE_KO_RT 2  // references per lane of the shared-y m3/joint sweep (64-reference groups)
#endif
#ifndef ENTE_CNT_MINB
#define ENTE_CNT_MINB 32
#endif
#ifndef ENTE_KNN_MINB
#define ENTE_KNN_MINB 32
#endif
// resident one-warp sweep CTAs per SM by layout width: 32 (64 registers)
// up to D = 7, fewer for wider layouts so their references stay in registers
__host__ __device__ constexpr int sweep_minb(int D, int cap) {
    return D <= 7 ? cap : (D <= 9 ? (cap < 28 ? cap : 28) : (D <= 11 ? (cap < 24 ? cap : 24)
                                                              : (D <= 13 ? (cap < 20 ? cap : 20) : 16)));
}
constexpr int kBlockSubs = 32;              // sub-tiles per walker block (one per lane)
constexpr int kKnnQ = 2;                    // kNN sub-tile boxes: 4 * kKnnQ columns from 0


// ---------------------------------------------------------------------------
// sweep tile t -> (chunk, first sorted reference): tile0[c] = first tile of
// chunk c (ascending, n_chunks + 1 entries); chunks without tiles repeat
// their successor's value, so the largest c with tile0[c] <= t is the owner.
// tile0[n_chunks + 1 + c] = the chunk's first tile index within the chunk
// (non-zero only for split searches, which sweep a range of references).
// ---------------------------------------------------------------------------
__device__ __forceinline__ TileRef tile_of(const int32_t *__restrict__ tile0, int n_chunks, int t,
                                           int refs = kWarpRefs) {
    int lo = 0, hi = n_chunks - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(tile0 + mid) <= t) lo = mid;
        else hi = mid - 1;
    }
    TileRef tr;
    tr.chunk = lo;
    tr.r0 = (t - __ldg(tile0 + lo) + __ldg(tile0 + n_chunks + 1 + lo)) * refs;
    return tr;
}

// ---------------------------------------------------------------------------
// register-level helpers for the fp32 sweeps
// TE layout columns: 0 = y_t, 1..DY = y-past, DY+1..D-1 = x-past
// (embedding.py:50-60).  Coordinates are held as packed pairs (0,1), (2,3)...
// so one FADD2 gives two differences.  Pairs [0, PG) cover columns 0..DY
// (the gate: y-past plus y_t), pairs [PG, NP) the rest.
// ---------------------------------------------------------------------------
template <int DY, int DX>
struct Lay {
    static constexpr int D = 1 + DY + DX;
    static constexpr int DP = (D + 3) & ~3;
    static constexpr int NP = (D + 1) / 2;     // coordinate pairs
    static constexpr int PG = (DY + 2) / 2;    // gate pairs: columns 0 .. 2*PG-1 >= DY
    static constexpr int NSLOT = DP <= 8 ? 8 : (DP <= 12 ? 6 : 4);  // ring slots per warp
};

template <int D>
__device__ __forceinline__ void load_ref(float2 (&nr)[(D + 1) / 2], const float *__restrict__ row,
                                         bool valid) {
#pragma unroll
    for (int p = 0; p < (D + 1) / 2; ++p) {
        const float a = valid ? row[2 * p] : 0.0f;
        const float b = (valid && 2 * p + 1 < D) ? row[2 * p + 1] : 0.0f;
        nr[p] = make_float2(-a, -b);
    }
}

// difference pairs [P0, P1) of ref (negated, packed) and candidate row (smem)
template <int D, int P0, int P1>
__device__ __forceinline__ void diff_pairs(const float2 (&nr)[(D + 1) / 2], const float2 *c,
                                           float (&a)[2 * ((D + 1) / 2)]) {
#pragma unroll
    for (int p = P0; p < P1; ++p) {
        if (2 * p + 1 < D) {
            const float2 d = __fadd2_rn(nr[p], c[p]);
            a[2 * p] = d.x;
            a[2 * p + 1] = d.y;
        } else {
            a[2 * p] = nr[p].x + c[p].x;
        }
    }
}

// max |a[c]| for c in [LO, HI) folded into acc (3-input FMNMX chain)
template <int LO, int HI, int N>
__device__ __forceinline__ float maxabs(const float (&a)[N], float acc) {
    int c = LO;
#pragma unroll
    for (; c + 1 < HI; c += 2) acc = fmaxf(fmaxf(acc, fabsf(a[c])), fabsf(a[c + 1]));
    if (c < HI) acc = fmaxf(acc, fabsf(a[c]));
    return acc;
}

template <int LO, int HI, int N>
__device__ __forceinline__ float maxabs0(const float (&a)[N]) {
    if constexpr (HI - LO <= 0) return 0.0f;
    else if constexpr (HI - LO == 1) return fabsf(a[LO]);
    else return maxabs<LO + 2, HI, N>(a, fmaxf(fabsf(a[LO]), fabsf(a[LO + 1])));
}

// Keep the S smallest values, ascending (new[s] = median(old[s-1], old[s], d));
// a no-op when d >= kd[S-1].
template <int S>
__device__ __forceinline__ void insert_sorted(float (&kd)[S], float d) {
#pragma unroll
    for (int s = S - 1; s >= 1; --s) kd[s] = fmaxf(kd[s - 1], fminf(kd[s], d));
    kd[0] = fminf(kd[0], d);
}

struct Band {
    float nlo, nt;  // -lo, -t
    float lo, hi, w;
};

__device__ __forceinline__ Band make_band(float t32, double delta) {
    Band b;
    const double two = 2.0 * delta;
    const float lo = __double2float_rd(__dsub_rd((double)t32, two));
    const float hi = __double2float_ru(__dadd_ru((double)t32, two));
    b.lo = lo;
    b.hi = hi;
    b.nlo = -lo;
    b.nt = -t32;
    // band width, rounded up: v in [lo, hi] => 0 <= fl(v - lo) <= w, so the
    // sweeps test |fl(v - lo)| <= w on the values they already subtract for
    // the counts (a superset: the exact flags are recomputed on a hit)
    b.w = __fsub_ru(hi, lo);
    return b;
}

// lane index read once into a register the compiler cannot rematerialise:
// with threadIdx.x it re-reads SR_TID (an S2R, ~20 cycles) inside the walk
// loops whenever registers are tight
#ifndef ENTE_PIN_LANE
#define ENTE_PIN_LANE 1
#endif
__device__ __forceinline__ int pinned_lane() {
#if ENTE_PIN_LANE
    int l;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
#else
    return threadIdx.x & 31;
#endif
}

__device__ __forceinline__ float warp_max_nonneg(float v) {
    return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(fmaxf(v, 0.0f))));
}

// ---------------------------------------------------------------------------
// Warp-private candidate stream.
//
// Each sweep CTA is ONE warp owning 32 * kRT (64) consecutive sorted
// references (kRT per lane).  It walks the chunk's 32-row sub-tiles home-first, then alternately
// below and above (nearest first in the Morton order, so kNN bounds shrink
// early).  Sub-tile boxes are tested 32 positions at a time, one per lane,
// with the next window's boxes prefetched into registers; needed sub-tiles
// are streamed into a ring of NSLOT shared-memory slots by the TMA engine
// (cp.async.bulk + mbarrier).  Warps never wait for each other.
// ---------------------------------------------------------------------------
// A sub-tile box: Q float4 quads of column minima, then Q of maxima
// (fbox layout per sub-tile: lo[4Q] | hi[4Q], float4 index st * 2Q).
#ifndef ENTE_GAP_FADD2
#define ENTE_GAP_FADD2 1
#endif

template <int Q>
struct Box {
    float4 lo[Q], hi[Q];
};

template <int Q>
__device__ __forceinline__ Box<Q> load_box(const float4 *__restrict__ fb, int st) {
    Box<Q> b;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        b.lo[q] = __ldg(fb + 2 * Q * st + q);
        b.hi[q] = __ldg(fb + 2 * Q * st + Q + q);
    }
    return b;
}

__device__ __forceinline__ float gap4(float4 lo, float4 hi, float4 blo, float4 bhi) {
#if ENTE_GAP_FADD2
    // two columns per FADD2 (same roundings as the scalar form)
    const float2 a = __fadd2_rn(make_float2(lo.x, lo.y), make_float2(-bhi.x, -bhi.y));
    const float2 b = __fadd2_rn(make_float2(blo.x, blo.y), make_float2(-hi.x, -hi.y));
    const float2 c = __fadd2_rn(make_float2(lo.z, lo.w), make_float2(-bhi.z, -bhi.w));
    const float2 d = __fadd2_rn(make_float2(blo.z, blo.w), make_float2(-hi.z, -hi.w));
    return fmaxf(fmaxf(fmaxf(fmaxf(a.x, a.y), fmaxf(b.x, b.y)), fmaxf(c.x, c.y)), fmaxf(d.x, d.y));
#else
    const float a = fmaxf(fmaxf(lo.x - bhi.x, blo.x - hi.x), fmaxf(lo.y - bhi.y, blo.y - hi.y));
    const float b = fmaxf(fmaxf(lo.z - bhi.z, blo.z - hi.z), fmaxf(lo.w - bhi.w, blo.w - hi.w));
    return fmaxf(a, b);
#endif
}

// Block walk over a chunk's sub-tiles in aligned blocks of kBlockSubs (= 32, one
// per lane): the home block first, then blocks alternately above and below
// it.  A block whose box (the union of its sub-tile boxes, block_box_kernel)
// is not within the bound is skipped with one warp-uniform test; otherwise
// every lane tests its sub-tile's box as before.  Every sub-tile is
// considered once.  Used by the m3 count sweep, whose bounds (the bands)
// are fixed: the order cannot change what is visited.  (The kNN passes keep the
// sub-tile-outward Walker: there the visiting order decides how fast the
// k-th distances shrink, and block order measured 34 % slower on C2.)
template <int Q>
struct BlockWalker {
    int nsub, nwin, hb, w;
    uint32_t mask;  // needed sub-tiles of the current block not yet issued
    int wst;        // per lane: sub-tile of the current block (-1: none)
    float wd;       // per lane: its box distance
    Box<Q> own;     // the warp's own box, identical in all lanes
    uint32_t need;  // per lane: refs_need() bits of the sub-tile last returned
    int ln;         // this lane
    const float4 *sb;  // this chunk's block boxes

    __device__ void init(const float4 *__restrict__ fb, const float4 *__restrict__ sbox, int wrow, int n,
                         int npad, int lane, int refs = kWarpRefs) {
        ln = lane;
        sb = sbox;
        const int h0 = wrow / kSub;
        const int nh = (min(wrow + refs, n) - wrow + kSub - 1) / kSub;
        nsub = npad / kSub;
        const int nblk = (nsub + kBlockSubs - 1) / kBlockSubs;
        hb = h0 / kBlockSubs;
        nwin = 1 + 2 * max(hb, nblk - 1 - hb);
        w = -1;
        mask = 0;
        own = load_box<Q>(fb, h0);
        for (int s = 1; s < nh; ++s) {
            const Box<Q> b = load_box<Q>(fb, h0 + s);
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                own.lo[q] = make_float4(fminf(own.lo[q].x, b.lo[q].x), fminf(own.lo[q].y, b.lo[q].y),
                                        fminf(own.lo[q].z, b.lo[q].z), fminf(own.lo[q].w, b.lo[q].w));
                own.hi[q] = make_float4(fmaxf(own.hi[q].x, b.hi[q].x), fmaxf(own.hi[q].y, b.hi[q].y),
                                        fmaxf(own.hi[q].z, b.hi[q].z), fmaxf(own.hi[q].w, b.hi[q].w));
            }
        }
    }

    __device__ float dist(const Box<Q> &b) const {
        float d = 0.0f;
#pragma unroll
        for (int q = 0; q < Q; ++q) d = fmaxf(d, gap4(b.lo[q], b.hi[q], own.lo[q], own.hi[q]));
        return d;
    }

    template <class RefTest>
    __device__ int next(const float4 *__restrict__ fb, float bound, bool strict,
                        RefTest &&refs_need) {
        const int lane = ln;
        for (;;) {
            while (mask == 0) {
                if (++w >= nwin) return -1;
                const int k = (w + 1) >> 1;
                const int blk = w == 0 ? hb : ((w & 1) ? hb + k : hb - k);
                if (blk < 0 || blk * kBlockSubs >= nsub) continue;
                const float bd = dist(load_box<Q>(sb, blk));  // warp-uniform
                if (!(strict ? (bd < bound) : (bd <= bound))) continue;
                const int st = blk * kBlockSubs + lane;
                wst = st < nsub ? st : -1;
                wd = wst >= 0 ? dist(load_box<Q>(fb, wst)) : INFINITY;
                mask = __ballot_sync(0xffffffffu, wst >= 0 && (strict ? (wd < bound) : (wd <= bound)));
            }
            const int b = __ffs(mask) - 1;
            mask &= mask - 1;
            const float d = __shfl_sync(0xffffffffu, wd, b);
            if (!(strict ? (d < bound) : (d <= bound))) continue;  // the bound may have shrunk
            const int st = __shfl_sync(0xffffffffu, wst, b);
            const uint32_t nm = (uint32_t)refs_need(load_box<Q>(fb, st));
            if (__any_sync(0xffffffffu, nm != 0u)) {
                need = nm;
                return st;
            }
        }
    }
};

template <int Q>
struct Walker {
    int h0, nh, nsub, npos;
    int base;       // first position of the evaluated window (-32 before the first)
    uint32_t mask;  // needed positions of that window not yet issued
    int wst;        // per lane: sub-tile at position base + lane (-1: none)
    float wd;       // per lane: its box distance
    int nst;        // per lane: sub-tile at position base + 32 + lane (prefetched)
    Box<Q> nb;      // its box
    Box<Q> own;     // the warp's own box, identical in all lanes
    uint32_t need;  // per lane: refs_need() bits of the sub-tile last returned
    int ln;         // this lane

    __device__ int sub_at(int pos) const {
        if (pos < nh) return h0 + pos;
        const int p = pos - nh, k = (p >> 1) + 1;
        const int s = (p & 1) ? h0 + nh - 1 + k : h0 - k;
        return (s >= 0 && s < nsub) ? s : -1;
    }

    __device__ void prefetch(const float4 *__restrict__ fb, int pos) {
        nst = pos < npos ? sub_at(pos) : -1;
        if (nst >= 0) nb = load_box<Q>(fb, nst);
    }

    __device__ void init(const float4 *__restrict__ fb, const float4 *__restrict__, int wrow, int n,
                         int npad, int lane, int refs = kWarpRefs) {
        ln = lane;
        h0 = wrow / kSub;
        nh = (min(wrow + refs, n) - wrow + kSub - 1) / kSub;
        nsub = npad / kSub;
        npos = nh + 2 * max(h0, nsub - h0 - nh);
        base = -32;
        mask = 0;
        own = load_box<Q>(fb, h0);
        for (int s = 1; s < nh; ++s) {
            const Box<Q> b = load_box<Q>(fb, h0 + s);
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                own.lo[q] = make_float4(fminf(own.lo[q].x, b.lo[q].x), fminf(own.lo[q].y, b.lo[q].y),
                                        fminf(own.lo[q].z, b.lo[q].z), fminf(own.lo[q].w, b.lo[q].w));
                own.hi[q] = make_float4(fmaxf(own.hi[q].x, b.hi[q].x), fmaxf(own.hi[q].y, b.hi[q].y),
                                        fmaxf(own.hi[q].z, b.hi[q].z), fmaxf(own.hi[q].w, b.hi[q].w));
            }
        }
        prefetch(fb, ln);
    }

    // fp32 box distance (a lower bound of every d32 between the two boxes:
    // fl is monotone, fl(x_j - x_i) >= fl(lo_j - hi_i))
    __device__ float dist(const Box<Q> &b) const {
        float d = 0.0f;
#pragma unroll
        for (int q = 0; q < Q; ++q) d = fmaxf(d, gap4(b.lo[q], b.hi[q], own.lo[q], own.hi[q]));
        return d;
    }

    // Next sub-tile whose box distance to the warp's box is below `bound`
    // (strict) or not above it, AND that some reference of the warp needs by
    // its own point-to-box distance (refs_need(box), evaluated per lane);
    // returns -1 when the walk is over.
    template <class RefTest>
    __device__ int next(const float4 *__restrict__ fb, float bound, bool strict,
                        RefTest &&refs_need) {
        const int lane = ln;
        for (;;) {
            while (mask == 0) {
                if (base + 32 >= npos) return -1;
                base += 32;
                wst = nst;
                wd = wst >= 0 ? dist(nb) : INFINITY;
                // (positions past the chunk never qualify, even for an infinite bound)
                mask = __ballot_sync(0xffffffffu, wst >= 0 && (strict ? (wd < bound) : (wd <= bound)));
                prefetch(fb, base + 32 + lane);
            }
            const int b = __ffs(mask) - 1;
            mask &= mask - 1;
            const float d = __shfl_sync(0xffffffffu, wd, b);
            if (!(strict ? (d < bound) : (d <= bound))) continue;  // the bound may have shrunk
            const int st = __shfl_sync(0xffffffffu, wst, b);
            const uint32_t nm = (uint32_t)refs_need(load_box<Q>(fb, st));
            if (__any_sync(0xffffffffu, nm != 0u)) {
                need = nm;
                return st;
            }
        }
    }
};

#ifndef ENTE_KNN_WA
#define ENTE_KNN_WA 2
#endif

// kNN walk: the sub-tile-outward Walker for its first ENTE_KNN_WA windows
// (the nearest Morton neighbours, which shrink the k-th distances fast),
// then the block walk of BlockWalker over the rest of the chunk, skipping
// the sub-tiles already visited.
template <int Q>
struct KnnWalker : Walker<Q> {
    int w;  // block window (-2: still in the sub-tile phase)
    const float4 *sb;

    __device__ void init(const float4 *__restrict__ fb, const float4 *__restrict__ sbox, int wrow, int n,
                         int npad, int lane, int refs = kWarpRefs) {
        Walker<Q>::init(fb, sbox, wrow, n, npad, lane, refs);
        this->npos = min(this->npos, 32 * ENTE_KNN_WA);
        w = -2;
        sb = sbox;
    }

    template <class RefTest>
    __device__ int next(const float4 *__restrict__ fb, float bound, bool strict,
                        RefTest &&refs_need) {
        const int h0 = this->h0, nh = this->nh, nsub = this->nsub;
        if (w == -2) {
            const int st = Walker<Q>::next(fb, bound, strict, refs_need);
            if (st >= 0 || nh + 2 * max(h0, nsub - h0 - nh) <= this->npos) return st;
            w = -1;
            this->mask = 0;
        }
        // sub-tiles the first phase visited: [vlo, vhi]
        const int pa = this->npos - nh;
        const int vlo = h0 - (pa + 1) / 2, vhi = h0 + nh - 1 + pa / 2;
        const int hb = h0 / kBlockSubs, nblk = (nsub + kBlockSubs - 1) / kBlockSubs;
        const int nwin = 1 + 2 * max(hb, nblk - 1 - hb);
        const int lane = this->ln;
        for (;;) {
            while (this->mask == 0) {
                if (++w >= nwin) return -1;
                const int k = (w + 1) >> 1;
                const int blk = w == 0 ? hb : ((w & 1) ? hb + k : hb - k);
                if (blk < 0 || blk * kBlockSubs >= nsub) continue;
                if (blk * kBlockSubs >= vlo && blk * kBlockSubs + kBlockSubs - 1 <= vhi) continue;
                const float bd = this->dist(load_box<Q>(sb, blk));  // warp-uniform
                if (!(strict ? (bd < bound) : (bd <= bound))) continue;
                const int st = blk * kBlockSubs + lane;
                this->wst = (st < nsub && (st < vlo || st > vhi)) ? st : -1;
                this->wd = this->wst >= 0 ? this->dist(load_box<Q>(fb, this->wst)) : INFINITY;
                this->mask = __ballot_sync(0xffffffffu, this->wst >= 0 &&
                                                            (strict ? (this->wd < bound) : (this->wd <= bound)));
            }
            const int b = __ffs(this->mask) - 1;
            this->mask &= this->mask - 1;
            const float d = __shfl_sync(0xffffffffu, this->wd, b);
            if (!(strict ? (d < bound) : (d <= bound))) continue;
            const int st = __shfl_sync(0xffffffffu, this->wst, b);
            const uint32_t nm = (uint32_t)refs_need(load_box<Q>(fb, st));
            if (__any_sync(0xffffffffu, nm != 0u)) {
                this->need = nm;
                return st;
            }
        }
    }
};

// fp32 distance from a reference (negated packed coordinates) to a sub-tile
// box over the columns F0 .. F0 + NC - 1 (box slot g = column - F0): a lower
// bound of the reference's fp32 distance to every row of the sub-tile over
// any column set containing them (fl monotone).
template <int F0, int NC, int NP, int Q>
__device__ __forceinline__ float point_box(const float2 (&nr)[NP], const Box<Q> &b) {
    float d = 0.0f;
    constexpr int NPAIR = (F0 % 2 == 0) ? NC / 2 : 0;
    // column pairs (box slots 2p, 2p+1 = columns F0 + 2p, F0 + 2p + 1) when the
    // box slots line up with the packed reference pairs: lo - x and hi - x of
    // two columns per FADD2 on adjacent registers (no operand moves), the
    // same roundings as the per-column form below
#pragma unroll
    for (int p = 0; p < NPAIR; ++p) {
        const int g = 2 * p, c = F0 + g;
        const float4 l4 = b.lo[g >> 2], h4 = b.hi[g >> 2];
        const float2 l = (g & 3) == 0 ? make_float2(l4.x, l4.y) : make_float2(l4.z, l4.w);
        const float2 h = (g & 3) == 0 ? make_float2(h4.x, h4.y) : make_float2(h4.z, h4.w);
        const float2 el = __fadd2_rn(l, nr[c >> 1]);  // lo - x
        const float2 eh = __fadd2_rn(h, nr[c >> 1]);  // hi - x
        d = fmaxf(fmaxf(d, el.x), el.y);
        d = fmaxf(fmaxf(d, -eh.x), -eh.y);
    }
#pragma unroll
    for (int g = 2 * NPAIR; g < NC; ++g) {
        const int c = F0 + g;  // column
        const float x = (c & 1) ? nr[c >> 1].y : nr[c >> 1].x;  // -x_c
        const float4 l4 = b.lo[g >> 2], h4 = b.hi[g >> 2];
        const float l = (g & 3) == 0 ? l4.x : (g & 3) == 1 ? l4.y : (g & 3) == 2 ? l4.z : l4.w;
        const float h = (g & 3) == 0 ? h4.x : (g & 3) == 1 ? h4.y : (g & 3) == 2 ? h4.z : h4.w;
        const float2 e = __fadd2_rn(make_float2(l, h), make_float2(x, x));  // lo-x, hi-x
        d = fmaxf(fmaxf(d, e.x), -e.y);
    }
    return d;
}

// the same lower bound over columns C0 .. C1-1 of a box whose slot g holds
// column g (the kNN-order boxes, columns 0 .. 4Q-1)
template <int C0, int C1, int NP, int Q>
__device__ __forceinline__ float point_box_cols(const float2 (&nr)[NP], const Box<Q> &b) {
    // a leading odd column alone, then column pairs (two columns per FADD2,
    // as in point_box), then a trailing odd column; bounds are constants
    constexpr int P0 = (C0 + 1) & ~1, NPAIR = (C1 - P0) / 2, T0 = P0 + 2 * NPAIR;
    float d = 0.0f;
    auto one = [&](int c) {  // (scalar adds: a packed one would need its operands moved)
        const float x = (c & 1) ? nr[c >> 1].y : nr[c >> 1].x;  // -x_c
        const float4 l4 = b.lo[c >> 2], h4 = b.hi[c >> 2];
        const float l = (c & 3) == 0 ? l4.x : (c & 3) == 1 ? l4.y : (c & 3) == 2 ? l4.z : l4.w;
        const float h = (c & 3) == 0 ? h4.x : (c & 3) == 1 ? h4.y : (c & 3) == 2 ? h4.z : h4.w;
        d = fmaxf(fmaxf(d, __fadd_rn(l, x)), -__fadd_rn(h, x));
    };
    if constexpr (C0 < P0 && C0 < C1) one(C0);
#pragma unroll
    for (int p = 0; p < NPAIR; ++p) {
        const int c = P0 + 2 * p;
        const float4 l4 = b.lo[c >> 2], h4 = b.hi[c >> 2];
        const float2 l = (c & 3) == 0 ? make_float2(l4.x, l4.y) : make_float2(l4.z, l4.w);
        const float2 h = (c & 3) == 0 ? make_float2(h4.x, h4.y) : make_float2(h4.z, h4.w);
        const float2 el = __fadd2_rn(l, nr[c >> 1]);
        const float2 eh = __fadd2_rn(h, nr[c >> 1]);
        d = fmaxf(fmaxf(d, el.x), el.y);
        d = fmaxf(fmaxf(d, -eh.x), -eh.y);
    }
    if constexpr (T0 < C1) one(T0);
    return d;
}

template <int DP, int NSLOT>
struct Ring {
    float buf[NSLOT][kSub * DP];
    uint64_t full[NSLOT];
};

// Shared memory of the compacted sweeps: the ring, then the references.
// The grouped rounds' last row prefetch reads up to 8 rows past the last
// ring slot (values never used); they land in `full` and `rs`, which are
// larger than that, so no padding is needed.
template <class RingT, class RefsT>
struct __align__(128) SweepSmem {
    RingT ring;
    RefsT rs;
};

template <int DP, int NSLOT>
__device__ __forceinline__ void ring_issue(Ring<DP, NSLOT> &ring, int slot, const float *src) {
    constexpr uint32_t bytes = kSub * DP * sizeof(float);
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&ring.full[slot], bytes);
    bulk_g2s(ring.buf[slot], src, bytes, &ring.full[slot]);
}

// ---------------------------------------------------------------------------
// pass 1: fp32 k-th neighbour distance (self included as the (k+1)-th slot)
// lane l owns sorted rows wrow + r*32 + l, r < kRT
// ---------------------------------------------------------------------------
template <int DY, int DX, int S>
__global__ void __launch_bounds__(32, S > 16 ? 24 : (S > 8 ? 16 : sweep_minb(1 + DY + DX, ENTE_KNN_MINB))) knn_pass_kernel(
    const float *__restrict__ pts32, const float *__restrict__ fbox,
    const ChunkInfo *__restrict__ info, const int32_t *__restrict__ tile0, int n_chunks, int k, int prune,
    const int32_t *__restrict__ kmap, float *__restrict__ t32_out, int32_t *__restrict__ L_out,
    unsigned long long *__restrict__ work) {
    using L = Lay<DY, DX>;
    constexpr int D = L::D, DP = L::DP, NP = L::NP, PG = L::PG;
    constexpr int NSLOT = L::NSLOT < ENTE_KNN_NSLOT ? L::NSLOT : ENTE_KNN_NSLOT;
    constexpr int NBC = D < 4 * kKnnQ ? D : 4 * kKnnQ;  // box columns 0 .. NBC-1
    __shared__ __align__(128) Ring<DP, NSLOT> ring;
    // k + 1 > 16 slots: the sorted lists live in shared memory ([ref][slot][lane],
    // conflict-free), only their last entry (the current k-th) in a register
    constexpr bool SL = S > 16;
    constexpr int SR = SL ? 1 : S;
    __shared__ float lst[SL ? kRT : 1][SL ? S : 1][32];
    const TileRef tr = tile_of(tile0, n_chunks, blockIdx.x);
    const ChunkInfo ci = info[tr.chunk];
    if (!ci.ok32) return;
    const int lane = pinned_lane();
    const float *cp = pts32 + ci.prow0 * DP;
    const float4 *fb = reinterpret_cast<const float4 *>(fbox) + (ci.prow0 / kSub) * 2 * kKnnQ;
    const int wrow = tr.r0;
    float2 ref[kRT][NP];
    float kd[kRT][SR];  // register list, or (SL) the current k-th only
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
        const int idx = wrow + r * 32 + lane;
        const bool valid = idx < ci.n;
        load_ref<D>(ref[r], cp + (int64_t)idx * DP, valid);
        if constexpr (SL) {
            for (int s = 0; s < S; ++s) lst[r][s][lane] = (!valid || s < S - (k + 1)) ? -INFINITY : INFINITY;
            kd[r][0] = valid ? INFINITY : -INFINITY;
        } else {
#pragma unroll
            for (int s = 0; s < S; ++s) kd[r][s] = (!valid || s < S - (k + 1)) ? -INFINITY : INFINITY;
        }
    }
    // sorted insertion of d < current k-th into reference slot r's list
    auto insert = [&](int r, float d) {
        if constexpr (SL) {
            int p = S - 1;
            while (p > 0 && lst[r][p - 1][lane] > d) {
                lst[r][p][lane] = lst[r][p - 1][lane];
                --p;
            }
            lst[r][p][lane] = d;
            kd[r][0] = lst[r][S - 1][lane];
        } else {
            insert_sorted<S>(kd[r], d);
        }
    };
    if (lane < NSLOT) mbar_init(&ring.full[lane], 1);
    fence_barrier_init();
    __syncwarp();
    KnnWalker<kKnnQ> wk;
    wk.init(fb, reinterpret_cast<const float4 *>(fbox) + ci.sbk, wrow, ci.n, ci.npad, lane);
    float bound = INFINITY;  // warp max of the current k-th distances
    auto refs_need = [&](const Box<kKnnQ> &b) {
        bool need = !prune;
#pragma unroll
        for (int r = 0; r < kRT; ++r) need |= point_box<0, NBC, NP, kKnnQ>(ref[r], b) < kd[r][SR - 1];
        return need;
    };
    int slot_st = -1;        // lane s: sub-tile in ring slot s
    int issued = 0;
    uint32_t nsub = 0;
    for (; issued < NSLOT; ++issued) {
        const int st = wk.next(fb, prune ? bound : INFINITY, true, refs_need);
        if (st < 0) break;
        if (lane == issued) slot_st = st;
        if (lane == 0) ring_issue(ring, issued, cp + (int64_t)st * kSub * DP);
    }
    for (int used = 0; used < issued; ++used) {
        const int slot = used % NSLOT;
        mbar_wait(&ring.full[slot], (uint32_t)(used / NSLOT) & 1u);
        const float4 *tile = reinterpret_cast<const float4 *>(ring.buf[slot]);
        constexpr int G = 2 * PG < D ? 2 * PG : D;  // gate columns 0 .. G-1
        constexpr int NQ = DP / 4;
        float4 nxt[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) nxt[q] = tile[q];
#pragma unroll 2
        for (int j = 0; j < kSub; ++j) {
            float4 cur[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) cur[q] = nxt[q];
            if (j + 1 < kSub) {  // prefetch the next candidate row
#pragma unroll
                for (int q = 0; q < NQ; ++q) nxt[q] = tile[(j + 1) * NQ + q];
            }
            const float2 *c = reinterpret_cast<const float2 *>(cur);
            float a[kRT][2 * NP];
            float dj[kRT];
            bool need = false;
#pragma unroll
            for (int r = 0; r < kRT; ++r) {
                diff_pairs<D, 0, PG>(ref[r], c, a[r]);
                dj[r] = maxabs0<0, G, 2 * NP>(a[r]);
                need |= dj[r] < kd[r][SR - 1];
            }
            if (__any_sync(0xffffffffu, need)) {
                bool ins = false;
#pragma unroll
                for (int r = 0; r < kRT; ++r) {
                    diff_pairs<D, PG, NP>(ref[r], c, a[r]);
                    dj[r] = maxabs<G, D, 2 * NP>(a[r], dj[r]);
                    ins |= dj[r] < kd[r][SR - 1];
                }
                if (ins) {
#pragma unroll
                    for (int r = 0; r < kRT; ++r)
                        if (SL ? dj[r] < kd[r][0] : true) insert(r, dj[r]);
                }
            }
        }
        nsub += kWarpRefs;  // every reference of the warp visits the sub-tile
        float wb = 0.0f;
#pragma unroll
        for (int r = 0; r < kRT; ++r) wb = fmaxf(wb, kd[r][SR - 1]);
        bound = warp_max_nonneg(wb);
        __syncwarp();
        const int st = wk.next(fb, prune ? bound : INFINITY, true, refs_need);
        if (st >= 0) {
            if (lane == issued % NSLOT) slot_st = st;
            if (lane == 0) ring_issue(ring, issued % NSLOT, cp + (int64_t)st * kSub * DP);
            ++issued;
        }
    }
    (void)slot_st;
    if (lane == 0) atomicAdd(work, (unsigned long long)nsub);
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
        const int idx = wrow + r * 32 + lane;
        if (idx >= ci.n) continue;
        const float t32 = kd[r][SR - 1];
        const float lo = __double2float_rd(__dsub_rd((double)t32, 2.0 * ci.delta));
        int Lc = 0;
        if constexpr (SL) {
            for (int s = 0; s < S; ++s) Lc += (lst[r][s][lane] > -INFINITY) && (lst[r][s][lane] < lo);
        } else {
#pragma unroll
            for (int s = 0; s < S; ++s) Lc += (kd[r][s] > -INFINITY) && (kd[r][s] < lo);
        }
        if (lo > 0.0f) Lc -= 1;  // the self pair (distance 0) was counted
        const int64_t orow = ci.row0 + (kmap ? kmap[ci.row0 + idx] : idx);  // count-order row
        t32_out[orow] = t32;
        L_out[orow] = Lc;
    }
}

// ---------------------------------------------------------------------------
// pass 1, compacted references (chunks >= kCompactMinRows, k + 1 <= 16).
//
// Same walk, boxes and result as knn_pass_kernel, organised like the count
// pass: the warp's 64 references and their sorted lists live in shared
// memory; for every streamed sub-tile only the references whose point-to-box
// distance is below their current k-th distance (about a quarter of them on
// embedded dynamics) ride the lanes, in grouped rounds (<= 8 / <= 16
// references: 4 / 2 lane groups over interleaved candidate rows).  A lane of
// group g > 0 starts from an empty list bounded by the reference's current
// k-th distance; at the end of the round the groups' lists are merged into
// group 0 by a shuffle tree (only when some lane found a closer row).
// ---------------------------------------------------------------------------
template <int DP, int S>
struct KnnRefs {
    float ref[32 * kRT][DP];  // fp32 centred coordinates
    float kd[S][32 * kRT];    // ascending lists ([slot][reference]: conflict-free)
    int slot[32 * kRT];       // compacted reference list of the current sub-tile
};

template <int DY, int DX, int S>
__global__ void __launch_bounds__(32, sweep_minb(1 + DY + DX, ENTE_KNN_MINB)) knn_compact_kernel(
    const float *__restrict__ pts32, const float *__restrict__ fbox,
    const ChunkInfo *__restrict__ info, const int32_t *__restrict__ tile0, int n_chunks, int k, int prune,
    const int32_t *__restrict__ kmap, float *__restrict__ t32_out, int32_t *__restrict__ L_out,
    unsigned long long *__restrict__ work) {
    static_assert(S <= 16, "register lists only");
    using L = Lay<DY, DX>;
    constexpr int D = L::D, DP = L::DP, NP = L::NP, PG = L::PG;
    constexpr int NSLOT = ENTE_KNNC_NSLOT;
    constexpr int NBC = D < 4 * kKnnQ ? D : 4 * kKnnQ;  // box columns 0 .. NBC-1
    constexpr int NQ = DP / 4;
    __shared__ SweepSmem<Ring<DP, NSLOT>, KnnRefs<DP, S>> sm;
    auto &ring = sm.ring;
    auto &rs = sm.rs;
    const TileRef tr = tile_of(tile0, n_chunks, blockIdx.x);
    const ChunkInfo ci = info[tr.chunk];
    if (!ci.ok32) return;
    const int lane = pinned_lane();
    const unsigned lt = (1u << lane) - 1u;
    const float *cp = pts32 + ci.prow0 * DP;
    const float4 *fb = reinterpret_cast<const float4 *>(fbox) + (ci.prow0 / kSub) * 2 * kKnnQ;
    const int wrow = tr.r0;
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
        const int ri = r * 32 + lane;
        const int idx = wrow + ri;
        const bool valid = idx < ci.n;
#pragma unroll
        for (int c = 0; c < DP; ++c) rs.ref[ri][c] = (valid && c < D) ? cp[(int64_t)idx * DP + c] : 0.0f;
#pragma unroll
        for (int s = 0; s < S; ++s) rs.kd[s][ri] = (!valid || s < S - (k + 1)) ? -INFINITY : INFINITY;
    }
#if ENTE_KNNC_REGREF
    // this lane's own references and current k-th distances in registers
    // (walker tests); the k-th values are refreshed after every sub-tile
    float2 myref[kRT][NP];
    float mythr[kRT];
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
        const int idx = wrow + r * 32 + lane;
        load_ref<D>(myref[r], cp + (int64_t)idx * DP, idx < ci.n);
        mythr[r] = idx < ci.n ? INFINITY : -INFINITY;
    }
#endif
    // this lane's references: point-to-box tests against their current k-th
    auto refs_need = [&](const Box<kKnnQ> &b) {
        uint32_t need = 0u;
#pragma unroll
        for (int r = 0; r < kRT; ++r) {
#if ENTE_KNNC_REGREF
            const float thr = mythr[r];
            const float2 (&nr)[NP] = myref[r];
#else
            const int ri = r * 32 + lane;
            const float thr = rs.kd[S - 1][ri];
            float2 nr[NP];
            const float2 *rr = reinterpret_cast<const float2 *>(rs.ref[ri]);
#pragma unroll
            for (int p = 0; p < NP; ++p) nr[p] = make_float2(-rr[p].x, -rr[p].y);
#endif
            // (a finished or padding reference has thr = -inf: no box distance is below it)
            need |= (prune ? point_box<0, NBC, NP, kKnnQ>(nr, b) < thr : thr > -INFINITY) ? (1u << r) : 0u;
        }
        return need;
    };
    auto warp_bound = [&]() {
        float wb = 0.0f;
#pragma unroll
        for (int r = 0; r < kRT; ++r) {
            const float t = rs.kd[S - 1][r * 32 + lane];
#if ENTE_KNNC_REGREF
            mythr[r] = t;
#endif
            wb = fmaxf(wb, t);
        }
        return warp_max_nonneg(wb);
    };
    if (lane < NSLOT) mbar_init(&ring.full[lane], 1);
    fence_barrier_init();
    __syncwarp();
    KnnWalker<kKnnQ> wk;
    wk.init(fb, reinterpret_cast<const float4 *>(fbox) + ci.sbk, wrow, ci.n, ci.npad, lane);
    float bound = INFINITY;  // warp max of the current k-th distances
    int slot_st = -1;
    uint32_t slot_need = 0u;
    int issued = 0;
    uint32_t nsub = 0;
    for (; issued < NSLOT; ++issued) {
        const int st = wk.next(fb, prune ? bound : INFINITY, true, refs_need);
        if (st < 0) break;
        if (lane == issued) slot_st = st;
        slot_need |= wk.need << (kRT * issued);
        if (lane == 0) ring_issue(ring, issued, cp + (int64_t)st * kSub * DP);
    }
    for (int used = 0; used < issued; ++used) {
        const int slot = used % NSLOT;
        const uint32_t nb = (slot_need >> (kRT * slot)) & ((1u << kRT) - 1u);
        int base = 0;
#pragma unroll
        for (int r = 0; r < kRT; ++r) {
            const uint32_t m = __ballot_sync(0xffffffffu, (nb >> r) & 1u);
            if ((nb >> r) & 1u) rs.slot[base + __popc(m & lt)] = r * 32 + lane;
            base += __popc(m);
        }
        const int nneed = base;
        __syncwarp();
        mbar_wait(&ring.full[slot], (uint32_t)(used / NSLOT) & 1u);
        const float4 *tile = reinterpret_cast<const float4 *>(ring.buf[slot]);
        auto run_round = [&](auto lgc, int round) {
            constexpr int LG = decltype(lgc)::value;
            constexpr int G = 1 << LG, PER = 32 >> LG, STRIDE = G * NQ;
            constexpr int STEPS = kSub >> LG;  // candidate rows per lane (even: kSub >= 16, G <= 8)
            static_assert(STEPS >= 2 && STEPS % 2 == 0, "row pairs");
            const int g = lane >> (5 - LG);
            const int it = lane & (PER - 1);
            const bool active = round + it < nneed;
            const int ri = active ? rs.slot[round + it] : 0;
            float2 ref[NP];
            {
                const float2 *rr = reinterpret_cast<const float2 *>(rs.ref[ri]);
#pragma unroll
                for (int p = 0; p < NP; ++p) ref[p] = make_float2(-rr[p].x, -rr[p].y);
            }
            float kd[S];
#pragma unroll
            for (int s = 0; s < S; ++s) kd[s] = !active ? -INFINITY : (g == 0 ? rs.kd[s][ri] : INFINITY);
            float thr = active ? rs.kd[S - 1][ri] : -INFINITY;  // rows at or beyond it cannot enter
            auto visit = [&](const float4 (&cur)[NQ]) {
                const float2 *c = reinterpret_cast<const float2 *>(cur);
                float a[2 * NP];
                // straight line: a warp vote on the gate columns rarely
                // skips a row once the round's lanes hold different
                // references, so every column is differenced (measured:
                // C2 kNN pass 33.6 -> 31.9 ms, C4 29.2 -> 26.5 ms)
                diff_pairs<D, 0, NP>(ref, c, a);
                const float dj = maxabs0<0, D, 2 * NP>(a);
                if (dj < thr) {
                    insert_sorted<S>(kd, dj);
                    thr = fminf(thr, kd[S - 1]);
                }
            };
            const float4 *pr = tile + g * NQ;
            float4 ra[NQ], rb[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) ra[q] = pr[q];
ENTE_UNROLL(ENTE_KNNC_UNROLL)
            for (int s = 0; s < STEPS; s += 2, pr += 2 * STRIDE) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) rb[q] = pr[STRIDE + q];
                visit(ra);
#pragma unroll
                for (int q = 0; q < NQ; ++q) ra[q] = pr[2 * STRIDE + q];  // may read past the ring (SweepSmem)
                visit(rb);
            }
            // merge the groups' lists into group 0 (tree; lists are ascending)
#pragma unroll
            for (int o = 16; o >= PER; o >>= 1) {
                const float p0 = __shfl_xor_sync(0xffffffffu, kd[0], o);
                const bool recv = (lane & o) == 0;
                if (__any_sync(0xffffffffu, recv && p0 < kd[S - 1])) {
                    float pv[S];
#pragma unroll
                    for (int s = 0; s < S; ++s) pv[s] = __shfl_xor_sync(0xffffffffu, kd[s], o);
                    if (recv) {
#pragma unroll
                        for (int s = 0; s < S; ++s) insert_sorted<S>(kd, pv[s]);
                    }
                }
            }
            if (active && g == 0) {
#pragma unroll
                for (int s = 0; s < S; ++s) rs.kd[s][ri] = kd[s];
            }
            __syncwarp();
        };
        for (int round = 0; round < nneed; round += 32) {
            const int m = nneed - round;
            if (m <= 8)
                run_round(std::integral_constant<int, 2>{}, round);
            else if (m <= 16)
                run_round(std::integral_constant<int, 1>{}, round);
            else
                run_round(std::integral_constant<int, 0>{}, round);
        }
        nsub += nneed;  // (reference, sub-tile) visits of compacted references
        bound = warp_bound();
        const int st = wk.next(fb, prune ? bound : INFINITY, true, refs_need);
        if (st >= 0) {
            const int ns = issued % NSLOT;
            if (lane == ns) slot_st = st;
            slot_need = (slot_need & ~(((1u << kRT) - 1u) << (kRT * ns))) | (wk.need << (kRT * ns));
            if (lane == 0) ring_issue(ring, ns, cp + (int64_t)st * kSub * DP);
            ++issued;
        }
    }
    (void)slot_st;
    if (lane == 0) atomicAdd(work, (unsigned long long)nsub);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
        const int ri = r * 32 + lane;
        const int idx = wrow + ri;
        if (idx >= ci.n) continue;
        const float t32 = rs.kd[S - 1][ri];
        const float lo = __double2float_rd(__dsub_rd((double)t32, 2.0 * ci.delta));
        int Lc = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) Lc += (rs.kd[s][ri] > -INFINITY) && (rs.kd[s][ri] < lo);
        if (lo > 0.0f) Lc -= 1;  // the self pair (distance 0) was counted
        const int64_t orow = ci.row0 + (kmap ? kmap[ci.row0 + idx] : idx);  // count-order row
        t32_out[orow] = t32;
        L_out[orow] = Lc;
    }
}

// ---------------------------------------------------------------------------
// pass 2, direct mapping (small chunks): two fixed references per lane
//   marginal 0 = y-past (A), 1 = y + y-past (m2), 2 = y-past + x-past (m3)
//   A <= every marginal and the joint, so A > hi settles a pair (outside
//   everywhere, no event) after the gate columns alone
// ---------------------------------------------------------------------------
template <int DY, int DX>
__global__ void __launch_bounds__(32, sweep_minb(1 + DY + DX, ENTE_CNT_MINB)) count_pass_direct_kernel(
    const float *__restrict__ pts32, const float *__restrict__ fbox,
    const ChunkInfo *__restrict__ info, const int32_t *__restrict__ tile0, int n_chunks,
    const float *__restrict__ t32_in, int64_t ws_rows, int prune, int32_t *__restrict__ cnt_out,
    uint32_t *__restrict__ ev, int32_t *__restrict__ ev_n, uint32_t fmask,
    unsigned long long *__restrict__ work) {
    using L = Lay<DY, DX>;
    constexpr int D = L::D, DP = L::DP, NP = L::NP, PG = L::PG, NSLOT = L::NSLOT;
    __shared__ __align__(128) Ring<DP, NSLOT> ring;
    const TileRef tr = tile_of(tile0, n_chunks, blockIdx.x);
    const ChunkInfo ci = info[tr.chunk];
    if (!ci.ok32) return;
    const int lane = pinned_lane();
    const float *cp = pts32 + ci.prow0 * DP;
    const float4 *fb = reinterpret_cast<const float4 *>(fbox) + (ci.prow0 / kSub) * 2;
    const int wrow = tr.r0;
    float2 ref[kRT][NP];
    Band band[kRT];
    uint32_t cA[kRT], c2[kRT], c3[kRT];
    int nev[kRT];
    float hmax = 0.0f;
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
        const int idx = wrow + r * 32 + lane;
        const bool valid = idx < ci.n;
        load_ref<D>(ref[r], cp + (int64_t)idx * DP, valid);
        band[r] = make_band(valid ? t32_in[ci.row0 + idx] : 0.0f, ci.delta);
        if (!valid) {  // empty band: never inside, never an event
            band[r].lo = -INFINITY;
            band[r].nlo = INFINITY;
            band[r].hi = -INFINITY;
            band[r].w = -1.0f;
        } else {
            hmax = fmaxf(hmax, band[r].hi);
        }
        cA[r] = c2[r] = c3[r] = 0;
        nev[r] = 0;
    }
    const float bound = warp_max_nonneg(hmax);
    constexpr int NG = DY < kGate ? DY : kGate;
    auto refs_need = [&](const Box<1> &b) {
        bool need = !prune;
#pragma unroll
        for (int r = 0; r < kRT; ++r) need |= point_box<1, NG, NP, 1>(ref[r], b) <= band[r].hi;
        return need;
    };
    if (lane < NSLOT) mbar_init(&ring.full[lane], 1);
    fence_barrier_init();
    __syncwarp();
    Walker<1> wk;
    wk.init(fb, reinterpret_cast<const float4 *>(fbox) + ci.sbg, wrow, ci.n, ci.npad, lane);
    int slot_st = -1;
    int issued = 0;
    uint32_t nsub = 0;
    for (; issued < NSLOT; ++issued) {
        const int st = wk.next(fb, prune ? bound : INFINITY, false, refs_need);
        if (st < 0) break;
        if (lane == issued) slot_st = st;
        if (lane == 0) ring_issue(ring, issued, cp + (int64_t)st * kSub * DP);
    }
    for (int used = 0; used < issued; ++used) {
        const int slot = used % NSLOT;
        const int cur_st = __shfl_sync(0xffffffffu, slot_st, slot);
        mbar_wait(&ring.full[slot], (uint32_t)(used / NSLOT) & 1u);
        const float4 *tile = reinterpret_cast<const float4 *>(ring.buf[slot]);
        constexpr int NQ = DP / 4;
        float4 nxt[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) nxt[q] = tile[q];
#pragma unroll 2
        for (int j = 0; j < kSub; ++j) {
            float4 cur[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) cur[q] = nxt[q];
            if (j + 1 < kSub) {  // prefetch the next candidate row
#pragma unroll
                for (int q = 0; q < NQ; ++q) nxt[q] = tile[(j + 1) * NQ + q];
            }
            const float2 *c = reinterpret_cast<const float2 *>(cur);
            float a[kRT][2 * NP];
            float vA[kRT];
            bool need[kRT];
#pragma unroll
            for (int r = 0; r < kRT; ++r) {
                diff_pairs<D, 0, PG>(ref[r], c, a[r]);
                vA[r] = maxabs0<1, 1 + DY, 2 * NP>(a[r]);
                need[r] = vA[r] <= band[r].hi;
            }
            // one warp vote per reference slot: the slots hold the two halves
            // of the warp's Morton-ordered group, so a candidate often matters
            // to one half only
#pragma unroll
            for (int r = 0; r < kRT; ++r) {
                if (!__any_sync(0xffffffffu, need[r])) continue;
                diff_pairs<D, PG, NP>(ref[r], c, a[r]);
                const float A = vA[r];
                const float m2 = fmaxf(A, fabsf(a[r][0]));
                const float m3 = maxabs<1 + DY, D, 2 * NP>(a[r], A);
                const float jd = fmaxf(m2, m3);
                // certain-inside counts: sign bit of (v - lo)
                const float2 e = __fadd2_rn(make_float2(A, m2), make_float2(band[r].nlo, band[r].nlo));
                const float2 e34 = __fadd2_rn(make_float2(m3, jd), make_float2(band[r].nlo, band[r].nlo));
                cA[r] += __float_as_uint(e.x) >> 31;
                c2[r] += __float_as_uint(e.y) >> 31;
                c3[r] += __float_as_uint(e34.x) >> 31;
                // conservative band test on the same differences: min |v - lo| <= w
                const float bm = fminf(fminf(fabsf(e.x), fabsf(e.y)), fminf(fabsf(e34.x), fabsf(e34.y)));
                if (bm <= band[r].w) {
                    const float lo = band[r].lo, hi = band[r].hi;
                    uint32_t f = ((A >= lo && A <= hi) ? 1u : 0u) | ((m2 >= lo && m2 <= hi) ? 2u : 0u) |
                                 ((m3 >= lo && m3 <= hi) ? 4u : 0u) | ((jd >= lo && jd <= hi) ? 8u : 0u);
                    f &= fmask;
                    if (f) {
                        const int idx = wrow + r * 32 + lane;
                        const int jg = cur_st * kSub + j;
                        if (nev[r] < kCap) ev[(ci.row0 + idx) * kCap + nev[r]] = (uint32_t)jg | (f << 28);
                        ++nev[r];
                    }
                }
            }
        }
        nsub += kWarpRefs;  // every reference of the warp visits the sub-tile
        __syncwarp();
        const int st = wk.next(fb, prune ? bound : INFINITY, false, refs_need);
        if (st >= 0) {
            if (lane == issued % NSLOT) slot_st = st;
            if (lane == 0) ring_issue(ring, issued % NSLOT, cp + (int64_t)st * kSub * DP);
            ++issued;
        }
    }
    if (lane == 0) atomicAdd(work, (unsigned long long)nsub);
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
        const int idx = wrow + r * 32 + lane;
        if (idx >= ci.n) continue;
        const uint32_t self = band[r].lo > 0.0f ? 1u : 0u;  // the self pair counted as inside
        const int64_t row = ci.row0 + idx;
        cnt_out[row] = (int32_t)(cA[r] - self);
        cnt_out[ws_rows + row] = (int32_t)(c2[r] - self);
        cnt_out[2 * ws_rows + row] = (int32_t)(c3[r] - self);
        ev_n[row] = nev[r];
    }
}

// ---------------------------------------------------------------------------
// pass 2: certain counts in the three TE marginals + band events
//   marginal 0 = y-past (A), 1 = y + y-past (m2), 2 = y-past + x-past (m3)
//   A <= every marginal and the joint, so A > hi settles a pair (outside
//   everywhere, no event) after the gate columns alone.
//
// References are compacted.  The warp's 64 references live in
// shared memory (coordinates, band, counts, event fill); for every streamed
// sub-tile the walker's per-reference point-to-box tests say which of them
// can have a pair inside the band (about a third of an evaluated sub-tile's
// references), and only those are packed onto the lanes, one per lane, in
// rounds of 32 -- most sub-tiles need one round instead of the two a fixed
// two-references-per-lane mapping costs.  Per round a lane reloads its
// reference from shared memory and folds its counts back afterwards.
// ---------------------------------------------------------------------------
template <int DP, int NSLOT, int RT = kRT>
struct CountRefs {
    float ref[32 * RT][DP];  // fp32 centred coordinates
    float lo[32 * RT], hi[32 * RT], w[32 * RT];
    uint32_t cnt[3][32 * RT];
    int nev[32 * RT];
    int slot[32 * RT];       // compacted reference list of the current sub-tile
};

// references per lane of the count sweeps: the KO sweep visits few rows per
// (reference, sub-tile) in the principal-axis order, so 128-reference groups
// amortise the walk better (C2 count sweep, ms: 64 refs 34.5, 96 31.8, 128 32.3, 256 44.3)
template <bool KO>
__host__ __device__ constexpr int count_rt() { return KO ? ENTE_KO_RT : kRT; }

// KO (shared-y TE batches): the same sweep over the kNN-order copy and its
// all-column boxes, counting only the y-past + x-past marginal (m3) and
// recording m3 / joint (jd) band events; the y marginals are counted once
// per point for the whole batch (shared_y.cu).  Pruning uses box columns
// 1 .. 4*kKnnQ-1 (column 0 is not in m3, which bounds jd from below).
template <int DY, int DX, bool KO>
__global__ void __launch_bounds__(32, sweep_minb(1 + DY + DX, ENTE_CNT_MINB)) count_pass_kernel(
    const float *__restrict__ pts32, const float *__restrict__ fbox,
    const ChunkInfo *__restrict__ info, const int32_t *__restrict__ tile0, int n_chunks,
    const float *__restrict__ t32_in, int64_t ws_rows, int prune, int32_t *__restrict__ cnt_out,
    uint32_t *__restrict__ ev, int32_t *__restrict__ ev_n, uint32_t fmask,
    unsigned long long *__restrict__ work) {
    using L = Lay<DY, DX>;
    constexpr int D = L::D, DP = L::DP, NP = L::NP, PG = L::PG;
    constexpr int NSLOT = L::NSLOT < ENTE_CNT_NSLOT ? L::NSLOT : ENTE_CNT_NSLOT;
    constexpr int RT = count_rt<KO>(), WR = 32 * RT;  // references per lane / per warp
    __shared__ SweepSmem<Ring<DP, NSLOT>, CountRefs<DP, NSLOT, RT>> sm;
    auto &ring = sm.ring;
    auto &rs = sm.rs;
    const TileRef tr = tile_of(tile0, n_chunks, blockIdx.x, WR);
    const ChunkInfo ci = info[tr.chunk];
    if (!ci.ok32) return;
    const int lane = pinned_lane();
    const unsigned lt = (1u << lane) - 1u;
    const float *cp = pts32 + ci.prow0 * DP;
    constexpr int Q = KO ? kKnnQ : 1;  // float4 quads per box half
    const float4 *fb = reinterpret_cast<const float4 *>(fbox) + (ci.prow0 / kSub) * 2 * Q;
    const int wrow = tr.r0;
    float myhi[RT];
    float hmax = 0.0f;
#pragma unroll
    for (int r = 0; r < RT; ++r) {
        const int ri = r * 32 + lane;
        const int idx = wrow + ri;
        const bool valid = idx < ci.n;
#pragma unroll
        for (int c = 0; c < DP; ++c) rs.ref[ri][c] = (valid && c < D) ? cp[(int64_t)idx * DP + c] : 0.0f;
        Band b = make_band(valid ? t32_in[ci.row0 + idx] : 0.0f, ci.delta);
        if (!valid) {  // empty band: never inside, never an event, never needed
            b.lo = -INFINITY;
            b.hi = -INFINITY;
            b.w = -1.0f;
            b.nt = 0.0f;
        } else {
            hmax = fmaxf(hmax, b.hi);
        }
        rs.lo[ri] = b.lo;
        rs.hi[ri] = b.hi;
        rs.w[ri] = b.w;
        // the reference box test's threshold: the band's upper end, or (no
        // pruning) +inf for a live reference and -inf for padding (d >= 0)
        myhi[r] = prune ? b.hi : (b.hi > -INFINITY ? INFINITY : -INFINITY);
        rs.cnt[0][ri] = rs.cnt[1][ri] = rs.cnt[2][ri] = 0u;
        rs.nev[ri] = 0;
    }
    const float bound = warp_max_nonneg(hmax);
    constexpr int NG = DY < kGate ? DY : kGate;
    constexpr int NBC = D < 4 * kKnnQ ? D : 4 * kKnnQ;  // KO: box columns 0 .. NBC-1
    // this lane's own references' gate columns (negated, packed), read back
    // from shared memory so they hold no registers through the rounds
    struct NegRef {
        float2 v[NP];
    };
    auto gate_ref = [&](int r) {
        NegRef nr;
        const float2 *rr = reinterpret_cast<const float2 *>(rs.ref[r * 32 + lane]);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const float2 v = (KO || p <= NG / 2) ? rr[p] : make_float2(0.0f, 0.0f);
            nr.v[p] = make_float2(-v.x, -v.y);
        }
        return nr;
    };
    auto refs_need = [&](const Box<Q> &b) {
        uint32_t need = 0u;
#pragma unroll
        for (int r = 0; r < RT; ++r) {
            float d;
            if constexpr (KO) d = point_box_cols<1, NBC, NP, Q>(gate_ref(r).v, b);
            else d = point_box<1, NG, NP, 1>(gate_ref(r).v, b);
            need |= d <= myhi[r] ? (1u << r) : 0u;
        }
        return need;
    };
    if (lane < NSLOT) mbar_init(&ring.full[lane], 1);
    fence_barrier_init();
    __syncwarp();
    // m3 sweep over the kNN order: block walk (its kNN-order sub-tiles are
    // scattered over m3 space, whole blocks fall outside the bands); the
    // gate-column count passes keep the sub-tile walk (block boxes over
    // four gate columns rarely exclude a block: C4 +0.4 %)
    std::conditional_t<KO, BlockWalker<Q>, Walker<Q>> wk;
    wk.init(fb, reinterpret_cast<const float4 *>(fbox) + (Q == 1 ? ci.sbg : ci.sbk), wrow, ci.n, ci.npad,
            lane, WR);
    if constexpr (KO) {  // column 0 is not an m3 column: the warp box spans it
        wk.own.lo[0].x = -INFINITY;
        wk.own.hi[0].x = INFINITY;
    }
    int slot_st = -1;
    uint32_t slot_need = 0u;  // RT bits per ring slot: this lane's needs of the issued sub-tiles
    int issued = 0;
    uint32_t nsub = 0;
    for (; issued < NSLOT; ++issued) {
        const int st = wk.next(fb, prune ? bound : INFINITY, false, refs_need);
        if (st < 0) break;
        if (lane == issued) slot_st = st;
        slot_need |= wk.need << (RT * issued);
        if (lane == 0) ring_issue(ring, issued, cp + (int64_t)st * kSub * DP);
    }
    for (int used = 0; used < issued; ++used) {
        const int slot = used % NSLOT;
        const int cur_st = __shfl_sync(0xffffffffu, slot_st, slot);
        const uint32_t nb = (slot_need >> (RT * slot)) & ((1u << RT) - 1u);
        // compact the references that need this sub-tile
        int base = 0;
#pragma unroll
        for (int r = 0; r < RT; ++r) {
            const uint32_t m = __ballot_sync(0xffffffffu, (nb >> r) & 1u);
            if ((nb >> r) & 1u) rs.slot[base + __popc(m & lt)] = r * 32 + lane;
            base += __popc(m);
        }
        const int nneed = base;
        __syncwarp();
        mbar_wait(&ring.full[slot], (uint32_t)(used / NSLOT) & 1u);
        const float4 *tile = reinterpret_cast<const float4 *>(ring.buf[slot]);
        constexpr int NQ = DP / 4;
        // Grouped rounds: with at most 8 (16) references left, the warp splits
        // into 4 (2) groups of lanes that share the round's references and
        // take every 4th (2nd) candidate row, so the round walks 8 (16) rows
        // instead of 32 (half the rounds hold <= 8 references).  LG = log2 of
        // the group count is a compile-time constant of each specialisation.
        auto run_round = [&](auto lgc, int round) {
            constexpr int LG = decltype(lgc)::value;
            constexpr int G = 1 << LG, PER = 32 >> LG, STRIDE = G * NQ;
            constexpr int STEPS = kSub >> LG;  // candidate rows per lane (even: kSub >= 16, G <= 8)
            static_assert(STEPS >= 2 && STEPS % 2 == 0, "row pairs");
            const int g = lane >> (5 - LG);  // group: candidate rows g, g + G, g + 2G, ...
            const int it = lane & (PER - 1);
            const bool active = round + it < nneed;
            const int ri = active ? rs.slot[round + it] : 0;
            float2 ref[NP];
            {
                const float2 *rr = reinterpret_cast<const float2 *>(rs.ref[ri]);
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    const float2 v = rr[p];
                    ref[p] = make_float2(-v.x, -v.y);
                }
            }
            const float lo = active ? rs.lo[ri] : -INFINITY;
            const float hi = active ? rs.hi[ri] : -INFINITY;
            const float nlo = -lo, wb = active ? rs.w[ri] : -1.0f;
            uint32_t cA = 0u, c2 = 0u, c3 = 0u;
            // one candidate row (sub-tile row j) against this lane's reference
            auto visit = [&](const float4 (&cur)[NQ], int j) {
                const float2 *c = reinterpret_cast<const float2 *>(cur);
                float a[2 * NP];
                // Straight line: about half of the (reference, row) pairs a
                // compacted round visits pass the y-past gate A <= hi, so a
                // warp vote on it almost never skips a row; all the columns
                // are differenced unconditionally.  jd = max(m2, m3) is one
                // of m2, m3, so the band test needs only A, m2, m3.
                diff_pairs<D, 0, NP>(ref, c, a);
                if constexpr (KO) {
                    const float m3 = maxabs0<1, D, 2 * NP>(a);
                    const float jd = fmaxf(m3, fabsf(a[0]));
                    const float2 e = __fadd2_rn(make_float2(m3, jd), make_float2(nlo, nlo));
                    c3 += __float_as_uint(e.x) >> 31;
                    if (fminf(fabsf(e.x), fabsf(e.y)) <= wb) {
                        uint32_t f = ((m3 >= lo && m3 <= hi) ? 4u : 0u) | ((jd >= lo && jd <= hi) ? 8u : 0u);
                        f &= fmask;
                        if (f) {
                            const int pos = atomicAdd(&rs.nev[ri], 1);
                            if (pos < kCap)
                                ev[(ci.row0 + wrow + ri) * kCap + pos] = (uint32_t)(cur_st * kSub + j) | (f << 28);
                        }
                    }
                    return;
                }
                const float A = maxabs0<1, 1 + DY, 2 * NP>(a);
                const float m2 = fmaxf(A, fabsf(a[0]));
                const float m3 = maxabs<1 + DY, D, 2 * NP>(a, A);
                const float2 e = __fadd2_rn(make_float2(A, m2), make_float2(nlo, nlo));
                const float e3 = __fadd_rn(m3, nlo);
                cA += __float_as_uint(e.x) >> 31;
                c2 += __float_as_uint(e.y) >> 31;
                c3 += __float_as_uint(e3) >> 31;
                const float bm = fminf(fminf(fabsf(e.x), fabsf(e.y)), fabsf(e3));
                if (bm <= wb) {
                    const float jd = fmaxf(m2, m3);
                    uint32_t f = ((A >= lo && A <= hi) ? 1u : 0u) | ((m2 >= lo && m2 <= hi) ? 2u : 0u) |
                                 ((m3 >= lo && m3 <= hi) ? 4u : 0u) | ((jd >= lo && jd <= hi) ? 8u : 0u);
                    f &= fmask;
                    if (f) {
                        const int pos = atomicAdd(&rs.nev[ri], 1);
                        if (pos < kCap)
                            ev[(ci.row0 + wrow + ri) * kCap + pos] = (uint32_t)(cur_st * kSub + j) | (f << 28);
                    }
                }
            };
            // ping-pong row registers: the next row's LDS overlaps this row's math
            const float4 *pr = tile + g * NQ;  // this lane's row s (loop-carried)
            float4 ra[NQ], rb[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) ra[q] = pr[q];
            // (KO rows are cheaper: two rows per loop trip measured 4 % faster)
            constexpr int kTrip = KO ? ENTE_KO_UNROLL : ENTE_CNT_UNROLL;
#pragma unroll kTrip
            for (int s = 0; s < STEPS; s += 2, pr += 2 * STRIDE) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) rb[q] = pr[STRIDE + q];
                visit(ra, s * G + g);
                // the last iteration may read G rows past the ring (SweepSmem)
#pragma unroll
                for (int q = 0; q < NQ; ++q) ra[q] = pr[2 * STRIDE + q];
                visit(rb, (s + 1) * G + g);
            }
            // fold the groups' counts onto group 0
#pragma unroll
            for (int o = PER; o < 32; o <<= 1) {
                cA += __shfl_xor_sync(0xffffffffu, cA, o);
                c2 += __shfl_xor_sync(0xffffffffu, c2, o);
                c3 += __shfl_xor_sync(0xffffffffu, c3, o);
            }
            if (active && g == 0) {
                rs.cnt[0][ri] += cA;
                rs.cnt[1][ri] += c2;
                rs.cnt[2][ri] += c3;
            }
            __syncwarp();
        };
        for (int round = 0; round < nneed; round += 32) {
            const int m = nneed - round;
            if (ENTE_CNT_GROUPS > 1 && m <= 4)
                run_round(std::integral_constant<int, 3>{}, round);
            else if (ENTE_CNT_GROUPS && m <= 8)
                run_round(std::integral_constant<int, 2>{}, round);
            else if (ENTE_CNT_GROUPS && m <= 16)
                run_round(std::integral_constant<int, 1>{}, round);
            else
                run_round(std::integral_constant<int, 0>{}, round);
        }
        nsub += nneed;  // (reference, sub-tile) visits of compacted references
        __syncwarp();
        const int st = wk.next(fb, prune ? bound : INFINITY, false, refs_need);
        if (st >= 0) {
            const int ns = issued % NSLOT;
            if (lane == ns) slot_st = st;
            slot_need = (slot_need & ~(((1u << RT) - 1u) << (RT * ns))) | (wk.need << (RT * ns));
            if (lane == 0) ring_issue(ring, ns, cp + (int64_t)st * kSub * DP);
            ++issued;
        }
    }
    if (lane == 0) atomicAdd(work, (unsigned long long)nsub);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < RT; ++r) {
        const int ri = r * 32 + lane;
        const int idx = wrow + ri;
        if (idx >= ci.n) continue;
        const uint32_t self = rs.lo[ri] > 0.0f ? 1u : 0u;  // the self pair counted as inside
        const int64_t row = ci.row0 + idx;
        cnt_out[row] = KO ? 0 : (int32_t)(rs.cnt[0][ri] - self);
        cnt_out[ws_rows + row] = KO ? 0 : (int32_t)(rs.cnt[1][ri] - self);
        cnt_out[2 * ws_rows + row] = (int32_t)(rs.cnt[2][ri] - self);
        ev_n[row] = rs.nev[ri];
    }
}

// ---------------------------------------------------------------------------
// resolve: fp64 certification of band events (sorted positions -> rows via perm)
// one thread per reference of a 128-reference tile
// ---------------------------------------------------------------------------
struct TeLayout {
    int dy;
    int nout;
    int slot[kMaxMarg];  // output o <- TE marginal slot (0, 1, 2)
};

__device__ __forceinline__ void te_dist64(const double *ref, const double *q, int dim, int dy,
                                          double &A, double &m2, double &m3, double &jd) {
    double a = 0.0, b = 0.0;
    for (int c = 1; c < dim; ++c) {
        const double v = fabs(__dsub_rn(ref[c], q[c]));
        if (c <= dy) a = fmax(a, v);
        else b = fmax(b, v);
    }
    const double y = fabs(__dsub_rn(ref[0], q[0]));
    A = a;
    m2 = fmax(a, y);
    m3 = fmax(a, b);
    jd = fmax(m2, m3);
}

// ---------------------------------------------------------------------------
// rescan: exact eps and counts for references whose band events overflowed
// (heavily tied data).  One warp per listed sorted row; the lanes take the
// 32 candidates of a sub-tile, sub-tiles are pruned by their gate boxes, and
// every candidate the fp32 filter cannot decide is settled in fp64 on the
// spot, so there is no per-point event limit:
//   A  eps = k-th smallest joint d64 over the candidates with d32 <= hiA,
//      hiA = up(t32 + 2 delta) (they include the true k nearest); per-lane
//      sorted fp64 lists, k rounds of warp-minimum extraction
//   B  with eps exact: v32 < lo = down(eps - delta) -> inside,
//      v32 > hi = up(eps + delta) -> outside, otherwise compare v64 < eps
// ---------------------------------------------------------------------------
constexpr int kRescanWarps = 4;

template <int DY, int DX, int S>
__global__ void __launch_bounds__(kRescanWarps * 32) rescan_kernel(
    const float *__restrict__ pts32, const float *__restrict__ fbox, const double *__restrict__ pts64,
    const double *__restrict__ pts64s, const ChunkInfo *__restrict__ info, int n_chunks,
    const int32_t *__restrict__ perm, const float *__restrict__ t32_in,
    const int64_t *__restrict__ list, const int32_t *__restrict__ list_n, int k, TeLayout lay,
    int64_t total_rows, double *__restrict__ out_eps, int32_t *__restrict__ out_counts) {
    using L = Lay<DY, DX>;
    constexpr int D = L::D, DP = L::DP, NP = L::NP;
    constexpr int NG = DY < kGate ? DY : kGate;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * kRescanWarps;
    const int64_t count = *list_n;
    for (int64_t it = (int64_t)blockIdx.x * kRescanWarps + (threadIdx.x >> 5); it < count;
         it += nwarps) {
        const int64_t srow = list[it];
        const int c = chunk_of_row(info, n_chunks, srow);
        const ChunkInfo ci = info[c];
        const int s = (int)(srow - ci.row0);  // sorted position of the reference
        const int64_t row = ci.row0 + perm[srow];
        const float *cp = pts32 + ci.prow0 * DP;
        const float4 *fb = reinterpret_cast<const float4 *>(fbox) + (ci.prow0 / kSub) * 2;
        const int nsub = ci.npad / kSub;
        float2 ref[NP];
        load_ref<D>(ref, cp + (int64_t)s * DP, true);
        double r64[D];
#pragma unroll
        // fp64 rows in the count order (coalesced per sub-tile), written for
        // every chunk with rescans by gather64_kernel
        const double *s64 = pts64s + ci.prow0 * D;
        for (int col = 0; col < D; ++col) r64[col] = s64[(int64_t)s * D + col];
        const double delta = ci.delta;
        const float hiA = __double2float_ru(__dadd_ru((double)t32_in[srow], 2.0 * delta));
        // ---- phase A: exact k-th joint distance
        double kd[S];
#pragma unroll
        for (int q = 0; q < S; ++q) kd[q] = (q < S - k) ? -INFINITY : INFINITY;
        for (int base = 0; base < nsub; base += 32) {
            const int st_l = base + lane;
            bool need = false;
            if (st_l < nsub) need = point_box<1, NG, NP, 1>(ref, load_box<1>(fb, st_l)) <= hiA;
            uint32_t m = __ballot_sync(0xffffffffu, need);
            while (m) {
                const int st = base + __ffs(m) - 1;
                m &= m - 1;
                const int j = st * kSub + lane;
                const float *q = cp + (int64_t)(lane < kSub ? j : st * kSub) * DP;
                float d = 0.0f;
#pragma unroll
                for (int col = 0; col < D; ++col) {
                    const float x = (col & 1) ? ref[col >> 1].y : ref[col >> 1].x;
                    d = fmaxf(d, fabsf(q[col] + x));
                }
                if (lane < kSub && j < ci.n && j != s && d <= hiA) {
                    const double *q64 = s64 + (int64_t)j * D;
                    double d64 = 0.0;
#pragma unroll
                    for (int col = 0; col < D; ++col) d64 = fmax(d64, fabs(__dsub_rn(r64[col], q64[col])));
                    if (d64 < kd[S - 1]) {
#pragma unroll
                        for (int q2 = S - 1; q2 >= 1; --q2) kd[q2] = fmax(kd[q2 - 1], fmin(kd[q2], d64));
                        kd[0] = fmin(kd[0], d64);
                    }
                }
            }
        }
        double eps = 0.0;
        for (int q = 0; q < k; ++q) {
            const double v = kd[S - k];
            double mn = v;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, off));
            const unsigned win = __ffs(__ballot_sync(0xffffffffu, v == mn)) - 1;
            if ((unsigned)lane == win) {
#pragma unroll
                for (int q2 = 0; q2 < S - 1; ++q2)
                    if (q2 >= S - k) kd[q2] = kd[q2 + 1];
                kd[S - 1] = INFINITY;
            }
            eps = mn;
        }
        // ---- phase B: strict counts in the three TE marginals
        const float lo = __double2float_rd(__dsub_rd(eps, delta));
        const float hi = __double2float_ru(__dadd_ru(eps, delta));
        int cnt[3] = {0, 0, 0};
        for (int base = 0; base < nsub; base += 32) {
            const int st_l = base + lane;
            bool need = false;
            if (st_l < nsub) need = point_box<1, NG, NP, 1>(ref, load_box<1>(fb, st_l)) <= hi;
            uint32_t m = __ballot_sync(0xffffffffu, need);
            while (m) {
                const int st = base + __ffs(m) - 1;
                m &= m - 1;
                const int j = st * kSub + lane;
                if (lane >= kSub || j >= ci.n || j == s) continue;
                const float *q = cp + (int64_t)j * DP;
                float a = 0.0f, b = 0.0f;
#pragma unroll
                for (int col = 1; col < D; ++col) {
                    const float x = (col & 1) ? ref[col >> 1].y : ref[col >> 1].x;
                    const float v = fabsf(q[col] + x);
                    if (col <= DY) a = fmaxf(a, v);
                    else b = fmaxf(b, v);
                }
                const float y = fabsf(q[0] + ref[0].x);
                const float v32[3] = {a, fmaxf(a, y), fmaxf(a, b)};
                bool amb = false;
#pragma unroll
                for (int o = 0; o < 3; ++o) {
                    cnt[o] += v32[o] < lo;
                    amb |= (v32[o] >= lo && v32[o] <= hi);
                }
                if (amb) {
                    double A, m2, m3, jd;
                    te_dist64(r64, s64 + (int64_t)j * D, D, DY, A, m2, m3, jd);
                    const double v64[3] = {A, m2, m3};
#pragma unroll
                    for (int o = 0; o < 3; ++o)
                        cnt[o] += (v32[o] >= lo && v32[o] <= hi) && (v64[o] < eps);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 3; ++o) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) cnt[o] += __shfl_xor_sync(0xffffffffu, cnt[o], off);
        }
        if (lane == 0) {
            out_eps[row] = eps;
            for (int o = 0; o < lay.nout; ++o) out_counts[o * total_rows + row] = cnt[lay.slot[o]];
        }
        __syncwarp();
    }
}

using KnnFn = void (*)(const float *, const float *, const ChunkInfo *, const int32_t *, int, int,
                       int, const int32_t *, float *, int32_t *, unsigned long long *);
using CountFn = void (*)(const float *, const float *, const ChunkInfo *, const int32_t *, int,
                         const float *, int64_t, int, int32_t *, uint32_t *, int32_t *, uint32_t,
                         unsigned long long *);

using RescanFn = void (*)(const float *, const float *, const double *, const double *,
                          const ChunkInfo *, int, const int32_t *, const float *, const int64_t *,
                          const int32_t *, int, TeLayout, int64_t, double *, int32_t *);


// Every kernel of one compiled (d_y, d_x) TE layout.
struct SweepSet {
    KnnFn knn[5];      // k + 1 <= 5, 8, 16 register slots; 32, 64 shared-memory slots
    KnnFn knn_compact[3];  // k + 1 <= 5, 8, 16, compacted references (chunks >= 4096 rows)
    CountFn compact;   // count pass, compacted references (chunks >= 4096 rows)
    CountFn direct;    // count pass, two references per lane (small chunks)
    CountFn count3;    // shared-y batches: m3 counts + m3/jd events on the kNN order (compacted)
    RescanFn rescan[5];  // k <= 4, 8, 16, 32, 64
};

template <int DY, int DX>
SweepSet make_sweep_set() {
    SweepSet s;
    s.knn[0] = knn_pass_kernel<DY, DX, 5>;
    s.knn[1] = knn_pass_kernel<DY, DX, 8>;
    s.knn[2] = knn_pass_kernel<DY, DX, 16>;
    s.knn[3] = knn_pass_kernel<DY, DX, 32>;
    s.knn[4] = knn_pass_kernel<DY, DX, 64>;
    s.knn_compact[0] = knn_compact_kernel<DY, DX, 5>;
    s.knn_compact[1] = knn_compact_kernel<DY, DX, 8>;
    s.knn_compact[2] = knn_compact_kernel<DY, DX, 16>;
    s.compact = count_pass_kernel<DY, DX, false>;
    s.count3 = count_pass_kernel<DY, DX, true>;
    s.direct = count_pass_direct_kernel<DY, DX>;
    s.rescan[0] = rescan_kernel<DY, DX, 4>;
    s.rescan[1] = rescan_kernel<DY, DX, 8>;
    s.rescan[2] = rescan_kernel<DY, DX, 16>;
    s.rescan[3] = rescan_kernel<DY, DX, 32>;
    s.rescan[4] = rescan_kernel<DY, DX, 64>;
    return s;
}

// the layout groups (sweeps_a/b/c.cu); false when (dy, dx) is not in the group
bool sweep_set_a(int dy, int dx, SweepSet &out);
bool sweep_set_b(int dy, int dx, SweepSet &out);
bool sweep_set_c(int dy, int dx, SweepSet &out);

inline bool find_sweep_set(int dy, int dx, SweepSet &out) {
    return sweep_set_a(dy, dx, out) || sweep_set_b(dy, dx, out) || sweep_set_c(dy, dx, out);
}

}  // namespace ente
