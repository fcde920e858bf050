// Exact batched max-norm kNN distances + strict marginal radius counts.
//
// Replaces ente.engine.batch_search (/root/reference/pkg/src/ente/engine.py:203-216):
// the reference sweeps every reference point over a first-coordinate sorted
// order in fp64 (_kth_sweep 70-123, _count_sweep 126-160).  Here the same
// exact fp64 answer is produced by an fp32 filter with a proven error bound
// and fp64 certification of the few pairs the filter cannot decide:
//
//   prep      column mean / min / max, bound
//             delta = 4 * 2^-24 * max|x - m| * (1 + 2^-20) >= |d32 - d64|
//   sort      per-chunk Morton order over the filter columns (the y-past
//             block: every contribution needs max|dy-past| inside the radius),
//             CTA radix sort; fp32 copy x32 = fl32(x - m) in that order plus
//             per-32 / per-128-row bounding boxes
//   pruning   a warp (128 sorted references) skips a 32-candidate sub-tile
//             when the fp32 box distance already exceeds its bound; boxes are
//             exact lower bounds of every d32 in them, so skipping is exact
//   pass 1    t32_i = k-th smallest fp32 distance (self excluded) via a
//             (k+1)-slot sorted register list; L_i = #{d32 < lo_i}
//   pass 2    per pair: the three TE marginal distances and the joint one;
//             d32 < lo_i counts as certainly inside, values inside the band
//             [lo_i, hi_i] = t32 -/+ 2 delta (directed rounding) are recorded
//             as events (<= kCap per point)
//   resolve   fp64 re-scoring of the events: eps_i = the (k - L_i)-th
//             smallest joint d64 among band events; marginal events inside
//             eps_i are added to the counts -> bit-identical to the reference
//   exact     warp-per-point fp64 scan (overflowed points, chunks whose
//             range defeats fp32, layouts without a compiled kernel)
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "profile.cuh"
#include "radix.cuh"

namespace ente {

// ---------------------------------------------------------------------------
// prep: column statistics, error bound, finiteness
// ---------------------------------------------------------------------------
constexpr int kSub = 32;                    // rows per sub-tile box (one warp of candidates)
constexpr int kSubPerStage = kTJ / kSub;    // sub-tiles per shared-memory stage
constexpr int kWarps = kNT / 32;            // warps per sweep CTA; warp w owns 128 refs

// per-chunk column statistics (fp64): mean, min, max of the raw values
struct ColStats {
    double mean[kMaxDim];
    double lo[kMaxDim];
    double hi[kMaxDim];
};

__global__ void __launch_bounds__(256) prep_kernel(const double *__restrict__ pts64, int dim,
                                                   ChunkInfo *__restrict__ info,
                                                   ColStats *__restrict__ stats,
                                                   int32_t *__restrict__ status, int want32) {
    const int c = blockIdx.x;
    const ChunkInfo ci = info[c];
    if (status[c] != ENTE_CHUNK_OK) return;
    __shared__ double red[3][256];
    __shared__ ColStats local;
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    const double *p = pts64 + ci.row0 * dim;
    ColStats *cs = &local;
    for (int col = 0; col < dim; ++col) {
        double s = 0.0, lo = INFINITY, hi = -INFINITY;
        for (int r = threadIdx.x; r < ci.n; r += blockDim.x) {
            const double v = p[(int64_t)r * dim + col];
            s += v;
            lo = fmin(lo, v);
            hi = fmax(hi, v);
            if (!isfinite(v)) bad = 1;
        }
        red[0][threadIdx.x] = s;
        red[1][threadIdx.x] = lo;
        red[2][threadIdx.x] = hi;
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (threadIdx.x < w) {
                red[0][threadIdx.x] += red[0][threadIdx.x + w];
                red[1][threadIdx.x] = fmin(red[1][threadIdx.x], red[1][threadIdx.x + w]);
                red[2][threadIdx.x] = fmax(red[2][threadIdx.x], red[2][threadIdx.x + w]);
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            cs->mean[col] = red[0][0] / ci.n;
            cs->lo[col] = red[1][0];
            cs->hi[col] = red[2][0];
        }
        __syncthreads();
    }
    if (bad) {
        if (threadIdx.x == 0) {
            status[c] = ENTE_CHUNK_NONFINITE;
            info[c].ok32 = 0;
        }
        return;
    }
    if (stats)
        for (int e = threadIdx.x; e < 3 * kMaxDim; e += blockDim.x)
            (&stats[c].mean[0])[e] = (&local.mean[0])[e];
    if (threadIdx.x == 0 && stats) {
        // spread s = max |fl64(x - m)| is attained at a column extreme
        double smax = 0.0;
        for (int col = 0; col < dim; ++col) {
            smax = fmax(smax, fabs(__dsub_rn(cs->lo[col], cs->mean[col])));
            smax = fmax(smax, fabs(__dsub_rn(cs->hi[col], cs->mean[col])));
        }
        // the fp32 path needs normal-range fp32 values
        const int ok = (smax > 1e-30) && (smax < 1e30);
        info[c].delta = 4.0 * 0x1p-24 * smax * (1.0 + 0x1p-20);
        info[c].ok32 = ok && want32;
    }
}

// ---------------------------------------------------------------------------
// sort: Morton order over the filter columns [f0, f0 + nf), stable radix
// ---------------------------------------------------------------------------
struct FilterCols {
    int f0, nf, bits;  // columns and Morton bits per column
};

__global__ void __launch_bounds__(kSortThreads) sort_kernel(
    const double *__restrict__ pts64, int dim, const ChunkInfo *__restrict__ info,
    const ColStats *__restrict__ stats, FilterCols fc, uint32_t *__restrict__ ka,
    uint32_t *__restrict__ kb, int32_t *__restrict__ va, int32_t *__restrict__ vb,
    int32_t *__restrict__ perm) {
    __shared__ SortSmem sm;
    __shared__ double qlo[kMaxDim], qscale[kMaxDim];
    const ChunkInfo ci = info[blockIdx.x];
    if (!ci.ok32) return;
    const ColStats *cs = stats + blockIdx.x;
    const uint32_t qmax = (1u << fc.bits) - 1u;
    if (threadIdx.x < fc.nf) {
        const int col = fc.f0 + threadIdx.x;
        const double span = cs->hi[col] - cs->lo[col];
        qlo[threadIdx.x] = cs->lo[col];
        qscale[threadIdx.x] = span > 0.0 ? (double)qmax / span : 0.0;
    }
    __syncthreads();
    const double *p = pts64 + ci.row0 * dim;
    uint32_t *k0 = ka + ci.row0, *k1 = kb + ci.row0;
    int32_t *v0 = va + ci.row0, *v1 = vb + ci.row0;
    for (int i = threadIdx.x; i < ci.n; i += kSortThreads) {
        uint32_t key = 0;
        uint32_t q[kMaxDim];
        for (int f = 0; f < fc.nf; ++f) {
            const double t = (p[(int64_t)i * dim + fc.f0 + f] - qlo[f]) * qscale[f];
            q[f] = (uint32_t)fmin(fmax(t, 0.0), (double)qmax);
        }
        for (int b = fc.bits - 1; b >= 0; --b)
            for (int f = 0; f < fc.nf; ++f) key = (key << 1) | ((q[f] >> b) & 1u);
        k0[i] = key;
        v0[i] = i;
    }
    __syncthreads();
    const int par = cta_radix_sort<uint32_t, int32_t>(k0, k1, v0, v1, ci.n, fc.nf * fc.bits, sm);
    const int32_t *res = par ? v1 : v0;
    for (int i = threadIdx.x; i < ci.n; i += kSortThreads) perm[ci.row0 + i] = res[i];
}

// ---------------------------------------------------------------------------
// gather: sorted fp32 rows (centred) + bounding boxes per 32 and 128 rows
// box layout: [lo[0..dp) | hi[0..dp)] per tile
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kTJ) gather_kernel(const double *__restrict__ pts64, int dim,
                                                     const ChunkInfo *__restrict__ info, int n_chunks,
                                                     const ColStats *__restrict__ stats,
                                                     const int32_t *__restrict__ perm, int dp,
                                                     float *__restrict__ pts32,
                                                     float *__restrict__ box32,
                                                     float *__restrict__ box128) {
    __shared__ float slo[kTJ / 32][kMaxDim], shi[kTJ / 32][kMaxDim];
    for (int cidx = blockIdx.y; cidx < n_chunks; cidx += gridDim.y) {
    const ChunkInfo ci = info[cidx];
    const int stage = blockIdx.x;
    if (!ci.ok32 || stage * kTJ >= ci.npad) continue;
    const ColStats *cs = stats + cidx;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s = stage * kTJ + threadIdx.x;
    const bool valid = s < ci.n;
    const int64_t orig = valid ? ci.row0 + perm[ci.row0 + s] : 0;
    float *q = pts32 + (ci.prow0 + s) * dp;
    const int64_t sub = ci.prow0 / kSub + stage * kSubPerStage + warp;
    for (int col = 0; col < dp; ++col) {
        float v = 0.0f;
        if (col < dim)
            v = valid ? __double2float_rn(__dsub_rn(pts64[orig * dim + col], cs->mean[col])) : INFINITY;
        q[col] = v;
        float lo = (valid && col < dim) ? v : INFINITY;
        float hi = (valid && col < dim) ? v : -INFINITY;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
        }
        if (lane == 0) {
            box32[sub * 2 * dp + col] = lo;
            box32[sub * 2 * dp + dp + col] = hi;
            if (col < kMaxDim) {
                slo[warp][col] = lo;
                shi[warp][col] = hi;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < dp) {
        const int col = threadIdx.x;
        float lo = INFINITY, hi = -INFINITY;
        for (int w = 0; w < kTJ / 32; ++w) {
            lo = fminf(lo, slo[w][col]);
            hi = fmaxf(hi, shi[w][col]);
        }
        const int64_t t = ci.prow0 / kTJ + stage;
        box128[t * 2 * dp + col] = lo;
        box128[t * 2 * dp + dp + col] = hi;
    }
    __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// register-level helpers for the fp32 sweeps
// ---------------------------------------------------------------------------
template <int D>
struct Ref {
    static constexpr int NP = (D + 1) / 2;
    float2 nr[NP];  // negated coordinates, packed for FADD2
};

template <int D>
__device__ __forceinline__ void load_ref(Ref<D> &ref, const float *__restrict__ row, bool valid) {
#pragma unroll
    for (int p = 0; p < Ref<D>::NP; ++p) {
        float a = valid ? row[2 * p] : 0.0f;
        float b = (valid && 2 * p + 1 < D) ? row[2 * p + 1] : 0.0f;
        ref.nr[p] = make_float2(-a, -b);
    }
}

template <int D>
struct Cand {
    static constexpr int DP = (D + 3) & ~3;
    float4 v[DP / 4];
    __device__ __forceinline__ float2 pair(int p) const {
        const float4 &q = v[p >> 1];
        return (p & 1) ? make_float2(q.z, q.w) : make_float2(q.x, q.y);
    }
    __device__ __forceinline__ float at(int c) const {
        const float4 &q = v[c >> 2];
        switch (c & 3) {
            case 0: return q.x;
            case 1: return q.y;
            case 2: return q.z;
            default: return q.w;
        }
    }
};

// signed differences x_ref - x_cand (sign irrelevant: only |.| is used)
template <int D>
__device__ __forceinline__ void diffs(const Ref<D> &ref, const Cand<D> &c, float (&a)[D]) {
#pragma unroll
    for (int p = 0; p < D / 2; ++p) {
        float2 d = __fadd2_rn(ref.nr[p], c.pair(p));
        a[2 * p] = d.x;
        a[2 * p + 1] = d.y;
    }
    if (D & 1) a[D - 1] = ref.nr[D / 2].x + c.at(D - 1);
}

// max |a[c]| for c in [LO, HI), folded into acc (3-input FMNMX chain)
template <int LO, int HI, int D>
__device__ __forceinline__ float maxabs(const float (&a)[D], float acc) {
    int c = LO;
#pragma unroll
    for (; c + 1 < HI; c += 2) acc = fmaxf(fmaxf(acc, fabsf(a[c])), fabsf(a[c + 1]));
    if (c < HI) acc = fmaxf(acc, fabsf(a[c]));
    return acc;
}

template <int LO, int HI, int D>
__device__ __forceinline__ float maxabs0(const float (&a)[D]) {
    if constexpr (HI - LO <= 0) return 0.0f;
    else if constexpr (HI - LO == 1) return fabsf(a[LO]);
    else return maxabs<LO + 2, HI, D>(a, fmaxf(fabsf(a[LO]), fabsf(a[LO + 1])));
}

// Keep the S smallest values, ascending (new[s] = median(old[s-1], old[s], d));
// a no-op when d >= kd[S-1].
template <int S>
__device__ __forceinline__ void insert_sorted(float (&kd)[S], float d) {
#pragma unroll
    for (int s = S - 1; s >= 1; --s) kd[s] = fmaxf(kd[s - 1], fminf(kd[s], d));
    kd[0] = fminf(kd[0], d);
}

// Shared-memory candidate ring fed by 1-D TMA bulk copies.
template <int DP>
struct Ring {
    float buf[2][kTJ * DP];
    uint64_t full[2];
};

template <int DP>
__device__ __forceinline__ void ring_issue(Ring<DP> &ring, int stage, const float *src) {
    constexpr uint32_t bytes = kTJ * DP * sizeof(float);
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&ring.full[stage], bytes);
    bulk_g2s(ring.buf[stage], src, bytes, &ring.full[stage]);
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
    const double w = fmax(__dsub_ru((double)t32, (double)lo), __dsub_ru((double)hi, (double)t32));
    b.lo = lo;
    b.hi = hi;
    b.nlo = -lo;
    b.nt = -t32;
    b.w = __double2float_ru(w);
    return b;
}

// ---------------------------------------------------------------------------
// traversal: candidate stages visited home-first, then alternately below and
// above (spatially nearest first in the Morton order, so kNN bounds shrink
// early); warp 0 evaluates 32 positions at a time and picks the first stage
// some warp still needs (its box distance below that warp's bound)
// ---------------------------------------------------------------------------
struct Trav {
    int h0, nh, nst, npos;
    __device__ void init(int r0, int n, int npad) {
        h0 = r0 / kTJ;
        nh = (min(r0 + kRefTile, n) - r0 + kTJ - 1) / kTJ;
        nst = npad / kTJ;
        npos = nh + 2 * max(h0, nst - h0 - nh);
    }
    __device__ int stage_at(int pos) const {
        if (pos < nh) return h0 + pos;
        const int p = pos - nh, k = (p >> 1) + 1;
        const int s = (p & 1) ? h0 + nh - 1 + k : h0 - k;
        return (s >= 0 && s < nst) ? s : -1;
    }
};

// fp32 box distance over columns [c0, c1): a lower bound of every d32 between
// the two boxes (fl is monotone: fl(x_j - x_i) >= fl(lo_j - hi_i))
template <int DP>
__device__ __forceinline__ float box_dist(const float *a, const float *b, int c0, int c1) {
    float m = 0.0f;
#pragma unroll
    for (int c = 0; c < DP; ++c) {
        if (c < c0 || c >= c1) continue;
        m = fmaxf(m, fmaxf(b[c] - a[DP + c], a[c] - b[DP + c]));
    }
    return m;
}

__device__ __forceinline__ float warp_max_nonneg(float v) {
    return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(fmaxf(v, 0.0f))));
}

// Warp 0: next stage to load (or -1).  strict: process iff dist < bound (kNN);
// otherwise iff dist <= bound (counts: the band is closed at hi).
template <int DP>
__device__ __forceinline__ int next_stage(const Trav &tv, int &spos, const float *box128,
                                          int64_t stage0, const float (*wbox)[2 * DP],
                                          const float *wbound, int c0, int c1, bool strict,
                                          int prune) {
    const int lane = threadIdx.x & 31;
    while (spos < tv.npos) {
        const int pos = spos + lane;
        const int st = pos < tv.npos ? tv.stage_at(pos) : -1;
        bool take = false;
        if (st >= 0) {
            if (!prune) {
                take = true;
            } else {
                const float *bb = box128 + (stage0 + st) * 2 * DP;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) {
                    const float d = box_dist<DP>(wbox[w], bb, c0, c1);
                    take |= strict ? (d < wbound[w]) : (d <= wbound[w]);
                }
            }
        }
        const unsigned hit = __ballot_sync(0xffffffffu, take);
        if (hit) {
            const int first = __ffs(hit) - 1;
            spos += first + 1;
            return __shfl_sync(0xffffffffu, st, first);
        }
        spos += 32;
    }
    return -1;
}

// ---------------------------------------------------------------------------
// pass 1: fp32 k-th neighbour distance (self included as the (k+1)-th slot)
// refs: warp w owns sorted rows r0 + w*128 + r*32 + lane, r < kRT
// ---------------------------------------------------------------------------
template <int D, int S>
__global__ void __launch_bounds__(kNT) knn_pass_kernel(
    const float *__restrict__ pts32, const float *__restrict__ box32,
    const float *__restrict__ box128, const ChunkInfo *__restrict__ info,
    const TileRef *__restrict__ tiles, int k, int prune, float *__restrict__ t32_out,
    int32_t *__restrict__ L_out, unsigned long long *__restrict__ work) {
    constexpr int DP = (D + 3) & ~3;
    __shared__ __align__(128) Ring<DP> ring;
    __shared__ float wbox[kWarps][2 * DP];
    __shared__ float wbound[kWarps];
    __shared__ int sid[2];
    const TileRef tr = tiles[blockIdx.x];
    const ChunkInfo ci = info[tr.chunk];
    if (!ci.ok32) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float *cp = pts32 + ci.prow0 * DP;
    const int64_t sub0 = ci.prow0 / kSub, stage0 = ci.prow0 / kTJ;
    Trav tv;
    tv.init(tr.r0, ci.n, ci.npad);
    const int wrow = tr.r0 + warp * kTJ;  // first sorted row of this warp
    const bool wvalid = wrow < ci.n;
    for (int e = lane; e < 2 * DP; e += 32)
        wbox[warp][e] = wvalid ? box128[(stage0 + wrow / kTJ) * 2 * DP + e]
                               : (e < DP ? INFINITY : -INFINITY);
    if (lane == 0) wbound[warp] = wvalid ? INFINITY : 0.0f;
    Ref<D> ref[kRT];
    float kd[kRT][S];
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
        const int idx = wrow + r * 32 + lane;
        const bool valid = idx < ci.n;
        load_ref<D>(ref[r], cp + (int64_t)idx * DP, valid);
#pragma unroll
        for (int s = 0; s < S; ++s)
            kd[r][s] = (!valid || s < S - (k + 1)) ? -INFINITY : INFINITY;
    }
    if (threadIdx.x == 0) {
        mbar_init(&ring.full[0], 1);
        mbar_init(&ring.full[1], 1);
        fence_barrier_init();
    }
    __syncthreads();
    int spos = 0;
    if (warp == 0) {
        for (int b = 0; b < 2; ++b) {
            const int st = next_stage<DP>(tv, spos, box128, stage0, wbox, wbound, 0, D, true, prune);
            if (lane == 0) {
                sid[b] = st;
                if (st >= 0) ring_issue(ring, b, cp + (int64_t)st * kTJ * DP);
            }
        }
    }
    __syncthreads();
    uint32_t uses = 0;  // bit b: parity of buffer b
    uint32_t nsub = 0;  // sub-tiles this warp evaluated
    for (int it = 0;; ++it) {
        const int b = it & 1;
        const int cur = sid[b];
        if (cur < 0) break;
        mbar_wait(&ring.full[b], (uses >> b) & 1u);
        uses ^= 1u << b;
        const float4 *tile = reinterpret_cast<const float4 *>(ring.buf[b]);
        for (int q = 0; q < kSubPerStage; ++q) {
            if (prune) {
                float wb = 0.0f;
#pragma unroll
                for (int r = 0; r < kRT; ++r) wb = fmaxf(wb, kd[r][S - 1]);
                wb = warp_max_nonneg(wb);
                const float bd = box_dist<DP>(wbox[warp], box32 + (sub0 + (int64_t)cur * kSubPerStage + q) * 2 * DP, 0, D);
                if (!(bd < wb)) continue;
            }
            ++nsub;
#pragma unroll 2
            for (int jj = 0; jj < kSub; ++jj) {
                const int j = q * kSub + jj;
                Cand<D> c;
#pragma unroll
                for (int v = 0; v < DP / 4; ++v) c.v[v] = tile[j * (DP / 4) + v];
                float d[kRT];
                bool any = false;
#pragma unroll
                for (int r = 0; r < kRT; ++r) {
                    float a[D];
                    diffs<D>(ref[r], c, a);
                    d[r] = maxabs0<0, D, D>(a);
                    any |= d[r] < kd[r][S - 1];
                }
                if (any) {
#pragma unroll
                    for (int r = 0; r < kRT; ++r) insert_sorted<S>(kd[r], d[r]);
                }
            }
        }
        {
            float wb = 0.0f;
#pragma unroll
            for (int r = 0; r < kRT; ++r) wb = fmaxf(wb, kd[r][S - 1]);
            wb = warp_max_nonneg(wb);
            if (lane == 0 && wvalid) wbound[warp] = wb;
        }
        __syncthreads();
        if (warp == 0) {
            const int st = next_stage<DP>(tv, spos, box128, stage0, wbox, wbound, 0, D, true, prune);
            if (lane == 0) {
                sid[b] = st;
                if (st >= 0) ring_issue(ring, b, cp + (int64_t)st * kTJ * DP);
            }
        }
        __syncthreads();
    }
    if (lane == 0 && wvalid) atomicAdd(work, (unsigned long long)nsub);
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
        const int idx = wrow + r * 32 + lane;
        if (idx >= ci.n) continue;
        const float t32 = kd[r][S - 1];
        const float lo = __double2float_rd(__dsub_rd((double)t32, 2.0 * ci.delta));
        int L = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) L += (kd[r][s] > -INFINITY) && (kd[r][s] < lo);
        if (lo > 0.0f) L -= 1;  // the self pair (distance 0) was counted
        t32_out[ci.row0 + idx] = t32;
        L_out[ci.row0 + idx] = L;
    }
}

// ---------------------------------------------------------------------------
// pass 2: certain counts in the three TE marginals + band events
//   columns: 0 = y_t, 1..DY = y-past, DY+1..D-1 = x-past (embedding.py:50-60)
//   marginal 0 = y-past (A), 1 = y + y-past, 2 = y-past + x-past
//   pruning uses the filter columns [f0, f0 + nf): a subset of every
//   requested marginal and of the joint, so their box distance bounds all
//   values that can count or fall in the band
// ---------------------------------------------------------------------------
template <int DY, int DX>
__global__ void __launch_bounds__(kNT) count_pass_kernel(
    const float *__restrict__ pts32, const float *__restrict__ box32,
    const float *__restrict__ box128, const ChunkInfo *__restrict__ info,
    const TileRef *__restrict__ tiles, const float *__restrict__ t32_in, int64_t ws_rows,
    FilterCols fc, int prune, int32_t *__restrict__ cnt_out, uint32_t *__restrict__ ev,
    int32_t *__restrict__ ev_n, uint32_t fmask, unsigned long long *__restrict__ work) {
    constexpr int D = 1 + DY + DX;
    constexpr int DP = (D + 3) & ~3;
    __shared__ __align__(128) Ring<DP> ring;
    __shared__ float wbox[kWarps][2 * DP];
    __shared__ float wbound[kWarps];
    __shared__ int sid[2];
    const TileRef tr = tiles[blockIdx.x];
    const ChunkInfo ci = info[tr.chunk];
    if (!ci.ok32) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float *cp = pts32 + ci.prow0 * DP;
    const int64_t sub0 = ci.prow0 / kSub, stage0 = ci.prow0 / kTJ;
    const int c0 = fc.f0, c1 = fc.f0 + fc.nf;
    Trav tv;
    tv.init(tr.r0, ci.n, ci.npad);
    const int wrow = tr.r0 + warp * kTJ;
    const bool wvalid = wrow < ci.n;
    for (int e = lane; e < 2 * DP; e += 32)
        wbox[warp][e] = wvalid ? box128[(stage0 + wrow / kTJ) * 2 * DP + e]
                               : (e < DP ? INFINITY : -INFINITY);
    Ref<D> ref[kRT];
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
    const float wb = warp_max_nonneg(hmax);
    if (lane == 0) wbound[warp] = wvalid ? wb : -1.0f;
    if (threadIdx.x == 0) {
        mbar_init(&ring.full[0], 1);
        mbar_init(&ring.full[1], 1);
        fence_barrier_init();
    }
    __syncthreads();
    int spos = 0;
    if (warp == 0) {
        for (int b = 0; b < 2; ++b) {
            const int st = next_stage<DP>(tv, spos, box128, stage0, wbox, wbound, c0, c1, false, prune);
            if (lane == 0) {
                sid[b] = st;
                if (st >= 0) ring_issue(ring, b, cp + (int64_t)st * kTJ * DP);
            }
        }
    }
    __syncthreads();
    uint32_t uses = 0;
    uint32_t nsub = 0;
    for (int it = 0;; ++it) {
        const int b = it & 1;
        const int cur = sid[b];
        if (cur < 0) break;
        mbar_wait(&ring.full[b], (uses >> b) & 1u);
        uses ^= 1u << b;
        const float4 *tile = reinterpret_cast<const float4 *>(ring.buf[b]);
        for (int q = 0; q < kSubPerStage; ++q) {
            if (prune) {
                const float bd = box_dist<DP>(wbox[warp], box32 + (sub0 + (int64_t)cur * kSubPerStage + q) * 2 * DP, c0, c1);
                if (!(bd <= wb) || !wvalid) continue;
            }
            ++nsub;
#pragma unroll 1
            for (int jj = 0; jj < kSub; ++jj) {
                const int j = q * kSub + jj;
                Cand<D> c;
#pragma unroll
                for (int v = 0; v < DP / 4; ++v) c.v[v] = tile[j * (DP / 4) + v];
                float vA[kRT], v2[kRT], v3[kRT], vj[kRT];
                bool any = false;
#pragma unroll
                for (int r = 0; r < kRT; ++r) {
                    float a[D];
                    diffs<D>(ref[r], c, a);
                    const float A = maxabs0<1, 1 + DY, D>(a);
                    const float m2 = fmaxf(A, fabsf(a[0]));
                    const float m3 = maxabs<1 + DY, D, D>(a, A);
                    const float jd = fmaxf(m2, m3);
                    // certain-inside counts: sign bit of (v - lo)
                    const float2 e = __fadd2_rn(make_float2(A, m2), make_float2(band[r].nlo, band[r].nlo));
                    const float e3 = m3 + band[r].nlo;
                    cA[r] += __float_as_uint(e.x) >> 31;
                    c2[r] += __float_as_uint(e.y) >> 31;
                    c3[r] += __float_as_uint(e3) >> 31;
                    // conservative band test: min |v - t| <= w
                    const float2 b1 = __fadd2_rn(make_float2(A, m2), make_float2(band[r].nt, band[r].nt));
                    const float2 b2 = __fadd2_rn(make_float2(m3, jd), make_float2(band[r].nt, band[r].nt));
                    const float bm = fminf(fminf(fabsf(b1.x), fabsf(b1.y)), fminf(fabsf(b2.x), fabsf(b2.y)));
                    any |= bm <= band[r].w;
                    vA[r] = A;
                    v2[r] = m2;
                    v3[r] = m3;
                    vj[r] = jd;
                }
                if (any) {
                    const int jg = cur * kTJ + j;
#pragma unroll
                    for (int r = 0; r < kRT; ++r) {
                        const float lo = band[r].lo, hi = band[r].hi;
                        uint32_t f = ((vA[r] >= lo && vA[r] <= hi) ? 1u : 0u) |
                                     ((v2[r] >= lo && v2[r] <= hi) ? 2u : 0u) |
                                     ((v3[r] >= lo && v3[r] <= hi) ? 4u : 0u) |
                                     ((vj[r] >= lo && vj[r] <= hi) ? 8u : 0u);
                        f &= fmask;
                        if (f) {
                            const int idx = wrow + r * 32 + lane;
                            if (nev[r] < kCap)
                                ev[(ci.row0 + idx) * kCap + nev[r]] = (uint32_t)jg | (f << 28);
                            ++nev[r];
                        }
                    }
                }
            }
        }
        __syncthreads();
        if (warp == 0) {
            const int st = next_stage<DP>(tv, spos, box128, stage0, wbox, wbound, c0, c1, false, prune);
            if (lane == 0) {
                sid[b] = st;
                if (st >= 0) ring_issue(ring, b, cp + (int64_t)st * kTJ * DP);
            }
        }
        __syncthreads();
    }
    if (lane == 0 && wvalid) atomicAdd(work, (unsigned long long)nsub);
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
// resolve: fp64 certification of band events (sorted positions -> rows via perm)
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

__global__ void __launch_bounds__(kNT) resolve_kernel(
    const double *__restrict__ pts64, int dim, const ChunkInfo *__restrict__ info,
    const TileRef *__restrict__ tiles, int k, TeLayout lay, const int32_t *__restrict__ perm,
    const int32_t *__restrict__ L_in, const int32_t *__restrict__ cnt_in,
    const uint32_t *__restrict__ ev, const int32_t *__restrict__ ev_n, int64_t ws_rows,
    int64_t total_rows, double *__restrict__ out_eps, int32_t *__restrict__ out_counts,
    int64_t *__restrict__ ovf_list, int32_t *__restrict__ ovf_n) {
    const TileRef tr = tiles[blockIdx.x];
    const ChunkInfo ci = info[tr.chunk];
    for (int r = 0; r < kRT; ++r) {
        const int s = tr.r0 + r * kNT + threadIdx.x;  // sorted position
        if (s >= ci.n) continue;
        const int64_t srow = ci.row0 + s;
        const int64_t row = ci.ok32 ? ci.row0 + perm[srow] : srow;
        const int ne = ci.ok32 ? ev_n[srow] : kCap + 1;
        const int need = ci.ok32 ? k - L_in[srow] : 0;
        bool fallback = !ci.ok32 || ne > kCap || need < 1;
        double eps = 0.0;
        int extra[3] = {0, 0, 0};
        if (!fallback) {
            double ref[kMaxDim];
            const double *rp = pts64 + row * dim;
            for (int c = 0; c < dim; ++c) ref[c] = rp[c];
            double dj[kCap];
            int nj = 0;
            for (int e = 0; e < ne; ++e) {
                const uint32_t w = ev[srow * kCap + e];
                const int j = (int)(w & 0x0FFFFFFFu);
                if (j == s || !(w >> 31)) continue;
                double A, m2, m3, jd;
                te_dist64(ref, pts64 + (ci.row0 + perm[ci.row0 + j]) * dim, dim, lay.dy, A, m2, m3, jd);
                int p = nj++;
                while (p > 0 && dj[p - 1] > jd) {
                    dj[p] = dj[p - 1];
                    --p;
                }
                dj[p] = jd;
            }
            if (need > nj) {
                fallback = true;
            } else {
                eps = dj[need - 1];
                for (int e = 0; e < ne; ++e) {
                    const uint32_t w = ev[srow * kCap + e];
                    const int j = (int)(w & 0x0FFFFFFFu);
                    const uint32_t f = (w >> 28) & 7u;
                    if (j == s || !f) continue;
                    double A, m2, m3, jd;
                    te_dist64(ref, pts64 + (ci.row0 + perm[ci.row0 + j]) * dim, dim, lay.dy, A, m2, m3, jd);
                    extra[0] += (f & 1u) && (A < eps);
                    extra[1] += (f & 2u) && (m2 < eps);
                    extra[2] += (f & 4u) && (m3 < eps);
                }
            }
        }
        if (fallback) {
            const int slot = atomicAdd(ovf_n, 1);
            ovf_list[slot] = row;
            continue;
        }
        out_eps[row] = eps;
        for (int o = 0; o < lay.nout; ++o) {
            const int sl = lay.slot[o];
            out_counts[o * total_rows + row] = cnt_in[sl * ws_rows + srow] + extra[sl];
        }
    }
}

// ---------------------------------------------------------------------------
// exact: one warp per point, fp64 scan, warp-shuffle top-k merge
// ---------------------------------------------------------------------------
struct Masks {
    uint32_t m[kMaxMarg];
    int n;
};

constexpr int kExactWarps = 8;  // warps per CTA

template <int S>
__global__ void __launch_bounds__(kExactWarps * 32) exact_kernel(
    const double *__restrict__ pts64, int dim, const ChunkInfo *__restrict__ info, int n_chunks,
    const int32_t *__restrict__ status, const int64_t *__restrict__ list,
    const int32_t *__restrict__ list_n, int64_t dense_n, int k, Masks masks, int64_t total_rows,
    const double *__restrict__ radii, double *__restrict__ out_eps, int32_t *__restrict__ out_counts) {
    __shared__ double sref[kExactWarps][kMaxDim];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t nwarps = (int64_t)gridDim.x * kExactWarps;
    const int64_t count = list ? (int64_t)*list_n : dense_n;
    for (int64_t it = (int64_t)blockIdx.x * kExactWarps + wib; it < count; it += nwarps) {
        const int64_t row = list ? list[it] : it;
        const int c = chunk_of_row(info, n_chunks, row);
        if (status[c] != ENTE_CHUNK_OK) continue;
        const ChunkInfo ci = info[c];
        if (row >= ci.row0 + ci.n) continue;  // a row between chunks
        const int idx = (int)(row - ci.row0);
        const double *rp = pts64 + row * dim;
        if (lane < dim) sref[wib][lane] = rp[lane];
        __syncwarp();
        double kd[S];
#pragma unroll
        for (int s = 0; s < S; ++s) kd[s] = (s < S - k) ? -INFINITY : INFINITY;
        for (int j = radii ? ci.n : lane; j < ci.n; j += 32) {
            if (j == idx) continue;
            const double *q = pts64 + (ci.row0 + j) * dim;
            double d = 0.0;
            for (int col = 0; col < dim; ++col) d = fmax(d, fabs(__dsub_rn(sref[wib][col], q[col])));
            if (d < kd[S - 1]) {
#pragma unroll
                for (int s = S - 1; s >= 1; --s) kd[s] = fmax(kd[s - 1], fmin(kd[s], d));
                kd[0] = fmin(kd[0], d);
            }
        }
        // k rounds of warp-wide minimum extraction
        double eps = radii ? radii[row] : 0.0;
        for (int q = 0; q < (radii ? 0 : k); ++q) {
            const double v = kd[S - k];
            double m = v;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, off));
            const unsigned win = __ffs(__ballot_sync(0xffffffffu, v == m)) - 1;
            if ((unsigned)lane == win) {
#pragma unroll
                for (int s = 0; s < S - 1; ++s)
                    if (s >= S - k) kd[s] = kd[s + 1];
                kd[S - 1] = INFINITY;
            }
            eps = m;
        }
        int cnt[kMaxMarg];
#pragma unroll
        for (int m = 0; m < kMaxMarg; ++m) cnt[m] = 0;
        for (int j = lane; j < ci.n; j += 32) {
            if (j == idx) continue;
            const double *q = pts64 + (ci.row0 + j) * dim;
            double dm[kMaxMarg];
#pragma unroll
            for (int m = 0; m < kMaxMarg; ++m) dm[m] = 0.0;
            for (int col = 0; col < dim; ++col) {
                const double v = fabs(__dsub_rn(sref[wib][col], q[col]));
#pragma unroll
                for (int m = 0; m < kMaxMarg; ++m)
                    if (m < masks.n && ((masks.m[m] >> col) & 1u)) dm[m] = fmax(dm[m], v);
            }
#pragma unroll
            for (int m = 0; m < kMaxMarg; ++m) cnt[m] += (m < masks.n) && (dm[m] < eps);
        }
#pragma unroll
        for (int m = 0; m < kMaxMarg; ++m) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) cnt[m] += __shfl_xor_sync(0xffffffffu, cnt[m], off);
        }
        if (lane == 0) {
            if (out_eps) out_eps[row] = eps;
            for (int m = 0; m < masks.n; ++m) out_counts[m * total_rows + row] = cnt[m];
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// host side: kernel tables and dispatch
// ---------------------------------------------------------------------------
using KnnFn = void (*)(const float *, const float *, const float *, const ChunkInfo *,
                       const TileRef *, int, int, float *, int32_t *, unsigned long long *);
using CountFn = void (*)(const float *, const float *, const float *, const ChunkInfo *,
                         const TileRef *, const float *, int64_t, FilterCols, int, int32_t *,
                         uint32_t *, int32_t *, uint32_t, unsigned long long *);

template <int D>
static KnnFn knn_for_slots(int slots) {
    if (slots <= 5) return knn_pass_kernel<D, 5>;
    if (slots <= 8) return knn_pass_kernel<D, 8>;
    if (slots <= 16) return knn_pass_kernel<D, 16>;
    return nullptr;
}

static KnnFn knn_table(int dim, int slots) {
    switch (dim) {
        case 3: return knn_for_slots<3>(slots);
        case 4: return knn_for_slots<4>(slots);
        case 5: return knn_for_slots<5>(slots);
        case 6: return knn_for_slots<6>(slots);
        case 7: return knn_for_slots<7>(slots);
        case 8: return knn_for_slots<8>(slots);
        case 9: return knn_for_slots<9>(slots);
        case 11: return knn_for_slots<11>(slots);
        case 13: return knn_for_slots<13>(slots);
        case 15: return knn_for_slots<15>(slots);
        case 17: return knn_for_slots<17>(slots);
        default: return nullptr;
    }
}

// (DY, DX) layouts with a compiled count kernel: TE embeddings d_y, d_x <= 3,
// the symmetric C3 sweep (1+2d) and the bench layout (marginal = first m cols).
#define ENTE_TE_LAYOUTS(X)                                                                  \
    X(1, 1) X(1, 2) X(2, 1) X(2, 2) X(1, 3) X(3, 1) X(2, 3) X(3, 2) X(3, 3) X(4, 4) X(5, 5) \
    X(6, 6) X(7, 7) X(8, 8) X(0, 2) X(1, 4) X(2, 4) X(3, 5) X(4, 6) X(5, 7) X(6, 8) X(7, 9)

static CountFn count_table(int dy, int dx) {
#define ENTE_CASE(a, b) \
    if (dy == a && dx == b) return count_pass_kernel<a, b>;
    ENTE_TE_LAYOUTS(ENTE_CASE)
#undef ENTE_CASE
    return nullptr;
}

struct Plan {
    bool fast = false;
    int dy = 0, dx = 0, slots = 0, dp = 0;
    TeLayout lay{};
    FilterCols fc{};
    int64_t total_rows = 0;
    int64_t total_prows = 0;
    int n_tiles = 0;
    int max_npad = 0;
};

// Map the requested marginals onto the TE layout [y | y-past(dy) | x-past(dx)].
static bool match_te_layout(int dim, const uint32_t *masks, int n_marg, int &dy_out,
                            TeLayout &lay) {
    const uint32_t all_but_0 = ((dim >= 32) ? 0xFFFFFFFFu : ((1u << dim) - 1u)) & ~1u;
    for (int dy = 0; dy < dim; ++dy) {
        const uint32_t yp = ((1u << (dy + 1)) - 1u) & ~1u;  // cols 1..dy
        const uint32_t yyp = (1u << (dy + 1)) - 1u;         // cols 0..dy
        bool ok = true;
        for (int m = 0; m < n_marg && ok; ++m) {
            if (dy >= 1 && masks[m] == yp) lay.slot[m] = 0;
            else if (masks[m] == yyp) lay.slot[m] = 1;
            else if (masks[m] == all_but_0) lay.slot[m] = 2;
            else ok = false;
        }
        if (ok && count_table(dy, dim - 1 - dy) != nullptr) {
            dy_out = dy;
            lay.dy = dy;
            lay.nout = n_marg;
            return true;
        }
    }
    return false;
}

// Filter columns: the intersection of every requested marginal with the
// joint, as a contiguous range (the TE marginals are ranges sharing y-past).
static FilterCols filter_cols(int dim, int dy, const TeLayout &lay) {
    int lo = 0, hi = dim;
    for (int o = 0; o < lay.nout; ++o) {
        switch (lay.slot[o]) {
            case 0: lo = std::max(lo, 1); hi = std::min(hi, dy + 1); break;
            case 1: hi = std::min(hi, dy + 1); break;
            default: lo = std::max(lo, 1); break;
        }
    }
    FilterCols fc{};
    fc.f0 = lo;
    fc.nf = std::max(0, hi - lo);
    fc.bits = fc.nf > 0 ? std::min(10, 30 / fc.nf) : 0;
    if (fc.nf > 0 && fc.bits == 0) fc.bits = 1;  // nf > 30: one bit per column
    if (fc.nf * fc.bits > 32) fc.nf = 32 / fc.bits;  // Morton over a prefix
    return fc;
}

static int exact_slots(int k) {
    if (k <= 4) return 4;
    if (k <= 8) return 8;
    if (k <= 16) return 16;
    if (k <= 32) return 32;
    if (k <= 64) return 64;
    return 0;
}

static Plan make_plan(const ente_chunk *chunks, int n_chunks, int dim, const uint32_t *masks,
                      int n_marg, int k) {
    Plan p;
    for (int c = 0; c < n_chunks; ++c) {
        p.total_rows = std::max(p.total_rows, chunks[c].row0 + chunks[c].n);
        const int npad = round_up(chunks[c].n, kTJ);
        p.total_prows += npad;
        p.max_npad = std::max(p.max_npad, npad);
        p.n_tiles += (chunks[c].n + kRefTile - 1) / kRefTile;
    }
    int dy = 0;
    TeLayout lay{};
    if (k + 1 <= 16 && knn_table(dim, k + 1) && match_te_layout(dim, masks, n_marg, dy, lay)) {
        p.fast = true;
        p.dy = dy;
        p.dx = dim - 1 - dy;
        p.slots = k + 1;
        p.dp = (dim + 3) & ~3;
        p.lay = lay;
        p.fc = filter_cols(dim, dy, lay);
    }
    return p;
}

struct SearchWs {
    ChunkInfo *info;
    ColStats *stats;
    TileRef *tiles;
    float *pts32;
    float *box32;
    float *box128;
    uint32_t *ka, *kb;
    int32_t *va, *vb;
    int32_t *perm;
    float *t32;
    int32_t *L;
    int32_t *cnt3;
    uint32_t *ev;
    int32_t *ev_n;
    int64_t *ovf;
    int32_t *ovf_n;
};

static SearchWs layout_ws(Arena &a, const Plan &p, int n_chunks) {
    SearchWs w{};
    w.info = a.take<ChunkInfo>(n_chunks);
    w.ovf_n = a.take<int32_t>(1);
    if (p.fast) {
        w.stats = a.take<ColStats>(n_chunks);
        w.tiles = a.take<TileRef>(p.n_tiles);
        w.pts32 = a.take<float>((size_t)p.total_prows * p.dp);
        w.box32 = a.take<float>((size_t)(p.total_prows / kSub) * 2 * p.dp);
        w.box128 = a.take<float>((size_t)(p.total_prows / kTJ) * 2 * p.dp);
        w.ka = a.take<uint32_t>(p.total_rows);
        w.kb = a.take<uint32_t>(p.total_rows);
        w.va = a.take<int32_t>(p.total_rows);
        w.vb = a.take<int32_t>(p.total_rows);
        w.perm = a.take<int32_t>(p.total_rows);
        w.t32 = a.take<float>(p.total_rows);
        w.L = a.take<int32_t>(p.total_rows);
        w.cnt3 = a.take<int32_t>((size_t)3 * p.total_rows);
        w.ev = a.take<uint32_t>((size_t)p.total_rows * kCap);
        w.ev_n = a.take<int32_t>(p.total_rows);
        w.ovf = a.take<int64_t>(p.total_rows);
    }
    return w;
}

static int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

template <int S>
static void launch_exact(cudaStream_t st, const double *pts64, int dim, const ChunkInfo *info,
                         int n_chunks, const int32_t *status, const int64_t *list,
                         const int32_t *list_n, int64_t dense_n, int k, Masks masks,
                         int64_t total_rows, double *out_eps, int32_t *out_counts,
                         const double *radii = nullptr) {
    int64_t blocks = list ? (int64_t)num_sms() * 8 : (dense_n + kExactWarps - 1) / kExactWarps;
    blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)num_sms() * 64));
    ENTE_LAUNCH("exact", st,
                exact_kernel<S><<<(unsigned)blocks, kExactWarps * 32, 0, st>>>(
                    pts64, dim, info, n_chunks, status, list, list_n, dense_n, k, masks,
                    total_rows, radii, out_eps, out_counts));
}

static void dispatch_exact(int k, cudaStream_t st, const double *pts64, int dim,
                           const ChunkInfo *info, int n_chunks, const int32_t *status,
                           const int64_t *list, const int32_t *list_n, int64_t dense_n, Masks masks,
                           int64_t total_rows, double *out_eps, int32_t *out_counts) {
    switch (exact_slots(k)) {
        case 4: launch_exact<4>(st, pts64, dim, info, n_chunks, status, list, list_n, dense_n, k, masks, total_rows, out_eps, out_counts); break;
        case 8: launch_exact<8>(st, pts64, dim, info, n_chunks, status, list, list_n, dense_n, k, masks, total_rows, out_eps, out_counts); break;
        case 16: launch_exact<16>(st, pts64, dim, info, n_chunks, status, list, list_n, dense_n, k, masks, total_rows, out_eps, out_counts); break;
        case 32: launch_exact<32>(st, pts64, dim, info, n_chunks, status, list, list_n, dense_n, k, masks, total_rows, out_eps, out_counts); break;
        default: launch_exact<64>(st, pts64, dim, info, n_chunks, status, list, list_n, dense_n, k, masks, total_rows, out_eps, out_counts); break;
    }
}

static int validate(const ente_chunk *chunks, int n_chunks, int dim, const uint32_t *masks,
                    int n_marg, int k) {
    if (n_chunks < 0 || (n_chunks > 0 && !chunks)) {
        set_error("ente_search: bad chunk list");
        return ENTE_ERR_ARG;
    }
    if (dim < 1 || dim > kMaxDim) {
        set_error("ente_search: dim=%d outside [1, %d]", dim, kMaxDim);
        return ENTE_ERR_ARG;
    }
    if (n_marg < 0 || n_marg > kMaxMarg || (n_marg > 0 && !masks)) {
        set_error("ente_search: n_marg=%d outside [0, %d]", n_marg, kMaxMarg);
        return ENTE_ERR_ARG;
    }
    const uint32_t full = dim >= 32 ? 0xFFFFFFFFu : ((1u << dim) - 1u);
    for (int m = 0; m < n_marg; ++m) {
        if (masks[m] == 0 || (masks[m] & ~full)) {
            set_error("ente_search: marginal %d mask 0x%x invalid for dim=%d", m, masks[m], dim);
            return ENTE_ERR_ARG;
        }
    }
    if (k < 1 || exact_slots(k) == 0) {
        set_error("ente_search: k=%d outside [1, 64]", k);
        return ENTE_ERR_ARG;
    }
    int64_t prev_end = 0;
    for (int c = 0; c < n_chunks; ++c) {
        if (chunks[c].n < 2 || chunks[c].row0 < prev_end || chunks[c].n > (1 << 28)) {
            set_error("ente_search: chunk %d (row0=%lld, n=%d) must have n in [2, 2^28] and "
                      "ascending, non-overlapping rows",
                      c, (long long)chunks[c].row0, chunks[c].n);
            return ENTE_ERR_ARG;
        }
        prev_end = chunks[c].row0 + chunks[c].n;
    }
    return ENTE_OK;
}

}  // namespace ente

using namespace ente;

extern "C" size_t ente_search_workspace_size(const ente_chunk *chunks, int n_chunks, int dim,
                                             int n_marg, int k) {
    (void)n_marg;
    uint32_t dummy[kMaxMarg] = {0};
    Plan p = make_plan(chunks, n_chunks, dim, dummy, 0, k);
    // size for the fast path whenever it could be taken
    if (k + 1 <= 16 && knn_table(dim, k + 1)) {
        p.fast = true;
        p.dp = (dim + 3) & ~3;
    }
    Arena a(nullptr, 0);
    layout_ws(a, p, n_chunks);
    return a.used + 256;
}

static int g_prune = -1;  // ENTE_PRUNE=0 disables box pruning (measurement only)

static int prune_enabled() {
    if (g_prune < 0) {
        const char *e = getenv("ENTE_PRUNE");
        g_prune = (e && e[0] == '0') ? 0 : 1;
    }
    return g_prune;
}

// Per-device running totals of evaluated sub-tiles ([0] knn, [1] count),
// accumulated by the sweeps themselves (one atomic per warp, no host sync).
static unsigned long long *g_dwork[64] = {nullptr};

static unsigned long long *device_work() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!g_dwork[dev]) {
        void *p = nullptr;
        if (cudaMalloc(&p, 2 * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
        cudaMemset(p, 0, 2 * sizeof(unsigned long long));
        g_dwork[dev] = static_cast<unsigned long long *>(p);
    }
    return g_dwork[dev];
}

extern "C" int ente_search(const double *pts64, int64_t total_rows, int dim,
                           const ente_chunk *chunks, int n_chunks, const uint32_t *marg_masks,
                           int n_marg, int k, double *out_eps, int32_t *out_counts,
                           int32_t *status, void *workspace, size_t ws_bytes, void *stream) {
    int rc = validate(chunks, n_chunks, dim, marg_masks, n_marg, k);
    if (rc != ENTE_OK) return rc;
    if (n_chunks == 0) return ENTE_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Plan p = make_plan(chunks, n_chunks, dim, marg_masks, n_marg, k);
    if (p.total_rows > total_rows) {
        set_error("ente_search: chunks reference row %lld beyond total_rows=%lld",
                  (long long)p.total_rows, (long long)total_rows);
        return ENTE_ERR_ARG;
    }
    const int64_t ws_rows = p.total_rows;  // stride of the workspace per-row arrays
    Arena a(workspace, ws_bytes);
    SearchWs w = layout_ws(a, p, n_chunks);
    if (!a.ok() || !w.info) {
        set_error("ente_search: workspace of %zu bytes too small (need %zu)", ws_bytes, a.used);
        return ENTE_ERR_WORKSPACE;
    }
    // host-side chunk table, tile list and k checks
    std::vector<ChunkInfo> hinfo(n_chunks);
    std::vector<int32_t> hstatus(n_chunks, ENTE_CHUNK_OK);
    std::vector<TileRef> htiles;
    int64_t prow = 0;
    for (int c = 0; c < n_chunks; ++c) {
        ChunkInfo &ci = hinfo[c];
        ci.row0 = chunks[c].row0;
        ci.n = chunks[c].n;
        ci.npad = round_up(ci.n, kTJ);
        ci.prow0 = prow;
        ci.delta = 0.0;
        ci.ok32 = 0;
        prow += ci.npad;
        if (k > ci.n - 1) hstatus[c] = ENTE_CHUNK_K_TOO_LARGE;
        if (p.fast && hstatus[c] == ENTE_CHUNK_OK)
            for (int r0 = 0; r0 < ci.n; r0 += kRefTile) htiles.push_back({c, r0});
    }
    ENTE_CUDA(cudaMemcpyAsync(w.info, hinfo.data(), sizeof(ChunkInfo) * n_chunks,
                              cudaMemcpyHostToDevice, st));
    ENTE_CUDA(cudaMemcpyAsync(status, hstatus.data(), sizeof(int32_t) * n_chunks,
                              cudaMemcpyHostToDevice, st));
    ENTE_CUDA(cudaMemsetAsync(w.ovf_n, 0, sizeof(int32_t), st));
    Masks masks{};
    masks.n = n_marg;
    for (int m = 0; m < n_marg; ++m) masks.m[m] = marg_masks[m];
    if (p.fast && !htiles.empty()) {
        const int prune = prune_enabled();
        unsigned long long *work = device_work();
        if (!work) {
            set_error("ente_search: cannot allocate the work counters");
            return ENTE_ERR_CUDA;
        }
        ENTE_LAUNCH("prep", st,
                    prep_kernel<<<n_chunks, 256, 0, st>>>(pts64, dim, w.info, w.stats, status, 1));
        ENTE_CUDA(cudaGetLastError());
        FilterCols sfc = p.fc;
        if (!prune) sfc.nf = 0;  // identity order
        ENTE_LAUNCH("sort", st,
                    sort_kernel<<<n_chunks, kSortThreads, 0, st>>>(pts64, dim, w.info, w.stats, sfc,
                                                                   w.ka, w.kb, w.va, w.vb, w.perm));
        ENTE_CUDA(cudaGetLastError());
        dim3 ggrid((unsigned)(p.max_npad / kTJ), (unsigned)std::min(n_chunks, 65535));
        ENTE_LAUNCH("gather", st,
                    gather_kernel<<<ggrid, kTJ, 0, st>>>(pts64, dim, w.info, n_chunks, w.stats,
                                                         w.perm, p.dp, w.pts32, w.box32,
                                                         w.box128));
        ENTE_CUDA(cudaGetLastError());
        ENTE_CUDA(cudaMemcpyAsync(w.tiles, htiles.data(), sizeof(TileRef) * htiles.size(),
                                  cudaMemcpyHostToDevice, st));
        const unsigned nt = (unsigned)htiles.size();
        ENTE_LAUNCH("knn_pass", st,
                    knn_table(dim, p.slots)<<<nt, kNT, 0, st>>>(w.pts32, w.box32, w.box128, w.info,
                                                               w.tiles, k, prune, w.t32, w.L,
                                                               work));
        ENTE_CUDA(cudaGetLastError());
        uint32_t fmask = 8u;
        for (int o = 0; o < p.lay.nout; ++o) fmask |= 1u << p.lay.slot[o];
        ENTE_LAUNCH("count_pass", st,
                    count_table(p.dy, p.dx)<<<nt, kNT, 0, st>>>(w.pts32, w.box32, w.box128, w.info,
                                                                w.tiles, w.t32, ws_rows, p.fc,
                                                                prune, w.cnt3, w.ev, w.ev_n, fmask,
                                                                work + 1));
        ENTE_CUDA(cudaGetLastError());
        ENTE_LAUNCH("resolve", st,
                    resolve_kernel<<<nt, kNT, 0, st>>>(pts64, dim, w.info, w.tiles, k, p.lay,
                                                       w.perm, w.L, w.cnt3, w.ev, w.ev_n, ws_rows,
                                                       total_rows, out_eps, out_counts, w.ovf,
                                                       w.ovf_n));
        ENTE_CUDA(cudaGetLastError());
        dispatch_exact(k, st, pts64, dim, w.info, n_chunks, status, w.ovf, w.ovf_n, 0, masks,
                       total_rows, out_eps, out_counts);
        ENTE_CUDA(cudaGetLastError());
    } else if (!p.fast) {
        ENTE_LAUNCH("prep", st,
                    prep_kernel<<<n_chunks, 256, 0, st>>>(pts64, dim, w.info, nullptr, status, 0));
        ENTE_CUDA(cudaGetLastError());
        dispatch_exact(k, st, pts64, dim, w.info, n_chunks, status, nullptr, nullptr, total_rows,
                       masks, total_rows, out_eps, out_counts);
        ENTE_CUDA(cudaGetLastError());
    }
    return ENTE_OK;
}

// Evaluated 32-candidate x 128-reference sub-tiles of the two sweeps on the
// current device since the last call (synchronises the device): the pruned
// work actually done.
extern "C" void ente_search_work(unsigned long long *knn_subtiles, unsigned long long *count_subtiles) {
    unsigned long long h[2] = {0, 0};
    unsigned long long *d = device_work();
    if (d && cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess)
        cudaMemset(d, 0, sizeof(h));
    *knn_subtiles = h[0];
    *count_subtiles = h[1];
}

extern "C" size_t ente_radius_counts_workspace_size(int n_chunks) {
    Arena a(nullptr, 0);
    a.take<ChunkInfo>(n_chunks);
    return a.used + 256;
}

// Strict radius counts for caller-given radii (reference radius_counts,
// engine.py:179-188): fp64 warp-per-point scan, one count array per marginal.
extern "C" int ente_radius_counts(const double *pts64, int64_t total_rows, int dim,
                                  const ente_chunk *chunks, int n_chunks, const uint32_t *marg_masks,
                                  int n_marg, const double *radii, int32_t *out_counts,
                                  int32_t *status, void *workspace, size_t ws_bytes, void *stream) {
    int rc = validate(chunks, n_chunks, dim, marg_masks, n_marg, 1);
    if (rc != ENTE_OK) return rc;
    if (n_chunks == 0 || n_marg == 0) return ENTE_OK;
    if (!radii || !out_counts) {
        set_error("ente_radius_counts: radii and out_counts are required");
        return ENTE_ERR_ARG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Arena a(workspace, ws_bytes);
    ChunkInfo *info = a.take<ChunkInfo>(n_chunks);
    if (!a.ok() || !info) {
        set_error("ente_radius_counts: workspace of %zu bytes too small (need %zu)", ws_bytes, a.used);
        return ENTE_ERR_WORKSPACE;
    }
    std::vector<ChunkInfo> hinfo(n_chunks);
    std::vector<int32_t> hstatus(n_chunks, ENTE_CHUNK_OK);
    for (int c = 0; c < n_chunks; ++c) {
        hinfo[c] = ChunkInfo{};
        hinfo[c].row0 = chunks[c].row0;
        hinfo[c].n = chunks[c].n;
        if (chunks[c].row0 + chunks[c].n > total_rows) {
            set_error("ente_radius_counts: chunk %d beyond total_rows", c);
            return ENTE_ERR_ARG;
        }
    }
    ENTE_CUDA(cudaMemcpyAsync(info, hinfo.data(), sizeof(ChunkInfo) * n_chunks, cudaMemcpyHostToDevice, st));
    ENTE_CUDA(cudaMemcpyAsync(status, hstatus.data(), sizeof(int32_t) * n_chunks, cudaMemcpyHostToDevice, st));
    Masks masks{};
    masks.n = n_marg;
    for (int m = 0; m < n_marg; ++m) masks.m[m] = marg_masks[m];
    launch_exact<4>(st, pts64, dim, info, n_chunks, status, nullptr, nullptr, total_rows, 1, masks,
                    total_rows, nullptr, out_counts, radii);
    ENTE_CUDA(cudaGetLastError());
    return ENTE_OK;
}
