// Shared-y marginal counts of a TE batch.
//
// In an analyze_pair batch every chunk pools the same target rows (r, t) of
// one window: the y columns (y_t, y-past) of chunk c's row i are those of
// original point p = phi_c(r) * w + t, phi_c the chunk's surrogate
// repetition permutation (identity for originals; u moves only x-past,
// embedding.py:109-115, inference.py:105-117).  The two y marginals of the
// KSG estimate, y-past (A) and y_t + y-past (m2), therefore count neighbours
// in ONE point set for the whole batch -- only the radius eps_c(i) and the
// tiny per-chunk jitter differ.  Instead of sweeping every chunk, each
// original point p is visited once:
//
//   queries  the C radii {eps_c(i_c(p))} of p, sorted (per-p radix sort);
//   walk     every q with D0(p, q) <= max radius + M, D0 the unjittered fp64
//            max-norm distance (Morton order over y-past, 32-row fp64 boxes);
//   count    for each q: queries with r > D0 + M count q for certain (one
//            +1 in a difference array), queries with r in [D0 - M, D0 + M]
//            are settled exactly on the jittered fp64 rows of that chunk,
//            |fl(a - b)| folded by max exactly as the reference
//            (engine.py:126-160), compared strictly with r.
//
// M bounds |D_c(p, q) - D0(p, q)|: the jitter moves every stored value by at
// most hw = amplitude * std (ksg.py:52-59) plus rounding, so M = 2 hw (1 +
// 1e-12) + 2^-48 (max|y| + hw) (host, shared_y_margin).  Every decision is
// exact; only the work changes: C2 visits ~2.5e3 neighbours per point once,
// instead of ~8e2 rows per point in every one of 2010 chunks.
#pragma once

#include "common.cuh"
#include "radix.cuh"

namespace ente {

#ifndef ENTE_SY_THREADS
#define ENTE_SY_THREADS 256
#endif
constexpr int kSyThreads = ENTE_SY_THREADS;
#ifndef ENTE_SY_QUEUE
#define ENTE_SY_QUEUE 1024
#endif
constexpr int kSyQueue = ENTE_SY_QUEUE;  // pending exact checks per CTA (shared memory)
constexpr int kSyMaxY = 9;  // y columns (1 + d_y), d_y <= 8

struct SyGeom {
    int reps, w, m, C;    // repetitions, window width, points (= rows per chunk), chunks
    int dd;               // y columns: 1 + d_y
    int nsub;             // 32-row subtiles of the sorted y0 copy
    double margin;
};

// query scatter: key[p * C + c] = high 32 bits of eps_c(i) (eps >= 0: bit
// order = value order; the key truncates the radius to r' <= r < r' (1 +
// 2^-20), which the count kernel's classification allows for), val = c, for
// row i of chunk c whose y-part is point p
// qs[p * C + c]: the point of chunk c's k-th neighbour of p (resolve's
// kstar, a chunk row mapped to its point) with its y-marginal verdicts in
// bits 30 (y-past distance < eps) and 31 (y_t + y-past), or all ones
__global__ void __launch_bounds__(256) sy_scatter_kernel(
    const ChunkInfo *__restrict__ info, const int32_t *__restrict__ chunk_perm,
    const int32_t *__restrict__ perms, SyGeom g, const double *__restrict__ eps,
    const uint32_t *__restrict__ kstar, uint32_t *__restrict__ key, int32_t *__restrict__ val,
    uint32_t *__restrict__ qs) {
    const int c = blockIdx.y;
    const int64_t row0 = info[c].row0;
    const int pi = chunk_perm[c];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.m; i += gridDim.x * blockDim.x) {
        const int r = i / g.w, t = i - r * g.w;
        const int pr = pi < 0 ? r : perms[(int64_t)pi * g.reps + r];
        const int64_t slot = (int64_t)(pr * g.w + t) * g.C + c;
        key[slot] = (uint32_t)((uint64_t)__double_as_longlong(eps[row0 + i]) >> 32);
        val[slot] = c;
        const uint32_t ks = kstar[row0 + i];
        uint32_t qv = 0xFFFFFFFFu;
        if (ks != 0xFFFFFFFFu) {
            const int qrow = (int)(ks & 0x0FFFFFFFu), qr = qrow / g.w, qt = qrow - qr * g.w;
            const int qpr = pi < 0 ? qr : perms[(int64_t)pi * g.reps + qr];
            qv = (uint32_t)(qpr * g.w + qt) | (ks & 0xC0000000u);
        }
        qs[slot] = qv;
    }
}

// per-point sort of the C query radii (one CTA per point)
template <int T>
__global__ void __launch_bounds__(T) sy_sort_kernel(uint32_t *__restrict__ ka, uint32_t *__restrict__ kb,
                                                    int32_t *__restrict__ va, int32_t *__restrict__ vb,
                                                    int C, int32_t *__restrict__ parity) {
    __shared__ SortSmemT<T> sm;
    const int64_t off = (int64_t)blockIdx.x * C;
    const int par = cta_radix_sort<T, uint32_t, int32_t>(ka + off, kb + off, va + off, vb + off, C, 32, sm);
    if (threadIdx.x == 0) parity[blockIdx.x] = par;
}

// Morton keys of the y0 points over the y-past columns (one CTA)
__global__ void __launch_bounds__(kSortThreads) sy_order_kernel(
    const double *__restrict__ y0, SyGeom g, uint32_t *__restrict__ ka, uint32_t *__restrict__ kb,
    int32_t *__restrict__ va, int32_t *__restrict__ vb, int32_t *__restrict__ yperm) {
    __shared__ SortSmem sm;
    __shared__ double lo[kSyMaxY], scale[kSyMaxY];
    const int nf = g.dd - 1 < 4 ? g.dd - 1 : 4;
    const int bits = nf > 0 ? (24 / nf < 16 ? 24 / nf : 16) : 0;
    const uint32_t qmax = (1u << bits) - 1u;
    __shared__ double red[2][kSortThreads / 32][4];
    {
        double a[4], b[4];
        for (int f = 0; f < 4; ++f) {
            a[f] = INFINITY;
            b[f] = -INFINITY;
        }
        for (int i = threadIdx.x; i < g.m; i += kSortThreads)
            for (int f = 0; f < nf; ++f) {
                const double v = y0[(int64_t)i * g.dd + 1 + f];
                a[f] = fmin(a[f], v);
                b[f] = fmax(b[f], v);
            }
        for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                a[f] = fmin(a[f], __shfl_xor_sync(0xffffffffu, a[f], o));
                b[f] = fmax(b[f], __shfl_xor_sync(0xffffffffu, b[f], o));
            }
        if ((threadIdx.x & 31) == 0)
            for (int f = 0; f < 4; ++f) {
                red[0][threadIdx.x >> 5][f] = a[f];
                red[1][threadIdx.x >> 5][f] = b[f];
            }
        __syncthreads();
        if (threadIdx.x < nf) {
            double lo_ = INFINITY, hi_ = -INFINITY;
            for (int w2 = 0; w2 < kSortThreads / 32; ++w2) {
                lo_ = fmin(lo_, red[0][w2][threadIdx.x]);
                hi_ = fmax(hi_, red[1][w2][threadIdx.x]);
            }
            lo[threadIdx.x] = lo_;
            scale[threadIdx.x] = hi_ > lo_ ? (double)qmax / (hi_ - lo_) : 0.0;
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < g.m; i += kSortThreads) {
        uint32_t q[4], key = 0;
        for (int f = 0; f < nf; ++f)
            q[f] = (uint32_t)fmin(fmax((y0[(int64_t)i * g.dd + 1 + f] - lo[f]) * scale[f], 0.0), (double)qmax);
        for (int b = bits - 1; b >= 0; --b)
            for (int f = 0; f < nf; ++f) key = (key << 1) | ((q[f] >> b) & 1u);
        ka[i] = key;
        va[i] = i;
    }
    __syncthreads();
    const int par = cta_radix_sort<kSortThreads, uint32_t, int32_t>(ka, kb, va, vb, g.m, nf * bits, sm);
    const int32_t *res = par ? vb : va;
    for (int i = threadIdx.x; i < g.m; i += kSortThreads) yperm[i] = res[i];
}

// sorted fp64 copy of y0 + per-32-row boxes over the y-past columns (lo | hi)
__global__ void __launch_bounds__(256) sy_gather_kernel(const double *__restrict__ y0, SyGeom g,
                                                        const int32_t *__restrict__ yperm,
                                                        double *__restrict__ ys, double *__restrict__ box) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool valid = s < g.m;
    const int p = valid ? yperm[s] : 0;
    for (int c = 0; c < g.dd; ++c) {
        const double v = valid ? y0[(int64_t)p * g.dd + c] : 0.0;
        if (valid) ys[(int64_t)s * g.dd + c] = v;
        if (c >= 1) {
            double a = valid ? v : INFINITY, b = valid ? v : -INFINITY;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
                b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
            }
            const int sub = s >> 5;
            if (lane == 0 && sub < g.nsub) {
                box[(int64_t)sub * 2 * (g.dd - 1) + (c - 1)] = a;
                box[(int64_t)sub * 2 * (g.dd - 1) + (g.dd - 1) + (c - 1)] = b;
            }
        }
    }
}

#ifndef ENTE_SY_BINS
#define ENTE_SY_BINS 2048
#endif
constexpr int kSyBins = ENTE_SY_BINS;  // lookup table over each point's radius range (uint16 entries)

__device__ __forceinline__ double sy_radius(uint32_t key) {  // truncated radius r' of a key
    return __longlong_as_double((long long)((uint64_t)key << 32));
}

// first k with r'[k] > x: the lookup table gives a start within a bin of the
// answer, a short scan finishes it (correct for any table entry: the array is
// sorted)
__device__ __forceinline__ int sy_upper(const uint32_t *key, const uint16_t *tab, int C, double r0,
                                        double inv_bw, double x) {
    if (!(x >= r0)) return 0;
    const double fb = (x - r0) * inv_bw;
    int k = tab[fb >= (double)(kSyBins - 1) ? kSyBins - 1 : (int)fb];
    while (k > 0 && sy_radius(key[k - 1]) > x) --k;
    while (k < C && sy_radius(key[k]) <= x) ++k;
    return k;
}

// One CTA per original point p: both y-marginal counts of p's row in every
// chunk.  out_counts[0 | 1][row] = y-past / y_t + y-past counts (the TE
// layout's slots 0 and 1, engine.py:191-200 with embedding.py:50-60).
//
// Radii are sorted by their high 32 bits (r' <= r < r'(1 + 2^-20)): query k
// counts q for certain when r'_k > D0 + M, never when r'_k < (D0 - M)(1 -
// 2^-19), and otherwise (rare: |r - D0| within M + 2^-20 r) q is settled on
// the jittered rows with the exact radius eps_c.
// PACK (m < 2^16 shared points): the two marginals' counters share one
// 32-bit word per query (y-past low half, y_t + y-past high half), and the
// exact additions likewise, so the CTA's shared memory drops by 16 B per
// query and four CTAs fit an SM instead of three.
template <bool PACK>
__global__ void __launch_bounds__(kSyThreads) sy_count_kernel(
    const double *__restrict__ y0, const double *__restrict__ ys, const int32_t *__restrict__ yperm,
    const double *__restrict__ box, SyGeom g, const uint32_t *__restrict__ ka,
    const uint32_t *__restrict__ kb, const int32_t *__restrict__ va, const int32_t *__restrict__ vb,
    const uint32_t *__restrict__ qs, const int32_t *__restrict__ parity, const ChunkInfo *__restrict__ info,
    const int32_t *__restrict__ chunk_perm, const int32_t *__restrict__ inv_perms,
    const double *__restrict__ pts64, int dim, const double *__restrict__ eps, int64_t total_rows,
    int32_t *__restrict__ out_counts) {
    extern __shared__ __align__(16) unsigned char sy_smem[];
    const int C = g.C;
    uint32_t *key = reinterpret_cast<uint32_t *>(sy_smem);
    int32_t *cid = reinterpret_cast<int32_t *>(key + C);
    int32_t *dA = cid + C;                    // C + 1 difference counters (y-past)
    int32_t *d2 = PACK ? dA : dA + C + 1;     // C + 1 (y_t + y-past)
    int32_t *xA = d2 + C + 1;                 // C exact additions
    int32_t *x2 = PACK ? xA : xA + C;
    uint32_t *qsm = reinterpret_cast<uint32_t *>(x2 + C);  // k-th neighbour records (C)
    // counter updates and reads (PACK: halves of one word)
    auto add_d = [&](int u, int which) {
        if constexpr (PACK) atomicAdd(reinterpret_cast<uint32_t *>(&dA[u]), which ? 0x10000u : 1u);
        else atomicAdd(which ? &d2[u] : &dA[u], 1);
    };
    auto add_x = [&](int k, int which) {
        if constexpr (PACK) atomicAdd(reinterpret_cast<uint32_t *>(&xA[k]), which ? 0x10000u : 1u);
        else atomicAdd(which ? &x2[k] : &xA[k], 1);
    };
    auto get = [&](const int32_t *lo, const int32_t *hi, int k, int which) -> int {
        if constexpr (PACK) {
            const uint32_t v = (uint32_t)lo[k];
            return which ? (int)(v >> 16) : (int)(v & 0xFFFFu);
        } else {
            return which ? hi[k] : lo[k];
        }
    };
    int32_t *list = reinterpret_cast<int32_t *>(qsm + C);  // queued subtiles (nsub)
    uint16_t *tab = reinterpret_cast<uint16_t *>(list + g.nsub);  // kSyBins
    __shared__ int nlist, wq_n[kSyThreads / 32];
    __shared__ uint32_t qk[kSyQueue];  // exact checks: k | which << 31
    __shared__ int32_t qq[kSyQueue];   // ... and the neighbour q
    __shared__ int wsum[kSyThreads / 32][2];
    const int p = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t off = (int64_t)p * C;
    const uint32_t *keys = parity[p] ? kb + off : ka + off;
    const int32_t *vals = parity[p] ? vb + off : va + off;
    for (int k = tid; k < C; k += kSyThreads) {
        key[k] = keys[k];
        cid[k] = vals[k];
        qsm[k] = qs[off + vals[k]];
        xA[k] = 0;
        x2[k] = 0;
    }
    for (int k = tid; k <= C; k += kSyThreads) {
        dA[k] = 0;
        d2[k] = 0;
    }
    if (tid == 0) nlist = 0;
    if (tid < kSyThreads / 32) wq_n[tid] = 0;
    double yp[kSyMaxY];
    for (int c = 0; c < g.dd; ++c) yp[c] = y0[(int64_t)p * g.dd + c];
    __syncthreads();
    const double r0 = sy_radius(key[0]);
    const double rmax = sy_radius(key[C - 1]) * (1.0 + 0x1p-19);  // >= every exact radius
    const double bw = (rmax - r0) / kSyBins;
    const double inv_bw = bw > 0.0 ? 1.0 / bw : 0.0;
    {  // tab[b] = first k with r'_k >= r0 + b bw: one search per thread, then a merge
        constexpr int PER = kSyBins / kSyThreads;
        const int b0 = tid * PER;
        double edge = r0 + b0 * bw;
        int lo = 0, hi = C;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sy_radius(key[mid]) >= edge) hi = mid;
            else lo = mid + 1;
        }
        for (int b = b0; b < b0 + PER; ++b) {
            edge = r0 + b * bw;
            while (lo < C && sy_radius(key[lo]) < edge) ++lo;
            tab[b] = (uint16_t)lo;
        }
    }
    const double R = rmax + g.margin;
    const int ny = g.dd - 1;
    // subtiles whose y-past box lies within R of p
    for (int s = tid; s < g.nsub; s += kSyThreads) {
        const double *b = box + (int64_t)s * 2 * ny;
        double d = 0.0;
        for (int c = 0; c < ny; ++c) d = fmax(d, fmax(b[c] - yp[1 + c], yp[1 + c] - b[ny + c]));
        if (d <= R) list[atomicAdd(&nlist, 1)] = s;
    }
    __syncthreads();
    const int nl = nlist;
    const int pr = p / g.w, pt = p - pr * g.w;
    auto row_in = [&](int c, int point_r, int point_t) -> int64_t {  // chunk row of a point
        const int pi = chunk_perm[c];
        const int rr = pi < 0 ? point_r : inv_perms[(int64_t)pi * g.reps + point_r];
        return info[c].row0 + (int64_t)rr * g.w + point_t;
    };
    // Exact checks are queued per warp and settled by the whole warp at once
    // (independent scattered reads of the jittered rows in flight together
    // instead of one lane's loop); no CTA barrier inside the walk.
    constexpr int QW = kSyQueue / (kSyThreads / 32);
    uint32_t *wqk = qk + warp * QW;
    int32_t *wqq = qq + warp * QW;
    auto check = [&](int k, int which, int q) {
        const int c = cid[k];
        const int64_t ip = row_in(c, pr, pt);
        const double *rp = pts64 + ip * dim;
        const double *rq = pts64 + row_in(c, q / g.w, q - (q / g.w) * g.w) * dim;
        double dd = 0.0;
        for (int col = which ? 0 : 1; col < g.dd; ++col) dd = fmax(dd, fabs(__dsub_rn(rp[col], rq[col])));
        if (dd < eps[ip]) add_x(k, which);
    };
    auto drain = [&]() {  // warp-uniform
        __syncwarp();
        const int n = wq_n[warp] < QW ? wq_n[warp] : QW;
        for (int e = lane; e < n; e += 32) check((int)(wqk[e] & 0x7FFFFFFFu), (int)(wqk[e] >> 31), wqq[e]);
        __syncwarp();
        if (lane == 0) wq_n[warp] = 0;
        __syncwarp();
    };
    for (int e = warp; e < nl; e += kSyThreads / 32) {
        const int sq = list[e] * 32 + lane;
        const int q = sq < g.m ? yperm[sq] : p;
        if (q != p) {
            const double *yq = ys + (int64_t)sq * g.dd;
            double a = 0.0;
            for (int c = 1; c < g.dd; ++c) a = fmax(a, fabs(__dsub_rn(yp[c], yq[c])));
            const double b2 = fmax(a, fabs(__dsub_rn(yp[0], yq[0])));
            for (int which = 0; which < 2; ++which) {
                const double d0 = which ? b2 : a;
                if (d0 - g.margin > rmax) continue;  // outside every query
                const int u = sy_upper(key, tab, C, r0, inv_bw, d0 + g.margin);
                if (u < C) add_d(u, which);
                // near the radius (r' >= (d0 - M)(1 - 2^-19)): exact, queued
                const double lo_x = (d0 - g.margin) * (1.0 - 0x1p-19);
                for (int k = u - 1; k >= 0 && sy_radius(key[k]) >= lo_x; --k) {
                    const uint32_t ks = qsm[k];
                    if ((ks & 0x3FFFFFFFu) == (uint32_t)q) {  // the k-th neighbour itself:
                        // its marginal distance is <= eps, equal unless resolve saw it below
                        if ((ks >> (30 + which)) & 1u) add_x(k, which);
                        continue;
                    }
                    const int slot = atomicAdd(&wq_n[warp], 1);
                    if (slot < QW) {
                        wqk[slot] = (uint32_t)k | ((uint32_t)which << 31);
                        wqq[slot] = q;
                    } else {
                        check(k, which, q);  // queue full: settle it in place
                    }
                }
            }
        }
        __syncwarp();
        if (wq_n[warp] >= QW / 2) drain();
    }
    drain();
    __syncthreads();
    // inclusive prefix sums of the difference arrays: every warp scans its
    // contiguous share of the C queries after one exchange of warp totals
    constexpr int NW = kSyThreads / 32;
    const int per = (C + NW - 1) / NW, k0 = warp * per, k1 = min(C, k0 + per);
    int sA = 0, s2 = 0;
    for (int k = k0 + lane; k < k1; k += 32) {
        sA += get(dA, d2, k, 0);
        s2 += get(dA, d2, k, 1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sA += __shfl_xor_sync(0xffffffffu, sA, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
        wsum[warp][0] = sA;
        wsum[warp][1] = s2;
    }
    __syncthreads();
    int runA = 0, run2 = 0;
    for (int w2 = 0; w2 < warp; ++w2) {
        runA += wsum[w2][0];
        run2 += wsum[w2][1];
    }
    for (int base = k0; base < k1; base += 32) {
        const int k = base + lane;
        int vA = k < k1 ? get(dA, d2, k, 0) : 0, v2 = k < k1 ? get(dA, d2, k, 1) : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int tA = __shfl_up_sync(0xffffffffu, vA, o), t2 = __shfl_up_sync(0xffffffffu, v2, o);
            if (lane >= o) {
                vA += tA;
                v2 += t2;
            }
        }
        if (k < k1) {
            const int c = cid[k];
            const int64_t row = row_in(c, pr, pt);
            out_counts[row] = runA + vA + get(xA, x2, k, 0);
            out_counts[total_rows + row] = run2 + v2 + get(xA, x2, k, 1);
        }
        runA += __shfl_sync(0xffffffffu, vA, 31);
        run2 += __shfl_sync(0xffffffffu, v2, 31);
    }
}

}  // namespace ente
