// Exact batched max-norm kNN distances + strict marginal radius counts.
//
// Replaces ente.engine.batch_search (/root/reference/pkg/src/ente/engine.py:203-216):
// the reference sweeps every reference point over a first-coordinate sorted
// order in fp64 (_kth_sweep 70-123, _count_sweep 126-160).  Here the same
// exact fp64 answer is produced by an fp32 filter with a proven error bound
// and fp64 certification of the few pairs the filter cannot decide:
//
//   prep      column mean / min / max, bound
//             delta = 4 * 2^-24 * max|x - m| * (1 + 2^-20) >= |d32 - d64|,
//             fp32 covariance -> principal axes (axes_kernel)
//   orders    count order: Morton over the y-past gate columns; kNN order:
//             Morton over the two principal axes when the chunk is
//             essentially 2-D, else the count order (CTA radix sorts); fp32
//             copies x32 = fl32(x - m) in both orders with per-32-row boxes
//   pruning   a sweep warp (64 sorted references) skips a 32-candidate
//             sub-tile when the fp32 box distance already exceeds its bound;
//             boxes are exact lower bounds of every d32 in them
//   pass 1    (sweeps.cuh) t32_i = k-th smallest fp32 distance (self
//             excluded) via a (k+1)-slot sorted list; L_i = #{d32 < lo_i}
//   pass 2    (sweeps.cuh) per pair: the three TE marginal distances and the
//             joint one; d32 < lo_i counts as certainly inside, values in the
//             band [lo_i, hi_i] = t32 -/+ 2 delta (directed rounding) are
//             recorded as events (<= kCap per point)
//   resolve   fp64 re-scoring of the events: eps_i = the (k - L_i)-th
//             smallest joint d64 among band events; marginal events inside
//             eps_i are added to the counts -> bit-identical to the reference
//   rescan    (sweeps.cuh) references whose events overflowed (ties): pruned
//             warp walk with fp64 on every undecided candidate
//   exact     warp-per-point fp64 scan (chunks whose range defeats fp32,
//             layouts without a compiled sweep)
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <mutex>
#include <set>
#include <vector>

#include "common.cuh"
#include "profile.cuh"
#include "radix.cuh"
#include "shared_y.cuh"
#include "sweeps.cuh"

namespace ente {

// ---------------------------------------------------------------------------
// prep: column statistics, error bound, finiteness
// ---------------------------------------------------------------------------
// fp32 row writer of the gathers: columns are collected in a float4 register
// and written as one 16-byte store per quad (rows are 16-B aligned, D padded
// to a multiple of 4) instead of one 4-byte store per column
#define STORE_COL(q4, col, v)                                   \
    do {                                                        \
        switch ((col) & 3) {                                    \
            case 0: quad.x = (v); break;                        \
            case 1: quad.y = (v); break;                        \
            case 2: quad.z = (v); break;                        \
            default: quad.w = (v); (q4)[(col) >> 2] = quad;     \
        }                                                       \
    } while (0)

// per-chunk column statistics (fp64): mean, min, max of the raw values
constexpr int kPcaCols = 8;  // principal axes over the first <= 8 columns

struct ColStats {
    double mean[kMaxDim];
    double lo[kMaxDim];
    double hi[kMaxDim];
    float axis[2][kPcaCols];  // the two leading principal axes (kNN order)
    int32_t use_pca;          // variance off the leading plane < kPcaResidual of lambda_1
    float cov[kPcaCols * (kPcaCols + 1) / 2];  // moments about the first row (prep)
    float x0[kPcaCols];                        // that row (fp32)
};

// The kNN pass sorts by the principal-axis Morton key only when the chunk is
// essentially two-dimensional (embedded low-dimensional dynamics, e.g. the
// Lorenz system: residual ~ 0.01); noise-driven AR data (residual >= 0.3)
// keeps the y-past Morton order of the count pass.
constexpr double kPcaResidual = 0.05;
constexpr int kPcaMinRows = 4096;

// Two leading eigenvectors of a symmetric P x P matrix by power iteration
// with deflation (P <= 8; ordering quality only, not exactness).
__device__ int principal_axes(double (&cov)[kPcaCols][kPcaCols], int P, float (&axis)[2][kPcaCols]) {
    double trace = 0.0, top = 0.0, lead = 0.0;
    for (int i = 0; i < P; ++i) trace += cov[i][i];
    for (int a = 0; a < 2; ++a) {
        double v[kPcaCols];
        for (int i = 0; i < kPcaCols; ++i) v[i] = (i < P) ? 1.0 + 0.1 * i + 0.37 * a * (i & 1) : 0.0;
        double lam = 0.0;
        for (int it = 0; it < 64; ++it) {
            double w[kPcaCols], nrm = 0.0;
            for (int i = 0; i < P; ++i) {
                w[i] = 0.0;
                for (int j = 0; j < P; ++j) w[i] += cov[i][j] * v[j];
                nrm += w[i] * w[i];
            }
            nrm = sqrt(nrm);
            if (!(nrm > 0.0)) break;
            double change = 0.0;
            for (int i = 0; i < P; ++i) {
                const double vi = w[i] / nrm;
                change = fmax(change, fabs(vi - v[i]));
                v[i] = vi;
            }
            lam = nrm;
            if (change < 1e-6) break;
        }
        for (int i = 0; i < kPcaCols; ++i) axis[a][i] = (i < P) ? (float)v[i] : 0.0f;
        for (int i = 0; i < P; ++i)
            for (int j = 0; j < P; ++j) cov[i][j] -= lam * v[i] * v[j];
        top += lam;
        if (a == 0) lead = lam;
    }
    return lead > 0.0 && (trace - top) < kPcaResidual * lead;
}

// One pass over the rows per group of 8 columns: fp64 sums / extrema, and
// (first group) the fp32 covariance about the chunk's first row for the
// principal axes.  The mean only centres the fp32 copy and enters the error
// bound through max|x - m|, so its summation order is free.
constexpr int kPrepThreadsBig = 256;   // CTA size for chunks of > kPrepSmallN rows
constexpr int kPrepThreadsSmall = 64;  // ... and for small chunks (C4: 500 rows)
constexpr int kPrepSmallN = 2048;
constexpr int kCovN = kPcaCols * (kPcaCols + 1) / 2;
constexpr int kCovStride = 4;  // covariance from rows 0, 4, 8, ...

template <int kPrepThreads>
__global__ void __launch_bounds__(kPrepThreads) prep_kernel(const double *__restrict__ pts64, int dim,
                                                            ChunkInfo *__restrict__ info,
                                                            ColStats *__restrict__ stats,
                                                            int32_t *__restrict__ status, int want32) {
    const int c = blockIdx.x;
    const ChunkInfo ci = info[c];
    if (status[c] != ENTE_CHUNK_OK) return;
    constexpr int kPrepWarps = kPrepThreads / 32;
    __shared__ double wred[3][kPrepWarps][8];
    __shared__ float wcov[kPrepWarps][kCovN];
    __shared__ ColStats local;
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    const double *p = pts64 + ci.row0 * dim;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int P = dim < kPcaCols ? dim : kPcaCols;
    for (int g0 = 0; g0 < dim; g0 += 8) {
        const int gn = dim - g0 < 8 ? dim - g0 : 8;
        double sum[8], lo[8], hi[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            sum[i] = 0.0;
            lo[i] = INFINITY;
            hi[i] = -INFINITY;
        }
        int nonfinite = 0;
        for (int r = threadIdx.x; r < ci.n; r += kPrepThreads) {
            double v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = i < gn ? p[(int64_t)r * dim + g0 + i] : 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                sum[i] += v[i];
                lo[i] = fmin(lo[i], v[i]);
                hi[i] = fmax(hi[i], v[i]);
                nonfinite |= !isfinite(v[i]);
            }
        }
        // second sweep for the covariance, kept apart so that neither loop
        // needs more than ~64 registers.  The axes only choose the kNN order
        // (never a result), so every kCovStride-th row suffices (the chunks
        // are not L2-resident); the sums are rescaled to n rows below.
        float cov[kCovN], x0[kPcaCols];
#pragma unroll
        for (int e = 0; e < kCovN; ++e) cov[e] = 0.0f;
#pragma unroll
        for (int i = 0; i < kPcaCols; ++i) x0[i] = (g0 == 0 && i < P) ? (float)p[i] : 0.0f;
        if (g0 == 0 && stats && ci.n >= kPcaMinRows) {
            for (int r = threadIdx.x * kCovStride; r < ci.n; r += kPrepThreads * kCovStride) {
                float x[kPcaCols];
#pragma unroll
                for (int i = 0; i < kPcaCols; ++i) x[i] = i < P ? (float)p[(int64_t)r * dim + i] - x0[i] : 0.0f;
                int e = 0;
#pragma unroll
                for (int i = 0; i < kPcaCols; ++i)
#pragma unroll
                    for (int j = 0; j <= i; ++j) cov[e++] += x[i] * x[j];
            }
        }
        if (nonfinite) bad = 1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            for (int off = 16; off > 0; off >>= 1) {
                sum[i] += __shfl_xor_sync(0xffffffffu, sum[i], off);
                lo[i] = fmin(lo[i], __shfl_xor_sync(0xffffffffu, lo[i], off));
                hi[i] = fmax(hi[i], __shfl_xor_sync(0xffffffffu, hi[i], off));
            }
            if (lane == 0) {
                wred[0][wid][i] = sum[i];
                wred[1][wid][i] = lo[i];
                wred[2][wid][i] = hi[i];
            }
        }
        if (g0 == 0 && stats) {
#pragma unroll
            for (int e = 0; e < kCovN; ++e) {
                float v = cov[e];
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane == 0) wcov[wid][e] = v;
            }
        }
        __syncthreads();
        if (threadIdx.x < gn) {
            const int i = threadIdx.x;
            double sm = 0.0, l = INFINITY, h = -INFINITY;
            for (int w = 0; w < kPrepWarps; ++w) {
                sm += wred[0][w][i];
                l = fmin(l, wred[1][w][i]);
                h = fmax(h, wred[2][w][i]);
            }
            local.mean[g0 + i] = sm / ci.n;
            local.lo[g0 + i] = l;
            local.hi[g0 + i] = h;
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
    const ColStats *cs = &local;
    if (stats) {
        for (int e = threadIdx.x; e < 3 * kMaxDim; e += blockDim.x)
            (&stats[c].mean[0])[e] = (&local.mean[0])[e];
        for (int e = threadIdx.x; e < kCovN; e += blockDim.x) {
            float v = 0.0f;
            for (int w = 0; w < kPrepWarps; ++w) v += wcov[w][e];
            stats[c].cov[e] = v * ((float)ci.n / (float)((ci.n + kCovStride - 1) / kCovStride));
        }
        if (threadIdx.x < kPcaCols) stats[c].x0[threadIdx.x] = threadIdx.x < P ? (float)p[threadIdx.x] : 0.0f;
    }
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

// principal axes of every chunk large enough to use them (one thread per
// chunk; the serial power iteration stays out of the prep CTAs)
__global__ void __launch_bounds__(128) axes_kernel(const ChunkInfo *__restrict__ info, int n_chunks,
                                                   int dim, ColStats *__restrict__ stats,
                                                   int allow_pca) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_chunks) return;
    const ChunkInfo ci = info[c];
    ColStats &cs = stats[c];
    cs.use_pca = 0;
    if (!allow_pca || !ci.ok32 || ci.n < kPcaMinRows) return;
    const int P = dim < kPcaCols ? dim : kPcaCols;
    // covariance about the mean from the moments about the first row
    double cov[kPcaCols][kPcaCols], d[kPcaCols];
    for (int i = 0; i < kPcaCols; ++i) d[i] = i < P ? cs.mean[i] - (double)cs.x0[i] : 0.0;
    int e = 0;
    for (int i = 0; i < kPcaCols; ++i)
        for (int j = 0; j <= i; ++j) {
            const double v = (double)cs.cov[e++] / ci.n - d[i] * d[j];
            cov[i][j] = cov[j][i] = (i < P && j < P) ? v : 0.0;
        }
    cs.use_pca = principal_axes(cov, P, cs.axis);
}

// ---------------------------------------------------------------------------
// sort: Morton order over the filter columns [f0, f0 + nf), stable radix
// ---------------------------------------------------------------------------
struct FilterCols {
    int f0, nf, bits;  // columns and Morton bits per column
    int skip_pca;      // chunks with principal axes need no filter order (kNN-order-only searches)
};

template <int T>
__global__ void __launch_bounds__(T) sort_kernel(
    const double *__restrict__ pts64, int dim, const ChunkInfo *__restrict__ info,
    const ColStats *__restrict__ stats, FilterCols fc, uint32_t *__restrict__ ka,
    uint32_t *__restrict__ kb, int32_t *__restrict__ va, int32_t *__restrict__ vb,
    int32_t *__restrict__ perm) {
    __shared__ SortSmemT<T> sm;
    __shared__ double qlo[kMaxDim], qscale[kMaxDim];
    const ChunkInfo ci = info[blockIdx.x];
    if (!ci.ok32) return;
    const ColStats *cs = stats + blockIdx.x;
    if (fc.skip_pca && cs->use_pca) return;
    const uint32_t qmax = (1u << fc.bits) - 1u;
    if (threadIdx.x < fc.nf) {
        const int col = fc.f0 + threadIdx.x;
        const double span = cs->hi[col] - cs->lo[col];
        qlo[threadIdx.x] = cs->lo[col];
        qscale[threadIdx.x] = span > 0.0 ? (double)qmax / span : 0.0;
    }
    __syncthreads();
    const double *p = pts64 + ci.row0 * dim;
    // small segments (the 128-thread instantiation) sort in shared memory
    constexpr bool SMS = T == kSortThreadsSmall;
    __shared__ uint32_t skey[SMS ? 2 : 1][SMS ? kSortSmallN : 1];
    __shared__ int32_t sval[SMS ? 2 : 1][SMS ? kSortSmallN : 1];
    uint32_t *k0 = SMS ? skey[0] : ka + ci.row0, *k1 = SMS ? skey[1] : kb + ci.row0;
    int32_t *v0 = SMS ? sval[0] : va + ci.row0, *v1 = SMS ? sval[1] : vb + ci.row0;
    for (int i = threadIdx.x; i < ci.n; i += T) {
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
    const int par = cta_radix_sort<T, uint32_t, int32_t>(k0, k1, v0, v1, ci.n, fc.nf * fc.bits, sm);
    const int32_t *res = par ? v1 : v0;
    for (int i = threadIdx.x; i < ci.n; i += T) perm[ci.row0 + i] = res[i];
}

// ---------------------------------------------------------------------------
// kNN order: Morton order of the projections on the chunk's two leading
// principal axes (12 bits each).  Embedded dynamics concentrate near a
// low-dimensional manifold; a 2-D order along it keeps 32-row sub-tiles
// compact in every column, which the kNN pass's all-column boxes exploit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t spread15(uint32_t v) {  // bits 0..14 -> even bits
    v &= 0x7FFFu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}

#ifndef ENTE_PCA_BITS
#define ENTE_PCA_BITS 8  // Morton bits per principal axis of the kNN order (12: same pruning, 3 radix passes)
#endif
template <int T>
__global__ void __launch_bounds__(T) sort_pca_kernel(
    const double *__restrict__ pts64, int dim, const ChunkInfo *__restrict__ info,
    const ColStats *__restrict__ stats, uint32_t *__restrict__ ka, uint32_t *__restrict__ kb,
    int32_t *__restrict__ va, int32_t *__restrict__ vb, const int32_t *__restrict__ cperm,
    int32_t *__restrict__ perm) {
    __shared__ SortSmemT<T> sm;
    __shared__ float red[4][(T / 32)];
    const ChunkInfo ci = info[blockIdx.x];
    if (!ci.ok32) return;
    const ColStats *cs = stats + blockIdx.x;
    if (!cs->use_pca) {  // keep the count pass's y-past Morton order
        for (int i = threadIdx.x; i < ci.n; i += T) perm[ci.row0 + i] = cperm[ci.row0 + i];
        return;
    }
    const int P = dim < kPcaCols ? dim : kPcaCols;
    const double *p = pts64 + ci.row0 * dim;
    constexpr bool SMS = T == kSortThreadsSmall;  // small segments sort in shared memory
    __shared__ uint32_t skey[SMS ? 2 : 1][SMS ? kSortSmallN : 1];
    __shared__ int32_t sval[SMS ? 2 : 1][SMS ? kSortSmallN : 1];
    uint32_t *k0 = SMS ? skey[0] : ka + ci.row0, *k1 = SMS ? skey[1] : kb + ci.row0;
    int32_t *v0 = SMS ? sval[0] : va + ci.row0, *v1 = SMS ? sval[1] : vb + ci.row0;
    float mn0 = INFINITY, mx0 = -INFINITY, mn1 = INFINITY, mx1 = -INFINITY;
    auto proj = [&](int i, float &z0, float &z1) {
        z0 = 0.0f;
        z1 = 0.0f;
        for (int c = 0; c < P; ++c) {
            const float x = (float)(p[(int64_t)i * dim + c] - cs->mean[c]);
            z0 += cs->axis[0][c] * x;
            z1 += cs->axis[1][c] * x;
        }
    };
    // one pass over the fp64 rows: projections parked in the key buffers
    for (int i = threadIdx.x; i < ci.n; i += T) {
        float z0, z1;
        proj(i, z0, z1);
        k0[i] = __float_as_uint(z0);
        k1[i] = __float_as_uint(z1);
        mn0 = fminf(mn0, z0);
        mx0 = fmaxf(mx0, z0);
        mn1 = fminf(mn1, z1);
        mx1 = fmaxf(mx1, z1);
    }
    for (int off = 16; off > 0; off >>= 1) {
        mn0 = fminf(mn0, __shfl_xor_sync(0xffffffffu, mn0, off));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
        mn1 = fminf(mn1, __shfl_xor_sync(0xffffffffu, mn1, off));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][wid] = mn0;
        red[1][wid] = mx0;
        red[2][wid] = mn1;
        red[3][wid] = mx1;
    }
    __syncthreads();
    for (int w = 0; w < (T / 32); ++w) {
        mn0 = fminf(mn0, red[0][w]);
        mx0 = fmaxf(mx0, red[1][w]);
        mn1 = fminf(mn1, red[2][w]);
        mx1 = fmaxf(mx1, red[3][w]);
    }
    const float q = (float)((1 << ENTE_PCA_BITS) - 1);  // bits per axis (radix passes = 2 bits / 8)
    const float s0 = mx0 > mn0 ? q / (mx0 - mn0) : 0.0f;
    const float s1 = mx1 > mn1 ? q / (mx1 - mn1) : 0.0f;
    for (int i = threadIdx.x; i < ci.n; i += T) {  // same thread, same i: no barrier needed
        const float z0 = __uint_as_float(k0[i]), z1 = __uint_as_float(k1[i]);
        const uint32_t a = (uint32_t)fminf(fmaxf((z0 - mn0) * s0, 0.0f), q);
        const uint32_t b = (uint32_t)fminf(fmaxf((z1 - mn1) * s1, 0.0f), q);
        k0[i] = (spread15(a) << 1) | spread15(b);
        v0[i] = i;
    }
    __syncthreads();
    const int par = cta_radix_sort<T, uint32_t, int32_t>(k0, k1, v0, v1, ci.n, 2 * ENTE_PCA_BITS, sm);
    const int32_t *res = par ? v1 : v0;
    for (int i = threadIdx.x; i < ci.n; i += T) perm[ci.row0 + i] = res[i];
}

// Block boxes: the union of each run of kBlockSubs sub-tile boxes of a chunk
// (one warp per block), stored after the sub-tile boxes at the chunk's
// ChunkInfo offset; the walkers test a whole block against their bound
// before loading its sub-tile boxes.
template <int Q>
__global__ void __launch_bounds__(256) block_box_kernel(const ChunkInfo *__restrict__ info, int n_chunks,
                                                        float4 *__restrict__ fbox, int knn) {
    const int lane = threadIdx.x & 31;
    const int blk = blockIdx.x * 8 + (threadIdx.x >> 5);
    for (int cidx = blockIdx.y; cidx < n_chunks; cidx += gridDim.y) {
        const ChunkInfo ci = info[cidx];
        const int nsub = ci.npad / kSub;
        if (!ci.ok32 || blk * kBlockSubs >= nsub) continue;
        const int sub = blk * kBlockSubs + lane;
        const float4 *fb = fbox + (ci.prow0 / kSub) * 2 * Q;
        float4 *out = fbox + (knn ? ci.sbk : ci.sbg) + (int64_t)blk * 2 * Q;
#pragma unroll
        for (int h = 0; h < 2 * Q; ++h) {  // h < Q: lo quads, else hi quads
            const bool lo = h < Q;
            float4 v = lane < kBlockSubs && sub < nsub
                           ? __ldg(fb + (int64_t)sub * 2 * Q + h)
                           : (lo ? make_float4(INFINITY, INFINITY, INFINITY, INFINITY)
                                 : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY));
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const float x = __shfl_xor_sync(0xffffffffu, v.x, off), y = __shfl_xor_sync(0xffffffffu, v.y, off);
                const float z = __shfl_xor_sync(0xffffffffu, v.z, off), t = __shfl_xor_sync(0xffffffffu, v.w, off);
                v = lo ? make_float4(fminf(v.x, x), fminf(v.y, y), fminf(v.z, z), fminf(v.w, t))
                       : make_float4(fmaxf(v.x, x), fmaxf(v.y, y), fmaxf(v.z, z), fmaxf(v.w, t));
            }
            if (lane == 0) out[h] = v;
        }
    }
}

// kNN copy: fp32 rows in the kNN order + boxes over columns 0 .. 4*kKnnQ-1
// (unused slots hold 0) + kmap (kNN position -> count-order position).
// Runs after gather_kernel, which fills inv (row -> count-order position).
__global__ void __launch_bounds__(kTJ) gather_knn_kernel(
    const double *__restrict__ pts64, int dim, const ChunkInfo *__restrict__ info, int n_chunks,
    const ColStats *__restrict__ stats, const int32_t *__restrict__ permk,
    const int32_t *__restrict__ inv, int dp, float *__restrict__ pts32, float *__restrict__ fbox,
    int32_t *__restrict__ kmap) {
    constexpr int NB = 4 * kKnnQ;
    for (int cidx = blockIdx.y; cidx < n_chunks; cidx += gridDim.y) {
        const ChunkInfo ci = info[cidx];
        const int stage = blockIdx.x;
        if (!ci.ok32 || stage * kTJ >= ci.npad) continue;
        const ColStats *cs = stats + cidx;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int s = stage * kTJ + threadIdx.x;
        const bool valid = s < ci.n;
        const int32_t o = valid ? permk[ci.row0 + s] : 0;
        const int64_t orig = ci.row0 + o;
        if (valid && kmap) kmap[ci.row0 + s] = inv[orig];
        float4 *q4 = reinterpret_cast<float4 *>(pts32 + (ci.prow0 + s) * dp);
        float4 quad = make_float4(0.f, 0.f, 0.f, 0.f);
        const int64_t sub = ci.prow0 / kSub + stage * (kTJ / kSub) + warp * (32 / kSub) + lane / kSub;
        for (int col = 0; col < dp; ++col) {
            float v = 0.0f;
            if (col < dim)
                v = valid ? __double2float_rn(__dsub_rn(pts64[orig * dim + col], cs->mean[col]))
                          : INFINITY;
            STORE_COL(q4, col, v);
            if (col < NB) {  // warp-uniform
                float lo = 0.0f, hi = 0.0f;
                if (col < dim) {
                    lo = valid ? v : INFINITY;
                    hi = valid ? v : -INFINITY;
#pragma unroll
                    for (int off = kSub / 2; off > 0; off >>= 1) {
                        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
                        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
                    }
                }
                if (lane % kSub == 0) {
                    fbox[sub * 2 * NB + col] = lo;
                    fbox[sub * 2 * NB + NB + col] = hi;
                }
            }
        }
        if (lane % kSub == 0)
            for (int col = dp; col < NB; ++col) fbox[sub * 2 * NB + col] = fbox[sub * 2 * NB + NB + col] = 0.0f;
    }
}


// ---------------------------------------------------------------------------
// gather: sorted fp32 rows (centred, D padded to DP) + per-32-row boxes over
// the gate columns (fbox layout per sub-tile: lo[kGate] | hi[kGate]; unused
// gate slots hold 0 so they add nothing to a box distance)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kTJ) gather_kernel(const double *__restrict__ pts64, int dim,
                                                     const ChunkInfo *__restrict__ info, int n_chunks,
                                                     const ColStats *__restrict__ stats,
                                                     const int32_t *__restrict__ perm, int dp,
                                                     FilterCols fc, float *__restrict__ pts32,
                                                     float *__restrict__ fbox,
                                                     int32_t *__restrict__ inv) {
    for (int cidx = blockIdx.y; cidx < n_chunks; cidx += gridDim.y) {
        const ChunkInfo ci = info[cidx];
        const int stage = blockIdx.x;
        if (!ci.ok32 || stage * kTJ >= ci.npad) continue;
        const ColStats *cs = stats + cidx;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int s = stage * kTJ + threadIdx.x;
        const bool valid = s < ci.n;
        const int64_t orig = valid ? ci.row0 + perm[ci.row0 + s] : 0;
        if (valid && inv) inv[orig] = s;
        float4 *q4 = reinterpret_cast<float4 *>(pts32 + (ci.prow0 + s) * dp);
        float4 quad = make_float4(0.f, 0.f, 0.f, 0.f);
        const int64_t sub = ci.prow0 / kSub + stage * (kTJ / kSub) + warp * (32 / kSub) + lane / kSub;
        for (int col = 0; col < dp; ++col) {
            float v = 0.0f;
            if (col < dim)
                v = valid ? __double2float_rn(__dsub_rn(pts64[orig * dim + col], cs->mean[col]))
                          : INFINITY;
            STORE_COL(q4, col, v);
            const int g = col - fc.f0;
            if (g >= 0 && g < kGate) {  // warp-uniform
                float lo = 0.0f, hi = 0.0f;
                if (g < fc.nf) {
                    lo = valid ? v : INFINITY;
                    hi = valid ? v : -INFINITY;
#pragma unroll
                    for (int off = kSub / 2; off > 0; off >>= 1) {
                        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
                        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
                    }
                }
                if (lane % kSub == 0) {
                    fbox[sub * 2 * kGate + g] = lo;
                    fbox[sub * 2 * kGate + kGate + g] = hi;
                }
            }
        }
        // gate slots beyond the columns (dim < f0 + kGate)
        if (lane % kSub == 0)
            for (int g = dim - fc.f0; g < kGate; ++g)
                if (g >= 0) fbox[sub * 2 * kGate + g] = fbox[sub * 2 * kGate + kGate + g] = 0.0f;
    }
}

// fp64 rows in the count order for chunks that have tie rescans (rs_flag):
// the rescan then reads candidate rows of a sub-tile as one coalesced block
// instead of one scattered row per lane
__global__ void __launch_bounds__(kTJ) gather64_kernel(const double *__restrict__ pts64, int dim,
                                                       const ChunkInfo *__restrict__ info, int n_chunks,
                                                       const int32_t *__restrict__ perm,
                                                       const int32_t *__restrict__ rs_flag,
                                                       double *__restrict__ pts64s) {
    for (int cidx = blockIdx.y; cidx < n_chunks; cidx += gridDim.y) {
        if (!rs_flag[cidx]) continue;
        const ChunkInfo ci = info[cidx];
        const int s = blockIdx.x * kTJ + threadIdx.x;
        if (s >= ci.n) continue;
        const double *src = pts64 + (ci.row0 + perm[ci.row0 + s]) * dim;
        double *dst = pts64s + (ci.prow0 + s) * dim;
        for (int c = 0; c < dim; ++c) dst[c] = src[c];
    }
}

__global__ void __launch_bounds__(kWarpRefs) resolve_kernel(
    const double *__restrict__ pts64, int dim, const ChunkInfo *__restrict__ info,
    const int32_t *__restrict__ tile0, int n_chunks, int k, TeLayout lay, const int32_t *__restrict__ perm,
    const int32_t *__restrict__ L_in, const int32_t *__restrict__ cnt_in,
    const uint32_t *__restrict__ ev, const int32_t *__restrict__ ev_n, int64_t ws_rows,
    int64_t total_rows, double *__restrict__ out_eps, int32_t *__restrict__ out_counts,
    int64_t *__restrict__ ovf_list, int32_t *__restrict__ ovf_n, int64_t *__restrict__ rs_list,
    int32_t *__restrict__ rs_n, int32_t *__restrict__ rs_flag, int allow_rescan,
    uint32_t *__restrict__ kstar) {
    const TileRef tr = tile_of(tile0, n_chunks, blockIdx.x);
    const ChunkInfo ci = info[tr.chunk];
    const int s = tr.r0 + threadIdx.x;  // sorted position
    if (s >= ci.n) return;
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
        int jj[kCap];
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
                jj[p] = jj[p - 1];
                --p;
            }
            dj[p] = jd;
            jj[p] = j;
        }
        if (need > nj) {
            fallback = true;
        } else {
            eps = dj[need - 1];
            if (kstar) {  // a neighbour at exactly eps, with its y-marginal verdicts (shared-y)
                const int qrow = perm[ci.row0 + jj[need - 1]];
                double A, m2, m3, jd;
                te_dist64(ref, pts64 + (ci.row0 + qrow) * dim, dim, lay.dy, A, m2, m3, jd);
                kstar[row] = (uint32_t)qrow | ((A < eps) ? 1u << 30 : 0u) | ((m2 < eps) ? 1u << 31 : 0u);
            }
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
        if (kstar) kstar[row] = 0xFFFFFFFFu;
        if (ci.ok32 && allow_rescan) {  // fp32 data usable: pruned warp rescan of the sorted row
            const int slot = atomicAdd(rs_n, 1);
            rs_list[slot] = srow;
            rs_flag[tr.chunk] = 1;
        } else {
            const int slot = atomicAdd(ovf_n, 1);
            ovf_list[slot] = row;
        }
        return;
    }
    out_eps[row] = eps;
    for (int o = 0; o < lay.nout; ++o) {
        const int sl = lay.slot[o];
        out_counts[o * total_rows + row] = cnt_in[sl * ws_rows + srow] + extra[sl];
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
// knn indices: the k nearest neighbours of every point in the canonical
// order ascending (fp64 max-norm distance, chunk-local index) -- the
// reference never returns them, so this order is the contract.
// One warp per point; with the fp32 kNN-order copy the walk skips sub-tiles
// whose all-column box lies beyond up(eps + delta) and compares d64 only for
// candidates with d32 <= that bound (every j with d64 <= eps qualifies);
// chunks without the fp32 copy are scanned in fp64.  Per-lane sorted
// (d, j) lists of S >= k slots, k rounds of lexicographic warp minima.
// ---------------------------------------------------------------------------
constexpr int kIdxWarps = 4;

__device__ __forceinline__ bool lex_less(double a, int ia, double b, int ib) {
    return a < b || (a == b && ia < ib);
}

template <int DP, int S>
__global__ void __launch_bounds__(kIdxWarps * 32) knn_index_kernel(
    const double *__restrict__ pts64, int dim, const ChunkInfo *__restrict__ info, int n_chunks,
    const int32_t *__restrict__ status, const float *__restrict__ pts32k,
    const float *__restrict__ fboxk, const int32_t *__restrict__ permk,
    const double *__restrict__ eps_in, int k, int64_t total_rows, int32_t *__restrict__ out_idx) {
    constexpr int NB = 4 * kKnnQ;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * kIdxWarps;
    for (int64_t it = (int64_t)blockIdx.x * kIdxWarps + (threadIdx.x >> 5); it < total_rows;
         it += nwarps) {
        const int c = chunk_of_row(info, n_chunks, it);
        const ChunkInfo ci = info[c];
        if (status[c] != ENTE_CHUNK_OK || it >= ci.row0 + ci.n) continue;
        const bool use32 = ci.ok32 && pts32k;
        // this warp's point: sorted position s (fp32 path) or local row
        const int s = (int)(it - ci.row0);
        const int local = use32 ? permk[it] : s;
        const int64_t row = ci.row0 + local;
        double r64[DP];
#pragma unroll
        for (int q = 0; q < DP; ++q) r64[q] = q < dim ? pts64[row * dim + q] : 0.0;
        const double eps = eps_in[row];
        double kd[S];
        int kj[S];
#pragma unroll
        for (int q = 0; q < S; ++q) {
            kd[q] = INFINITY;
            kj[q] = 0x7FFFFFFF;
        }
        auto consider = [&](int j_local) {
            const double *q64 = pts64 + (ci.row0 + j_local) * dim;
            double d = 0.0;
            for (int q = 0; q < dim; ++q) d = fmax(d, fabs(__dsub_rn(r64[q < DP ? q : 0], q64[q])));
            if (d <= eps && lex_less(d, j_local, kd[S - 1], kj[S - 1])) {
                int p = S - 1;
                while (p > 0 && lex_less(d, j_local, kd[p - 1], kj[p - 1])) {
                    kd[p] = kd[p - 1];
                    kj[p] = kj[p - 1];
                    --p;
                }
                kd[p] = d;
                kj[p] = j_local;
            }
        };
        if (use32) {
            const float *cp = pts32k + ci.prow0 * DP;
            const float4 *fb = reinterpret_cast<const float4 *>(fboxk) + (ci.prow0 / kSub) * 2 * kKnnQ;
            const int nsub = ci.npad / kSub;
            float ref[DP];
#pragma unroll
            for (int q = 0; q < DP; ++q) ref[q] = cp[(int64_t)s * DP + q];
            const float hi = __double2float_ru(__dadd_ru(eps, ci.delta));
            for (int base = 0; base < nsub; base += 32) {
                const int st_l = base + lane;
                bool need = false;
                if (st_l < nsub) {
                    const Box<kKnnQ> b = load_box<kKnnQ>(fb, st_l);
                    float d = 0.0f;
#pragma unroll
                    for (int g = 0; g < NB; ++g) {
                        const float4 l4 = b.lo[g >> 2], h4 = b.hi[g >> 2];
                        const float l = (g & 3) == 0 ? l4.x : (g & 3) == 1 ? l4.y : (g & 3) == 2 ? l4.z : l4.w;
                        const float h = (g & 3) == 0 ? h4.x : (g & 3) == 1 ? h4.y : (g & 3) == 2 ? h4.z : h4.w;
                        if (g < dim) d = fmaxf(d, fmaxf(l - ref[g < DP ? g : 0], ref[g < DP ? g : 0] - h));
                    }
                    need = d <= hi;
                }
                uint32_t m = __ballot_sync(0xffffffffu, need);
                while (m) {
                    const int st = base + __ffs(m) - 1;
                    m &= m - 1;
                    const int j = st * kSub + lane;
                    if (lane >= kSub || j >= ci.n || j == s) continue;
                    const float *q32 = cp + (int64_t)j * DP;
                    float d = 0.0f;
#pragma unroll
                    for (int q = 0; q < DP; ++q)
                        if (q < dim) d = fmaxf(d, fabsf(q32[q] - ref[q]));
                    if (d <= hi) consider(permk[ci.row0 + j]);
                }
            }
        } else {
            for (int j = lane; j < ci.n; j += 32)
                if (j != local) consider(j);
        }
        // k rounds of the lexicographic warp minimum
        for (int q = 0; q < k; ++q) {
            double bd = kd[0];
            int bj = kj[0];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double od = __shfl_xor_sync(0xffffffffu, bd, off);
                const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
                if (lex_less(od, oj, bd, bj)) {
                    bd = od;
                    bj = oj;
                }
            }
            if (kj[0] == bj && kd[0] == bd) {  // the owner pops its head
#pragma unroll
                for (int p = 0; p < S - 1; ++p) {
                    kd[p] = kd[p + 1];
                    kj[p] = kj[p + 1];
                }
                kd[S - 1] = INFINITY;
                kj[S - 1] = 0x7FFFFFFF;
            }
            if (lane == 0) out_idx[row * k + q] = bj;
        }
    }
}

// ---------------------------------------------------------------------------
// host side: kernel tables and dispatch
// ---------------------------------------------------------------------------
// Layout tables: the sweeps of every compiled (d_y, d_x) live in the
// sweeps_*.cu translation units (sweeps.cuh).
// Smallest chunk (padded rows of the batch's largest) for the compacted
// sweeps.  With grouped rounds they win even on 500-row chunks (C4: count
// pass 40.2 -> 31.2 ms), so the direct two-refs-per-lane sweeps are kept
// only for -DENTE_COMPACT_MIN_ROWS=<n> builds and k + 1 > 16.
#ifndef ENTE_COMPACT_MIN_ROWS
#define ENTE_COMPACT_MIN_ROWS 0
#endif
constexpr int kCompactMinRows = ENTE_COMPACT_MIN_ROWS;

#ifndef ENTE_KNN_COMPACT
#define ENTE_KNN_COMPACT 1
#endif

static KnnFn knn_table(int dy, int dx, int slots, int max_npad = 0) {
    SweepSet ss;
    if (!find_sweep_set(dy, dx, ss)) return nullptr;
    if (ENTE_KNN_COMPACT && max_npad >= kCompactMinRows && slots <= 16)
        return slots <= 5 ? ss.knn_compact[0] : slots <= 8 ? ss.knn_compact[1] : ss.knn_compact[2];
    return slots <= 5 ? ss.knn[0] : slots <= 8 ? ss.knn[1] : slots <= 16 ? ss.knn[2]
         : slots <= 32 ? ss.knn[3] : slots <= 64 ? ss.knn[4] : nullptr;
}

static RescanFn rescan_table(int dy, int dx, int k) {
    SweepSet ss;
    if (!find_sweep_set(dy, dx, ss)) return nullptr;
    return k <= 4 ? ss.rescan[0] : k <= 8 ? ss.rescan[1] : k <= 16 ? ss.rescan[2]
         : k <= 32 ? ss.rescan[3] : ss.rescan[4];
}

// The one-warp sweep CTAs are resident 32 per SM only with the whole
// 228 KB shared-memory carve-out (the count pass needs 6.1 KB + 1 KB
// reserved per CTA); ask for it once per kernel.
#ifndef ENTE_CARVEOUT
#define ENTE_CARVEOUT 1
#endif
static void prefer_shared(const void *fn) {
    static std::mutex mu;
    static std::set<const void *> done;
    if (!ENTE_CARVEOUT || !fn) return;
    std::lock_guard<std::mutex> lock(mu);
    if (done.insert(fn).second)
        cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)cudaSharedmemCarveoutMaxShared);
}

static CountFn count_table(int dy, int dx, int max_npad) {
    SweepSet ss;
    if (!find_sweep_set(dy, dx, ss)) return nullptr;
    return max_npad >= kCompactMinRows ? ss.compact : ss.direct;
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
    // with no marginals any layout of the right width serves (the gate is then
    // only a lower bound of the joint distance): prefer a 3-column gate block
    // (the Morton key and the gate boxes use up to kGate columns)
    int order[kMaxDim];
    int no = 0;
    if (n_marg == 0) {
        const int pref = dim - 1 < 3 ? dim - 1 : 3;
        for (int d = pref; d >= 1; --d) order[no++] = d;
        for (int d = pref + 1; d < dim; ++d) order[no++] = d;
    } else {
        for (int d = 0; d < dim; ++d) order[no++] = d;
    }
    for (int oi = 0; oi < no; ++oi) {
        const int dy = order[oi];
        const uint32_t yp = ((1u << (dy + 1)) - 1u) & ~1u;  // cols 1..dy
        const uint32_t yyp = (1u << (dy + 1)) - 1u;         // cols 0..dy
        bool ok = true;
        for (int m = 0; m < n_marg && ok; ++m) {
            if (dy >= 1 && masks[m] == yp) lay.slot[m] = 0;
            else if (masks[m] == yyp) lay.slot[m] = 1;
            else if (masks[m] == all_but_0) lay.slot[m] = 2;
            else ok = false;
        }
        if (ok && count_table(dy, dim - 1 - dy, 0) != nullptr) {
            dy_out = dy;
            lay.dy = dy;
            lay.nout = n_marg;
            return true;
        }
    }
    return false;
}

// Gate / filter columns: the y-past block [1, 1 + dy), a subset of every TE
// marginal and of the joint (embedding.py:50-60), capped at kGate columns
// for the Morton key and the sub-tile boxes.
static FilterCols filter_cols(int dy) {
    FilterCols fc{};
    fc.f0 = 1;
    fc.nf = std::min(dy, kGate);
    fc.bits = fc.nf > 0 ? std::min(16, 24 / fc.nf) : 0;  // 24-bit keys: three radix passes
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
        p.n_tiles += (chunks[c].n + kWarpRefs - 1) / kWarpRefs;
    }
    int dy = 0;
    TeLayout lay{};
    if (k + 1 <= 64 && match_te_layout(dim, masks, n_marg, dy, lay) &&
        knn_table(dy, dim - 1 - dy, k + 1)) {
        p.fast = true;
        p.dy = dy;
        p.dx = dim - 1 - dy;
        p.slots = k + 1;
        p.dp = (dim + 3) & ~3;
        p.lay = lay;
        p.fc = filter_cols(dy);
    }
    return p;
}

struct SearchWs {
    ChunkInfo *info;
    ColStats *stats;
    int32_t *tile0;
    float *pts32;
    float *fbox;
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
    int64_t *rs;
    int32_t *rs_n;
    int32_t *rs_flag;  // chunks with rescans
    double *pts64s;    // their fp64 rows in the count order
    // kNN order (principal-axis Morton)
    int32_t *permk, *kmap, *inv;
    float *pts32k, *fboxk;
};

// block boxes (unions of kBlockSubs consecutive sub-tile boxes, Walker) follow
// the sub-tile boxes in fbox / fboxk; chunk c's blocks start at block index
// prow0 / (kBlockSubs * kSub) + c, so chunks never share one
static int64_t block_boxes(const Plan &p, int n_chunks) {
    return p.total_prows / ((int64_t)kBlockSubs * kSub) + n_chunks + 1;
}

static SearchWs layout_ws(Arena &a, const Plan &p, int n_chunks) {
    SearchWs w{};
    w.info = a.take<ChunkInfo>(n_chunks);
    w.ovf_n = a.take<int32_t>(2);
    w.rs_n = w.ovf_n ? w.ovf_n + 1 : nullptr;
    if (p.fast) {
        w.stats = a.take<ColStats>(n_chunks);
        w.tile0 = a.take<int32_t>(2 * n_chunks + 1);
        w.pts32 = a.take<float>((size_t)p.total_prows * p.dp);
        w.fbox = a.take<float>((size_t)(p.total_prows / kSub + block_boxes(p, n_chunks)) * 2 * kGate);
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
        w.rs = a.take<int64_t>(p.total_rows);
        w.rs_flag = a.take<int32_t>(n_chunks);
        w.pts64s = a.take<double>((size_t)p.total_prows * p.dp);
        w.permk = a.take<int32_t>(p.total_rows);
        w.kmap = a.take<int32_t>(p.total_rows);
        w.inv = a.take<int32_t>(p.total_rows);
        w.pts32k = a.take<float>((size_t)p.total_prows * p.dp);
        w.fboxk = a.take<float>((size_t)(p.total_prows / kSub + block_boxes(p, n_chunks)) * 2 * 4 * kKnnQ);
    }
    return w;
}

static int launch_block_boxes(cudaStream_t st, const Plan &p, const SearchWs &w, int n_chunks, bool gate,
                              bool knn) {
    const int nblk = (int)((p.max_npad / kSub + kBlockSubs - 1) / kBlockSubs);
    dim3 grid((unsigned)((nblk + 7) / 8), (unsigned)std::min(n_chunks, 65535));
    if (gate) {
        ENTE_LAUNCH("block_box", st,
                    block_box_kernel<1><<<grid, 256, 0, st>>>(w.info, n_chunks,
                                                              reinterpret_cast<float4 *>(w.fbox), 0));
        ENTE_CUDA(cudaGetLastError());
    }
    if (knn) {
        ENTE_LAUNCH("block_box", st,
                    block_box_kernel<kKnnQ><<<grid, 256, 0, st>>>(w.info, n_chunks,
                                                                  reinterpret_cast<float4 *>(w.fboxk), 1));
        ENTE_CUDA(cudaGetLastError());
    }
    return ENTE_OK;
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

// prep -> principal axes -> both sort orders -> both fp32 copies with boxes
static int launch_orders(cudaStream_t st, const double *pts64, int dim, const Plan &p,
                         const SearchWs &w, int n_chunks, int32_t *status, int prune,
                         int allow_pca = 1, bool count_only = false, bool knn_only = false) {
        ENTE_LAUNCH("prep", st,
                    (p.max_npad <= kPrepSmallN ? prep_kernel<kPrepThreadsSmall> : prep_kernel<kPrepThreadsBig>)
                    <<<n_chunks, p.max_npad <= kPrepSmallN ? kPrepThreadsSmall : kPrepThreadsBig, 0, st>>>(
                        pts64, dim, w.info, w.stats, status, 1));
        ENTE_CUDA(cudaGetLastError());
        if (!count_only) {
            ENTE_LAUNCH("axes", st,
                        axes_kernel<<<(n_chunks + 127) / 128, 128, 0, st>>>(w.info, n_chunks, dim,
                                                                            w.stats, allow_pca));
            ENTE_CUDA(cudaGetLastError());
        }
        FilterCols sfc = p.fc;
        if (!prune) sfc.nf = 0;  // identity order
        sfc.skip_pca = knn_only ? 1 : 0;
        ENTE_LAUNCH("sort", st,
                    (p.max_npad <= kSortSmallN ? sort_kernel<kSortThreadsSmall> : sort_kernel<kSortThreads>)
                    <<<n_chunks, p.max_npad <= kSortSmallN ? kSortThreadsSmall : kSortThreads, 0, st>>>(pts64, dim, w.info, w.stats, sfc,
                                                                   w.ka, w.kb, w.va, w.vb, w.perm));
        ENTE_CUDA(cudaGetLastError());
        if (count_only) {  // the count order alone: no kNN-order copy
            dim3 ggrid((unsigned)(p.max_npad / kTJ), (unsigned)std::min(n_chunks, 65535));
            ENTE_LAUNCH("gather", st,
                        gather_kernel<<<ggrid, kTJ, 0, st>>>(pts64, dim, w.info, n_chunks, w.stats,
                                                             w.perm, p.dp, p.fc, w.pts32, w.fbox,
                                                             w.inv));
            ENTE_CUDA(cudaGetLastError());
            return ENTE_OK;
        }
        ENTE_LAUNCH("sort_pca", st,
                    (p.max_npad <= kSortSmallN ? sort_pca_kernel<kSortThreadsSmall> : sort_pca_kernel<kSortThreads>)
                    <<<n_chunks, p.max_npad <= kSortSmallN ? kSortThreadsSmall : kSortThreads, 0, st>>>(pts64, dim, w.info, w.stats,
                                                                       w.ka, w.kb, w.va, w.vb,
                                                                       w.perm, w.permk));
        ENTE_CUDA(cudaGetLastError());
        dim3 ggrid((unsigned)(p.max_npad / kTJ), (unsigned)std::min(n_chunks, 65535));
        if (!knn_only) {  // (shared-y batches sweep the kNN order only: no count-order copy)
            ENTE_LAUNCH("gather", st,
                        gather_kernel<<<ggrid, kTJ, 0, st>>>(pts64, dim, w.info, n_chunks, w.stats,
                                                             w.perm, p.dp, p.fc, w.pts32, w.fbox,
                                                             w.inv));
            ENTE_CUDA(cudaGetLastError());
        }
        ENTE_LAUNCH("gather_knn", st,
                    gather_knn_kernel<<<ggrid, kTJ, 0, st>>>(pts64, dim, w.info, n_chunks, w.stats,
                                                             w.permk, w.inv, p.dp, w.pts32k,
                                                             w.fboxk, knn_only ? nullptr : w.kmap));
        ENTE_CUDA(cudaGetLastError());
    // kNN-order block boxes: the kNN passes' KnnWalker and the shared-y m3
    // sweep's BlockWalker (the gate-column count passes walk sub-tiles)
    // (chunks of <= 32 sub-tiles never leave the KnnWalker's sub-tile phase)
    return launch_block_boxes(st, p, w, n_chunks, false, knn_only || p.max_npad / kSub > kBlockSubs);
}

// Uniform batches (every chunk n rows at row0 = base + c*n, no split: the TE
// pipeline's case) get their chunk table, status and tile map written on the
// device from a few scalars: no multi-MB host tables, and no pageable copy
// that would hold the host until the stream reaches it.
constexpr int kUniformMinChunks = 4096;  // smaller batches: host tables are cheap

struct UniformChunks {
    int64_t row0, stride, total_subs;
    int32_t n, npad, tiles, status;
};

__global__ void __launch_bounds__(256) uniform_chunks_kernel(UniformChunks u, int n_chunks,
                                                             ChunkInfo *__restrict__ info,
                                                             int32_t *__restrict__ status,
                                                             int32_t *__restrict__ tile0) {
    for (int c = blockIdx.x * 256 + threadIdx.x; c <= n_chunks; c += gridDim.x * 256) {
        if (c == n_chunks) {
            tile0[n_chunks] = n_chunks * u.tiles;
            continue;
        }
        ChunkInfo ci{};
        ci.row0 = u.row0 + (int64_t)c * u.stride;
        ci.n = u.n;
        ci.npad = u.npad;
        ci.prow0 = (int64_t)c * u.npad;
        ci.delta = 0.0;
        ci.ok32 = 0;
        ci.tile_lo = 0;
        const int64_t blk = ci.prow0 / ((int64_t)kBlockSubs * kSub) + c;
        ci.sbg = (int32_t)((u.total_subs + blk) * 2);
        ci.sbk = (int32_t)((u.total_subs + blk) * 2 * kKnnQ);
        info[c] = ci;
        status[c] = u.status;
        tile0[c] = c * u.tiles;
        tile0[n_chunks + 1 + c] = 0;
    }
}

// host chunk table + status (K_TOO_LARGE) + per-chunk first sweep tile;
// htile0 comes back empty when the tile map was written on the device
static int upload_chunks(cudaStream_t st, const ente_chunk *chunks, int n_chunks, int k,
                         const Plan &p, const SearchWs &w, int32_t *status,
                         std::vector<int32_t> &htile0, int32_t &ntiles, int split_index = 0,
                         int split_count = 1) {
    if (split_count == 1 && n_chunks >= kUniformMinChunks && w.tile0) {
        const int32_t n0 = chunks[0].n;
        const int64_t base = chunks[0].row0;
        bool uniform = true;
        for (int c = 1; c < n_chunks && uniform; ++c)
            uniform = chunks[c].n == n0 && chunks[c].row0 == base + (int64_t)c * n0;
        if (uniform) {
            UniformChunks u;
            u.row0 = base;
            u.stride = n0;
            u.n = n0;
            u.npad = (int32_t)round_up(n0, kTJ);
            u.total_subs = p.total_prows / kSub;
            u.status = k > n0 - 1 ? ENTE_CHUNK_K_TOO_LARGE : ENTE_CHUNK_OK;
            u.tiles = (p.fast && u.status == ENTE_CHUNK_OK) ? (n0 + kWarpRefs - 1) / kWarpRefs : 0;
            ntiles = n_chunks * u.tiles;
            htile0.clear();
            const unsigned blocks = (unsigned)std::min<int64_t>((n_chunks + 256) / 256, 1024);
            ENTE_LAUNCH("uniform_chunks", st,
                        uniform_chunks_kernel<<<blocks, 256, 0, st>>>(u, n_chunks, w.info, status, w.tile0));
            ENTE_CUDA(cudaGetLastError());
            ENTE_CUDA(cudaMemsetAsync(w.ovf_n, 0, 2 * sizeof(int32_t), st));
            if (w.rs_flag) ENTE_CUDA(cudaMemsetAsync(w.rs_flag, 0, sizeof(int32_t) * n_chunks, st));
            return ENTE_OK;
        }
    }
    std::vector<ChunkInfo> hinfo(n_chunks);
    std::vector<int32_t> hstatus(n_chunks, ENTE_CHUNK_OK);
    htile0.assign(2 * n_chunks + 1, 0);
    ntiles = 0;
    int64_t prow = 0;
    for (int c = 0; c < n_chunks; ++c) {
        ChunkInfo &ci = hinfo[c];
        ci.row0 = chunks[c].row0;
        ci.n = chunks[c].n;
        ci.npad = round_up(ci.n, kTJ);
        ci.prow0 = prow;
        ci.delta = 0.0;
        ci.ok32 = 0;
        ci.tile_lo = 0;
        {
            const int64_t blk = ci.prow0 / ((int64_t)kBlockSubs * kSub) + c;
            ci.sbg = (int32_t)((p.total_prows / kSub + blk) * 2);
            ci.sbk = (int32_t)((p.total_prows / kSub + blk) * 2 * kKnnQ);
        }
        prow += ci.npad;
        if (k > ci.n - 1) hstatus[c] = ENTE_CHUNK_K_TOO_LARGE;
        htile0[c] = ntiles;
        // this call's share of the chunk's sweep tiles (all of them unless split)
        const int64_t all = (ci.n + kWarpRefs - 1) / kWarpRefs;
        const int lo = (int)(all * split_index / split_count);
        const int hi = (int)(all * (split_index + 1) / split_count);
        ci.tile_lo = lo;
        htile0[n_chunks + 1 + c] = lo;
        if (p.fast && hstatus[c] == ENTE_CHUNK_OK) ntiles += hi - lo;
    }
    htile0[n_chunks] = ntiles;
    ENTE_CUDA(cudaMemcpyAsync(w.info, hinfo.data(), sizeof(ChunkInfo) * n_chunks,
                              cudaMemcpyHostToDevice, st));
    ENTE_CUDA(cudaMemcpyAsync(status, hstatus.data(), sizeof(int32_t) * n_chunks,
                              cudaMemcpyHostToDevice, st));
    ENTE_CUDA(cudaMemsetAsync(w.ovf_n, 0, 2 * sizeof(int32_t), st));
    if (w.rs_flag) ENTE_CUDA(cudaMemsetAsync(w.rs_flag, 0, sizeof(int32_t) * n_chunks, st));
    return ENTE_OK;
}

}  // namespace ente

using namespace ente;

static size_t radius_ws_size(const ente_chunk *chunks, int n_chunks, int max_mc);

extern "C" size_t ente_search_workspace_size(const ente_chunk *chunks, int n_chunks, int dim,
                                             int n_marg, int k) {
    (void)n_marg;
    uint32_t dummy[kMaxMarg] = {0};
    Plan p = make_plan(chunks, n_chunks, dim, dummy, 0, k);
    // size for the fast path whenever it could be taken
    if (k + 1 <= 64) {
        p.fast = true;
        p.dp = (dim + 3) & ~3;
    }
    Arena a(nullptr, 0);
    layout_ws(a, p, n_chunks);
    // marginals outside the TE layout run the generic radius path
    const size_t gen = n_marg > 0 ? radius_ws_size(chunks, n_chunks, std::min(dim, 17)) : 0;
    return std::max(a.used, gen) + 256;
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

// ---------------------------------------------------------------------------
// Generic marginal counts with given radii (reference radius_counts,
// engine.py:179-188, and _search_one's arbitrary marginal column lists,
// engine.py:191-200): the marginal's columns are copied into a dense fp64
// matrix laid out as a compiled TE layout [0 | gate (DY) | rest (DX)] whose
// slot-2 marginal (columns 1 .. D'-1) is exactly the marginal (zero columns
// pad it to a compiled width; they add nothing to a max-norm).  The count
// order, fp32 copy, boxes and count_pass sweep of the TE path then run
// unchanged with the band centred on fl32(r_i): |fl32(r) - r| <= u32 r, and
// for r <= 4 s that is <= delta, so v32 < lo => v64 < r and v32 > hi =>
// v64 > r still hold (for r > 4 s every pair is inside, which lo already
// says); band events are settled in fp64 by resolve_counts, overflowing
// references by the exact kernel.
// ---------------------------------------------------------------------------
struct MargCols {
    int n;
    int col[kMaxDim];
};

// dense [total_rows x dd] fp64: column 0 and columns > n hold 0
__global__ void __launch_bounds__(256) marg_dense_kernel(const double *__restrict__ pts64, int dim,
                                                         int64_t total_rows, MargCols mc, int dd,
                                                         double *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total_rows * dd;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / dd;
        const int c = (int)(i - row * dd);
        out[i] = (c >= 1 && c <= mc.n) ? pts64[row * dim + mc.col[c - 1]] : 0.0;
    }
}

// band centres in the count order: t32[sorted position] = fl32(radius of its row)
__global__ void __launch_bounds__(kWarpRefs) radii_t32_kernel(
    const ChunkInfo *__restrict__ info, const int32_t *__restrict__ tile0, int n_chunks,
    const int32_t *__restrict__ perm, const double *__restrict__ radii, float *__restrict__ t32) {
    const TileRef tr = tile_of(tile0, n_chunks, blockIdx.x);
    const ChunkInfo ci = info[tr.chunk];
    const int s = tr.r0 + threadIdx.x;
    if (s >= ci.n || !ci.ok32) return;
    const int64_t srow = ci.row0 + s;
    t32[srow] = __double2float_rn(radii[ci.row0 + perm[srow]]);
}

// certain count + fp64 settlement of the band events of the slot-2 marginal
__global__ void __launch_bounds__(kWarpRefs) resolve_counts_kernel(
    const double *__restrict__ dense, int dd, const ChunkInfo *__restrict__ info,
    const int32_t *__restrict__ tile0, int n_chunks, const int32_t *__restrict__ perm,
    const double *__restrict__ radii, const int32_t *__restrict__ cnt_in,
    const uint32_t *__restrict__ ev, const int32_t *__restrict__ ev_n, int64_t ws_rows,
    int32_t *__restrict__ out, int64_t *__restrict__ ovf_list, int32_t *__restrict__ ovf_n) {
    const TileRef tr = tile_of(tile0, n_chunks, blockIdx.x);
    const ChunkInfo ci = info[tr.chunk];
    const int s = tr.r0 + threadIdx.x;
    if (s >= ci.n) return;
    const int64_t srow = ci.row0 + s;
    const int64_t row = ci.ok32 ? ci.row0 + perm[srow] : srow;
    const int ne = ci.ok32 ? ev_n[srow] : kCap + 1;
    if (ne > kCap) {
        ovf_list[atomicAdd(ovf_n, 1)] = row;
        return;
    }
    const double r = radii[row];
    const double *rp = dense + row * dd;
    int cnt = cnt_in[2 * ws_rows + srow];
    for (int e = 0; e < ne; ++e) {
        const uint32_t w = ev[srow * kCap + e];
        const int j = (int)(w & 0x0FFFFFFFu);
        if (j == s || !((w >> 28) & 4u)) continue;
        const double *q = dense + (ci.row0 + perm[ci.row0 + j]) * dd;
        double d = 0.0;
        for (int c = 1; c < dd; ++c) d = fmax(d, fabs(__dsub_rn(rp[c], q[c])));
        cnt += d < r;
    }
    out[row] = cnt;
}

// compiled TE layout (DY, DX) whose columns 1 .. DY + DX hold an mc-column
// marginal: 1 <= DY <= min(mc, kGate), DY + DX >= mc, fewest columns, DY
// nearest 3 (the gate width the count order and boxes work best with)
static bool marg_layout(int mc, int &dy, int &dx) {
    static const int pref[4] = {3, 4, 2, 1};
    for (int t = mc; t + 1 <= 18; ++t)
        for (int y : pref) {
            if (y > mc || y > t) continue;
            if (count_table(y, t - y, 0) != nullptr) {
                dy = y;
                dx = t - y;
                return true;
            }
        }
    return false;
}

static Plan radius_plan(const ente_chunk *chunks, int n_chunks, int dy, int dx) {
    Plan p;
    for (int c = 0; c < n_chunks; ++c) {
        p.total_rows = std::max(p.total_rows, chunks[c].row0 + chunks[c].n);
        const int npad = round_up(chunks[c].n, kTJ);
        p.total_prows += npad;
        p.max_npad = std::max(p.max_npad, npad);
        p.n_tiles += (chunks[c].n + kWarpRefs - 1) / kWarpRefs;
    }
    p.fast = true;
    p.dy = dy;
    p.dx = dx;
    p.slots = 2;
    p.dp = (1 + dy + dx + 3) & ~3;
    p.lay.dy = dy;
    p.lay.nout = 1;
    p.lay.slot[0] = 2;
    p.fc = filter_cols(dy);
    return p;
}

// workspace of the generic radius path for marginals of up to max_mc columns
static size_t radius_ws_size(const ente_chunk *chunks, int n_chunks, int max_mc) {
    size_t need = 0;
    for (int mc = 1; mc <= max_mc; ++mc) {
        int dy, dx;
        if (!marg_layout(mc, dy, dx)) continue;
        Plan p = radius_plan(chunks, n_chunks, dy, dx);
        Arena a(nullptr, 0);
        layout_ws(a, p, n_chunks);
        a.take<double>((size_t)p.total_rows * (1 + dy + dx));
        need = std::max(need, a.used);
    }
    return need;
}

// counts of one marginal (mask) for the given radii; false when no compiled
// layout holds it (the caller then scans in fp64)
static int radius_fast(const double *pts64, int64_t total_rows, int dim, const ente_chunk *chunks,
                       int n_chunks, uint32_t mask, const double *radii, int32_t *out_counts,
                       int32_t *status, void *workspace, size_t ws_bytes, cudaStream_t st,
                       bool &done) {
    done = false;
    MargCols mc{};
    for (int c = 0; c < dim; ++c)
        if ((mask >> c) & 1u) mc.col[mc.n++] = c;
    int dy = 0, dx = 0;
    if (mc.n < 1 || !marg_layout(mc.n, dy, dx)) return ENTE_OK;
    const int dd = 1 + dy + dx;
    Plan p = radius_plan(chunks, n_chunks, dy, dx);
    Arena a(workspace, ws_bytes);
    SearchWs w = layout_ws(a, p, n_chunks);
    double *dense = a.take<double>((size_t)p.total_rows * dd);
    if (!a.ok() || !w.info || !dense) {
        set_error("ente_radius_counts: workspace of %zu bytes too small (need %zu)", ws_bytes, a.used);
        return ENTE_ERR_WORKSPACE;
    }
    std::vector<int32_t> htile0;
    int32_t ntiles = 0;
    int rc = upload_chunks(st, chunks, n_chunks, 1, p, w, status, htile0, ntiles);
    if (rc != ENTE_OK) return rc;
    if (!htile0.empty())
        ENTE_CUDA(cudaMemcpyAsync(w.tile0, htile0.data(), sizeof(int32_t) * (2 * n_chunks + 1),
                                  cudaMemcpyHostToDevice, st));
    {
        const int64_t elems = p.total_rows * dd;
        const unsigned blocks = (unsigned)std::min<int64_t>((elems + 255) / 256, (int64_t)num_sms() * 32);
        ENTE_LAUNCH("marg_dense", st,
                    marg_dense_kernel<<<std::max(1u, blocks), 256, 0, st>>>(pts64, dim, p.total_rows,
                                                                            mc, dd, dense));
        ENTE_CUDA(cudaGetLastError());
    }
    const int prune = prune_enabled();
    rc = launch_orders(st, dense, dd, p, w, n_chunks, status, prune, 0, true);
    if (rc != ENTE_OK) return rc;
    if (ntiles > 0) {
        unsigned long long *work = device_work();
        if (!work) {
            set_error("ente_radius_counts: cannot allocate the work counters");
            return ENTE_ERR_CUDA;
        }
        const unsigned nt = (unsigned)ntiles;
        ENTE_LAUNCH("radii_t32", st,
                    radii_t32_kernel<<<nt, kWarpRefs, 0, st>>>(w.info, w.tile0, n_chunks, w.perm, radii,
                                                               w.t32));
        ENTE_CUDA(cudaGetLastError());
        const CountFn count_fn = count_table(dy, dx, p.max_npad);
        prefer_shared(reinterpret_cast<const void *>(count_fn));
        ENTE_LAUNCH("count_pass", st,
                    count_fn<<<nt, 32, 0, st>>>(w.pts32, w.fbox, w.info, w.tile0, n_chunks, w.t32,
                                                p.total_rows, prune, w.cnt3, w.ev, w.ev_n, 4u,
                                                work + 1));
        ENTE_CUDA(cudaGetLastError());
        ENTE_LAUNCH("resolve_counts", st,
                    resolve_counts_kernel<<<nt, kWarpRefs, 0, st>>>(
                        dense, dd, w.info, w.tile0, n_chunks, w.perm, radii, w.cnt3, w.ev, w.ev_n,
                        p.total_rows, out_counts, w.ovf, w.ovf_n));
        ENTE_CUDA(cudaGetLastError());
        Masks masks{};
        masks.n = 1;
        masks.m[0] = mask;
        launch_exact<4>(st, pts64, dim, w.info, n_chunks, status, w.ovf, w.ovf_n, 0, 1, masks,
                        total_rows, nullptr, out_counts, radii);
        ENTE_CUDA(cudaGetLastError());
    }
    done = true;
    return ENTE_OK;
}

static int search_impl(const double *pts64, int64_t total_rows, int dim, const ente_chunk *chunks,
                       int n_chunks, const uint32_t *marg_masks, int n_marg, int k, double *out_eps,
                       int32_t *out_counts, int32_t *status, void *workspace, size_t ws_bytes,
                       void *stream, int split_index, int split_count) {
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
    if (!p.fast && n_marg > 0) {
        // marginals that are not the TE layout's: exact eps from the kNN fast path
        // (no marginals), then each marginal's counts with those radii
        uint32_t none[kMaxMarg] = {0};
        Plan pk = make_plan(chunks, n_chunks, dim, none, 0, k);
        bool fits = pk.fast;
        for (int m = 0; m < n_marg && fits; ++m) {
            int dy, dx;
            fits = marg_layout(__builtin_popcount(marg_masks[m]), dy, dx);
        }
        if (fits) {
            if (split_count > 1 && split_index != 0) return ENTE_OK;  // part 0 does it all
            rc = search_impl(pts64, total_rows, dim, chunks, n_chunks, marg_masks, 0, k, out_eps,
                             nullptr, status, workspace, ws_bytes, stream, 0, 1);
            if (rc != ENTE_OK) return rc;
            for (int m = 0; m < n_marg; ++m) {
                bool done = false;
                rc = radius_fast(pts64, total_rows, dim, chunks, n_chunks, marg_masks[m], out_eps,
                                 out_counts + (int64_t)m * total_rows, status, workspace, ws_bytes,
                                 st, done);
                if (rc != ENTE_OK) return rc;
            }
            return ENTE_OK;
        }
    }
    const int64_t ws_rows = p.total_rows;  // stride of the workspace per-row arrays
    Arena a(workspace, ws_bytes);
    SearchWs w = layout_ws(a, p, n_chunks);
    if (!a.ok() || !w.info) {
        set_error("ente_search: workspace of %zu bytes too small (need %zu)", ws_bytes, a.used);
        return ENTE_ERR_WORKSPACE;
    }
    // host-side chunk table, tile list and k checks
    std::vector<int32_t> htile0;
    int32_t ntiles = 0;
    rc = upload_chunks(st, chunks, n_chunks, k, p, w, status, htile0, ntiles, split_index,
                       split_count);
    if (rc != ENTE_OK) return rc;
    Masks masks{};
    masks.n = n_marg;
    for (int m = 0; m < n_marg; ++m) masks.m[m] = marg_masks[m];
    if (p.fast && ntiles > 0) {
        const int prune = prune_enabled();
        unsigned long long *work = device_work();
        if (!work) {
            set_error("ente_search: cannot allocate the work counters");
            return ENTE_ERR_CUDA;
        }
        // a split search keeps both sweeps in the count order, so every rank's
        // kNN pass covers exactly the references its count pass needs
        rc = launch_orders(st, pts64, dim, p, w, n_chunks, status, prune, split_count == 1);
        if (rc != ENTE_OK) return rc;
        if (!htile0.empty())
            ENTE_CUDA(cudaMemcpyAsync(w.tile0, htile0.data(), sizeof(int32_t) * (2 * n_chunks + 1),
                                      cudaMemcpyHostToDevice, st));
        const unsigned nt = (unsigned)ntiles;
        const KnnFn knn_fn = knn_table(p.dy, p.dx, p.slots, p.max_npad);
        const CountFn count_fn = count_table(p.dy, p.dx, p.max_npad);
        prefer_shared(reinterpret_cast<const void *>(knn_fn));
        prefer_shared(reinterpret_cast<const void *>(count_fn));
        ENTE_LAUNCH("knn_pass", st,
                    knn_fn<<<nt, 32, 0, st>>>(w.pts32k, w.fboxk, w.info,
                                                                     w.tile0, n_chunks, k, prune, w.kmap, w.t32,
                                                                     w.L, work));
        ENTE_CUDA(cudaGetLastError());
        uint32_t fmask = 8u;
        for (int o = 0; o < p.lay.nout; ++o) fmask |= 1u << p.lay.slot[o];
        ENTE_LAUNCH("count_pass", st,
                    count_fn<<<nt, 32, 0, st>>>(w.pts32, w.fbox, w.info, w.tile0, n_chunks,
                                                               w.t32, ws_rows, prune, w.cnt3, w.ev,
                                                               w.ev_n, fmask, work + 1));
        ENTE_CUDA(cudaGetLastError());
        ENTE_LAUNCH("resolve", st,
                    resolve_kernel<<<nt, kWarpRefs, 0, st>>>(pts64, dim, w.info, w.tile0, n_chunks, k, p.lay,
                                                       w.perm, w.L, w.cnt3, w.ev, w.ev_n, ws_rows,
                                                       total_rows, out_eps, out_counts, w.ovf,
                                                       w.ovf_n, w.rs, w.rs_n, w.rs_flag, 1, nullptr));
        ENTE_CUDA(cudaGetLastError());
        {
            dim3 ggrid((unsigned)(p.max_npad / kTJ), (unsigned)std::min(n_chunks, 65535));
            ENTE_LAUNCH("gather64", st,
                        gather64_kernel<<<ggrid, kTJ, 0, st>>>(pts64, dim, w.info, n_chunks, w.perm,
                                                               w.rs_flag, w.pts64s));
        }
        ENTE_CUDA(cudaGetLastError());
        {
            const unsigned rgrid = (unsigned)(num_sms() * 8);
            ENTE_LAUNCH("rescan", st,
                        rescan_table(p.dy, p.dx, k)<<<rgrid, kRescanWarps * 32, 0, st>>>(
                            w.pts32, w.fbox, pts64, w.pts64s, w.info, n_chunks, w.perm, w.t32, w.rs, w.rs_n,
                            k, p.lay, total_rows, out_eps, out_counts));
        }
        ENTE_CUDA(cudaGetLastError());
        dispatch_exact(k, st, pts64, dim, w.info, n_chunks, status, w.ovf, w.ovf_n, 0, masks,
                       total_rows, out_eps, out_counts);
        ENTE_CUDA(cudaGetLastError());
    } else if (!p.fast && split_index == 0) {  // (a split search: part 0 does it all)
        ENTE_LAUNCH("prep", st,
                    prep_kernel<kPrepThreadsBig><<<n_chunks, kPrepThreadsBig, 0, st>>>(pts64, dim, w.info, nullptr, status, 0));
        ENTE_CUDA(cudaGetLastError());
        dispatch_exact(k, st, pts64, dim, w.info, n_chunks, status, nullptr, nullptr, total_rows,
                       masks, total_rows, out_eps, out_counts);
        ENTE_CUDA(cudaGetLastError());
    }
    return ENTE_OK;
}

extern "C" int ente_search(const double *pts64, int64_t total_rows, int dim,
                           const ente_chunk *chunks, int n_chunks, const uint32_t *marg_masks,
                           int n_marg, int k, double *out_eps, int32_t *out_counts,
                           int32_t *status, void *workspace, size_t ws_bytes, void *stream) {
    return search_impl(pts64, total_rows, dim, chunks, n_chunks, marg_masks, n_marg, k, out_eps,
                       out_counts, status, workspace, ws_bytes, stream, 0, 1);
}

extern "C" int ente_search_split(const double *pts64, int64_t total_rows, int dim,
                                 const ente_chunk *chunks, int n_chunks,
                                 const uint32_t *marg_masks, int n_marg, int k, int split_index,
                                 int split_count, double *out_eps, int32_t *out_counts,
                                 int32_t *status, void *workspace, size_t ws_bytes, void *stream) {
    if (split_count < 1 || split_index < 0 || split_index >= split_count) {
        set_error("ente_search_split: split %d of %d", split_index, split_count);
        return ENTE_ERR_ARG;
    }
    return search_impl(pts64, total_rows, dim, chunks, n_chunks, marg_masks, n_marg, k, out_eps,
                       out_counts, status, workspace, ws_bytes, stream, split_index, split_count);
}

// ---------------------------------------------------------------------------
// Shared-y TE batches (shared_y.cuh): the kNN sweep, an m3 + joint-band sweep
// over the kNN order, fp64 resolve, and the y-marginal counts once per
// original point for the whole batch.
// ---------------------------------------------------------------------------
struct SyBufs {
    int32_t *chunk_perm, *va, *vb, *parity, *yva, *yvb, *yperm, *tile3;
    uint32_t *ka, *kb, *kstar, *qs;
    uint32_t *yka, *ykb;
    double *ys, *box;
};

static bool sy_pack(int64_t m) { return m < 65536; }  // counters fit 16-bit halves

static size_t sy_smem_bytes(int C, int nsub, bool pack) {
    const int halves = pack ? 1 : 2;
    return (size_t)C * 4 * 3 + halves * (size_t)(C + 1) * 4 + halves * (size_t)C * 4 +
           (size_t)nsub * 4 + (size_t)kSyBins * 2;
}

static SyBufs sy_layout(Arena &a, int64_t m, int C, int dd) {
    SyBufs b{};
    const int nsub = (int)((m + 31) / 32);
    b.chunk_perm = a.take<int32_t>(C);
    b.tile3 = a.take<int32_t>(2 * C + 1);
    b.ka = a.take<uint32_t>((size_t)m * C);
    b.kb = a.take<uint32_t>((size_t)m * C);
    b.va = a.take<int32_t>((size_t)m * C);
    b.vb = a.take<int32_t>((size_t)m * C);
    b.qs = a.take<uint32_t>((size_t)m * C);
    b.kstar = a.take<uint32_t>((size_t)m * C);
    b.parity = a.take<int32_t>(m);
    b.yka = a.take<uint32_t>(m);
    b.ykb = a.take<uint32_t>(m);
    b.yva = a.take<int32_t>(m);
    b.yvb = a.take<int32_t>(m);
    b.yperm = a.take<int32_t>(m);
    b.ys = a.take<double>((size_t)m * dd);
    b.box = a.take<double>((size_t)nsub * 2 * (dd - 1));
    return b;
}

static bool sy_usable(const Plan &p, int n_chunks, int64_t m, int k) {
    SweepSet ss;
    return p.fast && p.lay.nout == 3 && p.lay.slot[0] == 0 && p.lay.slot[1] == 1 && p.lay.slot[2] == 2 &&
           p.max_npad >= kCompactMinRows && k + 1 <= 16 && find_sweep_set(p.dy, p.dx, ss) &&
           ss.count3 != nullptr && 1 + p.dy <= kSyMaxY && n_chunks < 65535 &&
           sy_smem_bytes(n_chunks, (int)((m + 31) / 32), sy_pack(m)) <= 200 * 1024;
}

static void te_masks_of(int dy, int dim, uint32_t *masks) {
    masks[0] = ((1u << (dy + 1)) - 1u) & ~1u;                          // y-past
    masks[1] = (1u << (dy + 1)) - 1u;                                   // y_t + y-past
    masks[2] = ((dim >= 32) ? 0xFFFFFFFFu : ((1u << dim) - 1u)) & ~1u;  // y-past + x-past
}

extern "C" size_t ente_search_te_shared_workspace_size(const ente_chunk *chunks, int n_chunks, int dim,
                                                       int dy, int k) {
    uint32_t masks[3];
    te_masks_of(dy, dim, masks);
    Plan p = make_plan(chunks, n_chunks, dim, masks, 3, k);
    if (!p.fast) return ente_search_workspace_size(chunks, n_chunks, dim, 3, k);
    Arena a(nullptr, 0);
    layout_ws(a, p, n_chunks);
    const int64_t m = n_chunks > 0 ? chunks[0].n : 0;
    sy_layout(a, m, n_chunks, 1 + dy);
    return std::max(a.used, ente_search_workspace_size(chunks, n_chunks, dim, 3, k)) + 256;
}

extern "C" int ente_search_te_shared(const double *pts64, int64_t total_rows, int dim,
                                     const ente_chunk *chunks, int n_chunks, int dy, int k,
                                     const double *y0, int reps, int w, const int32_t *chunk_perm,
                                     const int32_t *perms, const int32_t *inv_perms, double margin,
                                     double *out_eps, int32_t *out_counts, int32_t *status,
                                     void *workspace, size_t ws_bytes, void *stream) {
    if (dy < 1 || dim - 1 - dy < 0 || reps < 1 || w < 1 || !y0 || !chunk_perm || !(margin >= 0.0)) {
        set_error("ente_search_te_shared: bad arguments");
        return ENTE_ERR_ARG;
    }
    uint32_t masks[3];
    te_masks_of(dy, dim, masks);
    int rc = validate(chunks, n_chunks, dim, masks, 3, k);
    if (rc != ENTE_OK) return rc;
    if (n_chunks == 0) return ENTE_OK;
    const int64_t m = (int64_t)reps * w;
    for (int c = 0; c < n_chunks; ++c)
        if (chunks[c].n != m) {
            set_error("ente_search_te_shared: chunk %d has %d rows, expected reps * w = %lld", c,
                      chunks[c].n, (long long)m);
            return ENTE_ERR_ARG;
        }
    Plan p = make_plan(chunks, n_chunks, dim, masks, 3, k);
    if (!sy_usable(p, n_chunks, m, k))  // the general search gives the same counts
        return search_impl(pts64, total_rows, dim, chunks, n_chunks, masks, 3, k, out_eps, out_counts,
                           status, workspace, ws_bytes, stream, 0, 1);
    if (p.total_rows > total_rows) {
        set_error("ente_search_te_shared: chunks reference rows beyond total_rows");
        return ENTE_ERR_ARG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t ws_rows = p.total_rows;
    Arena a(workspace, ws_bytes);
    SearchWs w_ = layout_ws(a, p, n_chunks);
    SyBufs b = sy_layout(a, m, n_chunks, 1 + dy);
    if (!a.ok() || !w_.info || !b.box) {
        set_error("ente_search_te_shared: workspace of %zu bytes too small (need %zu)", ws_bytes, a.used);
        return ENTE_ERR_WORKSPACE;
    }
    std::vector<int32_t> htile0;
    int32_t ntiles = 0;
    rc = upload_chunks(st, chunks, n_chunks, k, p, w_, status, htile0, ntiles);
    if (rc != ENTE_OK) return rc;
    const int prune = prune_enabled();
    unsigned long long *work = device_work();
    if (!work) {
        set_error("ente_search_te_shared: cannot allocate the work counters");
        return ENTE_ERR_CUDA;
    }
    rc = launch_orders(st, pts64, dim, p, w_, n_chunks, status, prune, 1, false, true);
    if (rc != ENTE_OK) return rc;
    if (!htile0.empty())
        ENTE_CUDA(cudaMemcpyAsync(w_.tile0, htile0.data(), sizeof(int32_t) * (2 * n_chunks + 1),
                                  cudaMemcpyHostToDevice, st));
    ENTE_CUDA(cudaMemcpyAsync(b.chunk_perm, chunk_perm, sizeof(int32_t) * n_chunks,
                              cudaMemcpyHostToDevice, st));
    SweepSet ss;
    find_sweep_set(p.dy, p.dx, ss);
    // the m3 / joint sweep takes groups of 32 * ENTE_KO_RT references
    constexpr int kWr3 = 32 * count_rt<true>();
    std::vector<int32_t> htile3(2 * n_chunks + 1, 0);
    int32_t ntiles3 = 0;
    for (int c = 0; c < n_chunks; ++c) {
        htile3[c] = ntiles3;
        if (k <= chunks[c].n - 1) ntiles3 += (chunks[c].n + kWr3 - 1) / kWr3;
    }
    htile3[n_chunks] = ntiles3;
    ENTE_CUDA(cudaMemcpyAsync(b.tile3, htile3.data(), sizeof(int32_t) * (2 * n_chunks + 1),
                              cudaMemcpyHostToDevice, st));
    if (ntiles > 0) {
        const unsigned nt = (unsigned)ntiles;
        const KnnFn knn_fn = knn_table(p.dy, p.dx, p.slots, p.max_npad);
        prefer_shared(reinterpret_cast<const void *>(knn_fn));
        prefer_shared(reinterpret_cast<const void *>(ss.count3));
        ENTE_LAUNCH("knn_pass", st,
                    knn_fn<<<nt, 32, 0, st>>>(w_.pts32k, w_.fboxk, w_.info, w_.tile0, n_chunks, k, prune,
                                              nullptr, w_.t32, w_.L, work));
        ENTE_CUDA(cudaGetLastError());
        ENTE_LAUNCH("count_pass", st,
                    ss.count3<<<(unsigned)ntiles3, 32, 0, st>>>(w_.pts32k, w_.fboxk, w_.info, b.tile3,
                                                               n_chunks, w_.t32,
                                                 ws_rows, prune, w_.cnt3, w_.ev, w_.ev_n, 4u | 8u,
                                                 work + 1));
        ENTE_CUDA(cudaGetLastError());
        ENTE_LAUNCH("resolve", st,
                    resolve_kernel<<<nt, kWarpRefs, 0, st>>>(pts64, dim, w_.info, w_.tile0, n_chunks, k,
                                                             p.lay, w_.permk, w_.L, w_.cnt3, w_.ev,
                                                             w_.ev_n, ws_rows, total_rows, out_eps,
                                                             out_counts, w_.ovf, w_.ovf_n, w_.rs,
                                                             w_.rs_n, w_.rs_flag, 0, b.kstar));
        ENTE_CUDA(cudaGetLastError());
    }
    Masks mk{};
    mk.n = 3;
    for (int i = 0; i < 3; ++i) mk.m[i] = masks[i];
    dispatch_exact(k, st, pts64, dim, w_.info, n_chunks, status, w_.ovf, w_.ovf_n, 0, mk, total_rows,
                   out_eps, out_counts);
    ENTE_CUDA(cudaGetLastError());
    // y-marginal counts once per original point
    SyGeom g;
    g.reps = reps;
    g.w = w;
    g.m = (int)m;
    g.C = n_chunks;
    g.dd = 1 + dy;
    g.nsub = (int)((m + 31) / 32);
    g.margin = margin;
    {
        dim3 grid((unsigned)std::min<int64_t>((m + 255) / 256, 1024), (unsigned)n_chunks);
        ENTE_LAUNCH("sy_scatter", st,
                    sy_scatter_kernel<<<grid, 256, 0, st>>>(w_.info, b.chunk_perm, perms, g, out_eps,
                                                             b.kstar, b.ka, b.va, b.qs));
        ENTE_CUDA(cudaGetLastError());
    }
    if (n_chunks <= kSortSmallN) {
        ENTE_LAUNCH("sy_sort", st,
                    sy_sort_kernel<kSortThreadsSmall><<<(unsigned)m, kSortThreadsSmall, 0, st>>>(
                        b.ka, b.kb, b.va, b.vb, n_chunks, b.parity));
    } else {
        ENTE_LAUNCH("sy_sort", st,
                    sy_sort_kernel<kSortThreads><<<(unsigned)m, kSortThreads, 0, st>>>(
                        b.ka, b.kb, b.va, b.vb, n_chunks, b.parity));
    }
    ENTE_CUDA(cudaGetLastError());
    ENTE_LAUNCH("sy_order", st,
                sy_order_kernel<<<1, kSortThreads, 0, st>>>(y0, g, b.yka, b.ykb, b.yva, b.yvb, b.yperm));
    ENTE_CUDA(cudaGetLastError());
    ENTE_LAUNCH("sy_gather", st,
                sy_gather_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(y0, g, b.yperm, b.ys, b.box));
    ENTE_CUDA(cudaGetLastError());
    const bool pack = sy_pack(m);
    const size_t smem = sy_smem_bytes(n_chunks, g.nsub, pack);
    auto kern = pack ? sy_count_kernel<true> : sy_count_kernel<false>;
    ENTE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ENTE_LAUNCH("sy_count", st,
                kern<<<(unsigned)m, kSyThreads, smem, st>>>(
                    y0, b.ys, b.yperm, b.box, g, b.ka, b.kb, b.va, b.vb, b.qs, b.parity, w_.info, b.chunk_perm,
                    inv_perms, pts64, dim, out_eps, total_rows, out_counts));
    ENTE_CUDA(cudaGetLastError());
    return ENTE_OK;
}

// Evaluated (reference, candidate) pairs of the two sweeps on the current
// device since the last call (synchronises the device): every (reference,
// sub-tile) visit the sweeps made -- compacted references of a sub-tile, or
// every reference of the warp in the direct variants -- times the sub-tile's
// rows.  This is the lane-level work; lanes left idle by partial rounds are
// not counted.
extern "C" void ente_search_work(unsigned long long *knn_pairs, unsigned long long *count_pairs) {
    unsigned long long h[2] = {0, 0};
    unsigned long long *d = device_work();
    if (d && cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess)
        cudaMemset(d, 0, sizeof(h));
    *knn_pairs = h[0] * (unsigned long long)kSub;
    *count_pairs = h[1] * (unsigned long long)kSub;
}


extern "C" int ente_knn_indices(const double *pts64, int64_t total_rows, int dim,
                                const ente_chunk *chunks, int n_chunks, int k,
                                const double *eps, int32_t *out_idx, int32_t *status,
                                void *workspace, size_t ws_bytes, void *stream) {
    int rc = validate(chunks, n_chunks, dim, nullptr, 0, k);
    if (rc != ENTE_OK) return rc;
    if (n_chunks == 0) return ENTE_OK;
    if (!eps || !out_idx) {
        set_error("ente_knn_indices: eps and out_idx are required");
        return ENTE_ERR_ARG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint32_t none[kMaxMarg] = {0};
    Plan p = make_plan(chunks, n_chunks, dim, none, 0, k);
    if (p.total_rows > total_rows) {
        set_error("ente_knn_indices: chunks reference row %lld beyond total_rows=%lld",
                  (long long)p.total_rows, (long long)total_rows);
        return ENTE_ERR_ARG;
    }
    Arena a(workspace, ws_bytes);
    SearchWs w = layout_ws(a, p, n_chunks);
    if (!a.ok() || !w.info) {
        set_error("ente_knn_indices: workspace of %zu bytes too small (need %zu)", ws_bytes, a.used);
        return ENTE_ERR_WORKSPACE;
    }
    std::vector<int32_t> htile0;
    int32_t ntiles = 0;
    rc = upload_chunks(st, chunks, n_chunks, k, p, w, status, htile0, ntiles);
    if (rc != ENTE_OK) return rc;
    if (p.fast && ntiles > 0) {
        rc = launch_orders(st, pts64, dim, p, w, n_chunks, status, 1);
        if (rc != ENTE_OK) return rc;
    } else {
        ENTE_LAUNCH("prep", st,
                    prep_kernel<kPrepThreadsBig><<<n_chunks, kPrepThreadsBig, 0, st>>>(pts64, dim, w.info, nullptr, status, 0));
        ENTE_CUDA(cudaGetLastError());
    }
    const float *p32 = p.fast ? w.pts32k : nullptr;
    const unsigned grid = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((p.total_rows + kIdxWarps - 1) / kIdxWarps, (int64_t)num_sms() * 64));
    const int dp = (dim + 3) & ~3;
    const int S = exact_slots(k);
#define ENTE_IDX(DPV, SV)                                                                        \
    if (dp == DPV && S == SV) {                                                                   \
        ENTE_LAUNCH("knn_index", st,                                                              \
                    knn_index_kernel<DPV, SV><<<grid, kIdxWarps * 32, 0, st>>>(                   \
                        pts64, dim, w.info, n_chunks, status, p32, w.fboxk, w.permk, eps, k,     \
                        p.total_rows, out_idx));                                                  \
        ENTE_CUDA(cudaGetLastError());                                                           \
        return ENTE_OK;                                                                           \
    }
#define ENTE_IDX_S(DPV) ENTE_IDX(DPV, 4) ENTE_IDX(DPV, 8) ENTE_IDX(DPV, 16) ENTE_IDX(DPV, 32) ENTE_IDX(DPV, 64)
    ENTE_IDX_S(4) ENTE_IDX_S(8) ENTE_IDX_S(12) ENTE_IDX_S(16) ENTE_IDX_S(20)
#undef ENTE_IDX_S
#undef ENTE_IDX
    set_error("ente_knn_indices: dim=%d is above the compiled maximum of 20", dim);
    return ENTE_ERR_ARG;
}

extern "C" int ente_search_path(int dim, const uint32_t *marg_masks, int n_marg, int k) {
    if (dim < 1 || dim > kMaxDim || n_marg < 0 || n_marg > kMaxMarg || k < 1) return 0;
    ente_chunk one{0, 1 << 16, 0};
    Plan p = make_plan(&one, 1, dim, marg_masks, n_marg, k);
    if (p.fast) return 1;
    uint32_t none[kMaxMarg] = {0};
    if (!make_plan(&one, 1, dim, none, 0, k).fast) return 0;
    for (int m = 0; m < n_marg; ++m) {
        int dy, dx;
        if (!marg_layout(__builtin_popcount(marg_masks[m]), dy, dx)) return 0;
    }
    return 2;
}

extern "C" size_t ente_radius_counts_workspace_size(const ente_chunk *chunks, int n_chunks,
                                                    int dim) {
    Arena a(nullptr, 0);
    a.take<ChunkInfo>(n_chunks);
    a.take<int32_t>(2);
    const size_t gen = (chunks && dim >= 1) ? radius_ws_size(chunks, n_chunks, std::min(dim, 17)) : 0;
    return std::max(a.used, gen) + 256;
}

// Strict radius counts for caller-given radii (reference radius_counts,
// engine.py:179-188), one count array per marginal: the generic fp32-filter
// sweep (radius_fast) for every marginal a compiled layout holds, the fp64
// warp-per-point scan for the others.
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
    for (int c = 0; c < n_chunks; ++c)
        if (chunks[c].row0 + chunks[c].n > total_rows) {
            set_error("ente_radius_counts: chunk %d beyond total_rows", c);
            return ENTE_ERR_ARG;
        }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Masks slow{};
    std::vector<int> slow_out;
    for (int m = 0; m < n_marg; ++m) {
        bool done = false;
        rc = radius_fast(pts64, total_rows, dim, chunks, n_chunks, marg_masks[m], radii,
                         out_counts + (int64_t)m * total_rows, status, workspace, ws_bytes, st, done);
        if (rc != ENTE_OK) return rc;
        if (!done) {
            slow.m[slow.n++] = marg_masks[m];
            slow_out.push_back(m);
        }
    }
    if (slow.n == 0) return ENTE_OK;
    // marginals no compiled layout holds (more than 17 columns): fp64 scan
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
    }
    ENTE_CUDA(cudaMemcpyAsync(info, hinfo.data(), sizeof(ChunkInfo) * n_chunks, cudaMemcpyHostToDevice, st));
    ENTE_CUDA(cudaMemcpyAsync(status, hstatus.data(), sizeof(int32_t) * n_chunks, cudaMemcpyHostToDevice, st));
    for (int i = 0; i < slow.n; ++i) {
        Masks one{};
        one.n = 1;
        one.m[0] = slow.m[i];
        launch_exact<4>(st, pts64, dim, info, n_chunks, status, nullptr, nullptr, total_rows, 1, one,
                        total_rows, nullptr, out_counts + (int64_t)slow_out[i] * total_rows, radii);
        ENTE_CUDA(cudaGetLastError());
    }
    return ENTE_OK;
}
