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
constexpr int kKnnQ = 2;                    // kNN sub-tile boxes: 4 * kKnnQ columns from 0

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
constexpr int kPrepThreads = 256;
constexpr int kPrepWarps = kPrepThreads / 32;
constexpr int kCovN = kPcaCols * (kPcaCols + 1) / 2;

__global__ void __launch_bounds__(kPrepThreads) prep_kernel(const double *__restrict__ pts64, int dim,
                                                            ChunkInfo *__restrict__ info,
                                                            ColStats *__restrict__ stats,
                                                            int32_t *__restrict__ status, int want32) {
    const int c = blockIdx.x;
    const ChunkInfo ci = info[c];
    if (status[c] != ENTE_CHUNK_OK) return;
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
        // second sweep over the (L2-resident) rows for the covariance, kept
        // apart so that neither loop needs more than ~64 registers
        float cov[kCovN], x0[kPcaCols];
#pragma unroll
        for (int e = 0; e < kCovN; ++e) cov[e] = 0.0f;
#pragma unroll
        for (int i = 0; i < kPcaCols; ++i) x0[i] = (g0 == 0 && i < P) ? (float)p[i] : 0.0f;
        if (g0 == 0 && stats && ci.n >= kPcaMinRows) {
            for (int r = threadIdx.x; r < ci.n; r += kPrepThreads) {
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
            stats[c].cov[e] = v;
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
    uint32_t *k0 = ka + ci.row0, *k1 = kb + ci.row0;
    int32_t *v0 = va + ci.row0, *v1 = vb + ci.row0;
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
    for (int i = threadIdx.x; i < ci.n; i += T) {
        float z0, z1;
        proj(i, z0, z1);
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
    const float q = 4095.0f;  // 12 bits per axis: 24-bit keys, three radix passes
    const float s0 = mx0 > mn0 ? q / (mx0 - mn0) : 0.0f;
    const float s1 = mx1 > mn1 ? q / (mx1 - mn1) : 0.0f;
    for (int i = threadIdx.x; i < ci.n; i += T) {
        float z0, z1;
        proj(i, z0, z1);
        const uint32_t a = (uint32_t)fminf(fmaxf((z0 - mn0) * s0, 0.0f), q);
        const uint32_t b = (uint32_t)fminf(fmaxf((z1 - mn1) * s1, 0.0f), q);
        k0[i] = (spread15(a) << 1) | spread15(b);
        v0[i] = i;
    }
    __syncthreads();
    const int par = cta_radix_sort<T, uint32_t, int32_t>(k0, k1, v0, v1, ci.n, 24, sm);
    const int32_t *res = par ? v1 : v0;
    for (int i = threadIdx.x; i < ci.n; i += T) perm[ci.row0 + i] = res[i];
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
        if (valid) kmap[ci.row0 + s] = inv[orig];
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

// ---------------------------------------------------------------------------
// sweep tile t -> (chunk, first sorted reference): tile0[c] = first tile of
// chunk c (ascending, n_chunks + 1 entries); chunks without tiles repeat
// their successor's value, so the largest c with tile0[c] <= t is the owner.
// tile0[n_chunks + 1 + c] = the chunk's first tile index within the chunk
// (non-zero only for split searches, which sweep a range of references).
// ---------------------------------------------------------------------------
__device__ __forceinline__ TileRef tile_of(const int32_t *__restrict__ tile0, int n_chunks, int t) {
    int lo = 0, hi = n_chunks - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(tile0 + mid) <= t) lo = mid;
        else hi = mid - 1;
    }
    TileRef tr;
    tr.chunk = lo;
    tr.r0 = (t - __ldg(tile0 + lo) + __ldg(tile0 + n_chunks + 1 + lo)) * kWarpRefs;
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
    const double w = fmax(__dsub_ru((double)t32, (double)lo), __dsub_ru((double)hi, (double)t32));
    b.lo = lo;
    b.hi = hi;
    b.nlo = -lo;
    b.nt = -t32;
    b.w = __double2float_ru(w);
    return b;
}

__device__ __forceinline__ float warp_max_nonneg(float v) {
    return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(fmaxf(v, 0.0f))));
}

// ---------------------------------------------------------------------------
// Warp-private candidate stream.
//
// Each sweep CTA is ONE warp owning 128 consecutive sorted references (4 per
// lane).  It walks the chunk's 32-row sub-tiles home-first, then alternately
// below and above (nearest first in the Morton order, so kNN bounds shrink
// early).  Sub-tile boxes are tested 32 positions at a time, one per lane,
// with the next window's boxes prefetched into registers; needed sub-tiles
// are streamed into a ring of NSLOT shared-memory slots by the TMA engine
// (cp.async.bulk + mbarrier).  Warps never wait for each other.
// ---------------------------------------------------------------------------
// A sub-tile box: Q float4 quads of column minima, then Q of maxima
// (fbox layout per sub-tile: lo[4Q] | hi[4Q], float4 index st * 2Q).
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
    const float a = fmaxf(fmaxf(lo.x - bhi.x, blo.x - hi.x), fmaxf(lo.y - bhi.y, blo.y - hi.y));
    const float b = fmaxf(fmaxf(lo.z - bhi.z, blo.z - hi.z), fmaxf(lo.w - bhi.w, blo.w - hi.w));
    return fmaxf(a, b);
}

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

    __device__ void init(const float4 *__restrict__ fb, int wrow, int n, int npad) {
        h0 = wrow / kSub;
        nh = (min(wrow + 32 * kRT, n) - wrow + kSub - 1) / kSub;
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
        prefetch(fb, (threadIdx.x & 31));
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
        const int lane = threadIdx.x & 31;
        for (;;) {
            while (mask == 0) {
                if (base + 32 >= npos) return -1;
                base += 32;
                wst = nst;
                wd = wst >= 0 ? dist(nb) : INFINITY;
                mask = __ballot_sync(0xffffffffu, strict ? (wd < bound) : (wd <= bound));
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

// fp32 distance from a reference (negated packed coordinates) to a sub-tile
// box over the columns F0 .. F0 + NC - 1 (box slot g = column - F0): a lower
// bound of the reference's fp32 distance to every row of the sub-tile over
// any column set containing them (fl monotone).
template <int F0, int NC, int NP, int Q>
__device__ __forceinline__ float point_box(const float2 (&nr)[NP], const Box<Q> &b) {
    float d = 0.0f;
#pragma unroll
    for (int g = 0; g < NC; ++g) {
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

template <int DP, int NSLOT>
struct Ring {
    float buf[NSLOT][kSub * DP];
    uint64_t full[NSLOT];
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
__global__ void __launch_bounds__(32, S > 8 ? 16 : sweep_minb(1 + DY + DX, ENTE_KNN_MINB)) knn_pass_kernel(
    const float *__restrict__ pts32, const float *__restrict__ fbox,
    const ChunkInfo *__restrict__ info, const int32_t *__restrict__ tile0, int n_chunks, int k, int prune,
    const int32_t *__restrict__ kmap, float *__restrict__ t32_out, int32_t *__restrict__ L_out,
    unsigned long long *__restrict__ work) {
    using L = Lay<DY, DX>;
    constexpr int D = L::D, DP = L::DP, NP = L::NP, PG = L::PG;
    constexpr int NSLOT = L::NSLOT < ENTE_KNN_NSLOT ? L::NSLOT : ENTE_KNN_NSLOT;
    constexpr int NBC = D < 4 * kKnnQ ? D : 4 * kKnnQ;  // box columns 0 .. NBC-1
    __shared__ __align__(128) Ring<DP, NSLOT> ring;
    const TileRef tr = tile_of(tile0, n_chunks, blockIdx.x);
    const ChunkInfo ci = info[tr.chunk];
    if (!ci.ok32) return;
    const int lane = threadIdx.x;
    const float *cp = pts32 + ci.prow0 * DP;
    const float4 *fb = reinterpret_cast<const float4 *>(fbox) + (ci.prow0 / kSub) * 2 * kKnnQ;
    const int wrow = tr.r0;
    float2 ref[kRT][NP];
    float kd[kRT][S];
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
        const int idx = wrow + r * 32 + lane;
        const bool valid = idx < ci.n;
        load_ref<D>(ref[r], cp + (int64_t)idx * DP, valid);
#pragma unroll
        for (int s = 0; s < S; ++s) kd[r][s] = (!valid || s < S - (k + 1)) ? -INFINITY : INFINITY;
    }
    if (lane < NSLOT) mbar_init(&ring.full[lane], 1);
    fence_barrier_init();
    __syncwarp();
    Walker<kKnnQ> wk;
    wk.init(fb, wrow, ci.n, ci.npad);
    float bound = INFINITY;  // warp max of the current k-th distances
    auto refs_need = [&](const Box<kKnnQ> &b) {
        bool need = !prune;
#pragma unroll
        for (int r = 0; r < kRT; ++r) need |= point_box<0, NBC, NP, kKnnQ>(ref[r], b) < kd[r][S - 1];
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
                need |= dj[r] < kd[r][S - 1];
            }
            if (__any_sync(0xffffffffu, need)) {
                bool ins = false;
#pragma unroll
                for (int r = 0; r < kRT; ++r) {
                    diff_pairs<D, PG, NP>(ref[r], c, a[r]);
                    dj[r] = maxabs<G, D, 2 * NP>(a[r], dj[r]);
                    ins |= dj[r] < kd[r][S - 1];
                }
                if (ins) {
#pragma unroll
                    for (int r = 0; r < kRT; ++r) insert_sorted<S>(kd[r], dj[r]);
                }
            }
        }
        ++nsub;
        float wb = 0.0f;
#pragma unroll
        for (int r = 0; r < kRT; ++r) wb = fmaxf(wb, kd[r][S - 1]);
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
        const float t32 = kd[r][S - 1];
        const float lo = __double2float_rd(__dsub_rd((double)t32, 2.0 * ci.delta));
        int Lc = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) Lc += (kd[r][s] > -INFINITY) && (kd[r][s] < lo);
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
    const int lane = threadIdx.x;
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
    wk.init(fb, wrow, ci.n, ci.npad);
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
                const float e3 = m3 + band[r].nlo;
                cA[r] += __float_as_uint(e.x) >> 31;
                c2[r] += __float_as_uint(e.y) >> 31;
                c3[r] += __float_as_uint(e3) >> 31;
                // conservative band test: min |v - t| <= w
                const float2 b1 = __fadd2_rn(make_float2(A, m2), make_float2(band[r].nt, band[r].nt));
                const float2 b2 = __fadd2_rn(make_float2(m3, jd), make_float2(band[r].nt, band[r].nt));
                const float bm = fminf(fminf(fabsf(b1.x), fabsf(b1.y)), fminf(fabsf(b2.x), fabsf(b2.y)));
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
        ++nsub;
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
template <int DP, int NSLOT>
struct CountRefs {
    float ref[32 * kRT][DP];  // fp32 centred coordinates
    float lo[32 * kRT], hi[32 * kRT], t[32 * kRT], w[32 * kRT];
    uint32_t cnt[3][32 * kRT];
    int nev[32 * kRT];
    int slot[32 * kRT];       // compacted reference list of the current sub-tile
};

template <int DY, int DX>
__global__ void __launch_bounds__(32, sweep_minb(1 + DY + DX, ENTE_CNT_MINB)) count_pass_kernel(
    const float *__restrict__ pts32, const float *__restrict__ fbox,
    const ChunkInfo *__restrict__ info, const int32_t *__restrict__ tile0, int n_chunks,
    const float *__restrict__ t32_in, int64_t ws_rows, int prune, int32_t *__restrict__ cnt_out,
    uint32_t *__restrict__ ev, int32_t *__restrict__ ev_n, uint32_t fmask,
    unsigned long long *__restrict__ work) {
    using L = Lay<DY, DX>;
    constexpr int D = L::D, DP = L::DP, NP = L::NP, PG = L::PG;
    constexpr int NSLOT = L::NSLOT < ENTE_CNT_NSLOT ? L::NSLOT : ENTE_CNT_NSLOT;
    __shared__ __align__(128) Ring<DP, NSLOT> ring;
    __shared__ __align__(16) CountRefs<DP, NSLOT> rs;
    const TileRef tr = tile_of(tile0, n_chunks, blockIdx.x);
    const ChunkInfo ci = info[tr.chunk];
    if (!ci.ok32) return;
    const int lane = threadIdx.x;
    const unsigned lt = (1u << lane) - 1u;
    const float *cp = pts32 + ci.prow0 * DP;
    const float4 *fb = reinterpret_cast<const float4 *>(fbox) + (ci.prow0 / kSub) * 2;
    const int wrow = tr.r0;
    float2 myref[kRT][NP];  // this lane's own references (walker tests)
    float myhi[kRT];
    float hmax = 0.0f;
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
        const int ri = r * 32 + lane;
        const int idx = wrow + ri;
        const bool valid = idx < ci.n;
        load_ref<D>(myref[r], cp + (int64_t)idx * DP, valid);
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
        rs.t[ri] = b.nt;
        rs.w[ri] = b.w;
        myhi[r] = b.hi;
        rs.cnt[0][ri] = rs.cnt[1][ri] = rs.cnt[2][ri] = 0u;
        rs.nev[ri] = 0;
    }
    const float bound = warp_max_nonneg(hmax);
    constexpr int NG = DY < kGate ? DY : kGate;
    auto refs_need = [&](const Box<1> &b) {
        uint32_t need = 0u;
#pragma unroll
        for (int r = 0; r < kRT; ++r)
            need |= ((!prune && myhi[r] > -INFINITY) || point_box<1, NG, NP, 1>(myref[r], b) <= myhi[r])
                        ? (1u << r) : 0u;
        return need;
    };
    if (lane < NSLOT) mbar_init(&ring.full[lane], 1);
    fence_barrier_init();
    __syncwarp();
    Walker<1> wk;
    wk.init(fb, wrow, ci.n, ci.npad);
    int slot_st = -1;
    uint32_t slot_need = 0u;  // kRT bits per ring slot: this lane's needs of the issued sub-tiles
    int issued = 0;
    uint32_t nsub = 0;
    for (; issued < NSLOT; ++issued) {
        const int st = wk.next(fb, prune ? bound : INFINITY, false, refs_need);
        if (st < 0) break;
        if (lane == issued) slot_st = st;
        slot_need |= wk.need << (kRT * issued);
        if (lane == 0) ring_issue(ring, issued, cp + (int64_t)st * kSub * DP);
    }
    for (int used = 0; used < issued; ++used) {
        const int slot = used % NSLOT;
        const int cur_st = __shfl_sync(0xffffffffu, slot_st, slot);
        const uint32_t nb = (slot_need >> (kRT * slot)) & ((1u << kRT) - 1u);
        // compact the references that need this sub-tile
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
        constexpr int NQ = DP / 4;
        for (int round = 0; round < nneed; round += 32) {
            const bool active = round + lane < nneed;
            const int ri = active ? rs.slot[round + lane] : 0;
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
            const float nlo = -lo, nt = rs.t[ri], wb = active ? rs.w[ri] : -1.0f;
            uint32_t cA = 0u, c2 = 0u, c3 = 0u;
            int nev = active ? rs.nev[ri] : 0;
            const int64_t evrow = (ci.row0 + wrow + ri) * kCap;
            // one candidate row against this lane's reference
            auto visit = [&](const float4 (&cur)[NQ], int j) {
                const float2 *c = reinterpret_cast<const float2 *>(cur);
                float a[2 * NP];
                diff_pairs<D, 0, PG>(ref, c, a);
                const float A = maxabs0<1, 1 + DY, 2 * NP>(a);
                if (!__any_sync(0xffffffffu, A <= hi)) return;
                diff_pairs<D, PG, NP>(ref, c, a);
                const float m2 = fmaxf(A, fabsf(a[0]));
                const float m3 = maxabs<1 + DY, D, 2 * NP>(a, A);
                const float jd = fmaxf(m2, m3);
                const float2 e = __fadd2_rn(make_float2(A, m2), make_float2(nlo, nlo));
                const float e3 = m3 + nlo;
                cA += __float_as_uint(e.x) >> 31;
                c2 += __float_as_uint(e.y) >> 31;
                c3 += __float_as_uint(e3) >> 31;
                const float2 b1 = __fadd2_rn(make_float2(A, m2), make_float2(nt, nt));
                const float2 b2 = __fadd2_rn(make_float2(m3, jd), make_float2(nt, nt));
                const float bm = fminf(fminf(fabsf(b1.x), fabsf(b1.y)), fminf(fabsf(b2.x), fabsf(b2.y)));
                if (bm <= wb) {
                    uint32_t f = ((A >= lo && A <= hi) ? 1u : 0u) | ((m2 >= lo && m2 <= hi) ? 2u : 0u) |
                                 ((m3 >= lo && m3 <= hi) ? 4u : 0u) | ((jd >= lo && jd <= hi) ? 8u : 0u);
                    f &= fmask;
                    if (f) {
                        if (nev < kCap) ev[evrow + nev] = (uint32_t)(cur_st * kSub + j) | (f << 28);
                        ++nev;
                    }
                }
            };
            // ping-pong row registers: the next row's LDS overlaps this row's math
            float4 ra[NQ], rb[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) ra[q] = tile[q];
            for (int j = 0; j < kSub; j += 2) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) rb[q] = tile[(j + 1) * NQ + q];
                visit(ra, j);
                if (j + 2 < kSub) {
#pragma unroll
                    for (int q = 0; q < NQ; ++q) ra[q] = tile[(j + 2) * NQ + q];
                }
                visit(rb, j + 1);
            }
            if (active) {
                rs.cnt[0][ri] += cA;
                rs.cnt[1][ri] += c2;
                rs.cnt[2][ri] += c3;
                rs.nev[ri] = nev;
            }
            __syncwarp();
        }
        ++nsub;
        __syncwarp();
        const int st = wk.next(fb, prune ? bound : INFINITY, false, refs_need);
        if (st >= 0) {
            const int ns = issued % NSLOT;
            if (lane == ns) slot_st = st;
            slot_need = (slot_need & ~(((1u << kRT) - 1u) << (kRT * ns))) | (wk.need << (kRT * ns));
            if (lane == 0) ring_issue(ring, ns, cp + (int64_t)st * kSub * DP);
            ++issued;
        }
    }
    if (lane == 0) atomicAdd(work, (unsigned long long)nsub);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
        const int ri = r * 32 + lane;
        const int idx = wrow + ri;
        if (idx >= ci.n) continue;
        const uint32_t self = rs.lo[ri] > 0.0f ? 1u : 0u;  // the self pair counted as inside
        const int64_t row = ci.row0 + idx;
        cnt_out[row] = (int32_t)(rs.cnt[0][ri] - self);
        cnt_out[ws_rows + row] = (int32_t)(rs.cnt[1][ri] - self);
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

__global__ void __launch_bounds__(kWarpRefs) resolve_kernel(
    const double *__restrict__ pts64, int dim, const ChunkInfo *__restrict__ info,
    const int32_t *__restrict__ tile0, int n_chunks, int k, TeLayout lay, const int32_t *__restrict__ perm,
    const int32_t *__restrict__ L_in, const int32_t *__restrict__ cnt_in,
    const uint32_t *__restrict__ ev, const int32_t *__restrict__ ev_n, int64_t ws_rows,
    int64_t total_rows, double *__restrict__ out_eps, int32_t *__restrict__ out_counts,
    int64_t *__restrict__ ovf_list, int32_t *__restrict__ ovf_n, int64_t *__restrict__ rs_list,
    int32_t *__restrict__ rs_n) {
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
        if (ci.ok32) {  // fp32 data usable: pruned warp rescan of the sorted row
            const int slot = atomicAdd(rs_n, 1);
            rs_list[slot] = srow;
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
    const ChunkInfo *__restrict__ info, int n_chunks, const int32_t *__restrict__ perm,
    const float *__restrict__ t32_in, const int64_t *__restrict__ list,
    const int32_t *__restrict__ list_n, int k, TeLayout lay, int64_t total_rows,
    double *__restrict__ out_eps, int32_t *__restrict__ out_counts) {
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
        for (int col = 0; col < D; ++col) r64[col] = pts64[row * D + col];
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
                    const double *q64 = pts64 + (ci.row0 + perm[ci.row0 + j]) * D;
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
                    te_dist64(r64, pts64 + (ci.row0 + perm[ci.row0 + j]) * D, D, DY, A, m2, m3, jd);
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
using KnnFn = void (*)(const float *, const float *, const ChunkInfo *, const int32_t *, int, int,
                       int, const int32_t *, float *, int32_t *, unsigned long long *);
using CountFn = void (*)(const float *, const float *, const ChunkInfo *, const int32_t *, int,
                         const float *, int64_t, int, int32_t *, uint32_t *, int32_t *, uint32_t,
                         unsigned long long *);

// (DY, DX) layouts with compiled sweeps: TE embeddings d_y, d_x <= 3, the
// symmetric C3 sweep (1+2d) and the bench layout (marginal = first m cols).
#define ENTE_TE_LAYOUTS(X)                                                                  \
    X(1, 1) X(1, 2) X(2, 1) X(2, 2) X(1, 3) X(3, 1) X(2, 3) X(3, 2) X(3, 3) X(4, 4) X(5, 5) \
    X(6, 6) X(7, 7) X(8, 8) X(0, 2) X(1, 4) X(2, 4) X(3, 5) X(4, 6) X(5, 7) X(6, 8) X(7, 9)

template <int DY, int DX>
static KnnFn knn_for_slots(int slots) {
    if (slots <= 5) return knn_pass_kernel<DY, DX, 5>;
    if (slots <= 8) return knn_pass_kernel<DY, DX, 8>;
    if (slots <= 16) return knn_pass_kernel<DY, DX, 16>;
    return nullptr;
}

static KnnFn knn_table(int dy, int dx, int slots) {
#define ENTE_CASE(a, b) \
    if (dy == a && dx == b) return knn_for_slots<a, b>(slots);
    ENTE_TE_LAYOUTS(ENTE_CASE)
#undef ENTE_CASE
    return nullptr;
}

using RescanFn = void (*)(const float *, const float *, const double *, const ChunkInfo *, int,
                          const int32_t *, const float *, const int64_t *, const int32_t *, int,
                          TeLayout, int64_t, double *, int32_t *);

template <int DY, int DX>
static RescanFn rescan_for_k(int k) {
    if (k <= 4) return rescan_kernel<DY, DX, 4>;
    if (k <= 8) return rescan_kernel<DY, DX, 8>;
    return rescan_kernel<DY, DX, 16>;
}

static RescanFn rescan_table(int dy, int dx, int k) {
#define ENTE_CASE(a, b) \
    if (dy == a && dx == b) return rescan_for_k<a, b>(k);
    ENTE_TE_LAYOUTS(ENTE_CASE)
#undef ENTE_CASE
    return nullptr;
}

// Chunks of a few sub-tiles: nearly every reference needs every sub-tile,
// so compaction only adds its overhead; the direct two-per-lane sweep wins.
constexpr int kCompactMinRows = 4096;

static CountFn count_table(int dy, int dx, int max_npad) {
#define ENTE_CASE(a, b) \
    if (dy == a && dx == b) \
        return max_npad >= kCompactMinRows ? count_pass_kernel<a, b> : count_pass_direct_kernel<a, b>;
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
    // with no marginals any layout of the right width serves (the gate is then
    // only a lower bound of the joint distance): prefer a y-past block
    for (int dy = n_marg == 0 ? 1 : 0; dy < dim; ++dy) {
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
    if (k + 1 <= 16 && match_te_layout(dim, masks, n_marg, dy, lay) &&
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
    // kNN order (principal-axis Morton)
    int32_t *permk, *kmap, *inv;
    float *pts32k, *fboxk;
};

static SearchWs layout_ws(Arena &a, const Plan &p, int n_chunks) {
    SearchWs w{};
    w.info = a.take<ChunkInfo>(n_chunks);
    w.ovf_n = a.take<int32_t>(2);
    w.rs_n = w.ovf_n ? w.ovf_n + 1 : nullptr;
    if (p.fast) {
        w.stats = a.take<ColStats>(n_chunks);
        w.tile0 = a.take<int32_t>(2 * n_chunks + 1);
        w.pts32 = a.take<float>((size_t)p.total_prows * p.dp);
        w.fbox = a.take<float>((size_t)(p.total_prows / kSub) * 2 * kGate);
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
        w.permk = a.take<int32_t>(p.total_rows);
        w.kmap = a.take<int32_t>(p.total_rows);
        w.inv = a.take<int32_t>(p.total_rows);
        w.pts32k = a.take<float>((size_t)p.total_prows * p.dp);
        w.fboxk = a.take<float>((size_t)(p.total_prows / kSub) * 2 * 4 * kKnnQ);
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

// prep -> principal axes -> both sort orders -> both fp32 copies with boxes
static int launch_orders(cudaStream_t st, const double *pts64, int dim, const Plan &p,
                         const SearchWs &w, int n_chunks, int32_t *status, int prune,
                         int allow_pca = 1) {
        ENTE_LAUNCH("prep", st,
                    prep_kernel<<<n_chunks, 256, 0, st>>>(pts64, dim, w.info, w.stats, status, 1));
        ENTE_CUDA(cudaGetLastError());
        ENTE_LAUNCH("axes", st,
                    axes_kernel<<<(n_chunks + 127) / 128, 128, 0, st>>>(w.info, n_chunks, dim, w.stats,
                                                                        allow_pca));
        ENTE_CUDA(cudaGetLastError());
        FilterCols sfc = p.fc;
        if (!prune) sfc.nf = 0;  // identity order
        ENTE_LAUNCH("sort", st,
                    (p.max_npad <= kSortSmallN ? sort_kernel<kSortThreadsSmall> : sort_kernel<kSortThreads>)
                    <<<n_chunks, p.max_npad <= kSortSmallN ? kSortThreadsSmall : kSortThreads, 0, st>>>(pts64, dim, w.info, w.stats, sfc,
                                                                   w.ka, w.kb, w.va, w.vb, w.perm));
        ENTE_CUDA(cudaGetLastError());
        ENTE_LAUNCH("sort_pca", st,
                    (p.max_npad <= kSortSmallN ? sort_pca_kernel<kSortThreadsSmall> : sort_pca_kernel<kSortThreads>)
                    <<<n_chunks, p.max_npad <= kSortSmallN ? kSortThreadsSmall : kSortThreads, 0, st>>>(pts64, dim, w.info, w.stats,
                                                                       w.ka, w.kb, w.va, w.vb,
                                                                       w.perm, w.permk));
        ENTE_CUDA(cudaGetLastError());
        dim3 ggrid((unsigned)(p.max_npad / kTJ), (unsigned)std::min(n_chunks, 65535));
        ENTE_LAUNCH("gather", st,
                    gather_kernel<<<ggrid, kTJ, 0, st>>>(pts64, dim, w.info, n_chunks, w.stats,
                                                         w.perm, p.dp, p.fc, w.pts32, w.fbox,
                                                         w.inv));
        ENTE_CUDA(cudaGetLastError());
        ENTE_LAUNCH("gather_knn", st,
                    gather_knn_kernel<<<ggrid, kTJ, 0, st>>>(pts64, dim, w.info, n_chunks, w.stats,
                                                             w.permk, w.inv, p.dp, w.pts32k,
                                                             w.fboxk, w.kmap));
        ENTE_CUDA(cudaGetLastError());
    return ENTE_OK;
}

// host chunk table + status (K_TOO_LARGE) + per-chunk first sweep tile
static int upload_chunks(cudaStream_t st, const ente_chunk *chunks, int n_chunks, int k,
                         const Plan &p, const SearchWs &w, int32_t *status,
                         std::vector<int32_t> &htile0, int32_t &ntiles, int split_index = 0,
                         int split_count = 1) {
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
    if (k + 1 <= 16) {
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
        ENTE_CUDA(cudaMemcpyAsync(w.tile0, htile0.data(), sizeof(int32_t) * (2 * n_chunks + 1),
                                  cudaMemcpyHostToDevice, st));
        const unsigned nt = (unsigned)ntiles;
        ENTE_LAUNCH("knn_pass", st,
                    knn_table(p.dy, p.dx, p.slots)<<<nt, 32, 0, st>>>(w.pts32k, w.fboxk, w.info,
                                                                     w.tile0, n_chunks, k, prune, w.kmap, w.t32,
                                                                     w.L, work));
        ENTE_CUDA(cudaGetLastError());
        uint32_t fmask = 8u;
        for (int o = 0; o < p.lay.nout; ++o) fmask |= 1u << p.lay.slot[o];
        ENTE_LAUNCH("count_pass", st,
                    count_table(p.dy, p.dx, p.max_npad)<<<nt, 32, 0, st>>>(w.pts32, w.fbox, w.info, w.tile0, n_chunks,
                                                               w.t32, ws_rows, prune, w.cnt3, w.ev,
                                                               w.ev_n, fmask, work + 1));
        ENTE_CUDA(cudaGetLastError());
        ENTE_LAUNCH("resolve", st,
                    resolve_kernel<<<nt, kWarpRefs, 0, st>>>(pts64, dim, w.info, w.tile0, n_chunks, k, p.lay,
                                                       w.perm, w.L, w.cnt3, w.ev, w.ev_n, ws_rows,
                                                       total_rows, out_eps, out_counts, w.ovf,
                                                       w.ovf_n, w.rs, w.rs_n));
        ENTE_CUDA(cudaGetLastError());
        {
            const unsigned rgrid = (unsigned)(num_sms() * 8);
            ENTE_LAUNCH("rescan", st,
                        rescan_table(p.dy, p.dx, k)<<<rgrid, kRescanWarps * 32, 0, st>>>(
                            w.pts32, w.fbox, pts64, w.info, n_chunks, w.perm, w.t32, w.rs, w.rs_n,
                            k, p.lay, total_rows, out_eps, out_counts));
        }
        ENTE_CUDA(cudaGetLastError());
        dispatch_exact(k, st, pts64, dim, w.info, n_chunks, status, w.ovf, w.ovf_n, 0, masks,
                       total_rows, out_eps, out_counts);
        ENTE_CUDA(cudaGetLastError());
    } else if (!p.fast && split_index == 0) {  // (a split search: part 0 does it all)
        ENTE_LAUNCH("prep", st,
                    prep_kernel<<<n_chunks, 256, 0, st>>>(pts64, dim, w.info, nullptr, status, 0));
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

// Evaluated (reference, candidate) pairs (whole sub-tiles x reference groups) of the two sweeps on the
// current device since the last call (synchronises the device): the pruned
// work actually done.
extern "C" void ente_search_work(unsigned long long *knn_pairs, unsigned long long *count_pairs) {
    unsigned long long h[2] = {0, 0};
    unsigned long long *d = device_work();
    if (d && cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess)
        cudaMemset(d, 0, sizeof(h));
    *knn_pairs = h[0] * (unsigned long long)(kSub * kWarpRefs);
    *count_pairs = h[1] * (unsigned long long)(kSub * kWarpRefs);
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
                    prep_kernel<<<n_chunks, 256, 0, st>>>(pts64, dim, w.info, nullptr, status, 0));
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
