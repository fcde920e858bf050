// Ragwitz local-predictor errors: the second kNN loop of the reference.
//
// Replaces ente.embedding._local_predictor_sq_errors
// (/root/reference/pkg/src/ente/embedding.py:123-165).  For every anchor
// (r0, t0) the k_pred nearest embedded points of the OTHER repetitions
// (max norm over the d delay coordinates, fp64) predict the next sample as
// the mean of their next samples; the output is the squared error.
//
// The reference scans candidates r2 ascending, t2 ascending and replaces
// only on strict improvement, inserting after equal distances: its k list is
// the first k candidates in lexicographic (distance, scan position) order,
// and the prediction sums their next samples in that order.  Here one warp
// per anchor: each lane keeps the k smallest (distance, position) pairs of
// its strided share of the scan, then k rounds of lexicographic warp minima
// rebuild the reference's ordered list; lane 0 sums in that order.
#include <cuda_runtime.h>

#include "common.cuh"
#include "profile.cuh"

namespace ente {

constexpr int kRagWarps = 4;
constexpr int kRagMaxK = 16;

template <int KS>
__global__ void __launch_bounds__(kRagWarps * 32) ragwitz_kernel(
    const double *__restrict__ values, int reps, int n_samp, int d, int tau,
    const int32_t *__restrict__ anchors_r, const int32_t *__restrict__ anchors_t, int n_anchor,
    int k_pred, double *__restrict__ out_err) {
    const int lane = threadIdx.x & 31;
    const int a = blockIdx.x * kRagWarps + (threadIdx.x >> 5);
    if (a >= n_anchor) return;
    const int r0 = anchors_r[a], t0 = anchors_t[a];
    const int span_lo = (d - 1) * tau;
    const int n_t = n_samp - 1 - span_lo;  // candidate t2 in [span_lo, n_samp - 2]
    const double *x0 = values + (int64_t)r0 * n_samp;
    double ref[16];
    for (int c = 0; c < d; ++c) ref[c] = x0[t0 - c * tau];
    double kd[KS];
    int64_t kp[KS];  // scan position (r2 * n_t + (t2 - span_lo))
    double kv[KS];
#pragma unroll
    for (int q = 0; q < KS; ++q) {
        kd[q] = INFINITY;
        kp[q] = INT64_MAX;
        kv[q] = 0.0;
    }
    const int64_t total = (int64_t)reps * n_t;
    for (int64_t pos = lane; pos < total; pos += 32) {
        const int r2 = (int)(pos / n_t);
        if (r2 == r0) continue;
        const int t2 = span_lo + (int)(pos - (int64_t)r2 * n_t);
        const double *x2 = values + (int64_t)r2 * n_samp;
        double dist = 0.0;
        for (int c = 0; c < d; ++c) dist = fmax(dist, fabs(__dsub_rn(ref[c], x2[t2 - c * tau])));
        // lexicographic (dist, pos): pos grows within a lane, so "<" on dist
        // alone inserts after equal distances, exactly like the reference
        if (dist < kd[KS - 1]) {
            int p = KS - 1;
            while (p > 0 && kd[p - 1] > dist) {
                kd[p] = kd[p - 1];
                kp[p] = kp[p - 1];
                kv[p] = kv[p - 1];
                --p;
            }
            kd[p] = dist;
            kp[p] = pos;
            kv[p] = x2[t2 + 1];
        }
    }
    double pred = 0.0;
    for (int q = 0; q < k_pred; ++q) {
        double bd = kd[0];
        int64_t bp = kp[0];
        double bv = kv[0];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, bd, off);
            const int64_t op = __shfl_xor_sync(0xffffffffu, bp, off);
            const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
            if (od < bd || (od == bd && op < bp)) {
                bd = od;
                bp = op;
                bv = ov;
            }
        }
        if (kp[0] == bp) {  // positions are unique: the owner pops its head
#pragma unroll
            for (int p = 0; p < KS - 1; ++p) {
                kd[p] = kd[p + 1];
                kp[p] = kp[p + 1];
                kv[p] = kv[p + 1];
            }
            kd[KS - 1] = INFINITY;
            kp[KS - 1] = INT64_MAX;
        }
        pred = __dadd_rn(pred, bv);  // numba: pred += best_v[q], q ascending
    }
    if (lane == 0) {
        pred = __ddiv_rn(pred, (double)k_pred);
        const double diff = __dsub_rn(pred, x0[t0 + 1]);
        out_err[a] = __dmul_rn(diff, diff);
    }
}

}  // namespace ente

using namespace ente;

extern "C" int ente_ragwitz_errors(const double *values, int reps, int n_samp, int d, int tau,
                                   const int32_t *anchors_r, const int32_t *anchors_t,
                                   int n_anchor, int k_pred, double *out_err, void *stream) {
    if (n_anchor == 0) return ENTE_OK;
    if (!values || !anchors_r || !anchors_t || !out_err || reps < 2 || n_samp < 2 || d < 1 ||
        d > 16 || tau < 1 || k_pred < 1 || k_pred > kRagMaxK || n_anchor < 0) {
        set_error("ente_ragwitz_errors: bad arguments (reps=%d, n=%d, d=%d, tau=%d, k=%d)", reps,
                  n_samp, d, tau, k_pred);
        return ENTE_ERR_ARG;
    }
    if ((int64_t)(reps - 1) * (n_samp - 1 - (d - 1) * tau) < k_pred) {
        set_error("ente_ragwitz_errors: fewer than k_pred candidates");
        return ENTE_ERR_ARG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned grid = (unsigned)((n_anchor + kRagWarps - 1) / kRagWarps);
    if (k_pred <= 4) {
        ENTE_LAUNCH("ragwitz", st,
                    ragwitz_kernel<4><<<grid, kRagWarps * 32, 0, st>>>(values, reps, n_samp, d, tau,
                                                                      anchors_r, anchors_t, n_anchor,
                                                                      k_pred, out_err));
    } else if (k_pred <= 8) {
        ENTE_LAUNCH("ragwitz", st,
                    ragwitz_kernel<8><<<grid, kRagWarps * 32, 0, st>>>(values, reps, n_samp, d, tau,
                                                                      anchors_r, anchors_t, n_anchor,
                                                                      k_pred, out_err));
    } else {
        ENTE_LAUNCH("ragwitz", st,
                    ragwitz_kernel<16><<<grid, kRagWarps * 32, 0, st>>>(values, reps, n_samp, d, tau,
                                                                       anchors_r, anchors_t, n_anchor,
                                                                       k_pred, out_err));
    }
    ENTE_CUDA(cudaGetLastError());
    return ENTE_OK;
}
