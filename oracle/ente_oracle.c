/*
 * ente_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker and the CPU
 * baseline of bench.py).  Nothing in paper_1401_4068_b200/ links or calls it.
 *
 * Plain-C restatement of the reference neighbour engine
 * (/root/reference/pkg/src/ente/engine.py):
 *
 *   oracle_stable_order   <- _prepared            engine.py:163-167
 *                            (np.argsort(key0, kind="stable"))
 *   oracle_kth_sweep      <- _kth_sweep           engine.py:70-123
 *   oracle_count_sweep    <- _count_sweep         engine.py:126-160
 *                            on the projection chunk of _search_one
 *                            engine.py:191-200 (column list instead of copy)
 *   oracle_kth_brute /    <- the O(n^2) oracles of pkg/tests/test_engine.py:29-52
 *   oracle_count_brute
 *
 * Arithmetic is IEEE fp64 with no contraction (compile with -ffp-contract=off),
 * matching numba's @njit without fastmath.  The sweep is parallel over points
 * with OpenMP; each point writes only its own slot, so the result does not
 * depend on the thread count (engine.py:12-15).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    double key;
    int64_t idx;
} keyed_t;

static int keyed_cmp(const void *a, const void *b) {
    const keyed_t *x = (const keyed_t *)a, *y = (const keyed_t *)b;
    if (x->key < y->key) return -1;
    if (x->key > y->key) return 1;
    /* equal keys keep input order: identical to a stable argsort */
    return (x->idx > y->idx) - (x->idx < y->idx);
}

/* order[p] = index of the p-th point by (column col0, input position). */
int oracle_stable_order(const double *pts, int64_t n, int dim, int col0, int64_t *order,
                        double *key_sorted) {
    keyed_t *buf = (keyed_t *)malloc(sizeof(keyed_t) * (size_t)n);
    if (!buf) return -1;
    for (int64_t i = 0; i < n; ++i) {
        buf[i].key = pts[i * dim + col0];
        buf[i].idx = i;
    }
    qsort(buf, (size_t)n, sizeof(keyed_t), keyed_cmp);
    for (int64_t p = 0; p < n; ++p) {
        order[p] = buf[p].idx;
        key_sorted[p] = buf[p].key;
    }
    free(buf);
    return 0;
}

int oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* k-th nearest neighbour max-norm distance of every point (self excluded). */
int oracle_kth_sweep(const double *pts, int64_t n, int dim, int k, double *eps) {
    if (k < 1 || k > n - 1 || k > 64) return -1;
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    double *key = (double *)malloc(sizeof(double) * (size_t)n);
    if (!order || !key) return -2;
    oracle_stable_order(pts, n, dim, 0, order, key);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t p = 0; p < n; ++p) {
        const int64_t i = order[p];
        const double *ref = pts + i * dim;
        double best[64];
        int have = 0;
        double bound = INFINITY;
        int64_t lo = p - 1, hi = p + 1;
        while (lo >= 0 || hi < n) {
            double gap_lo = lo >= 0 ? key[p] - key[lo] : INFINITY;
            double gap_hi = hi < n ? key[hi] - key[p] : INFINITY;
            if (have == k && gap_lo >= bound && gap_hi >= bound) break;
            int64_t j;
            if (gap_lo <= gap_hi) j = order[lo--];
            else j = order[hi++];
            const double *q = pts + j * dim;
            /* last coordinate first, abandon once the bound is reached */
            double d = 0.0;
            int rejected = 0;
            for (int c = dim - 1; c >= 0; --c) {
                double ad = fabs(ref[c] - q[c]);
                if (ad > d) {
                    d = ad;
                    if (have == k && d >= bound) {
                        rejected = 1;
                        break;
                    }
                }
            }
            if (rejected) continue;
            if (have < k) {
                int s = have++;
                while (s > 0 && best[s - 1] > d) {
                    best[s] = best[s - 1];
                    --s;
                }
                best[s] = d;
                if (have == k) bound = best[k - 1];
            } else if (d < bound) {
                int s = k - 1;
                while (s > 0 && best[s - 1] > d) {
                    best[s] = best[s - 1];
                    --s;
                }
                best[s] = d;
                bound = best[k - 1];
            }
        }
        eps[i] = best[k - 1];
    }
    free(order);
    free(key);
    return 0;
}

/* Strict within-radius counts in the projection onto cols[0..ncols).
 * The projection's first column is the sweep key (engine.py:198 builds the
 * projected Chunk, whose column 0 is cols[0]). */
int oracle_count_sweep(const double *pts, int64_t n, int dim, const int32_t *cols, int ncols,
                       const double *radii, int64_t *counts) {
    if (ncols < 1) return -1;
    for (int c = 0; c < ncols; ++c)
        if (cols[c] < 0 || cols[c] >= dim) return -1;
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    double *key = (double *)malloc(sizeof(double) * (size_t)n);
    if (!order || !key) return -2;
    oracle_stable_order(pts, n, dim, cols[0], order, key);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t p = 0; p < n; ++p) {
        const int64_t i = order[p];
        const double *ref = pts + i * dim;
        const double r = radii[i];
        int64_t total = 0;
        for (int dir = -1; dir <= 1; dir += 2) {
            for (int64_t q = p + dir; q >= 0 && q < n; q += dir) {
                double gap = dir < 0 ? key[p] - key[q] : key[q] - key[p];
                if (!(gap < r)) break;
                const double *o = pts + order[q] * dim;
                int inside = 1;
                for (int c = ncols - 1; c >= 1; --c) {
                    if (fabs(ref[cols[c]] - o[cols[c]]) >= r) {
                        inside = 0;
                        break;
                    }
                }
                total += inside;
            }
        }
        counts[i] = total;
    }
    free(order);
    free(key);
    return 0;
}

/* Independent O(n^2) statements (pkg/tests/test_engine.py:29-52). */
static double maxnorm(const double *a, const double *b, const int32_t *cols, int ncols) {
    double d = 0.0;
    for (int c = 0; c < ncols; ++c) {
        double ad = fabs(a[cols[c]] - b[cols[c]]);
        if (ad > d) d = ad;
    }
    return d;
}

static int cmp_double(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

int oracle_kth_brute(const double *pts, int64_t n, int dim, int k, double *eps) {
    if (k < 1 || k > n - 1) return -1;
    int32_t *cols = (int32_t *)malloc(sizeof(int32_t) * (size_t)dim);
    for (int c = 0; c < dim; ++c) cols[c] = c;
#pragma omp parallel
    {
        double *d = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < n; ++i) {
            int64_t m = 0;
            for (int64_t j = 0; j < n; ++j)
                if (j != i) d[m++] = maxnorm(pts + i * dim, pts + j * dim, cols, dim);
            qsort(d, (size_t)m, sizeof(double), cmp_double);
            eps[i] = d[k - 1];
        }
        free(d);
    }
    free(cols);
    return 0;
}

int oracle_count_brute(const double *pts, int64_t n, int dim, const int32_t *cols, int ncols,
                       const double *radii, int64_t *counts) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < n; ++i) {
        int64_t t = 0;
        for (int64_t j = 0; j < n; ++j)
            if (j != i && maxnorm(pts + i * dim, pts + j * dim, cols, ncols) < radii[i]) ++t;
        counts[i] = t;
    }
    return 0;
}
