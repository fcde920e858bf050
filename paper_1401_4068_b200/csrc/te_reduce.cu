// KSG TE reduction: te = psi(k) + mean(sort(psi(a+1) - psi(b+1) - psi(c+1))).
//
// Replaces ente.ksg.te_from_counts (/root/reference/pkg/src/ente/ksg.py:39-49).
// Bit-exact with the reference: the bracket is evaluated left to right from a
// table of scipy digamma values, sorted ascending (stable LSD radix sort on
// order-preserving 64-bit keys, one CTA per chunk), summed in numpy's
// pairwise order (pairwise_sum: < 8 sequential, <= 128 eight accumulators,
// else split at n/2 - (n/2) % 8) and divided by n.
#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"
#include "profile.cuh"
#include "radix.cuh"

namespace ente {


__device__ __forceinline__ uint64_t f64_key(double v) {
    const uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ double key_f64(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double((long long)b);
}

// numpy's pairwise_sum leaf (n <= 128): < 8 sequential, else eight
// accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail
__device__ double pairwise_leaf(const uint64_t *keys, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res = __dadd_rn(res, key_f64(keys[i]));
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = key_f64(keys[j]);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], key_f64(keys[i + j]));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, key_f64(keys[i]));
    return res;
}

// numpy's pairwise split: n > 128 -> (n2, n - n2), n2 = n/2 - (n/2) % 8
__device__ __forceinline__ int pairwise_split(int n) {
    int n2 = n / 2;
    return n2 - n2 % 8;
}

// Parallel replica of numpy's pairwise sum over the sorted keys: thread 0
// lists the leaves in depth-first order, all threads sum leaves, thread 0
// folds the leaf sums back up the same tree.  `scratch` holds >= 8 n bytes.
__device__ double pairwise_cta(const uint64_t *keys, int n, void *scratch, int *n_leaves) {
    int2 *leaf = reinterpret_cast<int2 *>(scratch);  // (offset, length)
    if (threadIdx.x == 0) {
        int stack_off[40], stack_n[40], sp = 0, nl = 0;
        stack_off[sp] = 0;
        stack_n[sp++] = n;
        while (sp) {
            --sp;
            const int off = stack_off[sp], m = stack_n[sp];
            if (m <= 128) {
                leaf[nl++] = make_int2(off, m);
            } else {
                const int m2 = pairwise_split(m);
                stack_off[sp] = off + m2;  // right pushed first: left pops first
                stack_n[sp++] = m - m2;
                stack_off[sp] = off;
                stack_n[sp++] = m2;
            }
        }
        *n_leaves = nl;
    }
    __syncthreads();
    const int nl = *n_leaves;
    double *val = reinterpret_cast<double *>(leaf + nl);
    for (int l = threadIdx.x; l < nl; l += blockDim.x) {
        const int2 d = leaf[l];
        val[l] = pairwise_leaf(keys + d.x, d.y);
    }
    __syncthreads();
    double res = 0.0;
    if (threadIdx.x == 0) {
        // post-order fold: the leaves come in DFS order, so a stack of
        // (pending right subtree size, left value) replays the recursion
        int st_n[40], st_state[40], sp = 0, next = 0;
        double st_left[40];
        double cur = 0.0;
        st_n[sp] = n;
        st_state[sp++] = 0;
        bool have = false;
        while (sp) {
            const int top = sp - 1;
            const int m = st_n[top];
            if (m <= 128) {  // leaf: its value goes to the parent
                cur = val[next++];
                --sp;
                have = true;
            } else if (st_state[top] == 0) {  // descend left
                st_state[top] = 1;
                st_n[sp] = pairwise_split(m);
                st_state[sp++] = 0;
                have = false;
                continue;
            } else if (st_state[top] == 1) {  // left done: keep it, descend right
                st_left[top] = cur;
                st_state[top] = 2;
                st_n[sp] = m - pairwise_split(m);
                st_state[sp++] = 0;
                have = false;
                continue;
            } else {  // both done
                cur = __dadd_rn(st_left[top], cur);
                --sp;
                have = true;
            }
            (void)have;
        }
        res = cur;
    }
    return res;
}

struct RedChunk {
    int64_t row0;
    int32_t n;
    int32_t pad_;
};

template <int T>
__global__ void __launch_bounds__(T) te_reduce_kernel(
    const int32_t *__restrict__ counts, int64_t total_rows, const RedChunk *__restrict__ chunks,
    const double *__restrict__ psi, int64_t table_len, double psi_k, uint64_t *__restrict__ ka,
    uint64_t *__restrict__ kb, double *__restrict__ out_te, RedChunk uniform) {
    __shared__ SortSmemT<T> sm;
    __shared__ int bad;
    __shared__ int n_leaves;
    // (uniform batches: chunk c at uniform.row0 + c * uniform.n, no table)
    const RedChunk ch = chunks ? chunks[blockIdx.x]
                               : RedChunk{uniform.row0 + (int64_t)blockIdx.x * uniform.n, uniform.n, 0};
    const int n = ch.n;
    constexpr bool SMS = T == kSortThreadsSmall;  // small segments sort in shared memory
    __shared__ uint64_t skey[SMS ? 2 : 1][SMS ? kSortSmallN : 1];
    uint64_t *src = SMS ? skey[0] : ka + ch.row0;
    uint64_t *dst = SMS ? skey[1] : kb + ch.row0;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += T) {
        const int64_t row = ch.row0 + i;
        const int a = counts[row], b = counts[total_rows + row], c = counts[2 * total_rows + row];
        double v = 0.0;
        if (a < 0 || b < 0 || c < 0 || a >= table_len || b >= table_len || c >= table_len) bad = 1;
        else v = __dsub_rn(__dsub_rn(psi[a], psi[b]), psi[c]);
        src[i] = f64_key(v);
    }
    __syncthreads();
    if (bad) {
        if (threadIdx.x == 0) out_te[blockIdx.x] = __longlong_as_double(0x7FF8000000000000ll);
        return;
    }
    // stable sort on the high 32 key bits (sign, exponent, 20 mantissa bits),
    // then every run of equal high halves is finished by an insertion sort on
    // the full key: runs are almost always one value or copies of one value
    // (equal brackets of equal count triples), so this halves the radix passes
    const int parity = cta_radix_sort<T, uint64_t, int>(src, dst, nullptr, nullptr, n, 32, sm, 32);
    uint64_t *sorted = parity ? dst : src;
    for (int i = threadIdx.x; i < n; i += T) {
        const uint32_t h = (uint32_t)(sorted[i] >> 32);
        if ((i > 0 && (uint32_t)(sorted[i - 1] >> 32) == h) || i + 1 >= n ||
            (uint32_t)(sorted[i + 1] >> 32) != h)
            continue;  // not the start of a run of length >= 2
        int e = i + 1;
        while (e < n && (uint32_t)(sorted[e] >> 32) == h) ++e;
        for (int a = i + 1; a < e; ++a) {
            const uint64_t key = sorted[a];
            int b = a - 1;
            while (b >= i && sorted[b] > key) {
                sorted[b + 1] = sorted[b];
                --b;
            }
            sorted[b + 1] = key;
        }
    }
    __syncthreads();
    const double sum = pairwise_cta(sorted, n, parity ? src : dst, &n_leaves);
    if (threadIdx.x == 0) out_te[blockIdx.x] = __dadd_rn(psi_k, __ddiv_rn(sum, (double)n));
}

}  // namespace ente

using namespace ente;

extern "C" size_t ente_te_reduce_workspace_size(const ente_chunk *chunks, int n_chunks) {
    int64_t rows = 0;
    for (int c = 0; c < n_chunks; ++c) rows = rows > chunks[c].row0 + chunks[c].n ? rows : chunks[c].row0 + chunks[c].n;
    Arena a(nullptr, 0);
    a.take<RedChunk>(n_chunks);
    a.take<uint64_t>(rows);
    a.take<uint64_t>(rows);
    return a.used + 256;
}

extern "C" int ente_te_reduce(const int32_t *counts, int64_t total_rows, const ente_chunk *chunks,
                              int n_chunks, const double *psi_table, int64_t table_len,
                              double psi_k, double *out_te, void *workspace, size_t ws_bytes,
                              void *stream) {
    if (n_chunks == 0) return ENTE_OK;
    if (n_chunks < 0 || !chunks || !counts || !psi_table || !out_te || table_len < 1) {
        set_error("ente_te_reduce: bad arguments");
        return ENTE_ERR_ARG;
    }
    int64_t rows = 0;
    int max_n = 0;
    std::vector<RedChunk> h(n_chunks);
    for (int c = 0; c < n_chunks; ++c) {
        if (chunks[c].n < 1 || chunks[c].row0 < 0 || chunks[c].row0 + chunks[c].n > total_rows) {
            set_error("ente_te_reduce: chunk %d outside the count rows", c);
            return ENTE_ERR_ARG;
        }
        h[c].row0 = chunks[c].row0;
        h[c].n = chunks[c].n;
        max_n = max_n > chunks[c].n ? max_n : chunks[c].n;
        rows = rows > chunks[c].row0 + chunks[c].n ? rows : chunks[c].row0 + chunks[c].n;
    }
    Arena a(workspace, ws_bytes);
    RedChunk *dch = a.take<RedChunk>(n_chunks);
    uint64_t *ka = a.take<uint64_t>(rows);
    uint64_t *kb = a.take<uint64_t>(rows);
    if (!a.ok() || !dch) {
        set_error("ente_te_reduce: workspace of %zu bytes too small (need %zu)", ws_bytes, a.used);
        return ENTE_ERR_WORKSPACE;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // uniform batches pass two scalars instead of the table (a pageable copy of
    // a few MB would hold the host until the stream reached it)
    bool uniform = n_chunks > 1;
    for (int c = 1; c < n_chunks && uniform; ++c)
        uniform = h[c].n == h[0].n && h[c].row0 == h[0].row0 + (int64_t)c * h[0].n;
    const RedChunk uni{h[0].row0, h[0].n, 0};
    if (!uniform)
        ENTE_CUDA(cudaMemcpyAsync(dch, h.data(), sizeof(RedChunk) * n_chunks, cudaMemcpyHostToDevice, st));
    ENTE_LAUNCH("te_reduce", st,
                (max_n <= kSortSmallN ? te_reduce_kernel<kSortThreadsSmall> : te_reduce_kernel<kSortThreads>)
                <<<n_chunks, max_n <= kSortSmallN ? kSortThreadsSmall : kSortThreads, 0, st>>>(counts, total_rows,
                                                                  uniform ? nullptr : dch,
                                                                  psi_table, table_len, psi_k, ka,
                                                                  kb, out_te, uni));
    ENTE_CUDA(cudaGetLastError());
    return ENTE_OK;
}
