/*
 * ente_b200.h -- C ABI of the B200-native ensemble-TE hot path.
 *
 * The reference (`ente`, /root/reference/pkg/src/ente) is pure Python with no
 * FFI; its boundary is the Python functions listed beside each entry point.
 * These entry points are what a ctypes binding of that boundary calls (see
 * INTEGRATION.md).  Conventions:
 *
 *   - every array argument marked [dev] is a DEVICE pointer owned by the
 *     caller; [host] arrays are read before the call returns;
 *   - every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and does not synchronise unless stated;
 *   - scratch memory comes from the caller through (workspace, ws_bytes),
 *     sized by the matching *_workspace_size() call;
 *   - the return value is ENTE_OK or a negative ente_status; the message of
 *     the last failure on the calling thread is ente_last_error();
 *   - per-chunk outcomes are reported in status[] (ente_chunk_status) and are
 *     mapped by the host onto the reference exception types
 *     (exceptions.py: ShapeMismatch, KTooLarge, DegenerateData).
 *
 * Point matrices are row-major [rows x dim] fp64 exactly as numpy lays out
 * a C-contiguous `Chunk.points` (engine.py:53-59); chunk c owns rows
 * [row0, row0 + n).
 */
#ifndef ENTE_B200_H
#define ENTE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ENTE_OK = 0,
    ENTE_ERR_ARG = -1,      /* invalid argument (shape, k, dim, ...) */
    ENTE_ERR_CUDA = -2,     /* a CUDA runtime call failed */
    ENTE_ERR_WORKSPACE = -3 /* workspace smaller than *_workspace_size() */
} ente_status;

typedef enum {
    ENTE_CHUNK_OK = 0,
    ENTE_CHUNK_K_TOO_LARGE = 1, /* KTooLarge: k not in [1, n-1] (engine.py:173-174) */
    ENTE_CHUNK_NONFINITE = 2,   /* ShapeMismatch: non-finite values (engine.py:57-58) */
    ENTE_CHUNK_DEGENERATE = 3   /* DegenerateData: ptp == 0 in every column (ksg.py:80-81) */
} ente_chunk_status;

/* One search problem: rows [row0, row0 + n) of the batch point matrix. */
typedef struct {
    int64_t row0;
    int32_t n;
    int32_t reserved;
} ente_chunk;

/* Library version string and the CUDA arch it was built for. */
const char *ente_version(void);
/* Message of the last failing call on this thread ("" if none). */
const char *ente_last_error(void);

/* ---------------------------------------------------------------------------
 * ente_search -- exact k-th nearest-neighbour max-norm distances and strict
 * marginal radius counts for a batch of chunks sharing `dim`.
 *
 * Replaces: ente.engine.batch_search          engine.py:203-216
 *           (knn_kth_distances engine.py:170-176, radius_counts 179-188,
 *            _search_one 191-200)
 *
 *   pts64        [dev]  [total_rows x dim] fp64, row-major
 *   chunks       [host] n_chunks descriptors
 *   marg_masks   [host] n_marg column bitmasks (bit c = column c), 1..8
 *                       masks, dim <= 32; a marginal is the max-norm over
 *                       its columns (engine.py:194-199)
 *   k                   neighbour order, 1 <= k <= n-1 for every chunk
 *   out_eps      [dev]  [total_rows] fp64 kth_distance, bit-identical to the
 *                       reference's fp64 sweep
 *   out_counts   [dev]  [n_marg x total_rows] int32 strict counts
 *   status       [dev]  [n_chunks] int32 ente_chunk_status
 *
 * Chunks with status != OK have undefined outputs.
 * ------------------------------------------------------------------------- */
size_t ente_search_workspace_size(const ente_chunk *chunks, int n_chunks, int dim, int n_marg,
                                  int k);
int ente_search(const double *pts64, int64_t total_rows, int dim, const ente_chunk *chunks,
               int n_chunks, const uint32_t *marg_masks, int n_marg, int k, double *out_eps,
               int32_t *out_counts, int32_t *status, void *workspace, size_t ws_bytes,
               void *stream);

/* ---------------------------------------------------------------------------
 * ente_search_split -- ente_search for part `split_index` of `split_count`:
 * every chunk's references (in the search's own spatial order) are cut into
 * split_count contiguous tile ranges and only this part's references get
 * kth_distance / counts written; all other output rows are left untouched.
 *
 * The multi-GPU path for fewer chunks than GPUs: every rank
 * runs the same chunks with its own split_index into zeroed outputs, and
 * one sum all-reduce (exact: x + 0 = x) assembles the full result.  The
 * parts are deterministic, disjoint and cover every row; both sweeps stay in
 * one spatial order so each part is self-contained.
 * ------------------------------------------------------------------------- */
int ente_search_split(const double *pts64, int64_t total_rows, int dim, const ente_chunk *chunks,
                      int n_chunks, const uint32_t *marg_masks, int n_marg, int k,
                      int split_index, int split_count, double *out_eps, int32_t *out_counts,
                      int32_t *status, void *workspace, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * ente_knn_indices -- the k nearest neighbours of every point, in the
 * canonical order ascending (fp64 max-norm distance, chunk-local index).
 *
 * No reference counterpart: ente.engine returns only kth_distance
 * (engine.py:62-67, 170-176; SURVEY 8c "index parity unpinned"), so this
 * order is the contract, pinned by an O(n^2) oracle (oracle/oracle.py
 * knn_indices).  `eps` must be the exact kth distances of the same points
 * (the out_eps of an ente_search call with the same chunks and k).
 *
 *   eps          [dev]  [total_rows] fp64
 *   out_idx      [dev]  [total_rows x k] int32 chunk-local row indices
 *   status       [dev]  [n_chunks] int32 (K_TOO_LARGE / NONFINITE as ente_search)
 *   workspace           sized by ente_search_workspace_size(chunks, n, dim, 0, k)
 * ------------------------------------------------------------------------- */
int ente_knn_indices(const double *pts64, int64_t total_rows, int dim, const ente_chunk *chunks,
                     int n_chunks, int k, const double *eps, int32_t *out_idx, int32_t *status,
                     void *workspace, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * ente_ragwitz_errors -- squared errors of the cross-repetition local
 * predictor for (dim, delay) candidate embeddings (Ragwitz criterion).
 *
 * Replaces: ente.embedding._local_predictor_sq_errors  embedding.py:123-165
 *           (caller: optimize_embedding embedding.py:168-210)
 *
 *   values       [dev]  [reps x n_samp] fp64 ensemble, repetition-major
 *   anchors_r/t  [dev]  [n_anchor] int32 repetition and 0-based index of the
 *                       anchor's most recent embedded sample
 *   k_pred              neighbours averaged, 1..16
 *   out_err      [dev]  [n_anchor] fp64 (prediction - next sample)^2,
 *                       bit-identical to the reference
 * ------------------------------------------------------------------------- */
int ente_ragwitz_errors(const double *values, int reps, int n_samp, int d, int tau,
                        const int32_t *anchors_r, const int32_t *anchors_t, int n_anchor,
                        int k_pred, double *out_err, void *stream);

/* ---------------------------------------------------------------------------
 * ente_radius_counts -- strict counts #{j != i : maxnorm_marg(p_i, p_j) < r_i}
 * for caller-given radii (fp64, exact), one count array per marginal.  Every
 * marginal of <= 17 columns runs the fp32-filter count sweep (the marginal
 * copied into a compiled layout, fp64 settlement of the band); wider ones
 * the fp64 scan.  ente_search uses the same path for marginal lists that are
 * not the TE layout (arbitrary column subsets, engine.py:191-200).
 *
 * Replaces: ente.engine.radius_counts         engine.py:179-188
 *
 *   radii        [dev]  [total_rows] fp64, >= 0 (the host raises ShapeMismatch
 *                       for negative radii, engine.py:185-186)
 *   out_counts   [dev]  [n_marg x total_rows] int32
 *   workspace           ente_radius_counts_workspace_size(chunks, n_chunks, dim)
 * ------------------------------------------------------------------------- */
size_t ente_radius_counts_workspace_size(const ente_chunk *chunks, int n_chunks, int dim);
int ente_radius_counts(const double *pts64, int64_t total_rows, int dim, const ente_chunk *chunks,
                       int n_chunks, const uint32_t *marg_masks, int n_marg, const double *radii,
                       int32_t *out_counts, int32_t *status, void *workspace, size_t ws_bytes,
                       void *stream);

/* ente_search_path -- which engine ente_search runs for this layout:
 * 1 the TE-layout fp32 sweeps, 2 the kNN sweep + generic marginal count
 * sweeps, 0 the fp64 warp-per-point scan (O(n^2), no pruning) -- so hosts can
 * report the slow case instead of taking it silently. */
int ente_search_path(int dim, const uint32_t *marg_masks, int n_marg, int k);

/* ---------------------------------------------------------------------------
 * ente_search_te_shared -- ente_search for a TE batch whose chunks all pool
 * the same target rows (r, t) of one window: chunk c's row r * w + t takes
 * its y columns (y_t, y-past) from repetition perms[chunk_perm[c]][r]
 * (identity for chunk_perm[c] = -1) -- every (u, surrogate) chunk of one
 * analyze_pair window.  Same outputs as ente_search with the three TE
 * marginals; the two y marginals are counted once per original point for the
 * whole batch (shared_y.cuh), the joint / y-past + x-past ones by the sweeps.
 * Falls back to ente_search when the batch does not qualify.
 *
 * Replaces: ente.ksg.estimate_te_batch's batch_search call (ksg.py:83) for the
 *           bundles of analyze_pair (inference.py:147,173)
 *
 *   y0           [dev]  [reps * w x (1 + dy)] fp64 unjittered y columns, row p = r * w + t
 *   chunk_perm   [host] n_chunks surrogate indices (-1 = original data)
 *   perms, inv_perms [dev] [n_perm x reps] int32 permutations and their inverses
 *   margin       >= |D_c(p, q) - D0(p, q)| for every chunk c: 2 x the jitter
 *                half width (amplitude x std) plus rounding (host computes it)
 * ------------------------------------------------------------------------- */
size_t ente_search_te_shared_workspace_size(const ente_chunk *chunks, int n_chunks, int dim, int dy,
                                            int k);
int ente_search_te_shared(const double *pts64, int64_t total_rows, int dim, const ente_chunk *chunks,
                          int n_chunks, int dy, int k, const double *y0, int reps, int w,
                          const int32_t *chunk_perm, const int32_t *perms, const int32_t *inv_perms,
                          double margin, double *out_eps, int32_t *out_counts, int32_t *status,
                          void *workspace, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * ente_jitter -- tie-breaking jitter, in place:
 *   pts += U(-1, 1) * (amplitude * std(pts, axis=0))     per chunk
 * with numpy's exact arithmetic: column std as a sequential row-order sum
 * (mean, squared deviations, /n, sqrt), U(-1,1) = -1 + 2 * ((raw >> 11) * 2^-53)
 * from the chunk's PCG64 stream in C order (element r*dim + c).  Also flags
 * degenerate chunks (ptp == 0 in every column after jitter, ksg.py:80-81)
 * and non-finite values (engine.py:57-58) in status.
 *
 * Replaces: ente.ksg._jittered_joint          ksg.py:52-59
 *
 *   pcg_state    [host] n_chunks x 4 uint64: {state_hi, state_lo, inc_hi,
 *                       inc_lo} = np.random.PCG64(seed).state before any draw
 *   amplitude           jitter amplitude; <= 0 skips the jitter but still
 *                       runs the checks
 * Batches of >= 4096 chunks with one n at row0 = base + c*n copy pcg_state
 * as given (then the chunk table is built on the device): pass pinned memory
 * to keep the host free, and keep it unchanged until the stream has run. 
 * ------------------------------------------------------------------------- */
int ente_jitter(double *pts64, int dim, const ente_chunk *chunks, int n_chunks,
                const uint64_t *pcg_state, double amplitude, int32_t *status, void *workspace,
                size_t ws_bytes, void *stream);
size_t ente_jitter_workspace_size(int n_chunks, int dim);

/* ---------------------------------------------------------------------------
 * ente_pack_te -- build the joint point matrix of every (u, surrogate) chunk
 * of an analyze_pair call directly from the two ensembles:
 *   joint row (r, t') = [ y(phi(r), t') | y-past(phi(r), t'-1) | x-past(r, t'-u) ]
 * rows repetition-outer / time-inner, phi = identity for originals.
 *
 * Replaces: ente.embedding.assemble_pointsets  embedding.py:75-120
 *           ente.inference._permuted_bundle    inference.py:105-117
 *
 *   x, y         [dev]  [reps x n_samples] fp64 source / target ensembles
 *   items        [host] n_items x 2 int32: {u, perm_index (-1 = original)}
 *   perms        [dev]  [n_perm x reps] int32 repetition permutations
 *   out          [dev]  [n_items * reps * w x (1 + dy + dx)] fp64
 * Window t_lo..t_hi is 1-based inclusive; callers validate IndexUnderflow.
 * ------------------------------------------------------------------------- */
int ente_pack_te(const double *x, const double *y, int reps, int n_samples, int dx, int tau_x,
                 int dy, int tau_y, int t_lo, int t_hi, const int32_t *items, int n_items,
                 const int32_t *perms, double *out, void *stream);

/* ente_pack_te_items -- the same gather with a window per item (the delay
 * scan x surrogates x time points of a non-stationary analysis in one
 * launch): items [host] n_items x 3 int32 {u, perm_index, t_lo}, every
 * window w samples wide.  Replaces one assemble_pointsets call per
 * (window, u) (embedding.py:75-120). */
int ente_pack_te_items(const double *x, const double *y, int reps, int n_samples, int dx,
                       int tau_x, int dy, int tau_y, int w, const int32_t *items, int n_items,
                       const int32_t *perms, double *out, void *stream);

/* ---------------------------------------------------------------------------
 * ente_te_reduce -- KSG transfer entropy of each TE-layout chunk:
 *   te = psi(k) + mean(sort(psi(a+1) - psi(b+1) - psi(c+1)))
 * with numpy's exact order: bracket evaluated left to right, ascending sort,
 * numpy pairwise summation (blocks of 8, PW_BLOCKSIZE 128), division by n.
 *
 * Replaces: ente.ksg.te_from_counts           ksg.py:39-49
 *
 *   counts       [dev]  [3 x total_rows] int32: n_ypast, n_y_ypast,
 *                       n_ypast_xpast (the layout ente_search writes for the
 *                       marginal masks of PointSetBundle, embedding.py:50-60)
 *   psi_table    [dev]  psi(m + 1) for m = 0 .. table_len-1 (scipy values)
 *   psi_k               psi(k)
 *   out_te       [dev]  [n_chunks] fp64
 * ------------------------------------------------------------------------- */
size_t ente_te_reduce_workspace_size(const ente_chunk *chunks, int n_chunks);
int ente_te_reduce(const int32_t *counts, int64_t total_rows, const ente_chunk *chunks,
                   int n_chunks, const double *psi_table, int64_t table_len, double psi_k,
                   double *out_te, void *workspace, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Random streams of the surrogate test (host code, no device work).
 *
 * ente_seed_states -- PCG64 state of np.random.default_rng(SeedSequence(e))
 * for n_items entropy word lists e_i = words[offsets[i] .. offsets[i+1])
 * (numpy's uint32 coercion of the seed, e.g. (seed, u, idx + 1) -> 3 words):
 * out [host] n_items x 4 uint64 {state_hi, state_lo, inc_hi, inc_lo}, the
 * pcg_state layout of ente_jitter.
 *
 * Replaces: np.random.default_rng(SeedSequence((seed, u, 0|idx+1)))
 *           inference.py:148,171-172 -> ksg.py:55
 *
 * ente_draw_permutations -- per entropy list i, the permutation of range(reps)
 * drawn by np.random.default_rng(SeedSequence(e_i)).permutation(reps),
 * redrawn from the same generator while strict and some phi(r) == r:
 * out [host] n_perms x reps int32.  strict with reps < 2 is ENTE_ERR_ARG
 * (InvalidPermutation in the reference).
 *
 * Replaces: ente.inference.draw_permutation   inference.py:41-49
 *           ente.inference._surrogate_seed    inference.py:101-102
 * ------------------------------------------------------------------------- */
int ente_seed_states(const uint32_t *words, const int64_t *offsets, int64_t n_items,
                     uint64_t *out);
int ente_draw_permutations(const uint32_t *words, const int64_t *offsets, int64_t n_perms,
                           int reps, int strict, int32_t *out);
/* ente_seed_states_cols -- ente_seed_states for the entropy lists
 * prefix + (cols[0][i], ..., cols[n_cols-1][i]) (each value one uint32 word,
 * 0 <= v < 2^32; n_prefix + n_cols <= 16): the tuple seeds
 * SeedSequence((seed, u, 0|idx+1)) of every jitter stream without building
 * a word list per item.  cols [host] n_cols x n_items int64, row-major. */
int ente_seed_states_cols(const uint32_t *prefix, int n_prefix, const int64_t *cols, int n_cols,
                          int64_t n_items, uint64_t *out);

/* ente_host_gather -- multi-threaded concatenation of n host buffers
 * (srcs[i], bytes[i]) into dst (pinned staging for one H2D copy of a batch).
 * Replaces the per-chunk host copies of batch_search's inputs
 * (engine.py:203-216 loops over chunks one at a time). */
int ente_host_gather(const void *const *srcs, const int64_t *bytes, int64_t n, void *dst);

/* ---------------------------------------------------------------------------
 * Instrumentation (no reference counterpart: the reference only has
 * time.perf_counter around whole calls, bench.py:71-81).
 *
 * ente_launch_count   kernels launched by this library since load
 * ente_profile_enable when on, every launch is bracketed by CUDA events on
 *                     its own stream; ente_profile_read synchronises them and
 *                     returns per-kernel launch counts and total milliseconds
 *                     (names as consecutive NUL-terminated strings); returns
 *                     the number of kernels seen
 * ente_microbench_pce pair-coordinate evaluations per second of the ideal
 *                     FADD2 + FMNMX3 inner loop (the measured fp32 ceiling)
 * ------------------------------------------------------------------------- */
int64_t ente_launch_count(void);
void ente_profile_enable(int on);
void ente_profile_reset(void);
int ente_profile_read(char *names, size_t names_len, int64_t *launches, double *ms,
                      int max_kernels);
int ente_microbench_pce(int iters, int blocks, double *pce_per_s, void *stream);
/* (reference, candidate) pairs the two sweeps evaluated on the current device
 * since the last call: each (reference, 32-row sub-tile) visit counts 32
 * pairs (lane-level work; pruning skips the rest, idle lanes of partial
 * rounds are not counted); synchronises */
void ente_search_work(unsigned long long *knn_pairs, unsigned long long *count_pairs);

#ifdef __cplusplus
}
#endif

#endif /* ENTE_B200_H */
