// Tie-breaking jitter replica + degenerate / finiteness checks.
//
// Replaces ente.ksg._jittered_joint (/root/reference/pkg/src/ente/ksg.py:52-59)
// and the checks of estimate_te_batch (ksg.py:80-81) / Chunk (engine.py:57-58).
// numpy arithmetic is reproduced exactly:
//   std   : column mean = sequential row-order sum / M; squared deviations
//           summed sequentially / M; sqrt (numpy _var/_std over axis 0)
//   U(-1,1): -1.0 + 2.0 * ((raw >> 11) * 2^-53), raw = PCG64 XSL-RR output
//           of the state AFTER each LCG step, elements in C order
//   update: x + (u * (amplitude * std)), two roundings, no FMA
#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"
#include "profile.cuh"

namespace ente {

struct U128 {
    uint64_t hi, lo;
};

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
    return r;
}

__device__ __forceinline__ U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}

// PCG_DEFAULT_MULTIPLIER_128 (numpy's PCG64)
__device__ __constant__ U128 kPcgMult = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};

__device__ __forceinline__ uint64_t pcg_output(U128 s) {
    const uint64_t x = s.hi ^ s.lo;
    const unsigned rot = (unsigned)(s.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

// state after `delta` LCG steps
__device__ U128 pcg_advance(U128 state, U128 inc, uint64_t delta) {
    U128 acc_mult = {0ull, 1ull}, acc_plus = {0ull, 0ull};
    U128 cur_mult = kPcgMult, cur_plus = inc;
    while (delta) {
        if (delta & 1ull) {
            acc_mult = mul128(acc_mult, cur_mult);
            acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
        }
        cur_plus = mul128(add128(cur_mult, U128{0ull, 1ull}), cur_plus);
        cur_mult = mul128(cur_mult, cur_mult);
        delta >>= 1;
    }
    return add128(mul128(acc_mult, state), acc_plus);
}

struct JitChunk {
    int64_t row0;
    int32_t n;
    int32_t pad_;
    U128 state, inc;
};

// One warp per chunk: numpy's sequential axis-0 sums, one lane per column.
// Blocks of 32 rows are loaded coalesced (lane l takes elements l, l + 32,
// ... of the block) into shared memory, the next block's loads overlapping
// this block's dependent fp64 additions; the column lanes then add the
// block's rows in row order, exactly as numpy does.
template <int DM>
__global__ void __launch_bounds__(32) jitter_std_kernel(const double *__restrict__ pts, int dim,
                                                        const JitChunk *__restrict__ ch,
                                                        double amplitude,
                                                        double *__restrict__ half_width) {
    __shared__ double buf[32 * DM];
    const JitChunk c = ch[blockIdx.x];
    const int lane = threadIdx.x;
    const double *p = pts + c.row0 * dim;
    const int64_t total = (int64_t)c.n * dim;
    const int per = 32 * dim;  // elements per 32-row block
    const int nblk = (c.n + 31) / 32;
    double reg[DM];
    auto load = [&](int b) {
        const int64_t e0 = (int64_t)b * per + lane;
#pragma unroll
        for (int i = 0; i < DM; ++i) {
            const int64_t e = e0 + 32 * i;
            reg[i] = (i < dim && e < total) ? p[e] : 0.0;
        }
    };
    auto stash = [&]() {
        __syncwarp();
#pragma unroll
        for (int i = 0; i < DM; ++i)
            if (i < dim) buf[32 * i + lane] = reg[i];
        __syncwarp();
    };
    // pass 1: sequential sum -> mean
    double sum = 0.0;
    load(0);
    for (int b = 0; b < nblk; ++b) {
        stash();
        if (b + 1 < nblk) load(b + 1);
        const int rows = min(32, c.n - 32 * b);
        if (lane < dim) {
#pragma unroll 8
            for (int r = 0; r < rows; ++r) sum = __dadd_rn(sum, buf[r * dim + lane]);
        }
    }
    const double mean = __ddiv_rn(sum, (double)c.n);
    // pass 2: sequential sum of squared deviations
    double v = 0.0;
    load(0);
    for (int b = 0; b < nblk; ++b) {
        stash();
        if (b + 1 < nblk) load(b + 1);
        const int rows = min(32, c.n - 32 * b);
        if (lane < dim) {
#pragma unroll 8
            for (int r = 0; r < rows; ++r) {
                const double d = __dsub_rn(buf[r * dim + lane], mean);
                v = __dadd_rn(v, __dmul_rn(d, d));
            }
        }
    }
    if (lane < dim) {
        const double sd = __dsqrt_rn(__ddiv_rn(v, (double)c.n));
        half_width[(int64_t)blockIdx.x * kMaxDim + lane] = __dmul_rn(amplitude, sd);
    }
}

// Element e of a chunk (C order) takes the PCG64 output after step e + 1.
// Threads own elements e0 + t + kJitThreads * i (coalesced); each advances
// its state by kJitThreads steps with one precomputed affine LCG jump.
constexpr int kJitPerThread = 64;
constexpr int kJitUniformMin = 4096;  // smaller batches: the host table is cheap

template <int kJitThreads>
__global__ void __launch_bounds__(kJitThreads) jitter_apply_kernel(double *__restrict__ pts, int dim,
                                                                   const JitChunk *__restrict__ ch,
                                                                   const double *__restrict__ half_width,
                                                                   int n_chunks) {
    for (int ci = blockIdx.y; ci < n_chunks; ci += gridDim.y) {  // grid.y <= 65535
        const JitChunk c = ch[ci];
        const int64_t total = (int64_t)c.n * dim;
        const int64_t base = (int64_t)blockIdx.x * kJitThreads * kJitPerThread;
        if (base >= total) continue;
        int64_t e = base + threadIdx.x;
        // jump of kJitThreads steps: s' = A s + C
        U128 A = {0ull, 1ull}, C = {0ull, 0ull};
        {
            U128 m = kPcgMult, plus = c.inc;
            uint64_t d = kJitThreads;
            while (d) {
                if (d & 1ull) {
                    A = mul128(A, m);
                    C = add128(mul128(C, m), plus);
                }
                plus = mul128(add128(m, U128{0ull, 1ull}), plus);
                m = mul128(m, m);
                d >>= 1;
            }
        }
        U128 s = pcg_advance(c.state, c.inc, (uint64_t)e + 1);  // state after step e + 1
        double *p = pts + c.row0 * dim;
        const double *hw = half_width + (int64_t)ci * kMaxDim;
        int col = (int)(e % dim);            // column of element e, stepped without division
        const int dcol = kJitThreads % dim;
        for (int i = 0; i < kJitPerThread && e < total; ++i, e += kJitThreads) {
            const uint64_t raw = pcg_output(s);
            const double u01 = (double)(raw >> 11) * 0x1p-53;
            const double u = __dadd_rn(-1.0, 2.0 * u01);
            p[e] = __dadd_rn(p[e], __dmul_rn(u, hw[col]));
            s = add128(mul128(A, s), C);
            col += dcol;
            if (col >= dim) col -= dim;
        }
    }
}

// status: non-finite beats degenerate (np.ptp of a NaN column is NaN != 0);
// one pass over the rows, per-thread column extrema (dim <= kMaxDim)
template <int T>
__global__ void __launch_bounds__(T) check_kernel(const double *__restrict__ pts, int dim,
                                                    const JitChunk *__restrict__ ch,
                                                    int32_t *__restrict__ status) {
    constexpr int NW = T / 32;
    __shared__ double wmin[NW][kMaxDim], wmax[NW][kMaxDim];
    __shared__ int bad;
    const JitChunk c = ch[blockIdx.x];
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    const double *p = pts + c.row0 * dim;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int lbad = 0;
    for (int g0 = 0; g0 < dim; g0 += 8) {
        const int gn = dim - g0 < 8 ? dim - g0 : 8;
        double a[8], b[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            a[i] = INFINITY;
            b[i] = -INFINITY;
        }
        for (int r = threadIdx.x; r < c.n; r += blockDim.x) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (i < gn) {
                    const double v = p[(int64_t)r * dim + g0 + i];
                    lbad |= !isfinite(v);
                    a[i] = fmin(a[i], v);
                    b[i] = fmax(b[i], v);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            for (int off = 16; off > 0; off >>= 1) {
                a[i] = fmin(a[i], __shfl_xor_sync(0xffffffffu, a[i], off));
                b[i] = fmax(b[i], __shfl_xor_sync(0xffffffffu, b[i], off));
            }
            if (lane == 0 && i < gn) {
                wmin[warp][g0 + i] = a[i];
                wmax[warp][g0 + i] = b[i];
            }
        }
    }
    if (lbad) bad = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
        int st = ENTE_CHUNK_OK;
        if (bad) {
            st = ENTE_CHUNK_NONFINITE;
        } else {
            double ptp_max = 0.0;
            for (int q = 0; q < dim; ++q) {
                double a = wmin[0][q], b = wmax[0][q];
                for (int w = 1; w < NW; ++w) {
                    a = fmin(a, wmin[w][q]);
                    b = fmax(b, wmax[w][q]);
                }
                ptp_max = fmax(ptp_max, b - a);
            }
            if (ptp_max == 0.0) st = ENTE_CHUNK_DEGENERATE;
        }
        if (status[blockIdx.x] == ENTE_CHUNK_OK) status[blockIdx.x] = st;
    }
}

struct JitWs {
    JitChunk *ch;
    double *hw;
    uint64_t *raw;  // PCG64 states as given (uniform batches)
};

static JitWs jit_layout(Arena &a, int n_chunks) {
    JitWs w;
    w.ch = a.take<JitChunk>(n_chunks);
    w.hw = a.take<double>((size_t)n_chunks * kMaxDim);
    w.raw = a.take<uint64_t>((size_t)n_chunks * 4);
    return w;
}

// uniform batches (chunk c = rows [row0 + c*n, +n)): the chunk table is built
// on the device from the PCG64 states copied as they are -- from pinned
// memory that copy does not hold the host, unlike a pageable multi-MB table
__global__ void __launch_bounds__(256) jit_uniform_kernel(JitChunk *__restrict__ ch,
                                                          const uint64_t *__restrict__ raw, int n_chunks,
                                                          int64_t row0, int n, int have_states) {
    for (int c = blockIdx.x * 256 + threadIdx.x; c < n_chunks; c += gridDim.x * 256) {
        JitChunk j{};
        j.row0 = row0 + (int64_t)c * n;
        j.n = n;
        if (have_states) {
            j.state = {raw[4 * c + 0], raw[4 * c + 1]};
            j.inc = {raw[4 * c + 2], raw[4 * c + 3]};
        }
        ch[c] = j;
    }
}

}  // namespace ente

using namespace ente;

extern "C" size_t ente_jitter_workspace_size(int n_chunks, int dim) {
    (void)dim;
    Arena a(nullptr, 0);
    jit_layout(a, n_chunks);
    return a.used + 256;
}

extern "C" int ente_jitter(double *pts64, int dim, const ente_chunk *chunks, int n_chunks,
                           const uint64_t *pcg_state, double amplitude, int32_t *status,
                           void *workspace, size_t ws_bytes, void *stream) {
    if (n_chunks == 0) return ENTE_OK;
    if (dim < 1 || dim > kMaxDim || n_chunks < 0 || !chunks || !pts64 || !status) {
        set_error("ente_jitter: bad arguments (dim=%d, n_chunks=%d)", dim, n_chunks);
        return ENTE_ERR_ARG;
    }
    if (amplitude > 0 && !pcg_state) {
        set_error("ente_jitter: PCG64 states required when amplitude > 0");
        return ENTE_ERR_ARG;
    }
    Arena a(workspace, ws_bytes);
    JitWs w = jit_layout(a, n_chunks);
    if (!a.ok() || !w.ch) {
        set_error("ente_jitter: workspace of %zu bytes too small (need %zu)", ws_bytes, a.used);
        return ENTE_ERR_WORKSPACE;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    bool uniform = n_chunks >= kJitUniformMin;
    for (int c = 1; c < n_chunks && uniform; ++c)
        uniform = chunks[c].n == chunks[0].n && chunks[c].row0 == chunks[0].row0 + (int64_t)c * chunks[0].n;
    if (uniform && chunks[0].n < 1) uniform = false;
    std::vector<JitChunk> h(uniform ? 0 : n_chunks);
    int max_n = uniform ? chunks[0].n : 0;
    if (uniform) {
        if (pcg_state)
            ENTE_CUDA(cudaMemcpyAsync(w.raw, pcg_state, sizeof(uint64_t) * 4 * (size_t)n_chunks,
                                      cudaMemcpyHostToDevice, st));
        const unsigned blocks = (unsigned)std::min(1024, (n_chunks + 255) / 256);
        ENTE_LAUNCH("jitter_table", st,
                    jit_uniform_kernel<<<blocks, 256, 0, st>>>(w.ch, w.raw, n_chunks, chunks[0].row0,
                                                               chunks[0].n, pcg_state ? 1 : 0));
        ENTE_CUDA(cudaGetLastError());
    }
    for (int c = 0; c < n_chunks && !uniform; ++c) {
        if (chunks[c].n < 1) {
            set_error("ente_jitter: chunk %d has n=%d", c, chunks[c].n);
            return ENTE_ERR_ARG;
        }
        h[c].row0 = chunks[c].row0;
        h[c].n = chunks[c].n;
        if (pcg_state) {
            h[c].state = {pcg_state[4 * c + 0], pcg_state[4 * c + 1]};
            h[c].inc = {pcg_state[4 * c + 2], pcg_state[4 * c + 3]};
        }
        max_n = max_n > chunks[c].n ? max_n : chunks[c].n;
    }
    if (!uniform)
        ENTE_CUDA(cudaMemcpyAsync(w.ch, h.data(), sizeof(JitChunk) * n_chunks, cudaMemcpyHostToDevice, st));
    if (amplitude > 0) {
        if (dim <= 8)
            ENTE_LAUNCH("jitter_std", st,
                        jitter_std_kernel<8><<<n_chunks, 32, 0, st>>>(pts64, dim, w.ch, amplitude, w.hw));
        else
            ENTE_LAUNCH("jitter_std", st,
                        jitter_std_kernel<kMaxDim><<<n_chunks, 32, 0, st>>>(pts64, dim, w.ch, amplitude, w.hw));
        ENTE_CUDA(cudaGetLastError());
        // small chunks: 64 threads, so the per-thread jump-ahead set-up is
        // amortised over more elements
        const int T = (int64_t)max_n * dim <= 64 * kJitPerThread ? 64 : 256;
        const int64_t per_block = (int64_t)T * kJitPerThread;
        const int64_t gx = ((int64_t)max_n * dim + per_block - 1) / per_block;
        dim3 grid((unsigned)gx, (unsigned)(n_chunks < 65535 ? n_chunks : 65535));
        if (T == 64)
            ENTE_LAUNCH("jitter_apply", st,
                        jitter_apply_kernel<64><<<grid, 64, 0, st>>>(pts64, dim, w.ch, w.hw, n_chunks));
        else
            ENTE_LAUNCH("jitter_apply", st,
                        jitter_apply_kernel<256><<<grid, 256, 0, st>>>(pts64, dim, w.ch, w.hw, n_chunks));
        ENTE_CUDA(cudaGetLastError());
    }
    if (max_n <= 2048)  // small chunks: 64-thread CTAs, many per SM
        ENTE_LAUNCH("check", st, check_kernel<64><<<n_chunks, 64, 0, st>>>(pts64, dim, w.ch, status));
    else
        ENTE_LAUNCH("check", st, check_kernel<256><<<n_chunks, 256, 0, st>>>(pts64, dim, w.ch, status));
    ENTE_CUDA(cudaGetLastError());
    return ENTE_OK;
}
