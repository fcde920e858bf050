// Chunk packing straight from device-resident ensembles.
//
// Replaces ente.embedding.assemble_pointsets (embedding.py:75-120) and
// ente.inference._permuted_bundle (inference.py:105-117): every (u, surrogate)
// chunk of an analyze_pair call is gathered in one launch.  Row (r, t') of an
// item holds
//     [ y(phi(r), t') | y(phi(r), t'-1-j*tau_y), j < d_y | x(r, t'-u-j*tau_x), j < d_x ]
// with 1-based t' in [t_lo, t_hi], repetition-outer / time-inner, and
// phi = the item's repetition permutation (identity for the original data):
// shuffling the target's repetitions permutes only the y columns.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "profile.cuh"

namespace ente {

struct PackItem {
    int32_t u;
    int32_t perm;
    int32_t t_lo;  // 1-based first sample of the item's window
    int32_t pad_;
};

// One thread per output row gathers it into shared memory; the CTA's rows
// (contiguous in the output) are then written back with coalesced stores.
constexpr int kPackThreads = 256;

__global__ void __launch_bounds__(kPackThreads) pack_te_kernel(
    const double *__restrict__ x, const double *__restrict__ y, int reps, int n_samples, int dx,
    int tau_x, int dy, int tau_y, int w, const PackItem *__restrict__ items, int n_items,
    const int32_t *__restrict__ perms, double *__restrict__ out) {
    extern __shared__ double stage[];  // [kPackThreads * dim]
    const int64_t rows = (int64_t)reps * w;
    const int64_t row0 = (int64_t)blockIdx.x * kPackThreads;
    const int64_t row = row0 + threadIdx.x;
    const bool valid = row < rows;
    const int r = valid ? (int)(row / w) : 0;
    const int dim = 1 + dy + dx;
    const int nrow = (int)(rows - row0 < kPackThreads ? rows - row0 : kPackThreads);
    for (int item = blockIdx.y; item < n_items; item += gridDim.y) {  // grid.y <= 65535
        const PackItem it = items[item];
        if (valid) {
            const int tp = it.t_lo + (int)(row - (int64_t)r * w);  // 1-based t'
            const int ry = it.perm >= 0 ? perms[(int64_t)it.perm * reps + r] : r;
            double *o = stage + threadIdx.x * dim;
            const double *yr = y + (int64_t)ry * n_samples;
            const double *xr = x + (int64_t)r * n_samples;
            o[0] = yr[tp - 1];
            for (int j = 0; j < dy; ++j) o[1 + j] = yr[tp - 2 - j * tau_y];
            for (int j = 0; j < dx; ++j) o[1 + dy + j] = xr[tp - 1 - it.u - j * tau_x];
        }
        __syncthreads();
        double *dst = out + ((int64_t)item * rows + row0) * dim;
        for (int e = threadIdx.x; e < nrow * dim; e += kPackThreads) dst[e] = stage[e];
        __syncthreads();
    }
}

}  // namespace ente

using namespace ente;

// Per-(device, stream) grow-only item table.  Calls on one stream are
// ordered, so a later copy into the table lands after the earlier kernel
// that read it; concurrent streams get separate tables.
static PackItem *item_table(int n, cudaStream_t st) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, std::pair<PackItem *, int>> tabs;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto &t = tabs[{dev, st}];
    if (t.second < n) {
        if (t.first) cudaFree(t.first);  // synchronises: rare (growth only)
        t.first = nullptr;
        t.second = 0;
        const int want = n < 4096 ? 4096 : n + n / 2;
        void *p = nullptr;
        if (cudaMalloc(&p, sizeof(PackItem) * (size_t)want) != cudaSuccess) return nullptr;
        t.first = static_cast<PackItem *>(p);
        t.second = want;
    }
    return t.first;
}

extern "C" int ente_pack_te_items(const double *x, const double *y, int reps, int n_samples,
                                  int dx, int tau_x, int dy, int tau_y, int w,
                                  const int32_t *items, int n_items, const int32_t *perms,
                                  double *out, void *stream) {
    if (n_items == 0) return ENTE_OK;
    if (!x || !y || !out || !items || reps < 1 || n_samples < 1 || dx < 1 || dy < 1 || tau_x < 1 ||
        tau_y < 1 || w < 1 || n_items < 0 || 1 + dx + dy > kMaxDim) {
        set_error("ente_pack_te: bad arguments");
        return ENTE_ERR_ARG;
    }
    std::vector<PackItem> h(n_items);
    for (int i = 0; i < n_items; ++i) {
        const int u = items[3 * i], perm = items[3 * i + 1], t_lo = items[3 * i + 2];
        if (perm >= 0 && !perms) {
            set_error("ente_pack_te: item %d needs a permutation table", i);
            return ENTE_ERR_ARG;
        }
        // every sample read must exist (the host raises IndexUnderflow first)
        if (u < 0 || t_lo - 1 - (dy - 1) * tau_y < 1 || t_lo - u - (dx - 1) * tau_x < 1 ||
            t_lo + w - 1 > n_samples) {
            set_error("ente_pack_te: item %d (u=%d, window start %d) outside the ensemble", i, u,
                      t_lo);
            return ENTE_ERR_ARG;
        }
        h[i] = PackItem{u, perm, t_lo, 0};
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // items travel through a per-device, grow-only device table with a
    // stream-ordered copy (no per-call allocation: stream-ordered
    // allocations are trimmed at every synchronisation, which cost
    // 10-600 ms per call)
    PackItem *ditems = item_table(n_items, st);
    if (!ditems) {
        set_error("ente_pack_te: cannot allocate the item table (%d items)", n_items);
        return ENTE_ERR_CUDA;
    }
    ENTE_CUDA(cudaMemcpyAsync(ditems, h.data(), sizeof(PackItem) * n_items, cudaMemcpyHostToDevice, st));
    const int64_t rows = (int64_t)reps * w;
    dim3 grid((unsigned)((rows + kPackThreads - 1) / kPackThreads),
              (unsigned)(n_items < 65535 ? n_items : 65535));
    const size_t smem = sizeof(double) * kPackThreads * (size_t)(1 + dx + dy);  // <= 64 KB
    static std::once_flag smem_once;
    std::call_once(smem_once, [] {
        cudaFuncSetAttribute(pack_te_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(double) * kPackThreads * kMaxDim));
    });
    ENTE_LAUNCH("pack_te", st,
                pack_te_kernel<<<grid, kPackThreads, smem, st>>>(x, y, reps, n_samples, dx, tau_x, dy,
                                                                 tau_y, w, ditems, n_items, perms, out));
    ENTE_CUDA(cudaGetLastError());
    // (a pageable-source cudaMemcpyAsync has staged h before returning)
    return ENTE_OK;
}

extern "C" int ente_pack_te(const double *x, const double *y, int reps, int n_samples, int dx,
                            int tau_x, int dy, int tau_y, int t_lo, int t_hi, const int32_t *items,
                            int n_items, const int32_t *perms, double *out, void *stream) {
    if (n_items == 0) return ENTE_OK;
    if (!items || n_items < 0 || t_hi < t_lo) {
        set_error("ente_pack_te: bad arguments");
        return ENTE_ERR_ARG;
    }
    std::vector<int32_t> it3(3 * (size_t)n_items);
    for (int i = 0; i < n_items; ++i) {
        it3[3 * i] = items[2 * i];
        it3[3 * i + 1] = items[2 * i + 1];
        it3[3 * i + 2] = t_lo;
    }
    return ente_pack_te_items(x, y, reps, n_samples, dx, tau_x, dy, tau_y, t_hi - t_lo + 1,
                              it3.data(), n_items, perms, out, stream);
}
