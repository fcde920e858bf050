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

#include <vector>

#include "common.cuh"
#include "profile.cuh"

namespace ente {

struct PackItem {
    int32_t u;
    int32_t perm;
};

__global__ void __launch_bounds__(256) pack_te_kernel(
    const double *__restrict__ x, const double *__restrict__ y, int reps, int n_samples, int dx,
    int tau_x, int dy, int tau_y, int t_lo, int w, const PackItem *__restrict__ items, int n_items,
    const int32_t *__restrict__ perms, double *__restrict__ out) {
    const int64_t rows = (int64_t)reps * w;
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= rows) return;
    for (int item = blockIdx.y; item < n_items; item += gridDim.y) {  // grid.y <= 65535
    const PackItem it = items[item];
    const int r = (int)(row / w);
    const int tp = t_lo + (int)(row - (int64_t)r * w);  // 1-based t'
    const int ry = it.perm >= 0 ? perms[(int64_t)it.perm * reps + r] : r;
    const int dim = 1 + dy + dx;
    double *o = out + ((int64_t)item * rows + row) * dim;
    const double *yr = y + (int64_t)ry * n_samples;
    const double *xr = x + (int64_t)r * n_samples;
    o[0] = yr[tp - 1];
    for (int j = 0; j < dy; ++j) o[1 + j] = yr[tp - 2 - j * tau_y];
    for (int j = 0; j < dx; ++j) o[1 + dy + j] = xr[tp - 1 - it.u - j * tau_x];
    }
}

}  // namespace ente

using namespace ente;

extern "C" int ente_pack_te(const double *x, const double *y, int reps, int n_samples, int dx,
                            int tau_x, int dy, int tau_y, int t_lo, int t_hi, const int32_t *items,
                            int n_items, const int32_t *perms, double *out, void *stream) {
    if (n_items == 0) return ENTE_OK;
    const int w = t_hi - t_lo + 1;
    if (!x || !y || !out || !items || reps < 1 || n_samples < 1 || dx < 1 || dy < 1 || tau_x < 1 ||
        tau_y < 1 || w < 1 || t_hi > n_samples || n_items < 0 || 1 + dx + dy > kMaxDim) {
        set_error("ente_pack_te: bad arguments");
        return ENTE_ERR_ARG;
    }
    // the earliest sample read must exist (IndexUnderflow is raised by the host)
    int max_u = 0;
    for (int i = 0; i < n_items; ++i) {
        if (items[2 * i + 1] >= 0 && !perms) {
            set_error("ente_pack_te: item %d needs a permutation table", i);
            return ENTE_ERR_ARG;
        }
        max_u = max_u > items[2 * i] ? max_u : items[2 * i];
    }
    if (t_lo - 1 - (dy - 1) * tau_y < 1 || t_lo - max_u - (dx - 1) * tau_x < 1) {
        set_error("ente_pack_te: window start %d underflows the embedding", t_lo);
        return ENTE_ERR_ARG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // items travel as kernel-visible memory via a small device copy
    PackItem *ditems = nullptr;
    ENTE_CUDA(cudaMallocAsync(&ditems, sizeof(PackItem) * n_items, st));
    ENTE_CUDA(cudaMemcpyAsync(ditems, items, sizeof(PackItem) * n_items, cudaMemcpyHostToDevice, st));
    const int64_t rows = (int64_t)reps * w;
    dim3 grid((unsigned)((rows + 255) / 256), (unsigned)(n_items < 65535 ? n_items : 65535));
    ENTE_LAUNCH("pack_te", st,
                pack_te_kernel<<<grid, 256, 0, st>>>(x, y, reps, n_samples, dx, tau_x, dy, tau_y,
                                                     t_lo, w, ditems, n_items, perms, out));
    ENTE_CUDA(cudaGetLastError());
    ENTE_CUDA(cudaFreeAsync(ditems, st));
    return ENTE_OK;
}
