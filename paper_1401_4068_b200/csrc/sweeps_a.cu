// Sweep instantiations, layout group A: d_y, d_x <= 3 and the symmetric 4/5 embeddings
#include "sweeps.cuh"

namespace ente {

bool sweep_set_a(int dy, int dx, SweepSet &out) {
#define ENTE_CASE(a, b)                  \
    if (dy == a && dx == b) {            \
        out = make_sweep_set<a, b>();    \
        return true;                     \
    }
    ENTE_CASE(1, 1) ENTE_CASE(1, 2) ENTE_CASE(2, 1) ENTE_CASE(2, 2) ENTE_CASE(1, 3) ENTE_CASE(3, 1) ENTE_CASE(2, 3) ENTE_CASE(3, 2) ENTE_CASE(3, 3) ENTE_CASE(4, 4) ENTE_CASE(5, 5)
#undef ENTE_CASE
    return false;
}

}  // namespace ente
