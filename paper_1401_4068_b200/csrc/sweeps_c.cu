// Sweep instantiations, layout group C: the remaining d_y, d_x <= 5 combinations
#include "sweeps.cuh"

namespace ente {

bool sweep_set_c(int dy, int dx, SweepSet &out) {
#define ENTE_CASE(a, b)                  \
    if (dy == a && dx == b) {            \
        out = make_sweep_set<a, b>();    \
        return true;                     \
    }
    ENTE_CASE(4, 1) ENTE_CASE(4, 2) ENTE_CASE(4, 3) ENTE_CASE(4, 13) ENTE_CASE(3, 4) ENTE_CASE(1, 5) ENTE_CASE(5, 1) ENTE_CASE(2, 5) ENTE_CASE(5, 2) ENTE_CASE(5, 3) ENTE_CASE(4, 5) ENTE_CASE(5, 4)
#undef ENTE_CASE
    return false;
}

}  // namespace ente
