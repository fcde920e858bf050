// Sweep instantiations, layout group B: wide C3 / bench layouts and the remaining d_y, d_x <= 5 combinations
#include "sweeps.cuh"

namespace ente {

bool sweep_set_b(int dy, int dx, SweepSet &out) {
#define ENTE_CASE(a, b)                  \
    if (dy == a && dx == b) {            \
        out = make_sweep_set<a, b>();    \
        return true;                     \
    }
    ENTE_CASE(6, 6) ENTE_CASE(7, 7) ENTE_CASE(8, 8) ENTE_CASE(0, 2) ENTE_CASE(4, 6) ENTE_CASE(5, 7) ENTE_CASE(6, 8) ENTE_CASE(7, 9) ENTE_CASE(4, 1) ENTE_CASE(4, 2) ENTE_CASE(4, 3) ENTE_CASE(3, 4) ENTE_CASE(1, 5) ENTE_CASE(5, 1) ENTE_CASE(2, 5) ENTE_CASE(5, 2) ENTE_CASE(5, 3) ENTE_CASE(4, 5) ENTE_CASE(5, 4)
#undef ENTE_CASE
    return false;
}

}  // namespace ente
