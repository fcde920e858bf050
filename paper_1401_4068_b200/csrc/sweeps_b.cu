// Sweep instantiations, layout group B: wide C3 / bench layouts
#include "sweeps.cuh"

namespace ente {

bool sweep_set_b(int dy, int dx, SweepSet &out) {
#define ENTE_CASE(a, b)                  \
    if (dy == a && dx == b) {            \
        out = make_sweep_set<a, b>();    \
        return true;                     \
    }
    ENTE_CASE(1, 4) ENTE_CASE(2, 4) ENTE_CASE(3, 5) ENTE_CASE(6, 6) ENTE_CASE(7, 7) ENTE_CASE(8, 8) ENTE_CASE(0, 2) ENTE_CASE(4, 6) ENTE_CASE(5, 7) ENTE_CASE(6, 8) ENTE_CASE(7, 9)
#undef ENTE_CASE
    return false;
}

}  // namespace ente
