// Host-side staging helpers of the C ABI (no device code).
#include <string.h>

#include "ente_b200.h"
#include "hostutil.cuh"

namespace ente {
void set_error(const char *fmt, ...);
}

extern "C" int ente_host_gather(const void *const *srcs, const int64_t *bytes, int64_t n, void *dst) {
    if (n < 0 || (n > 0 && (!srcs || !bytes || !dst))) {
        ente::set_error("ente_host_gather: bad arguments");
        return ENTE_ERR_ARG;
    }
    std::vector<int64_t> off((size_t)n + 1, 0);
    for (int64_t i = 0; i < n; ++i) {
        if (bytes[i] < 0) {
            ente::set_error("ente_host_gather: negative size");
            return ENTE_ERR_ARG;
        }
        off[i + 1] = off[i] + bytes[i];
    }
    // split by bytes, not by count: chunks may differ in size
    const int64_t total = off[n];
    const int64_t parts = std::max<int64_t>(1, std::min<int64_t>(64, total >> 22));  // >= 4 MB each
    char *d = static_cast<char *>(dst);
    ente::parallel_for(parts, 1, [&](int64_t lo, int64_t hi) {
        for (int64_t p = lo; p < hi; ++p) {
            const int64_t b0 = total * p / parts, b1 = total * (p + 1) / parts;
            int64_t i = std::upper_bound(off.begin(), off.end(), b0) - off.begin() - 1;
            for (int64_t pos = b0; pos < b1 && i < n; ++i) {
                const int64_t s = std::max(pos, off[i]), e = std::min(b1, off[i + 1]);
                if (e > s) memcpy(d + s, static_cast<const char *>(srcs[i]) + (s - off[i]), (size_t)(e - s));
                pos = e;
            }
        }
    });
    return ENTE_OK;
}
