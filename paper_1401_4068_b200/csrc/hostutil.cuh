// Host-side helpers of the C ABI (no device code).
#pragma once

#include <stdint.h>

#include <algorithm>
#include <thread>
#include <vector>

namespace ente {

// f(lo, hi) over [0, n) split across the host's hardware threads (one range
// per thread, at least `grain` items each)
template <class F>
void parallel_for(int64_t n, int64_t grain, F &&f) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t nt = std::min<int64_t>(hw, (n + grain - 1) / grain);
    if (nt <= 1) {
        f(0, n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t per = (n + nt - 1) / nt;
    for (int64_t t = 0; t < nt; ++t) {
        const int64_t lo = t * per, hi = std::min(n, lo + per);
        if (lo < hi) th.emplace_back([&f, lo, hi] { f(lo, hi); });
    }
    for (auto &t : th) t.join();
}

}  // namespace ente
