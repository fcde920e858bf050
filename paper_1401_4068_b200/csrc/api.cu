// C-ABI glue: error reporting and version string.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "profile.cuh"

namespace ente {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

struct KernelStats {
    int64_t launches = 0;
    double ms = 0.0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    cudaEvent_t open = nullptr;
};

static std::atomic<int64_t> g_launches{0};
static std::atomic<int> g_profiling{0};
static std::mutex g_mu;
static std::map<std::string, KernelStats> g_stats;
static std::vector<cudaEvent_t> g_pool;

static cudaEvent_t take_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

void prof_begin(const char *name, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!g_profiling.load(std::memory_order_relaxed)) return;
    std::lock_guard<std::mutex> lk(g_mu);
    KernelStats &ks = g_stats[name];
    ks.open = take_event();
    cudaEventRecord(ks.open, st);
}

void prof_end(const char *name, cudaStream_t st) {
    if (!g_profiling.load(std::memory_order_relaxed)) return;
    std::lock_guard<std::mutex> lk(g_mu);
    KernelStats &ks = g_stats[name];
    if (!ks.open) return;
    cudaEvent_t stop = take_event();
    cudaEventRecord(stop, st);
    ks.pending.emplace_back(ks.open, stop);
    ks.open = nullptr;
    ks.launches += 1;
}

bool ente_profile_enabled() { return g_profiling.load(std::memory_order_relaxed) != 0; }

}  // namespace ente

using namespace ente;

extern "C" int64_t ente_launch_count(void) { return g_launches.load(); }

extern "C" void ente_profile_enable(int on) { g_profiling.store(on ? 1 : 0); }

extern "C" void ente_profile_reset(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto &kv : g_stats)
        for (auto &pr : kv.second.pending) {
            g_pool.push_back(pr.first);
            g_pool.push_back(pr.second);
        }
    g_stats.clear();
}

extern "C" int ente_profile_read(char *names, size_t names_len, int64_t *launches, double *ms,
                                 int max_kernels) {
    std::lock_guard<std::mutex> lk(g_mu);
    int i = 0;
    size_t off = 0;
    for (auto &kv : g_stats) {
        KernelStats &ks = kv.second;
        for (auto &pr : ks.pending) {
            float t = 0.0f;
            if (cudaEventSynchronize(pr.second) == cudaSuccess &&
                cudaEventElapsedTime(&t, pr.first, pr.second) == cudaSuccess)
                ks.ms += t;
            g_pool.push_back(pr.first);
            g_pool.push_back(pr.second);
        }
        ks.pending.clear();
        if (i < max_kernels) {
            launches[i] = ks.launches;
            ms[i] = ks.ms;
            const size_t len = kv.first.size() + 1;
            if (names && off + len <= names_len) {
                memcpy(names + off, kv.first.c_str(), len);
                off += len;
            }
        }
        ++i;
    }
    return i;
}

extern "C" const char *ente_last_error(void) { return g_err; }

extern "C" const char *ente_version(void) { return "ente_b200 0.1.0 sm_100a"; }
