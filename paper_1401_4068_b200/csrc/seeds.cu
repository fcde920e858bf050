// Host-side (C++) surrogate-permutation and jitter-seed generation.
//
// The reference derives every random stream of analyze_pair from numpy:
//   jitter    default_rng(SeedSequence((seed, u, 0 | idx + 1)))   inference.py:148,171-172, ksg.py:55
//   surrogate default_rng(SeedSequence((seed, idx))).permutation(R),
//             redrawn until phi(r) != r for all r (strict)          inference.py:41-49,101-102,161-164
// Python pays ~26 us per SeedSequence + PCG64 construction and ~50-200 us
// per permutation; a C2 analyze_pair needs 2010 streams and 200
// permutations.  This file restates the published algorithms so the host
// prep is a few microseconds per item:
//   SeedSequence  numpy/random/bit_generator.pyx (entropy words, pool of 4
//                 uint32 mixed with hashmix/mix, generate_state)
//   PCG64         numpy/random/src/pcg64 (128-bit LCG, seeding
//                 pcg_setseq_128_srandom_r, XSL-RR output, 32-bit halves
//                 buffered by next_uint32)
//   permutation   Generator.permutation(int) = shuffle(arange(R)): for
//                 i = R-1 .. 1 swap(i, random_interval(i)), random_interval
//                 = masked rejection on next_uint32 (next_uint64 above 2^32)
// Pinned bit-for-bit against numpy by tests/test_seeds.py.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "ente_b200.h"
#include "hostutil.cuh"

namespace ente {
void set_error(const char *fmt, ...);
}

namespace {

// --- SeedSequence ---------------------------------------------------------
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kXShift = 16, kPool = 4;

inline uint32_t hashmix(uint32_t v, uint32_t &hc) {
    v ^= hc;
    hc *= kMultA;
    v *= hc;
    v ^= v >> kXShift;
    return v;
}

inline uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = kMixL * x - kMixR * y;
    r ^= r >> kXShift;
    return r;
}

// generate_state(4, uint64) of SeedSequence(entropy words)
void seed_sequence_state(const uint32_t *ent, int64_t n_ent, uint64_t out[4]) {
    uint32_t pool[kPool];
    uint32_t hc = kInitA;
    for (int i = 0; i < kPool; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u, hc);
    for (int s = 0; s < kPool; ++s)
        for (int d = 0; d < kPool; ++d)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
    for (int64_t s = kPool; s < n_ent; ++s)
        for (int d = 0; d < kPool; ++d) pool[d] = mix(pool[d], hashmix(ent[s], hc));
    uint32_t hb = kInitB;
    uint32_t w[8];
    for (int i = 0; i < 8; ++i) {
        uint32_t v = pool[i % kPool];
        v ^= hb;
        hb *= kMultB;
        v *= hb;
        v ^= v >> kXShift;
        w[i] = v;
    }
    for (int i = 0; i < 4; ++i) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

// --- PCG64 ----------------------------------------------------------------
typedef unsigned __int128 u128;
const u128 kPcgMult = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;

struct Pcg64 {
    u128 state, inc;
    bool has32 = false;
    uint32_t buf32 = 0;

    // PCG64(SeedSequence): pcg64_set_seed(seed = s[0..1], inc = s[2..3])
    void seed(const uint64_t s[4]) {
        const u128 init = ((u128)s[0] << 64) | s[1];
        const u128 seq = ((u128)s[2] << 64) | s[3];
        state = 0;
        inc = (seq << 1) | 1u;
        state = state * kPcgMult + inc;
        state += init;
        state = state * kPcgMult + inc;
    }
    uint64_t next64() {
        state = state * kPcgMult + inc;
        const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
        const unsigned rot = (unsigned)(state >> 122);
        return (x >> rot) | (x << ((64u - rot) & 63u));
    }
    uint32_t next32() {
        if (has32) {
            has32 = false;
            return buf32;
        }
        const uint64_t v = next64();
        has32 = true;
        buf32 = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    uint64_t interval(uint64_t max) {
        if (max == 0) return 0;
        uint64_t mask = max;
        mask |= mask >> 1;
        mask |= mask >> 2;
        mask |= mask >> 4;
        mask |= mask >> 8;
        mask |= mask >> 16;
        mask |= mask >> 32;
        uint64_t v;
        if (max <= 0xffffffffull) {
            while ((v = (next32() & mask)) > max) {
            }
        } else {
            while ((v = (next64() & mask)) > max) {
            }
        }
        return v;
    }
};

}  // namespace

extern "C" {

int ente_seed_states(const uint32_t *words, const int64_t *offsets, int64_t n_items,
                     uint64_t *out) {
    if (n_items < 0 || (n_items > 0 && (!words || !offsets || !out))) {
        ente::set_error("ente_seed_states: bad arguments");
        return ENTE_ERR_ARG;
    }
    for (int64_t i = 0; i < n_items; ++i)
        if (offsets[i + 1] < offsets[i]) {
            ente::set_error("ente_seed_states: offsets must be non-decreasing");
            return ENTE_ERR_ARG;
        }
    ente::parallel_for(n_items, 4096, [&](int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            uint64_t s[4];
            seed_sequence_state(words + offsets[i], offsets[i + 1] - offsets[i], s);
            Pcg64 g;
            g.seed(s);
            out[4 * i + 0] = (uint64_t)(g.state >> 64);
            out[4 * i + 1] = (uint64_t)g.state;
            out[4 * i + 2] = (uint64_t)(g.inc >> 64);
            out[4 * i + 3] = (uint64_t)g.inc;
        }
    });
    return ENTE_OK;
}

int ente_seed_states_cols(const uint32_t *prefix, int n_prefix, const int64_t *cols, int n_cols,
                          int64_t n_items, uint64_t *out) {
    if (n_items < 0 || n_prefix < 0 || n_cols < 0 || n_prefix + n_cols > 16 || n_prefix + n_cols < 1 ||
        (n_items > 0 && (!out || (n_prefix && !prefix) || (n_cols && !cols)))) {
        ente::set_error("ente_seed_states_cols: bad arguments");
        return ENTE_ERR_ARG;
    }
    for (int64_t j = 0; j < (int64_t)n_cols * n_items; ++j)
        if (cols[j] < 0 || cols[j] > 0xffffffffll) {
            ente::set_error("ente_seed_states_cols: column value outside one uint32 word");
            return ENTE_ERR_ARG;
        }
    ente::parallel_for(n_items, 8192, [&](int64_t lo, int64_t hi) {
        uint32_t ent[16];
        for (int j = 0; j < n_prefix; ++j) ent[j] = prefix[j];
        for (int64_t i = lo; i < hi; ++i) {
            for (int j = 0; j < n_cols; ++j) ent[n_prefix + j] = (uint32_t)cols[(int64_t)j * n_items + i];
            uint64_t s[4];
            seed_sequence_state(ent, n_prefix + n_cols, s);
            Pcg64 g;
            g.seed(s);
            out[4 * i + 0] = (uint64_t)(g.state >> 64);
            out[4 * i + 1] = (uint64_t)g.state;
            out[4 * i + 2] = (uint64_t)(g.inc >> 64);
            out[4 * i + 3] = (uint64_t)g.inc;
        }
    });
    return ENTE_OK;
}

int ente_draw_permutations(const uint32_t *words, const int64_t *offsets, int64_t n_perms,
                           int reps, int strict, int32_t *out) {
    if (n_perms < 0 || reps < 0 || (n_perms > 0 && (!words || !offsets || !out))) {
        ente::set_error("ente_draw_permutations: bad arguments");
        return ENTE_ERR_ARG;
    }
    if (strict && reps < 2 && n_perms > 0) {
        ente::set_error("strict permutation needs R >= 2");
        return ENTE_ERR_ARG;
    }
    ente::parallel_for(n_perms, 16, [&](int64_t lo, int64_t hi) {
        std::vector<int64_t> a((size_t)reps);
        for (int64_t p = lo; p < hi; ++p) {
            uint64_t s[4];
            seed_sequence_state(words + offsets[p], offsets[p + 1] - offsets[p], s);
            Pcg64 g;
            g.seed(s);
            for (;;) {
                for (int r = 0; r < reps; ++r) a[r] = r;
                for (int64_t i = reps - 1; i >= 1; --i) {
                    const int64_t j = (int64_t)g.interval((uint64_t)i);
                    std::swap(a[i], a[j]);
                }
                bool fixed = false;
                for (int r = 0; r < reps && !fixed; ++r) fixed = a[r] == r;
                if (!strict || !fixed) break;
            }
            for (int r = 0; r < reps; ++r) out[p * reps + r] = (int32_t)a[r];
        }
    });
    return ENTE_OK;
}

}  // extern "C"
