// Host-side insertion order: numpy's Generator.permutation(n) on a PCG64
// stream, restated so the build's order comes out as int32 directly (the
// reference draws it with numpy, vamana.py:141-143).  Same algorithm as
// numpy (pcg64 XSL-RR 128/64 output, 32-bit draws buffered in halves,
// Fisher-Yates from the top with masked rejection sampling), so the order is
// identical for the same stream state.
#include <cstdint>

#include "../../include/peakann_b200.h"

namespace {

typedef unsigned __int128 u128;

struct Pcg64 {
    u128 state, inc;
    int has_uint32;
    uint32_t uinteger;

    uint64_t next64() {
        const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
        state = state * mult + inc;
        const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
        const unsigned rot = (unsigned)(hi >> 58);
        const uint64_t x = hi ^ lo;
        return (x >> rot) | (x << ((64 - rot) & 63));
    }
    uint32_t next32() {
        if (has_uint32) {
            has_uint32 = 0;
            return uinteger;
        }
        const uint64_t v = next64();
        has_uint32 = 1;
        uinteger = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    // uniform in [0, max] by masked rejection
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
        if (max <= 0xffffffffULL) {
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

extern "C" int pk_pcg64_permutation(const uint64_t* state, int has_uint32, uint32_t uinteger, int64_t n,
                                    int32_t* out, uint64_t* state_out) {
    if (n < 0 || (n > 0 && !out) || !state) return 2;
    Pcg64 g;
    g.state = ((u128)state[0] << 64) | state[1];
    g.inc = ((u128)state[2] << 64) | state[3];
    g.has_uint32 = has_uint32;
    g.uinteger = uinteger;
    for (int64_t i = 0; i < n; ++i) out[i] = (int32_t)i;
    for (int64_t i = n - 1; i >= 1; --i) {
        const int64_t j = (int64_t)g.interval((uint64_t)i);
        const int32_t t = out[i];
        out[i] = out[j];
        out[j] = t;
    }
    if (state_out) {
        state_out[0] = (uint64_t)(g.state >> 64);
        state_out[1] = (uint64_t)g.state;
        state_out[2] = (uint64_t)g.has_uint32;
        state_out[3] = (uint64_t)g.uinteger;
    }
    return 0;
}
