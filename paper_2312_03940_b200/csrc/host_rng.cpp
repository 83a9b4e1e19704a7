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

// ---- PointSet validation ---------------------------------------------------------------
// Index of the first non-finite float in x[0, count) (row-major), -1 if all are
// finite.  Scanned by all host threads (the reference's np.isfinite check,
// core.py:17-54, is the same predicate).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

static int64_t first_nonfinite(const float* x, int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
        uint32_t b;
        std::memcpy(&b, x + i, 4);
        if ((b & 0x7f800000u) == 0x7f800000u) return i;  // inf or nan: all-ones exponent
    }
    return -1;
}

extern "C" int pk_find_nonfinite(const float* x, int64_t count, int64_t* first_bad) {
    if (!first_bad || (count > 0 && !x)) return 2;
    const int64_t chunk = 1 << 20;
    int nt = (int)std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), (count + chunk - 1) / chunk);
    if (nt <= 1) {
        *first_bad = first_nonfinite(x, 0, count);
        return 0;
    }
    std::vector<int64_t> res(nt, -1);
    std::vector<std::thread> th;
    const int64_t per = (count + nt - 1) / nt;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            const int64_t lo = t * per, hi = std::min(count, lo + per);
            if (lo < hi) res[t] = first_nonfinite(x, lo, hi);
        });
    for (auto& h : th) h.join();
    *first_bad = -1;
    for (int t = 0; t < nt; ++t)
        if (res[t] >= 0) {
            *first_bad = res[t];
            break;
        }
    return 0;
}
