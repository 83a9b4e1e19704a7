// Shared device helpers for the peakann-b200 kernels (sm_100a).
//
// Conventions (mirroring /root/reference/pkg/src/peakann/_kernels.py:1-11):
//  * coordinates are float32, stored row-major with rows padded to `dp`
//    floats (dp % 4 == 0, padding is zero, which adds exactly +0.0 to any
//    squared distance);
//  * squared distances are float64 and every ordering is the key
//    (squared distance, id), compared lexicographically;
//  * ids are int32 on device (n < 2^31), int64 at the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#define PK_FULL 0xffffffffu
#define PK_VIS 0x80000000u   // visited flag, stored in bit 31 of a beam id
#define PK_APX 0x40000000u   // lazy keys: the stored distance is an approximation (bit 30) ...
#define PK_A32 0x20000000u   // ... from the fp32 screen (bit 29 set) or the float64 one (clear)
#define PK_LAZYF 0x60000000u // both lazy-key flags
#define PK_IDMASK 0x1fffffffu
#define PK_IDAPX 0x7fffffffu // id + lazy-key flags (visit-log entries)

// Phase timers of the beam walk (diagnostics build only: nvcc -DPK_PHASE_TIMERS;
// tools/variant.sh): clock64 cycles per phase summed over warps (lane 0) into
// pk_phase_cycles[] -- 0 expand (next entry, adjacency row, seen filter),
// 1 row prefetch, 2 fp32 screens, 3 resolve, 4 merge, 5 emit, 6 seeding.
// One copy per translation unit (no relocatable device code): knn.cu's holds
// the query walks (pk_phase_timers), build.cu's the build searches
// (pk_phase_timers_build).
#ifdef PK_PHASE_TIMERS
static __device__ unsigned long long pk_phase_cycles[8];
#define PK_PT_BEGIN long long _pt0 = clock64();
#define PK_PT_END(ph)                                                                             \
    do {                                                                                          \
        if ((threadIdx.x & 31) == 0) atomicAdd(&pk_phase_cycles[ph], (unsigned long long)(clock64() - _pt0)); \
    } while (0)
#define PK_PT_NEXT(ph) \
    do {               \
        PK_PT_END(ph); \
        _pt0 = clock64(); \
    } while (0)
#else
#define PK_PT_BEGIN
#define PK_PT_END(ph) do { } while (0)
#define PK_PT_NEXT(ph) do { } while (0)
#endif

namespace pk {

constexpr int kWarp = 32;

// ---- error reporting -------------------------------------------------------
// Device-side sticky error word (bit flags), read back by the host driver.
enum DeviceError : unsigned {
    ERR_VISIT_OVERFLOW = 1u,   // build visit log exceeded its capacity
    ERR_CAND_OVERFLOW = 2u,    // candidate buffer exceeded its capacity
    ERR_BEAM_CAPACITY = 4u,    // L larger than the kernel's beam capacity
};

// ---- keys --------------------------------------------------------------------
// Squared distances are >= 0, so their IEEE bit patterns order like the values.
__device__ __forceinline__ unsigned long long dbits(double d) {
    return (unsigned long long)__double_as_longlong(d);
}
__device__ __forceinline__ bool key_lt(double da, unsigned ia, double db, unsigned ib) {
    return da < db || (da == db && ia < ib);
}
__device__ __forceinline__ bool key_eq(double da, unsigned ia, double db, unsigned ib) {
    return da == db && ia == ib;
}

__device__ __forceinline__ int next_pow2_dev(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ float4 ldg4(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}

// Per-query "seen" table: H = 2^hbits 16-bit slots as H/4 sets of 4 ways.  A
// set is picked by the id's low (hbits - 2) bits and each way stores the
// quotient id >> (hbits - 2), which reconstructs the id exactly, so nothing is
// ever reported seen falsely.  One 64-bit load reads a whole set (no probe
// loop, no divergence); a full set overwrites a pseudo-random way (lossy): a
// lost id only costs a re-evaluation.  Needs (n-1) >> (hbits-2) < 0xffff
// (choose_hash enforces it); 0xffff marks an empty way.
constexpr unsigned short kSeenEmpty = 0xffffu;

__device__ __forceinline__ bool seen_or_insert(unsigned short* hash, unsigned mask, int hbits, unsigned id) {
    const int sbits = hbits - 2;
    const unsigned set = id & (mask >> 2);
    const unsigned tag = id >> sbits;
    const uint2 v = reinterpret_cast<const uint2*>(hash)[set];
    const unsigned t2 = tag | (tag << 16);
    if (__vcmpeq2(v.x, t2) | __vcmpeq2(v.y, t2)) return true;
    const unsigned ex = __vcmpeq2(v.x, 0xffffffffu), ey = __vcmpeq2(v.y, 0xffffffffu);
    const unsigned way = ex ? ((ex & 0xffffu) ? 0u : 1u) : ey ? ((ey & 0xffffu) ? 2u : 3u) : ((tag ^ (id >> 5)) & 3u);
    hash[4 * set + way] = (unsigned short)tag;
    return false;
}

// seen_or_insert in two steps, so the set loads of several ids can be issued
// together (one round trip when the table lives in global memory): the second
// id's view of a shared set may miss the first id's insert, which can only
// lose an entry (a re-evaluation), never report an unseen id as seen
__device__ __forceinline__ uint2 seen_load(const unsigned short* hash, unsigned mask, unsigned id) {
    return reinterpret_cast<const uint2*>(hash)[id & (mask >> 2)];
}
__device__ __forceinline__ bool seen_apply(unsigned short* hash, unsigned mask, int hbits, unsigned id, uint2 v) {
    const unsigned set = id & (mask >> 2);
    const unsigned tag = id >> (hbits - 2);
    const unsigned t2 = tag | (tag << 16);
    if (__vcmpeq2(v.x, t2) | __vcmpeq2(v.y, t2)) return true;
    const unsigned ex = __vcmpeq2(v.x, 0xffffffffu), ey = __vcmpeq2(v.y, 0xffffffffu);
    const unsigned way = ex ? ((ex & 0xffffu) ? 0u : 1u) : ey ? ((ey & 0xffffu) ? 2u : 3u) : ((tag ^ (id >> 5)) & 3u);
    hash[4 * set + way] = (unsigned short)tag;
    return false;
}

// ---- mbarrier + bulk copy (tensor-core kernels; row ring of the float beam searches) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// global -> shared bulk copy (TMA engine, no tensor map): bytes % 16 == 0, both sides 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}

// ---- distance policies ---------------------------------------------------------
//
// Both policies return, for lane i < c, the squared distance between the query
// and candidate row `cid` (the id held by lane i), as a double that is
// bit-identical to the reference's sequential float64 accumulation
// (_kernels.py:21-28):
//
//  * Seq64: each lane walks its candidate's coordinates t = 0..d-1 in order,
//    acc = acc + diff*diff with the product and the sum rounded separately
//    (__dmul_rn / __dadd_rn, never contracted to an FMA: for coordinates of
//    different magnitude diff carries more than 26 bits and its square is not
//    exact, so an FMA would round differently from the reference's numba code).
//    The result is the reference's value for any float32 data.
//  * Exact32: lanes split the dimensions and reduce float32 partial sums across
//    the warp.  Only used when the point set is integer-valued with
//    d * (2*max|x|)^2 < 2^24 (checked on upload): every partial sum is then an
//    integer below 2^24, so each float32 operation is exact in any order and
//    equals the float64 reference bit for bit.
//
// Query vectors: member queries read float32 rows (converted exactly to
// float64, as `data[i].astype(np.float64)` does); free vector queries pass
// float64 coordinates and always use Seq64.

struct Seq64Member {
    const float* q;  // query row (dp floats), global
    int dp;
    __device__ __forceinline__ double eval_one(const float* __restrict__ X, int id) const {
        const float* r = X + (size_t)id * dp;
        double acc = 0.0;
#pragma unroll 4
        for (int t = 0; t < dp; t += 4) {
            float4 x = ldg4(r + t);
            float4 y = ldg4(q + t);
            double a = (double)y.x - (double)x.x; acc = __dadd_rn(acc, __dmul_rn(a, a));
            double b = (double)y.y - (double)x.y; acc = __dadd_rn(acc, __dmul_rn(b, b));
            double c = (double)y.z - (double)x.z; acc = __dadd_rn(acc, __dmul_rn(c, c));
            double e = (double)y.w - (double)x.w; acc = __dadd_rn(acc, __dmul_rn(e, e));
        }
        return acc;
    }
    // lane i < c: distance to its own cid
    __device__ __forceinline__ double eval(const float* __restrict__ X, int cid, int c) const {
        return lane_id() < c ? eval_one(X, cid) : 0.0;
    }
};

struct Seq64Vector {
    const double* q;  // float64 query (dp entries, zero padded), global
    int dp;
    __device__ __forceinline__ double eval_one(const float* __restrict__ X, int id) const {
        const float* r = X + (size_t)id * dp;
        double acc = 0.0;
#pragma unroll 4
        for (int t = 0; t < dp; t += 4) {
            float4 x = ldg4(r + t);
            double a = __ldg(q + t) - (double)x.x; acc = __dadd_rn(acc, __dmul_rn(a, a));
            double b = __ldg(q + t + 1) - (double)x.y; acc = __dadd_rn(acc, __dmul_rn(b, b));
            double c = __ldg(q + t + 2) - (double)x.z; acc = __dadd_rn(acc, __dmul_rn(c, c));
            double e = __ldg(q + t + 3) - (double)x.w; acc = __dadd_rn(acc, __dmul_rn(e, e));
        }
        return acc;
    }
    __device__ __forceinline__ double eval(const float* __restrict__ X, int cid, int c) const {
        return lane_id() < c ? eval_one(X, cid) : 0.0;
    }
};

// Exact32: QV float4 query slices per lane cover dims [4*lane + 128*v].
template <int QV>
struct Exact32 {
    float4 q[QV];
    int dp;

    __device__ __forceinline__ void load(const float* qrow, int dp_) {
        dp = dp_;
        const int lane = lane_id();
#pragma unroll
        for (int v = 0; v < QV; ++v) {
            int col = 4 * lane + 128 * v;
            q[v] = col < dp ? ldg4(qrow + col) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }

    __device__ __forceinline__ float partial(const float* __restrict__ X, int id) const {
        const float* r = X + (size_t)id * dp;
        const int lane = lane_id();
        float acc = 0.f;
#pragma unroll
        for (int v = 0; v < QV; ++v) {
            int col = 4 * lane + 128 * v;
            if (col < dp) {
                float4 x = ldg4(r + col);
                float a = q[v].x - x.x, b = q[v].y - x.y, c = q[v].z - x.z, e = q[v].w - x.w;
                acc = fmaf(a, a, acc);
                acc = fmaf(b, b, acc);
                acc = fmaf(c, c, acc);
                acc = fmaf(e, e, acc);
            }
        }
        return acc;
    }

    // Groups of 8 candidates: 8 independent row loads in flight, then a
    // transposed butterfly (3 halving stages + 2 plain stages) leaves the sum of
    // candidate j in lanes 4j..4j+3.
    __device__ __forceinline__ double eval(const float* __restrict__ X, int cid, int c) const {
        const int lane = lane_id();
        double mine = 0.0;
        for (int g = 0; g < c; g += 8) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int id = __shfl_sync(PK_FULL, cid, (g + j) & 31);
                v[j] = (g + j < c) ? partial(X, id) : 0.f;
            }
#pragma unroll
            for (int s = 16, h = 4; s >= 4; s >>= 1, h >>= 1) {
                const bool up = lane & s;
#pragma unroll
                for (int j = 0; j < h; ++j) {
                    float send = up ? v[j] : v[j + h];
                    float keep = up ? v[j + h] : v[j];
                    v[j] = keep + __shfl_xor_sync(PK_FULL, send, s);
                }
            }
            v[0] += __shfl_xor_sync(PK_FULL, v[0], 2);
            v[0] += __shfl_xor_sync(PK_FULL, v[0], 1);
            // candidate index held by this lane: bits (4,3,2) of lane
            float got = __shfl_sync(PK_FULL, v[0], ((lane - g) & 7) << 2);
            if (lane >= g && lane < g + 8 && lane < c) mine = (double)got;
        }
        return mine;
    }
};

// ExactU8: integer coordinates spanning at most 255 are stored as bytes
// (x - min), four per 32-bit word, rows of `dw` words.  |a - b| per byte
// (__vabsdiffu4) and its square summed by __dp4a are exact integer
// arithmetic, identical to the reference's float64 value (every term and sum
// is an integer far below 2^53).  Four lanes per candidate: lane quarter
// sub = lane & 3 owns words 32*v + 8*sub .. +8 of every row (v < QW), so one
// pass evaluates 8 candidates with two 128-bit loads per lane and a 2-step
// reduction (rows with dw % 8 != 0 use guarded scalar loads).
template <int QW>
struct ExactU8 {
    const unsigned* X8;
    unsigned q[8 * QW];
    int dw;

    __device__ __forceinline__ void fetch(const unsigned* r, unsigned (&o)[8 * QW]) const {
        const int sub = lane_id() & 3;
#pragma unroll
        for (int v = 0; v < QW; ++v) {
            const int w0 = 32 * v + 8 * sub;
            if ((dw & 7) == 0) {
                if (w0 < dw) {
                    const uint4 a = __ldg(reinterpret_cast<const uint4*>(r + w0));
                    const uint4 b = __ldg(reinterpret_cast<const uint4*>(r + w0 + 4));
                    o[8 * v + 0] = a.x; o[8 * v + 1] = a.y; o[8 * v + 2] = a.z; o[8 * v + 3] = a.w;
                    o[8 * v + 4] = b.x; o[8 * v + 5] = b.y; o[8 * v + 6] = b.z; o[8 * v + 7] = b.w;
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) o[8 * v + i] = 0u;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) o[8 * v + i] = w0 + i < dw ? __ldg(r + w0 + i) : 0u;
            }
        }
    }

    __device__ __forceinline__ void load(const unsigned* X8_, int dw_, unsigned id) {
        X8 = X8_;
        dw = dw_;
        fetch(X8 + (size_t)id * dw, q);
    }

    __device__ __forceinline__ unsigned partial(int id) const {
        unsigned x[8 * QW];
        fetch(X8 + (size_t)id * dw, x);
        unsigned a0 = 0u, a1 = 0u;
#pragma unroll
        for (int i = 0; i < 8 * QW; i += 2) {
            const unsigned e = __vabsdiffu4(q[i], x[i]);
            const unsigned f = __vabsdiffu4(q[i + 1], x[i + 1]);
            a0 = __dp4a(e, e, a0);
            a1 = __dp4a(f, f, a1);
        }
        return a0 + a1;
    }

    __device__ __forceinline__ double eval(const float* __restrict__, int cid, int c) const {
        const int lane = lane_id();
        double mine = 0.0;
        for (int g = 0; g < c; g += 8) {
            const int gi = g + (lane >> 2);
            const int id = __shfl_sync(PK_FULL, cid, gi & 31);
            unsigned s = gi < c ? partial(id) : 0u;
            s += __shfl_xor_sync(PK_FULL, s, 1);
            s += __shfl_xor_sync(PK_FULL, s, 2);
            const unsigned got = __shfl_sync(PK_FULL, s, ((lane - g) & 7) << 2);
            if (lane >= g && lane < g + 8 && lane < c) mine = (double)got;
        }
        return mine;
    }
};

// one full u8 row pair, sequential over words (prune on staged rows)
__device__ __forceinline__ unsigned u8_row_dist(const unsigned* a, const unsigned* b, int dw) {
    unsigned acc0 = 0u, acc1 = 0u;
    int w = 0;
    for (; w + 1 < dw; w += 2) {
        unsigned x = __vabsdiffu4(a[w], b[w]);
        unsigned y = __vabsdiffu4(a[w + 1], b[w + 1]);
        acc0 = __dp4a(x, x, acc0);
        acc1 = __dp4a(y, y, acc1);
    }
    if (w < dw) {
        unsigned x = __vabsdiffu4(a[w], b[w]);
        acc0 = __dp4a(x, x, acc0);
    }
    return acc0 + acc1;
}

// ---- policy selection --------------------------------------------------------------
// point data as seen by the kernels: float32 rows (always) and, in the u8
// mode, the packed byte rows
struct DataRef {
    const float* X;
    int dp;
    const unsigned* X8;
    int dw;
    int screen = 1;  // float data: decide RobustPrune kill tests from the fp32 screen when certain
};

constexpr int MODE_SEQ64 = 0;
constexpr int MODE_EXACT32 = 1;
constexpr int MODE_EXACT_U8 = 2;

// Seq64 member query with an fp32 pre-screen for the beam searches: screen()
// is a warp-cooperative fp32 squared distance (same value on every lane,
// within kScreenEps relative of the exact one when dp <= 128 * QV), used only
// to drop candidates that provably cannot enter a full beam; every distance
// that is stored or compared exactly still comes from eval_one().
template <int QV>
struct Seq64Screened : Seq64Member {
    static constexpr int kQV = QV;
    float4 qr[QV];  // this lane's query slices (chunks lane + 32 j), held in registers
    __device__ __forceinline__ void load_query() {
        const float4* a = reinterpret_cast<const float4*>(q);
        const int nv = dp >> 2, lane = lane_id();
#pragma unroll
        for (int j = 0; j < QV; ++j) {
            const int f = lane + 32 * j;
            qr[j] = f < nv ? __ldg(a + f) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    __device__ __forceinline__ float screen(const float* __restrict__ X, unsigned id) const {
        const float4* r = reinterpret_cast<const float4*>(X + (size_t)id * dp);
        const int nv = dp >> 2, lane = lane_id();
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < QV; ++j) {
            const int f = lane + 32 * j;
            if (f < nv) {
                const float4 y = qr[j], x = __ldg(r + f);
                const float d0 = y.x - x.x, d1 = y.y - x.y, d2 = y.z - x.z, d3 = y.w - x.w;
                acc = fmaf(d0, d0, acc);
                acc = fmaf(d1, d1, acc);
                acc = fmaf(d2, d2, acc);
                acc = fmaf(d3, d3, acc);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(PK_FULL, acc, o);
        return acc;
    }
    // screen() of a row staged in shared memory (row ring, beam.cuh): the same
    // arithmetic in the same order, so the same value as screen()
    __device__ __forceinline__ float screen_smem(const float4* __restrict__ r) const {
        const int nv = dp >> 2, lane = lane_id();
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < QV; ++j) {
            const int f = lane + 32 * j;
            if (f < nv) {
                const float4 y = qr[j], x = r[f];
                const float d0 = y.x - x.x, d1 = y.y - x.y, d2 = y.z - x.z, d3 = y.w - x.w;
                acc = fmaf(d0, d0, acc);
                acc = fmaf(d1, d1, acc);
                acc = fmaf(d2, d2, acc);
                acc = fmaf(d3, d3, acc);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(PK_FULL, acc, o);
        return acc;
    }
    // Warp-cooperative float64 value of the squared distance (lazy keys): each
    // lane accumulates its 4*QV coordinates with fma, then an xor butterfly
    // (commutative adds: every lane ends with the same value).  Within
    // (4*QV + 8) * 2^-53 relative of the exact sum, so within kLazyEps of the
    // reference's sequential value (<= 2*dp roundings of 2^-53 each).
    __device__ __forceinline__ double dscreen(const float* __restrict__ X, unsigned id) const {
        const float4* r = reinterpret_cast<const float4*>(X + (size_t)id * dp);
        const int nv = dp >> 2, lane = lane_id();
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < QV; ++j) {
            const int f = lane + 32 * j;
            if (f < nv) {
                const float4 y = qr[j], x = __ldg(r + f);
                const double d0 = (double)y.x - (double)x.x, d1 = (double)y.y - (double)x.y;
                const double d2 = (double)y.z - (double)x.z, d3 = (double)y.w - (double)x.w;
                acc = fma(d0, d0, acc);
                acc = fma(d1, d1, acc);
                acc = fma(d2, d2, acc);
                acc = fma(d3, d3, acc);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(PK_FULL, acc, o);
        return acc;
    }
};

// distance policies whose values are exact integers below 2^32 (packed keys)
template <class D>
struct int_keys {
    static constexpr bool value = false;
};
template <int QV>
struct int_keys<Exact32<QV>> {
    static constexpr bool value = true;
};
template <int QV>
struct int_keys<ExactU8<QV>> {
    static constexpr bool value = true;
};

template <class D>
struct has_screen {
    static constexpr bool value = false;
};
template <int QV>
struct has_screen<Seq64Screened<QV>> {
    static constexpr bool value = true;
};

// Seq64Screened whose beam search stages candidate rows through the shared-memory
// row ring (beam.cuh: ring_screens) instead of loading them into registers
template <int QV>
struct Seq64Ring : Seq64Screened<QV> {};
template <int QV>
struct has_screen<Seq64Ring<QV>> {
    static constexpr bool value = true;
};
template <class D>
struct uses_ring {
    static constexpr bool value = false;
};
template <int QV>
struct uses_ring<Seq64Ring<QV>> {
    static constexpr bool value = true;
};

template <int MODE, int QV, bool RING = false>
struct DistFor;
template <int QV, bool RING>
struct DistFor<MODE_SEQ64, QV, RING> {
    using T = typename std::conditional<RING, Seq64Ring<QV>, Seq64Screened<QV>>::type;
    __device__ static T make(const DataRef& D, unsigned id) {
        T t;
        t.q = D.X + (size_t)id * D.dp;
        t.dp = D.dp;
        t.load_query();
        return t;
    }
};
template <int QV>
struct DistFor<MODE_EXACT32, QV, false> {
    using T = Exact32<QV>;
    __device__ static T make(const DataRef& D, unsigned id) {
        T t;
        t.load(D.X + (size_t)id * D.dp, D.dp);
        return t;
    }
};
template <int QV>
struct DistFor<MODE_EXACT_U8, QV, false> {
    using T = ExactU8<QV>;
    __device__ static T make(const DataRef& D, unsigned id) {
        T t;
        t.load(D.X8, D.dw, id);
        return t;
    }
};

// fp32 screening of float data (SEQ64 mode): the pick row is spread over the
// warp as float4 chunks (lane l holds chunks l, l + 32, ...; QV = ceil(dp/128));
// dist() is a warp-cooperative fp32 sum of (p_i - x_i)^2 with an xor-butterfly
// reduction, so every lane gets the same value.  All terms are non-negative:
// the result is within 40 * 2^-24 relative of the exact sum (<= 32 fma steps
// per lane + 5 tree levels + the rounding of each difference), which callers
// widen to kScreenEps before deciding anything without the exact value.
constexpr double kScreenEps = 1e-5;

template <int QV>
struct Fp32Pick {
    float4 v[QV];
    __device__ __forceinline__ void load(const float* __restrict__ X, int dp, unsigned id) {
        const float4* r = reinterpret_cast<const float4*>(X + (size_t)id * dp);
        const int nv = dp >> 2, lane = lane_id();
#pragma unroll
        for (int j = 0; j < QV; ++j) {
            const int f = lane + 32 * j;
            v[j] = f < nv ? __ldg(r + f) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    __device__ __forceinline__ float partial(const float* __restrict__ X, int dp, unsigned id) const {
        const float4* r = reinterpret_cast<const float4*>(X + (size_t)id * dp);
        const int nv = dp >> 2, lane = lane_id();
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < QV; ++j) {
            const int f = lane + 32 * j;
            if (f < nv) {
                const float4 x = __ldg(r + f);
                const float a = v[j].x - x.x, b = v[j].y - x.y, c = v[j].z - x.z, d = v[j].w - x.w;
                acc = fmaf(a, a, acc);
                acc = fmaf(b, b, acc);
                acc = fmaf(c, c, acc);
                acc = fmaf(d, d, acc);
            }
        }
        return acc;
    }
    __device__ __forceinline__ static float reduce(float s) {
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(PK_FULL, s, o);
        return s;
    }
};

// Lazy keys (beam searches on float data).  A beam entry stores one of
//  * the fp32 warp-cooperative value a32 (Seq64Screened::screen; PK_APX|PK_A32):
//    within (4*QV + 7) * 2^-24 <= 2.4e-6 relative of the exact sum for
//    QV <= 8 when 1e-20 < a32 < 1e30 (no fp32 underflow / overflow), so the
//    reference's sequential value D lies in [a (1 - kEps32), a (1 + kEps32)];
//  * the float64 warp-cooperative value a64 (dscreen; PK_APX): both a64 and D
//    are within 2*dp + 4*QV + 8 roundings of 2^-53 of the exact sum (< 2.4e-13
//    for dp <= 1024), so D lies in [a (1 - kEps64), a (1 + kEps64)].  Every
//    nonzero term is >= 2^-298 (the smallest fp32 difference, squared): no
//    float64 underflow, and a64 == 0 means D == 0 exactly;
//  * the exact value D (no flag).
// Two keys whose intervals are disjoint are ordered by their stored values;
// overlapping ones are refined one level at a time until they are not.
constexpr double kEps32 = 4e-6;
constexpr double kEps64 = 1e-12;
__device__ __forceinline__ double key_eps(unsigned i) {
    return (i & PK_APX) ? ((i & PK_A32) ? kEps32 : kEps64) : 0.0;
}
__device__ __forceinline__ double key_lo(double v, unsigned i) { return v * (1.0 - key_eps(i)); }
__device__ __forceinline__ double key_hi(double v, unsigned i) { return v * (1.0 + key_eps(i)); }
// is (va, ia) < (vb, ib) certain from the two intervals?
__device__ __forceinline__ bool key_certain_lt(double va, unsigned ia, double vb, unsigned ib) {
    if (!((ia | ib) & PK_APX)) return key_lt(va, ia & PK_IDMASK, vb, ib & PK_IDMASK);
    return key_hi(va, ia) < key_lo(vb, ib);
}
// fp32 screen values usable as level-1 lazy keys
__device__ __forceinline__ bool screen_usable(float s) { return s > 1e-20f && s < 1e30f; }

// Verdict of "alpha2 * d <= k" from a screened d~ (fp32): 1 = true, 0 = false,
// 2 = too close to call (the caller computes the exact float64 distance).
__device__ __forceinline__ int screen_le(double alpha2, float dscr, double k) {
    const double d = (double)dscr;
    if (!(d > 1e-20) || !(d < 1e30) || !(k > 1e-20)) return 2;
    const double a = alpha2 * d;
    if (a * (1.0 + kScreenEps) < k) return 1;
    if (a * (1.0 - kScreenEps) > k) return 0;
    return 2;
}

// functor: id -> distance policy object for that query row
template <int MODE, int QV, bool RING = false>
struct MakeAt {
    DataRef D;
    __device__ typename DistFor<MODE, QV, RING>::T operator()(unsigned id) const {
        return DistFor<MODE, QV, RING>::make(D, id);
    }
};

// ---- warp utilities --------------------------------------------------------------
__device__ __forceinline__ int warp_excl_prefix(unsigned ballot) {
    return __popc(ballot & ((1u << lane_id()) - 1u));
}

// The take-th smallest of vals[0, s) (u32, in shared memory) by a radix
// select, 4 passes of 8 bits with a 256-bin histogram in `bins`; on return
// `need` = how many entries equal to the result belong to the take smallest.
__device__ __forceinline__ unsigned warp_radix_kth(const unsigned* vals, int s, int take, unsigned* bins, int& need) {
    const int lane = lane_id();
    unsigned prefix = 0u;
    need = take;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int x = lane; x < 256; x += 32) bins[x] = 0u;
        __syncwarp();
        for (int x = lane; x < s; x += 32) {
            const unsigned v = vals[x];
            if (shift == 24 || (v >> (shift + 8)) == prefix) atomicAdd(bins + ((v >> shift) & 255u), 1u);
        }
        __syncwarp();
        // lane l owns bins 8l .. 8l + 7
        unsigned c[8], tot = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            c[i] = bins[8 * lane + i];
            tot += c[i];
        }
        unsigned incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_up_sync(PK_FULL, incl, o);
            if (lane >= o) incl += v;
        }
        const unsigned excl = incl - tot;
        const bool here = excl < (unsigned)need && incl >= (unsigned)need;
        const int src = __ffs(__ballot_sync(PK_FULL, here)) - 1;
        int bin = 0;
        unsigned before = 0u;
        if (lane == src) {
            unsigned acc = excl;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (acc + c[i] >= (unsigned)need) {
                    bin = 8 * lane + i;
                    break;
                }
                acc += c[i];
            }
            before = acc;
        }
        bin = __shfl_sync(PK_FULL, bin, src);
        before = __shfl_sync(PK_FULL, before, src);
        need -= (int)before;
        prefix = (prefix << 8) | (unsigned)bin;
        __syncwarp();
    }
    return prefix;
}

}  // namespace pk
