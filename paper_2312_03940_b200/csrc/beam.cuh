// Warp-level greedy beam search, candidate sorting and RobustPrune.
//
// One warp owns one query.  The semantics are those of the reference
// (_kernels.py:125-212): seed with the start set, repeatedly expand the
// closest unvisited beam entry, insert every neighbour not yet in the beam,
// keep the best L by (dist, id), stop when every beam entry is visited.
//
// Two reorganisations keep the output bit-identical while doing less work
// (SURVEY.md §0.4, §0.11):
//  * the neighbours of one expansion are inserted as one batch (a merge of up
//    to 32 sorted candidates into the sorted beam).  Top-L of a union is
//    associative, so the batch merge equals sequential inserts;
//  * a node whose distance was already evaluated is not evaluated again.  The
//    reference re-evaluates evicted / rejected nodes, but their key is above
//    the beam's L-th key, which never increases once the beam is full, so they
//    can never re-enter.  The "seen" table is lossy (direct-mapped, ids may be
//    overwritten), which only costs re-evaluations; a re-evaluated node that
//    is still in the beam is recognised by its identical key and dropped.
//    Start points never need re-evaluation after seeding, so a bitmap of the
//    start set skips them exactly.
//
// Output rule (member queries): sorted(visited U unvisited beam) is the
// final beam followed by the evicted visited entries, so the first kk
// non-self entries are the beam minus the query itself plus, when the query
// sits in a full beam and kk == L, the best evicted visited entry.
#pragma once

#include "common.cuh"

namespace pk {

struct BeamSmem {
    double* bd;       // [Lcap] squared distances, (dist,id)-sorted
    unsigned* bi;     // [Lcap] ids | PK_VIS
    unsigned short* hash;  // [hmask+1] lossy seen table (common.cuh), 0xffff = empty
    unsigned hmask;
    int hbits;
    int* spos;        // [32] scratch: sorted insert positions
    unsigned* cbuf;   // [kCbuf] scratch: compacted candidate ids
    // row ring (float data, lazy keys): candidate rows staged by bulk copies
    float4* ring = nullptr;            // [ring_s][dp / 4]
    unsigned long long* bars = nullptr;  // [ring_s] mbarriers, one per slot
    int ring_s = 0;                    // slots (a power of two), 0 = no ring
};

constexpr int kCbuf = 64;  // compacted-candidate buffer (ids) per warp

// per-warp layout: bd[L] | bi[L] | (8-aligned) hash[H] (u16) | spos[32] | cbuf[kCbuf]
// (host side: beam_smem_bytes in api.cuh)
__device__ __forceinline__ BeamSmem carve_beam(unsigned char* base, int L, int H) {
    BeamSmem s;
    s.bd = reinterpret_cast<double*>(base);
    s.bi = reinterpret_cast<unsigned*>(base + (size_t)L * 8);
    const size_t hoff = ((size_t)L * 12 + 7) & ~(size_t)7;  // 8-byte aligned sets
    s.hash = reinterpret_cast<unsigned short*>(base + hoff);
    s.hmask = (unsigned)H - 1u;
    s.hbits = __ffs(H) - 1;
    const size_t tail = (hoff + (size_t)H * 2 + 15) & ~(size_t)15;
    s.spos = reinterpret_cast<int*>(base + tail);
    s.cbuf = reinterpret_cast<unsigned*>(base + tail + 128);
    return s;
}

// Beams wider than shared memory (doubling rounds that reach k ~ 16k and
// beyond; the reference doubles up to n - 1, dependent.py:118-126): the
// sorted beam bd[L] | bi[L] lives in a per-warp global slab, the seen table
// and the scratch stay in shared memory.  The walk is the same code on
// generic pointers, so the result is the same as the in-smem beam.
// smem layout: hash[H] (u16) | spos[32] | cbuf[kCbuf] (host: spill_smem_bytes)
__device__ __forceinline__ BeamSmem carve_beam_spill(unsigned char* base, unsigned char* slab, int L, int H) {
    BeamSmem s;
    s.bd = reinterpret_cast<double*>(slab);
    s.bi = reinterpret_cast<unsigned*>(slab + (size_t)L * 8);
    s.hash = reinterpret_cast<unsigned short*>(base);
    s.hmask = (unsigned)H - 1u;
    s.hbits = __ffs(H) - 1;
    const size_t tail = ((size_t)H * 2 + 15) & ~(size_t)15;
    s.spos = reinterpret_cast<int*>(base + tail);
    s.cbuf = reinterpret_cast<unsigned*>(base + tail + 128);
    return s;
}

// Row ring behind a warp's beam state (host: ring_smem_bytes in api.cuh):
// rows[ring_s][dp] f32 | bars[ring_s] u64, at `base` (16-byte aligned).  The
// fp32 screens of the lazy-key searches read whole candidate rows; a warp that
// loads them through registers gets one 4 KB row per ~1.1 us whatever it keeps
// in flight (tools/gather_probe2.cu), the bulk-copy engine delivers the same
// rows into shared memory 2-3 times faster and needs no registers for the rows
// in flight.  Lane 0 initialises the barriers once per kernel.
// Seen table in a per-warp global slab (L2-resident: 8 KB per warp), beam and
// scratch in shared memory: frees the shared memory the row ring needs without
// giving up resident warps.  One L2 round trip per expansion instead of a
// shared-memory one; the table is only ever touched by its own warp.
// smem layout: bd[L] | bi[L] | spos[32] | cbuf[kCbuf]  (host: beam_smem_bytes(L, 0))
__device__ __forceinline__ BeamSmem carve_beam_gh(unsigned char* base, unsigned char* slab, int L, int H) {
    BeamSmem s = carve_beam(base, L, 0);
    s.hash = reinterpret_cast<unsigned short*>(slab);
    s.hmask = (unsigned)H - 1u;
    s.hbits = __ffs(H) - 1;
    return s;
}

__device__ __forceinline__ size_t ring_smem_bytes_dev(int dp, int slots) {
    return ((size_t)slots * dp * 4 + (size_t)slots * 8 + 15) & ~(size_t)15;
}
__device__ __forceinline__ void carve_ring(BeamSmem& s, unsigned char* base, int dp, int slots) {
    s.ring_s = slots;
    if (!slots) return;
    s.ring = reinterpret_cast<float4*>(base);
    s.bars = reinterpret_cast<unsigned long long*>(base + (size_t)slots * dp * 4);
    if (lane_id() == 0) {
        for (int i = 0; i < slots; ++i) mbar_init(s.bars + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
}

struct SearchParams {
    const float* X;          // (n, dp)
    int dp;
    const int* adj;          // (n, R)
    int R;
    const int* deg;          // (n,)
    const int* starts;       // (s,)
    int s;
    const unsigned* X8;        // packed u8 rows (u8 mode only)
    int dw;
    int screen = 1;            // float data: fp32 pre-screen against a full beam (PK_SCREEN)
    unsigned* ubm = nullptr;   // counting mode: per-warp bitmaps of evaluated ids (exact unique count)
    int uwords = 0;            // 32-bit words per bitmap
    long long n_points = 0;    // n (bitmap size in counting mode)
    int prefetch = 1;          // L1 prefetch of the next expansion's adjacency row
    int prefetch_rows = 1;     // float data: L2 prefetch of every candidate row of an expansion (PK_PREFETCH_ROWS)
    int ring = 0;              // float data, lazy keys: slots of the per-warp row ring (0 = rows through registers)
    int* ticket = nullptr;     // dynamic work assignment: next unprocessed position of the launch (zeroed before it)
    unsigned char* ghash = nullptr;  // seen tables in global memory (carve_beam_gh): [warps][ghash_stride]
    size_t ghash_stride = 0;
    int lazy = 1;              // float data: lazy keys (fp32 screen values until a decision needs the exact one)
    int seed_only = 0;         // profiling aid (PK_SEED_ONLY): stop after seeding
    int seed_select = 1;       // exact integer modes: seed by selection instead of merges (PK_SEED_SELECT)
    // seeded beams per point id ([n][L] slots, [n] lengths): the build saves the
    // beam each inserted point starts its search from; a later search of the same
    // member query with the same L and start list starts from it instead of
    // seeding again (same start list + same L = same seeded beam)
    double* seed_bd = nullptr;
    unsigned* seed_bi = nullptr;
    int* seed_bl = nullptr;
    int seed_save = 0, seed_load = 0;
    // tensor-core pre-screen of the start set (tc_seed_mask): [n][seed_mw] bits,
    // set = the start may be among the point's take nearest
    const unsigned* seed_mask = nullptr;
    int seed_mw = 0;
    // exact integer start distances (u8 d = 128 builds, u8_seed_table): [n][s]
    const unsigned* seed_tab = nullptr;
    __device__ DataRef data() const { return DataRef{X, dp, X8, dw}; }
};

// Next position of a launch for this warp: a ticket from the shared counter
// (searches differ in length, so a static stride leaves most warps idle while
// the slowest finish their share), or the static stride without one.
__device__ __forceinline__ int next_position(int* ticket, int prev, int stride) {
    if (!ticket) return prev + stride;
    int v = 0;
    if (lane_id() == 0) v = atomicAdd(ticket, 1);
    return __shfl_sync(PK_FULL, v, 0);
}

// The same for kernels that give one item to a block: thread 0 takes a ticket,
// the block reads it after the next __syncthreads.  Items differ in cost
// (reverse groups of 65 .. 8,192 candidates), so a static stride leaves blocks
// idle at the end of a launch.  `ticket` null: static stride.
struct BlockTickets {
    int* slot;  // two shared ints, alternating
    int par;
    int stat;   // static position (no ticket counter)
    __device__ int first(int* ticket) {
        par = 0;
        stat = blockIdx.x;
        if (!ticket) return stat;
        if (threadIdx.x == 0) slot[0] = atomicAdd(ticket, 1);
        __syncthreads();
        return slot[0];
    }
    // call at the top of an item (takes the following item's ticket) ...
    __device__ void take_next(int* ticket) {
        if (!ticket) {
            stat += gridDim.x;
            return;
        }
        par ^= 1;
        if (threadIdx.x == 0) slot[par] = atomicAdd(ticket, 1);
    }
    // ... and at its end, after a __syncthreads
    __device__ int next(int* ticket) const { return ticket ? slot[par] : stat; }
};

// strictly increasing start list (every warp checks once per launch)
__device__ __forceinline__ bool starts_increasing(const SearchParams& P) {
    bool ok = true;
    for (int i = lane_id(); i + 1 < P.s; i += 32)
        if (!(__ldg(P.starts + i) < __ldg(P.starts + i + 1))) ok = false;
    return __all_sync(PK_FULL, ok);
}

template <class Dist>
struct WarpBeam {
    BeamSmem sm;
    int L;
    int bl;        // beam length (warp-uniform)
    int cursor;    // every entry below cursor is visited
    double ev_d;   // best evicted visited entry (warp-uniform; PK_APX in ev_i for a lazy key)
    unsigned ev_i;
    // optional visit log (build)
    unsigned* vlog_i;
    double* vlog_d;
    int vcap;
    int vl;
    unsigned* err;
    long long evals;  // distance evaluations (lane 0 count)
    unsigned qid = 0xffffffffu;  // member query id where known (build searches)
    unsigned* ubm;    // counting mode only: this warp's bitmap of evaluated ids
    long long uniq;   // distinct ids evaluated (the roofline's U)
    unsigned rt = 0;  // row ring: rows consumed so far by this warp (slot and barrier phase; survives init())
    bool lazy;        // lazy keys (float data, set by seed())
    long long exact;  // exact float64 evaluations in lazy mode (lane 0 count)

    __device__ void init(const BeamSmem& s_, int L_, unsigned* vi, double* vd, int vcap_, unsigned* err_) {
        sm = s_;
        L = L_;
        bl = 0;
        cursor = 0;
        ev_d = __longlong_as_double(0x7ff0000000000000LL);
        ev_i = 0xffffffffu;
        vlog_i = vi;
        vlog_d = vd;
        vcap = vcap_;
        vl = 0;
        err = err_;
        evals = 0;
        ubm = nullptr;
        uniq = 0;
        lazy = false;
        exact = 0;
        unsigned* h32 = reinterpret_cast<unsigned*>(sm.hash);
        for (unsigned h = lane_id(); h <= sm.hmask / 2; h += 32) h32[h] = 0xffffffffu;
        __syncwarp();
    }

    // Exact integer modes store the packed key (dist << 32 | id) in the bd slot
    // (one 64-bit compare per ordering decision instead of a float64 compare and
    // an id compare); dist_of() turns a stored slot back into the distance.
    __device__ __forceinline__ static double dist_of(double slot) {
        if constexpr (int_keys<Dist>::value)
            return (double)(unsigned)((unsigned long long)__double_as_longlong(slot) >> 32);
        else
            return slot;
    }
    __device__ __forceinline__ static unsigned long long kbits(double slot) {
        return (unsigned long long)__double_as_longlong(slot);
    }

    // Merge the candidates held by lanes with `valid` into the beam.
    // CheckDups: equal keys inside the batch are possible (duplicate start ids
    // in a user start list) -- keep the lowest lane.  Graph neighbours of one
    // expansion are distinct, so the walk skips that pass.
    template <bool CheckDups>
    __device__ void merge(double cd, unsigned cidf, bool valid) {
        const int lane = lane_id();
        double* bd = sm.bd;
        unsigned* bi = sm.bi;
        const unsigned cid = cidf & PK_IDMASK;  // cidf may carry PK_APX (stored with the entry)
        int pos = 0;
        bool keep = valid;
        // exact modes: distances are integers < 2^32, (dist, id) packs into one u64
        const unsigned long long mk = int_keys<Dist>::value ? ((unsigned long long)(unsigned)cd << 32) | cid : 0ull;
        if constexpr (int_keys<Dist>::value) {
            if (keep && bl == L && !(mk < kbits(bd[L - 1]))) keep = false;
            if (!__any_sync(PK_FULL, keep)) return;
            if (keep) {
                int lo = 0, hi = bl;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (kbits(bd[mid]) < mk) lo = mid + 1;
                    else hi = mid;
                }
                pos = lo;
                if (pos < bl && kbits(bd[pos]) == mk) keep = false;
            }
        } else {
            // a full beam rejects anything not better than its worst entry
            if (keep && bl == L && !key_lt(cd, cid, bd[L - 1], bi[L - 1] & PK_IDMASK)) keep = false;
            if (!__any_sync(PK_FULL, keep)) return;
            if (keep) {
                int lo = 0, hi = bl;
                while (lo < hi) {
                    int mid = (lo + hi) >> 1;
                    if (key_lt(bd[mid], bi[mid] & PK_IDMASK, cd, cid)) lo = mid + 1;
                    else hi = mid;
                }
                pos = lo;
                if (pos < bl && bd[pos] == cd && (bi[pos] & PK_IDMASK) == cid) keep = false;
            }
        }
        unsigned fb = __ballot_sync(PK_FULL, keep);
        if (!fb) return;
        if (CheckDups) {
            bool dupl = false;
            for (unsigned b = fb; b; b &= b - 1) {
                int j = __ffs(b) - 1;
                double dj = __shfl_sync(PK_FULL, cd, j);
                unsigned ij = __shfl_sync(PK_FULL, cid, j);
                if (j < lane && key_eq(dj, ij, cd, cid)) dupl = true;
            }
            keep = keep && !dupl;
            fb = __ballot_sync(PK_FULL, keep);
        }
        int rank = 0;
        if constexpr (int_keys<Dist>::value) {
            for (unsigned b = fb; b; b &= b - 1) {
                const unsigned long long kj = __shfl_sync(PK_FULL, mk, __ffs(b) - 1);
                rank += kj < mk;
            }
        } else {
            for (unsigned b = fb; b; b &= b - 1) {
                int j = __ffs(b) - 1;
                double dj = __shfl_sync(PK_FULL, cd, j);
                unsigned ij = __shfl_sync(PK_FULL, cid, j);
                if (key_lt(dj, ij, cd, cid)) ++rank;
            }
        }
        const int c = __popc(fb);
        if (keep) sm.spos[rank] = pos;
        __syncwarp();
        const int minpos = sm.spos[0];
        const int nbl = min(L, bl + c);
        // best evicted visited entry: every entry evicted by a merge is above
        // every key left in the beam, and the beam's L-th key never increases,
        // so later evictions are always below earlier ones -- the best one is
        // the lowest-positioned visited entry of the latest evicting merge (no
        // key comparison, so it also holds for lazy keys)
        int evn = 0x7fffffff;
        double evd = 0.0;
        unsigned evi = 0u;
        // shift the tail [minpos, bl) right, top-down in chunks of 32
        for (int top = bl - 1; top >= minpos; top -= 32) {
            const int e = top - lane;
            const bool act = e >= minpos;
            double de = 0.0;
            unsigned ie = 0;
            int ne = 0;
            if (act) {
                de = bd[e];
                ie = bi[e];
                int lo = 0, hi = c;
                while (lo < hi) {
                    int mid = (lo + hi) >> 1;
                    if (sm.spos[mid] <= e) lo = mid + 1;
                    else hi = mid;
                }
                ne = e + lo;
            }
            __syncwarp();
            if (act) {
                if (ne < L) {
                    bd[ne] = de;
                    bi[ne] = ie;
                } else if ((ie & PK_VIS) && ne < evn) {
                    evn = ne;
                    evd = de;
                    evi = ie & ~PK_VIS;
                }
            }
            __syncwarp();
        }
        if (__any_sync(PK_FULL, evn != 0x7fffffff)) {
            int mev = evn;
#pragma unroll
            for (int s = 16; s; s >>= 1) mev = min(mev, __shfl_xor_sync(PK_FULL, mev, s));
            const int src = __ffs(__ballot_sync(PK_FULL, evn == mev)) - 1;
            ev_d = __shfl_sync(PK_FULL, evd, src);
            ev_i = __shfl_sync(PK_FULL, evi, src);
        }
        const int np = pos + rank;
        if (keep && np < L) {
            bd[np] = int_keys<Dist>::value ? __longlong_as_double((long long)mk) : cd;
            bi[np] = cidf;
        }
        int mn = (keep && np < L) ? np : 0x7fffffff;
#pragma unroll
        for (int s = 16; s; s >>= 1) mn = min(mn, __shfl_xor_sync(PK_FULL, mn, s));
        if (mn < cursor) cursor = mn;
        bl = nbl;
        __syncwarp();
    }

    // ---- lazy keys (float data) -------------------------------------------------
    // Lane i < cnt: the level-1 lazy key of candidate cid (fp32 screen value,
    // PK_APX|PK_A32 in cidf); where the fp32 value is unusable (underflow /
    // overflow) the float64 one (PK_APX, or exact when it is 0).
    // fp32 screens through the row ring: every lane of `mask` holds a row id and
    // gets its row's screen value (other lanes keep `mine`).  Rows stream through
    // the ring_s slots: the lane that holds an id issues its bulk copy, the warp
    // waits for the oldest slot, screens it from shared memory and hands the slot
    // to the next row, so ring_s rows are in flight until the last ones drain.
    template <class D>
    __device__ float ring_screens(const SearchParams& P, const D& dist, unsigned id, unsigned mask, float mine) {
        const int lane = lane_id();
        const int S = sm.ring_s, nv = P.dp >> 2;
        const unsigned bytes = (unsigned)P.dp * 4u;
        const int sh = 31 - __clz(S);
        unsigned pend = mask;  // rows not requested yet
        unsigned ti = rt;      // next request's sequence number
        auto issue = [&]() {
            const int j = __ffs(pend) - 1;
            pend &= pend - 1u;
            if (lane == j) {
                const int slot = (int)(ti & (unsigned)(S - 1));
                mbar_expect_tx(sm.bars + slot, bytes);
                bulk_g2s(sm.ring + (size_t)slot * nv, P.X + (size_t)id * P.dp, bytes, sm.bars + slot);
            }
            ++ti;
        };
        for (int i = 0; i < S && pend; ++i) issue();
        for (unsigned w = mask; w; w &= w - 1u) {
            const int j = __ffs(w) - 1;
            const int slot = (int)(rt & (unsigned)(S - 1));
            mbar_wait(sm.bars + slot, (rt >> sh) & 1u);
            const float v = dist.screen_smem(sm.ring + (size_t)slot * nv);
            if (lane == j) mine = v;
            ++rt;
            __syncwarp();  // every lane has read the slot before it is refilled
            if (pend) issue();
        }
        return mine;
    }

    template <class D>
    __device__ double approx(const SearchParams& P, const D& dist, unsigned cid, int cnt, unsigned& cidf) {
        const int lane = lane_id();
        float mine = 0.f;
        if constexpr (uses_ring<D>::value) {
            mine = ring_screens(P, dist, cid, cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u), 0.f);
        } else {
            for (int j = 0; j < cnt; j += 2) {
                const int j1 = j + 1 < cnt ? j + 1 : j;
                const float s0 = dist.screen(P.X, __shfl_sync(PK_FULL, cid, j));
                const float s1 = dist.screen(P.X, __shfl_sync(PK_FULL, cid, j1));
                if (lane == j) mine = s0;
                if (lane == j1) mine = s1;
            }
        }
        double v = (double)mine;
        cidf = cid | PK_APX | PK_A32;
        const unsigned bad = __ballot_sync(PK_FULL, lane < cnt && !screen_usable(mine));
        for (unsigned b = bad; b; b &= b - 1) {
            const int j = __ffs(b) - 1;
            const double d64 = dist.dscreen(P.X, __shfl_sync(PK_FULL, cid, j));
            if (lane == j) {
                v = d64;
                cidf = d64 == 0.0 ? cid : (cid | PK_APX);
            }
        }
        return v;
    }

    // One refinement step of a lazy key: A32 -> A64 (warp-cooperative float64,
    // `coop` lanes one at a time) or A64 -> exact (lane-parallel sequential
    // float64, `seq` lanes).  Lane j refines (v, f) of row id.
    template <class D>
    __device__ void refine(const SearchParams& P, const D& dist, unsigned coop, unsigned seq, unsigned id, double& v,
                           unsigned& f) {
        const int lane = lane_id();
        for (unsigned b = coop; b; b &= b - 1) {
            const int j = __ffs(b) - 1;
            const double d64 = dist.dscreen(P.X, __shfl_sync(PK_FULL, id, j));
            if (lane == j) {
                v = d64;
                f = d64 == 0.0 ? (f & ~PK_LAZYF) : ((f & ~PK_A32) | PK_APX);
            }
        }
        if (seq) {
            if ((seq >> lane) & 1u) {
                v = dist.eval_one(P.X, (int)id);
                f &= ~PK_LAZYF;
            }
            if (lane == 0) exact += __popc(seq);
        }
    }

    // Make every ordering decision of the coming merge certain.  Candidates
    // certainly above the worst entry of a full beam, and ids already in the
    // beam (lossy seen table), are dropped.  Every other lazy key that is in an
    // uncertain pair -- candidate vs beam entry, candidate vs candidate, and
    // (after a refinement moved a beam key) adjacent beam entries -- is refined
    // one level, until no uncertain pair is left.  Afterwards key_lt on the
    // stored values is the exact (dist, id) order of every pair merge() compares.
    template <class D>
    __device__ void resolve(const SearchParams& P, const D& dist, double& cd, unsigned& cidf, bool& valid) {
        const int lane = lane_id();
        unsigned* bi = sm.bi;
        double* bd = sm.bd;
        int* work = sm.spos;  // beam positions to refine (merge() reuses spos afterwards)
        const unsigned cid = cidf & PK_IDMASK;
        bool dirty = false;   // a beam key was refined: re-check adjacent beam pairs
        for (;;) {
            const double clo = key_lo(cd, cidf), chi = key_hi(cd, cidf);
            int first = 0, last = 0;
            if (valid) {
                // lo and hi are non-decreasing along the beam (adjacent pairs are certain)
                int lo = 0, hi = bl;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (key_hi(bd[mid], bi[mid]) < clo) lo = mid + 1;
                    else hi = mid;
                }
                first = lo;
                hi = bl;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (key_lo(bd[mid], bi[mid]) <= chi) lo = mid + 1;
                    else hi = mid;
                }
                last = lo;
                if (bl == L && first == bl) {
                    valid = false;  // certainly above the worst entry of the full beam
                } else {
                    for (int e = first; e < last; ++e)
                        if ((bi[e] & PK_IDMASK) == cid) valid = false;  // already in the beam
                }
            }
            const bool capx = valid && (cidf & PK_APX);
            // candidate vs beam: an overlapping pair is uncertain unless both are exact
            bool own = false;
            if (capx && first < last) own = true;
            // candidate vs candidate
            const unsigned vb = __ballot_sync(PK_FULL, valid);
            for (unsigned b = vb; b; b &= b - 1) {
                const int j = __ffs(b) - 1;
                const double dj = __shfl_sync(PK_FULL, cd, j);
                const unsigned fj = __shfl_sync(PK_FULL, cidf, j);
                if (capx && j != lane && !key_certain_lt(dj, fj, cd, cidf) && !key_certain_lt(cd, cidf, dj, fj))
                    own = true;
            }
            // beam entries to refine: lazy entries overlapping a valid candidate
            int nw = 0;
            int e = valid ? first : last;
            for (;;) {
                while (e < last && !(bi[e] & PK_APX)) ++e;
                const bool has = e < last;
                const unsigned hb = __ballot_sync(PK_FULL, has);
                if (!hb) break;
                const int at = nw + warp_excl_prefix(hb);
                if (has && at < 32) work[at] = e;
                nw = min(32, nw + __popc(hb));
                if (has) ++e;
                if (nw >= 32) break;
            }
            // after a refinement of beam keys: adjacent beam pairs that became uncertain
            if (dirty) {
                for (int base = 0; base + 1 < bl && nw < 32; base += 32) {
                    const int x = base + lane;
                    bool unc = false;
                    if (x + 1 < bl) unc = !key_certain_lt(bd[x], bi[x], bd[x + 1], bi[x + 1]);
                    const unsigned ub = __ballot_sync(PK_FULL, unc);
                    // refine both lazy members of each uncertain pair
                    const bool w0 = unc && (bi[x] & PK_APX), w1 = unc && (bi[x + 1] & PK_APX);
                    const unsigned b0 = __ballot_sync(PK_FULL, w0), b1 = __ballot_sync(PK_FULL, w1);
                    int at = nw + warp_excl_prefix(b0);
                    if (w0 && at < 32) work[at] = x;
                    nw = min(32, nw + __popc(b0));
                    at = nw + warp_excl_prefix(b1);
                    if (w1 && at < 32) work[at] = x + 1;
                    nw = min(32, nw + __popc(b1));
                    (void)ub;
                }
            }
            const unsigned ob = __ballot_sync(PK_FULL, own);
            if (!ob && !nw) break;
            __syncwarp();
            // refine the candidates
            {
                const unsigned coop = __ballot_sync(PK_FULL, own && (cidf & PK_A32));
                const unsigned seq = ob & ~coop;
                double v = cd;
                unsigned f = cidf;
                refine(P, dist, coop, seq, cid, v, f);
                if (own) {
                    cd = v;
                    cidf = f;
                }
            }
            // refine the listed beam entries (lane j takes work[j]; duplicates refine twice, harmlessly)
            if (nw) {
                const int pos = lane < nw ? work[lane] : 0;
                unsigned f = lane < nw ? bi[pos] : 0u;
                double v = lane < nw ? bd[pos] : 0.0;
                const bool lz = lane < nw && (f & PK_APX);
                const unsigned coop = __ballot_sync(PK_FULL, lz && (f & PK_A32));
                const unsigned seq = __ballot_sync(PK_FULL, lz) & ~coop;
                refine(P, dist, coop, seq, f & PK_IDMASK, v, f);
                __syncwarp();
                if (lz) {
                    bd[pos] = v;
                    bi[pos] = f;
                }
                __syncwarp();
                dirty = true;
            }
        }
    }

    // lazy-mode batch insert: approx -> resolve -> merge
    template <bool CheckDups, class D>
    __device__ void insert_lazy(const SearchParams& P, const D& dist, unsigned cid, int cnt) {
        unsigned cidf;
        PK_PT_BEGIN
        double v = approx(P, dist, cid, cnt, cidf);
        PK_PT_NEXT(2);
        bool valid = lane_id() < cnt;
        resolve(P, dist, v, cidf, valid);
        PK_PT_NEXT(3);
        merge<CheckDups>(v, cidf, valid);
        PK_PT_END(4);
    }

    // build: exact distances for the visit-log entries logged with lazy keys
    template <class D>
    __device__ void finalize_log(const SearchParams& P, const D& dist) {
        const int lane = lane_id();
        const int nl = min(vl, vcap);
        for (int x = lane; x - lane < nl; x += 32) {
            const unsigned id = x < nl ? vlog_i[x] : 0u;
            const bool apx = x < nl && (id & PK_APX);
            const unsigned nb_ = __ballot_sync(PK_FULL, apx);
            if (lane == 0) exact += __popc(nb_);
            if (apx) {
                vlog_d[x] = dist.eval_one(P.X, (int)(id & PK_IDMASK));
                vlog_i[x] = id & PK_IDMASK;
            }
        }
        __syncwarp();
    }

    // counting mode: mark the ids held by lanes < cnt, count the first sightings
    __device__ void count_unique(unsigned id, int cnt) {
        if (!ubm) return;
        const int lane = lane_id();
        bool fresh = false;
        if (lane < cnt) fresh = !(atomicOr(ubm + (id >> 5), 1u << (id & 31)) & (1u << (id & 31)));
        const unsigned b = __ballot_sync(PK_FULL, fresh);
        uniq += __popc(b);
    }
    __device__ void begin_counting(unsigned* bm, int words) {
        ubm = bm;
        if (!bm) return;
        for (int w = lane_id(); w < words; w += 32) bm[w] = 0u;
        __syncwarp();
        __threadfence_block();
    }

    // Seed with the start set (batch insert of ceil(s/32) chunks).  `unique`:
    // the start list is strictly increasing (sample_starts' sorted draw), so a
    // batch cannot hold equal keys and the duplicate pass of merge is skipped.
    template <class D>
    __device__ void seed(const SearchParams& P, const D& dist, bool hash_starts, bool unique) {
        const int lane = lane_id();
        if constexpr (has_screen<D>::value) lazy = P.screen && P.lazy && P.dp <= 128 * D::kQV;
        if constexpr (has_screen<D>::value) {
            if (lazy && unique && !hash_starts && P.s > 64 && P.seed_select && L >= 128 &&
                2 * P.s <= (int)sm.hmask + 1) {
                if (seed_select_lazy(P, dist)) return;
            }
        }
        if constexpr (int_keys<D>::value) {
            // needs: L a power of two >= 128 (the 1 KB histogram lives in bd), the
            // s u32 distances fit the seen table
            if (unique && !hash_starts && P.s > 32 && P.seed_select && L >= 128 && (L & (L - 1)) == 0 &&
                2 * P.s <= (int)sm.hmask + 1) {
                seed_select(P, dist);
                return;
            }
        }
        for (int b = 0; b < P.s; b += 32) {
            const int cnt = min(32, P.s - b);
            unsigned id = lane < cnt ? (unsigned)P.starts[b + lane] : 0u;
            if (hash_starts && lane < cnt) seen_or_insert(sm.hash, sm.hmask, sm.hbits, id);
            count_unique(id, cnt);
            if constexpr (has_screen<D>::value) {
                if (lazy) {
                    if (lane == 0) evals += cnt;
                    if (unique) insert_lazy<false>(P, dist, id, cnt);
                    else insert_lazy<true>(P, dist, id, cnt);
                    continue;
                }
            }
            double dd = dist.eval(P.X, (int)id, cnt);
            if (lane == 0) evals += cnt;
            if (unique) merge<false>(dd, id, lane < cnt);
            else merge<true>(dd, id, lane < cnt);
        }
    }

    __device__ unsigned radix_kth(const unsigned* vals, int s, int take, unsigned* bins, int& need) {
        return warp_radix_kth(vals, s, take, bins, need);
    }

    // Seeding by selection for lazy keys (float data, strictly increasing start
    // list): every start's fp32 screen value a goes to the (still empty) seen
    // table, the take-th smallest value T is found by a radix select, and only
    // the starts with a (1 - eps) <= T (1 + eps) -- every other start is
    // certainly above the take-th key -- are inserted (resolve + merge, 32 at a
    // time).  Top-L is associative, so the beam equals the one after inserting
    // all starts.  Returns false (nothing changed) if a screen value is unusable.
    template <class D>
    __device__ bool seed_select_lazy(const SearchParams& P, const D& dist) {
        const int lane = lane_id();
        const int s = P.s;
        unsigned* asc = reinterpret_cast<unsigned*>(sm.hash);  // [s] fp32 screen values (bits)
        unsigned* bins = reinterpret_cast<unsigned*>(sm.bd);   // [256] histogram (L >= 128)
        // tensor-core pre-screen (tc_seed_mask): only the starts whose low bound is
        // not above the take-th high bound get an fp32 screen
        const unsigned* mrow = nullptr;
        if (P.seed_mask) mrow = P.seed_mask + (size_t)((dist.q - P.X) / P.dp) * P.seed_mw;
        bool bad = false;
        for (int b = 0; b < s; b += 32) {
            const int cnt = min(32, s - b);
            const unsigned id = lane < cnt ? (unsigned)P.starts[b + lane] : 0u;
            bool want = lane < cnt;
            if (mrow) want = want && ((mrow[b >> 5] >> lane) & 1u);
            unsigned wm = __ballot_sync(PK_FULL, want);
            float mine = __uint_as_float(0x7f800000u);
            if constexpr (uses_ring<D>::value) {
                mine = ring_screens(P, dist, id, wm, mine);
                wm = 0u;
            }
            while (wm) {
                const int j = __ffs(wm) - 1;
                wm &= wm - 1u;
                const int j1 = wm ? __ffs(wm) - 1 : j;
                if (wm) wm &= wm - 1u;
                const float s0 = dist.screen(P.X, __shfl_sync(PK_FULL, id, j));
                const float s1 = dist.screen(P.X, __shfl_sync(PK_FULL, id, j1));
                if (lane == j) mine = s0;
                if (lane == j1) mine = s1;
            }
            __syncwarp();
            if (lane < cnt) {
                if (want) bad |= !screen_usable(mine);
                asc[b + lane] = want ? __float_as_uint(mine) : 0x7f800000u;
            }
        }
        const bool any_bad = __any_sync(PK_FULL, bad);
        if (!any_bad) {
            for (int b = 0; b < s; b += 32) count_unique(lane < min(32, s - b) ? (unsigned)P.starts[b + lane] : 0u,
                                                         min(32, s - b));
            if (lane == 0) evals += s;
            __syncwarp();
            const int take = min(L, s);
            int need = 0;
            const unsigned T = radix_kth(asc, s, take, bins, need);
            const double thr = (double)__uint_as_float(T) * (1.0 + kEps32) / (1.0 - kEps32);
            // candidates in index order, staged in cbuf (start-list positions):
            // each chunk appends <= 32, full groups of 32 are inserted at once
            int nc = 0;
            auto insert = [&](int cnt) {
                __syncwarp();
                const unsigned xi = lane < cnt ? sm.cbuf[lane] : 0u;
                unsigned cidf = lane < cnt ? ((unsigned)P.starts[xi] | PK_APX | PK_A32) : 0u;
                double v = lane < cnt ? (double)__uint_as_float(asc[xi]) : 0.0;
                bool valid = lane < cnt;
                const unsigned rest = lane + cnt < nc ? sm.cbuf[lane + cnt] : 0u;
                __syncwarp();
                if (lane + cnt < nc) sm.cbuf[lane] = rest;
                nc -= cnt;
                __syncwarp();
                resolve(P, dist, v, cidf, valid);
                merge<false>(v, cidf, valid);
            };
            for (int b = 0; b < s; b += 32) {
                const int x = b + lane;
                const bool cand = x < s && (double)__uint_as_float(asc[x]) <= thr;
                const unsigned cb = __ballot_sync(PK_FULL, cand);
                if (cand) sm.cbuf[nc + __popc(cb & ((1u << lane) - 1u))] = (unsigned)x;
                nc += __popc(cb);
                if (nc >= 32) insert(32);
            }
            if (nc > 0) insert(nc);
        }
        // the seen table was scratch: empty it again
        unsigned* h32 = reinterpret_cast<unsigned*>(sm.hash);
        for (unsigned h = lane_id(); h <= sm.hmask / 2; h += 32) h32[h] = 0xffffffffu;
        __syncwarp();
        return !any_bad;
    }

    // Seeding by selection (exact integer modes, strictly increasing start list):
    // the beam after merging every start is the sorted top-min(L, s) of their
    // keys (dist, id); id order = start-list order, so the keys are (dist,
    // index).  Distances go to the (still empty) seen table as u32 scratch, a
    // radix select on dist (4 passes of 8 bits, histogram in the bd area) finds
    // the L-th key, the selected entries are packed into bd and sorted (warp
    // bitonic over L), and the seen table is cleared again.  Replaces ceil(s/32)
    // merges of a growing beam.
    template <class D>
    __device__ void seed_select(const SearchParams& P, const D& dist) {
        const int lane = lane_id();
        const int s = P.s;
        unsigned* dsc = reinterpret_cast<unsigned*>(sm.hash);  // [s] seed distances
        unsigned* bins = reinterpret_cast<unsigned*>(sm.bd);   // [256] histogram
        if (P.seed_tab && qid != 0xffffffffu) {
            // precomputed on the integer tensor cores: the same exact distances
            const unsigned* row = P.seed_tab + (size_t)qid * s;
            for (int x = lane; x < s; x += 32) dsc[x] = __ldg(row + x);
        } else {
            for (int b = 0; b < s; b += 32) {
                const int cnt = min(32, s - b);
                const unsigned id = lane < cnt ? (unsigned)P.starts[b + lane] : 0u;
                count_unique(id, cnt);
                const double dd = dist.eval(P.X, (int)id, cnt);
                if (lane == 0) evals += cnt;
                if (lane < cnt) dsc[b + lane] = (unsigned)dd;
            }
        }
        __syncwarp();
        const int take = min(L, s);
        int need = take;
        const unsigned T = radix_kth(dsc, s, take, bins, need);  // `need` entries equal to T are taken
        // collect in index order: every d < T, the first `need` with d == T
        unsigned long long* bk = reinterpret_cast<unsigned long long*>(sm.bd);
        int got = 0, eq = 0;
        for (int b = 0; b < s; b += 32) {
            const int x = b + lane;
            const unsigned v = x < s ? dsc[x] : 0xffffffffu;
            const bool isq = x < s && v == T;
            const unsigned qb = __ballot_sync(PK_FULL, isq);
            const bool sel = x < s && (v < T || (isq && eq + __popc(qb & ((1u << lane) - 1u)) < need));
            const unsigned sb = __ballot_sync(PK_FULL, sel);
            if (sel) {
                const unsigned id = (unsigned)P.starts[x];
                bk[got + __popc(sb & ((1u << lane) - 1u))] = ((unsigned long long)v << 32) | id;
            }
            got += __popc(sb);
            eq += __popc(qb);
        }
        __syncwarp();
        // pad to L (a power of two) and sort the packed keys
        for (int x = take + lane; x < L; x += 32) bk[x] = ~0ull;
        __syncwarp();
        for (int k = 2; k <= L; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = lane; i < L; i += 32) {
                    const int x = i ^ j;
                    if (x > i) {
                        const unsigned long long a = bk[i], b = bk[x];
                        if ((b < a) == ((i & k) == 0)) {
                            bk[i] = b;
                            bk[x] = a;
                        }
                    }
                }
                __syncwarp();
            }
        for (int x = lane; x < take; x += 32) sm.bi[x] = (unsigned)(bk[x] & 0xffffffffull);
        bl = take;
        cursor = 0;
        // the seen table was scratch: empty it again
        unsigned* h32 = reinterpret_cast<unsigned*>(sm.hash);
        for (unsigned h = lane_id(); h <= sm.hmask / 2; h += 32) h32[h] = 0xffffffffu;
        __syncwarp();
    }

    // seeded-beam cache (SearchParams::seed_*): save after seed(), load instead of it
    __device__ void save_seed(const SearchParams& P, unsigned q) {
        const size_t o = (size_t)q * L;
        for (int x = lane_id(); x < bl; x += 32) {
            P.seed_bd[o + x] = sm.bd[x];
            P.seed_bi[o + x] = sm.bi[x];
        }
        if (lane_id() == 0) P.seed_bl[q] = bl;
    }
    template <class D>
    __device__ void load_seed(const SearchParams& P, const D&, unsigned q) {
        if constexpr (has_screen<D>::value) lazy = P.screen && P.lazy && P.dp <= 128 * D::kQV;
        const size_t o = (size_t)q * L;
        bl = P.seed_bl[q];
        for (int x = lane_id(); x < bl; x += 32) {
            sm.bd[x] = P.seed_bd[o + x];
            sm.bi[x] = P.seed_bi[o + x];
        }
        cursor = 0;
        __syncwarp();
    }

    // First unvisited beam position at or after the cursor, -1 if none.
    __device__ int next_unvisited() {
        const int lane = lane_id();
        for (int base = cursor; base < bl; base += 32) {
            int e = base + lane;
            bool unv = e < bl && !(sm.bi[e] & PK_VIS);
            unsigned b = __ballot_sync(PK_FULL, unv);
            if (b) return base + __ffs(b) - 1;
        }
        return -1;
    }

    // Run the walk to completion.
    template <class D>
    __device__ void walk(const SearchParams& P, const D& dist) {
        const int lane = lane_id();
        for (;;) {
            PK_PT_BEGIN
            const int pos = next_unvisited();
            if (pos < 0) break;
            const unsigned pf = sm.bi[pos] & PK_IDAPX;
            const unsigned p = pf & PK_IDMASK;
            const double pd = dist_of(sm.bd[pos]);
            __syncwarp();
            if (lane == 0) {
                sm.bi[pos] = pf | PK_VIS;
                if (vlog_i) {
                    if (vl < vcap) {
                        vlog_i[vl] = pf;
                        vlog_d[vl] = pd;
                    } else {
                        atomicOr(err, ERR_VISIT_OVERFLOW);
                    }
                }
            }
            ++vl;
            cursor = pos + 1;
            __syncwarp();
            const int* row = P.adj + (size_t)p * P.R;
            // the degree and the first 64 row slots are loaded together (slots
            // past the degree are masked), so the two loads do not serialise
            int w_a = lane < P.R ? __ldg(row + lane) : -1;
            int w_b = lane + 32 < P.R ? __ldg(row + lane + 32) : -1;
            const int nd = __ldg(P.deg + p);
            if (nd == 0) {
                // empty row (early build batches: most start points are not inserted
                // yet): expanding it changes nothing, and neither does expanding the
                // following unvisited entries with empty rows -- visit that run at once
                visit_empty_run(P);
                continue;
            }
            if (P.prefetch) {
                // prefetch the adjacency row of the next unvisited entry: it is
                // the next expansion unless this one inserts something closer
                const int pn = next_unvisited();
                if (pn >= 0 && lane < 2) {
                    const int* nrow = P.adj + (size_t)(sm.bi[pn] & PK_IDMASK) * P.R + 32 * lane;
                    if (32 * lane < P.R) asm volatile("prefetch.global.L1 [%0];" ::"l"(nrow));
                }
            }
            int c = 0;
            // ring kernels (seen table in global memory): the sets of the first 64
            // slots are read together, one L2 round trip instead of two
            uint2 v_a = make_uint2(0u, 0u), v_b = v_a;
            if constexpr (uses_ring<D>::value) {
                if (lane >= nd) w_a = -1;
                if (lane + 32 >= nd) w_b = -1;
                if (w_a >= 0) v_a = seen_load(sm.hash, sm.hmask, (unsigned)w_a);
                if (w_b >= 0) v_b = seen_load(sm.hash, sm.hmask, (unsigned)w_b);
            }
            for (int e0 = 0; e0 < nd; e0 += 32) {
                int w = e0 + lane < nd ? (e0 == 0 ? w_a : e0 == 32 ? w_b : __ldg(row + e0 + lane)) : -1;
                bool cand = w >= 0;
                if (cand) {
                    bool seen;
                    if constexpr (uses_ring<D>::value)
                        seen = e0 == 0   ? seen_apply(sm.hash, sm.hmask, sm.hbits, (unsigned)w, v_a)
                               : e0 == 32 ? seen_apply(sm.hash, sm.hmask, sm.hbits, (unsigned)w, v_b)
                                          : seen_or_insert(sm.hash, sm.hmask, sm.hbits, (unsigned)w);
                    else
                        seen = seen_or_insert(sm.hash, sm.hmask, sm.hbits, (unsigned)w);
                    if (seen) cand = false;
                }
                unsigned b = __ballot_sync(PK_FULL, cand);
                const int nb = __popc(b);
                if (c + nb > kCbuf) {  // very wide rows: flush before the buffer overflows
                    flush(P, dist, c);
                    c = 0;
                }
                if (cand) sm.cbuf[c + warp_excl_prefix(b)] = (unsigned)w;
                c += nb;
            }
            __syncwarp();
            PK_PT_END(0);
            flush(P, dist, c);
        }
    }

    // Visit, in beam order, the unvisited entries from the cursor on whose rows
    // are empty, up to the first unvisited entry with a non-empty row.
    __device__ void visit_empty_run(const SearchParams& P) {
        const int lane = lane_id();
        for (int base = cursor; base < bl; base += 32) {
            const int e = base + lane;
            const unsigned iv = e < bl ? sm.bi[e] : PK_VIS;
            const bool unv = !(iv & PK_VIS);
            const int dg = unv ? __ldg(P.deg + (iv & PK_IDMASK)) : 0;
            const unsigned stop = __ballot_sync(PK_FULL, unv && dg > 0);
            const unsigned before = stop ? (1u << (__ffs(stop) - 1)) - 1u : 0xffffffffu;
            const unsigned run = __ballot_sync(PK_FULL, unv && dg == 0) & before;
            if ((run >> lane) & 1u) {
                sm.bi[e] = iv | PK_VIS;
                if (vlog_i) {
                    const int at = vl + __popc(run & ((1u << lane) - 1u));
                    if (at < vcap) {
                        vlog_i[at] = iv & PK_IDAPX;
                        vlog_d[at] = dist_of(sm.bd[e]);
                    } else {
                        atomicOr(err, ERR_VISIT_OVERFLOW);
                    }
                }
            }
            vl += __popc(run);
            if (stop) {
                cursor = base + __ffs(stop) - 1;
                break;
            }
            cursor = min(base + 32, bl);
        }
        __syncwarp();
    }

    // Ask L2 for every row of this batch of candidates at once (lane l takes
    // 128-byte line l of each row).  The fp32 screens then read the rows two at
    // a time -- all the registers allow -- and find them on their way from HBM
    // instead of issuing one HBM round trip per pair.
    __device__ void prefetch_rows(const SearchParams& P, unsigned cid, int cnt) {
        const int lane = lane_id();
        const int lines = (P.dp * 4 + 127) >> 7;
        for (int j = 0; j < cnt; ++j) {
            const unsigned id = __shfl_sync(PK_FULL, cid, j);
            const char* r = reinterpret_cast<const char*>(P.X + (size_t)id * P.dp);
            for (int l = lane; l < lines; l += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(r + ((size_t)l << 7)));
        }
    }

    // evaluate and merge the c candidates staged in cbuf
    template <class D>
    __device__ void flush(const SearchParams& P, const D& dist, int c) {
        const int lane = lane_id();
        __syncwarp();
        for (int g = 0; g < c; g += 32) {
            int cnt = min(32, c - g);
            unsigned cid = lane < cnt ? sm.cbuf[g + lane] : 0u;
            if (lane == 0) evals += cnt;
            count_unique(cid, cnt);
            if constexpr (has_screen<D>::value) {
                if (lazy) {
                    PK_PT_BEGIN
                    if constexpr (!uses_ring<D>::value)
                        if (P.prefetch_rows && cnt > 2) prefetch_rows(P, cid, cnt);
                    PK_PT_END(1);
                    insert_lazy<false>(P, dist, cid, cnt);
                    continue;
                }
            }
            if constexpr (has_screen<D>::value) {
                // float data, full beam: drop the candidates whose fp32 lower bound
                // already exceeds the worst key (they would be rejected by merge);
                // only the rest pay the sequential float64 evaluation
                if (bl == L && P.screen && P.dp >= 256 && P.dp <= 128 * D::kQV) {
                    const double wd = sm.bd[L - 1];
                    bool drop = false;
                    if constexpr (uses_ring<D>::value) {
                        const float sv = ring_screens(P, dist, cid, cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u), 0.f);
                        drop = lane < cnt && sv > 1e-20f && sv < 1e30f && (double)sv * (1.0 - kScreenEps) > wd;
                    } else {
                        for (int j = 0; j < cnt; j += 2) {
                            const int j1 = j + 1 < cnt ? j + 1 : j;
                            const float s0 = dist.screen(P.X, __shfl_sync(PK_FULL, cid, j));
                            const float s1 = dist.screen(P.X, __shfl_sync(PK_FULL, cid, j1));
                            if (lane == j && s0 > 1e-20f && s0 < 1e30f && (double)s0 * (1.0 - kScreenEps) > wd) drop = true;
                            if (lane == j1 && s1 > 1e-20f && s1 < 1e30f && (double)s1 * (1.0 - kScreenEps) > wd) drop = true;
                        }
                    }
                    const bool keep = lane < cnt && !drop;
                    const unsigned b = __ballot_sync(PK_FULL, keep);
                    cnt = __popc(b);
                    if (!cnt) continue;
                    __syncwarp();
                    if (keep) sm.cbuf[g + warp_excl_prefix(b)] = cid;
                    __syncwarp();
                    cid = lane < cnt ? sm.cbuf[g + lane] : 0u;
                }
            }
            double dd = dist.eval(P.X, (int)cid, cnt);
            merge<false>(dd, cid, lane < cnt);
        }
        __syncwarp();
    }

    // Member-query output: first kk entries of the beam without `self`, then
    // the best evicted visited entry if still short.  Returns the count.
    __device__ int emit(unsigned self, int kk, long long* out_ids, double* out_d) {
        return emit(self, kk, out_ids, out_d, [](unsigned) { return 0.0; });
    }
    // lazy keys: emitted entries get their exact value from exact_of(id)
    template <class F>
    __device__ int emit(unsigned self, int kk, long long* out_ids, double* out_d, const F& exact_of) {
        const int lane = lane_id();
        int got = 0;
        for (int base = 0; base < bl && got < kk; base += 32) {
            int e = base + lane;
            const unsigned f = e < bl ? sm.bi[e] : 0u;
            unsigned id = e < bl ? (f & PK_IDMASK) : self;
            bool ok = e < bl && id != self;
            unsigned b = __ballot_sync(PK_FULL, ok);
            int o = got + warp_excl_prefix(b);
            const bool out = ok && o < kk;
            const bool apx = out && (f & PK_APX);
            double v = e < bl ? dist_of(sm.bd[e]) : 0.0;
            if (__any_sync(PK_FULL, apx)) {
                if (apx) v = exact_of(id);
                const unsigned nb_ = __ballot_sync(PK_FULL, apx);
            if (lane == 0) exact += __popc(nb_);
            }
            if (out) {
                out_ids[o] = id;
                out_d[o] = v;
            }
            got += __popc(b);
        }
        got = min(got, kk);
        // best evicted visited entry (warp-uniform, see merge)
        const double bd_ = ev_d;
        const unsigned bi_ = ev_i;
        if (got < kk && bi_ != 0xffffffffu && (bi_ & PK_IDMASK) != self) {
            if (lane == 0) {
                out_ids[got] = bi_ & PK_IDMASK;
                out_d[got] = (bi_ & PK_APX) ? exact_of(bi_ & PK_IDMASK) : dist_of(bd_);
            }
            ++got;
        }
        return got;
    }
};

// ---- warp bitonic sort of (dist, id) keys in shared memory ----------------------
// P must be a power of two; entries beyond the live count must hold (+inf, ~0).
__device__ __forceinline__ void warp_sort(double* kd, unsigned* ki, int P) {
    const int lane = lane_id();
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < P; i += 32) {
                int x = i ^ j;
                if (x > i) {
                    double a = kd[i], b = kd[x];
                    unsigned ia = ki[i], ib = ki[x];
                    bool asc = (i & k) == 0;
                    bool gt = key_lt(b, ib, a, ia);
                    if (gt == asc) {
                        kd[i] = b; kd[x] = a;
                        ki[i] = ib; ki[x] = ia;
                    }
                }
            }
            __syncwarp();
        }
    }
}

// Same sort carrying a 16-bit payload (the staged-row slot of each key).
__device__ __forceinline__ void warp_sort_pos(double* kd, unsigned* ki, unsigned short* kp, int P) {
    const int lane = lane_id();
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < P; i += 32) {
                int x = i ^ j;
                if (x > i) {
                    double a = kd[i], b = kd[x];
                    unsigned ia = ki[i], ib = ki[x];
                    bool asc = (i & k) == 0;
                    if (key_lt(b, ib, a, ia) == asc) {
                        kd[i] = b; kd[x] = a;
                        ki[i] = ib; ki[x] = ia;
                        unsigned short pa = kp[i];
                        kp[i] = kp[x];
                        kp[x] = pa;
                    }
                }
            }
            __syncwarp();
        }
    }
}

__device__ __forceinline__ int warp_unique_pos(double* kd, unsigned* ki, unsigned short* kp, int c, unsigned self) {
    const int lane = lane_id();
    int out = 0;
    for (int base = 0; base < c; base += 32) {
        int i = base + lane;
        double d = 0.0;
        unsigned id = self;
        unsigned short ps = 0;
        bool keep = false;
        if (i < c) {
            d = kd[i];
            id = ki[i];
            ps = kp[i];
            keep = id != self && !(i > 0 && ki[i - 1] == id && kd[i - 1] == d);
        }
        unsigned b = __ballot_sync(PK_FULL, keep);
        __syncwarp();
        if (keep) {
            int o = out + warp_excl_prefix(b);
            kd[o] = d;
            ki[o] = id;
            kp[o] = ps;
        }
        out += __popc(b);
        __syncwarp();
    }
    return out;
}

// Drop duplicate keys (same id => same dist) and `self`, in place; returns count.
__device__ __forceinline__ int warp_unique(double* kd, unsigned* ki, int c, unsigned self) {
    const int lane = lane_id();
    int out = 0;
    for (int base = 0; base < c; base += 32) {
        int i = base + lane;
        double d = 0.0;
        unsigned id = self;
        bool keep = false;
        if (i < c) {
            d = kd[i];
            id = ki[i];
            keep = id != self && !(i > 0 && ki[i - 1] == id && kd[i - 1] == d);
        }
        unsigned b = __ballot_sync(PK_FULL, keep);
        __syncwarp();
        if (keep) {
            int o = out + warp_excl_prefix(b);
            kd[o] = d;
            ki[o] = id;
        }
        out += __popc(b);
        __syncwarp();
    }
    return out;
}

// RobustPrune over (dist,id)-sorted candidates kd/ki[0..c) (_kernels.py:290-315):
// take the closest alive candidate p*, kill every later u with
// alpha2 * d(p*, u) <= d(p, u); stop after R picks.  `alive` is c bytes of
// scratch.  Writes the picks to out[0..sel) and returns sel.
template <class MakeDist>
__device__ int warp_prune(const float* __restrict__ X, const double* kd, const unsigned* ki, int c,
                          double alpha2, int R, unsigned char* alive, unsigned* cbuf, int* out,
                          const MakeDist& make, long long* evals) {
    const int lane = lane_id();
    for (int i = lane; i < c; i += 32) alive[i] = 1;
    __syncwarp();
    int sel = 0;
    int t = 0;
    while (sel < R) {
        // next alive position >= t
        int nt = -1;
        for (int base = t; base < c; base += 32) {
            int i = base + lane;
            unsigned b = __ballot_sync(PK_FULL, i < c && alive[i]);
            if (b) { nt = base + __ffs(b) - 1; break; }
        }
        if (nt < 0) break;
        t = nt;
        const unsigned ps = ki[t];
        if (lane == 0) out[sel] = (int)ps;
        ++sel;
        if (sel >= R) break;
        auto dist = make(ps);
        for (int base = t + 1; base < c; base += 32) {
            int u = base + lane;
            bool a = u < c && alive[u];
            unsigned b = __ballot_sync(PK_FULL, a);
            const int cnt = __popc(b);
            if (!cnt) continue;
            if (a) cbuf[warp_excl_prefix(b)] = (unsigned)u;
            __syncwarp();
            unsigned uu = lane < cnt ? cbuf[lane] : 0u;
            __syncwarp();
            double duv = dist.eval(X, (int)(lane < cnt ? ki[uu] : ki[t]), cnt);
            if (lane == 0) *evals += cnt;
            if (lane < cnt && alpha2 * duv <= kd[uu]) alive[uu] = 0;
            __syncwarp();
        }
        ++t;
    }
    __syncwarp();
    return sel;
}

// One warp's share of a kill pass for pick `ps` (float data): the alive
// candidates in 32-position chunks base = first, first + stride, ... < end are
// screened with the fp32 distance (two per step, independent loads and
// reductions overlap); pairs screen_le cannot call are queued in cbuf (32
// entries) and evaluated in the reference's float64 order, one lane each.
// Returns the number of distance evaluations.
template <int QV>
__device__ long long screened_kill_pass(const float* __restrict__ X, int dp, unsigned ps, const Fp32Pick<QV>& pick,
                                        const double* kd, const unsigned* ki, unsigned char* alive, unsigned* cbuf,
                                        double alpha2, int first, int end, int stride) {
    const int lane = lane_id();
    int nunc = 0;
    long long nev = 0;
    auto flush = [&]() {
        __syncwarp();
        if (nunc) {
            const Seq64Member dx{X + (size_t)ps * dp, dp};
            const unsigned uu = lane < nunc ? cbuf[lane] : 0u;
            const double duv = dx.eval(X, (int)(lane < nunc ? ki[uu] : ps), nunc);
            if (lane < nunc && alpha2 * duv <= kd[uu]) alive[uu] = 0;
            nev += nunc;
        }
        nunc = 0;
        __syncwarp();
    };
    for (int base = first; base < end; base += stride) {
        const int u = base + lane;
        unsigned b = __ballot_sync(PK_FULL, u < end && alive[u]);
        while (b) {
            const int j0 = __ffs(b) - 1;
            b &= b - 1;
            const int j1 = b ? __ffs(b) - 1 : -1;
            if (b) b &= b - 1;
            const int u0 = base + j0, u1 = j1 >= 0 ? base + j1 : u0;
            const float p0 = pick.partial(X, dp, ki[u0]);
            const float p1 = pick.partial(X, dp, ki[u1]);
            const float s0 = Fp32Pick<QV>::reduce(p0), s1 = Fp32Pick<QV>::reduce(p1);
            const int v0 = screen_le(alpha2, s0, kd[u0]);
            const int v1 = j1 >= 0 ? screen_le(alpha2, s1, kd[u1]) : 0;
            nev += 1 + (j1 >= 0);
            if (lane == 0) {
                if (v0 == 1) alive[u0] = 0;
                if (v1 == 1) alive[u1] = 0;
            }
            if (v0 == 2) {
                if (lane == 0) cbuf[nunc] = (unsigned)u0;
                ++nunc;
            }
            if (v1 == 2) {
                if (lane == 0) cbuf[nunc] = (unsigned)u1;
                ++nunc;
            }
            if (nunc >= 31) flush();
        }
    }
    flush();
    return nev;
}

// RobustPrune for float data (SEQ64): same picks as warp_prune, every kill test
// alpha2 * d(pick, u) <= d(p, u) decided by screened_kill_pass.
template <int QV>
__device__ int warp_prune_seq64s(const float* __restrict__ X, int dp, const double* kd, const unsigned* ki, int c,
                                 double alpha2, int R, unsigned char* alive, unsigned* cbuf, int* out,
                                 long long* evals) {
    const int lane = lane_id();
    for (int i = lane; i < c; i += 32) alive[i] = 1;
    __syncwarp();
    int sel = 0;
    int t = 0;
    while (sel < R) {
        int nt = -1;
        for (int base = t; base < c; base += 32) {
            const int i = base + lane;
            const unsigned b = __ballot_sync(PK_FULL, i < c && alive[i]);
            if (b) {
                nt = base + __ffs(b) - 1;
                break;
            }
        }
        if (nt < 0) break;
        t = nt;
        const unsigned ps = ki[t];
        if (lane == 0) out[sel] = (int)ps;
        ++sel;
        if (sel >= R) break;
        Fp32Pick<QV> pick;
        pick.load(X, dp, ps);
        const long long nev = screened_kill_pass<QV>(X, dp, ps, pick, kd, ki, alive, cbuf, alpha2, t + 1, c, 32);
        if (lane == 0) *evals += nev;
        ++t;
    }
    __syncwarp();
    return sel;
}

// Copy the u8 rows of candidates ki[0..S) into shared memory (row stride rs
// words, rs = dw + 1 so lanes reading different rows hit different banks).
__device__ __forceinline__ void stage_u8_rows(const unsigned* __restrict__ X8, int dw, const unsigned* ki, int S,
                                              unsigned* rows, int rs) {
    const int lane = lane_id();
    int x = 0;
    for (; x + 4 <= S; x += 4) {
        const unsigned i0 = ki[x], i1 = ki[x + 1], i2 = ki[x + 2], i3 = ki[x + 3];
        for (int w = lane; w < dw; w += 32) {
            unsigned a = __ldg(X8 + (size_t)i0 * dw + w);
            unsigned b = __ldg(X8 + (size_t)i1 * dw + w);
            unsigned c = __ldg(X8 + (size_t)i2 * dw + w);
            unsigned d = __ldg(X8 + (size_t)i3 * dw + w);
            rows[(x + 0) * rs + w] = a;
            rows[(x + 1) * rs + w] = b;
            rows[(x + 2) * rs + w] = c;
            rows[(x + 3) * rs + w] = d;
        }
    }
    for (; x < S; ++x)
        for (int w = lane; w < dw; w += 32) rows[x * rs + w] = __ldg(X8 + (size_t)ki[x] * dw + w);
    __syncwarp();
}

// ---- d = 128 fast path (dw == 32 words per u8 row) ------------------------------
// Squared distances as |a|^2 + |b|^2 - 2 a.b: one __dp4a per word instead of
// absdiff + dp4a, the query row held in registers, rows read as 128-bit LDS.
// Staged rows use a 36-word stride (16-byte aligned, conflict-free per
// quarter warp); nrm[slot] holds each staged row's |x|^2.  All exact integers.
constexpr int kRs32 = 36;

__device__ __forceinline__ void load_row32(const unsigned* r, uint4 (&q)[8]) {
    const uint4* v = reinterpret_cast<const uint4*>(r);
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = v[i];
}

__device__ __forceinline__ unsigned dot32(const uint4 (&q)[8], const unsigned* r) {
    const uint4* v = reinterpret_cast<const uint4*>(r);
    unsigned a0 = 0u, a1 = 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint4 x = v[i];
        a0 = __dp4a(q[i].x, x.x, a0);
        a1 = __dp4a(q[i].y, x.y, a1);
        a0 = __dp4a(q[i].z, x.z, a0);
        a1 = __dp4a(q[i].w, x.w, a1);
    }
    return a0 + a1;
}

__device__ __forceinline__ unsigned norm32(const unsigned* r) {
    uint4 q[8];
    load_row32(r, q);
    return dot32(q, r);
}

// stage rows ki[0..S) (stride kRs32) and their norms
__device__ __forceinline__ void stage_u8_rows32(const unsigned* __restrict__ X8, const unsigned* ki, int S,
                                                unsigned* rows, unsigned* nrm) {
    const int lane = lane_id();
    // cp.async (LDGSTS): every row of the batch in flight at once, no registers;
    // lane l copies 16-byte chunk l % 8 of row x + l / 8
    const int chunk = lane & 7;
    for (int x = lane >> 3; x < S; x += 4) {
        const unsigned* src = X8 + (size_t)ki[x] * 32 + chunk * 4;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(rows + (size_t)x * kRs32 + chunk * 4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
    for (int r = lane; r < S; r += 32) nrm[r] = norm32(rows + (size_t)r * kRs32);
    __syncwarp();
}

// RobustPrune, d = 128 u8 rows: as warp_prune_u8, dot-product form
static __device__ int warp_prune_u8_32(const unsigned* __restrict__ X8, const double* kd, const unsigned* ki,
                                       const unsigned short* kp, int c, double alpha2, int R, unsigned char* alive,
                                       unsigned* cbuf, int* out, const unsigned* rows, const unsigned* nrm, int S,
                                       long long* evals) {
    const int lane = lane_id();
    for (int i = lane; i < c; i += 32) alive[i] = 1;
    __syncwarp();
    int sel = 0;
    int t = 0;
    while (sel < R) {
        int nt = -1;
        for (int base = t; base < c; base += 32) {
            int i = base + lane;
            unsigned b = __ballot_sync(PK_FULL, i < c && alive[i]);
            if (b) { nt = base + __ffs(b) - 1; break; }
        }
        if (nt < 0) break;
        t = nt;
        if (lane == 0) out[sel] = (int)ki[t];
        ++sel;
        if (sel >= R) break;
        const bool tin = kp[t] < S;
        const unsigned* rt = tin ? rows + (size_t)kp[t] * kRs32 : X8 + (size_t)ki[t] * 32;
        uint4 q[8];
        load_row32(rt, q);
        const unsigned nt_ = tin ? nrm[kp[t]] : dot32(q, rt);
        int nq = 0;
        auto run = [&](int cnt) {
            __syncwarp();
            if (lane < cnt) {
                const int u = (int)cbuf[lane];
                unsigned du;
                if (kp[u] < S) {
                    du = nt_ + nrm[kp[u]] - 2u * dot32(q, rows + (size_t)kp[u] * kRs32);
                } else {
                    const unsigned* ru = X8 + (size_t)ki[u] * 32;
                    du = nt_ + norm32(ru) - 2u * dot32(q, ru);
                }
                if (alpha2 * (double)du <= kd[u]) alive[u] = 0;
            }
            if (lane == 0) *evals += cnt;
            __syncwarp();
        };
        for (int base = t + 1; base < c; base += 32) {
            const int u = base + lane;
            const bool a = u < c && alive[u];
            const unsigned b = __ballot_sync(PK_FULL, a);
            const int k = __popc(b);
            if (nq + k > 32) {
                run(nq);
                nq = 0;
            }
            if (a) cbuf[nq + warp_excl_prefix(b)] = (unsigned)u;
            nq += k;
        }
        if (nq) run(nq);
        ++t;
    }
    __syncwarp();
    return sel;
}

// RobustPrune on u8 rows staged in shared memory (rows >= S come from
// global memory).  Same picks as warp_prune: one lane per candidate u, the
// whole row pair evaluated sequentially with exact integer dp4a arithmetic.
// Alive candidates after the current pick are queued 32 at a time so every
// lane has work.
// kp[u] = staged row slot of candidate u (rows[kp[u]] if kp[u] < S, else the
// row is read from global memory by id).
static __device__ int warp_prune_u8(const unsigned* __restrict__ X8, int dw, const double* kd, const unsigned* ki,
                                    const unsigned short* kp, int c, double alpha2, int R, unsigned char* alive,
                                    unsigned* cbuf, int* out, const unsigned* rows, int rs, int S, long long* evals) {
    const int lane = lane_id();
    for (int i = lane; i < c; i += 32) alive[i] = 1;
    __syncwarp();
    int sel = 0;
    int t = 0;
    while (sel < R) {
        int nt = -1;
        for (int base = t; base < c; base += 32) {
            int i = base + lane;
            unsigned b = __ballot_sync(PK_FULL, i < c && alive[i]);
            if (b) { nt = base + __ffs(b) - 1; break; }
        }
        if (nt < 0) break;
        t = nt;
        if (lane == 0) out[sel] = (int)ki[t];
        ++sel;
        if (sel >= R) break;
        const unsigned* rt = kp[t] < S ? rows + (size_t)kp[t] * rs : X8 + (size_t)ki[t] * dw;
        int nq = 0;
        auto run = [&](int cnt) {
            __syncwarp();
            if (lane < cnt) {
                const int u = (int)cbuf[lane];
                const unsigned* ru = kp[u] < S ? rows + (size_t)kp[u] * rs : X8 + (size_t)ki[u] * dw;
                const unsigned duv = u8_row_dist(rt, ru, dw);
                if (alpha2 * (double)duv <= kd[u]) alive[u] = 0;
            }
            if (lane == 0) *evals += cnt;
            __syncwarp();
        };
        for (int base = t + 1; base < c; base += 32) {
            const int u = base + lane;
            const bool a = u < c && alive[u];
            const unsigned b = __ballot_sync(PK_FULL, a);
            const int k = __popc(b);
            if (nq + k > 32) {
                run(nq);
                nq = 0;
            }
            if (a) cbuf[nq + warp_excl_prefix(b)] = (unsigned)u;
            nq += k;
        }
        if (nq) run(nq);
        ++t;
    }
    __syncwarp();
    return sel;
}

}  // namespace pk
