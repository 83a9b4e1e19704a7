// Vamana graph construction on device (vamana.py:106-172, _kernels.py:338-415).
//
// Per batch [lo, lo + 2^b) of the insertion order:
//   1. build_batch_kernel   -- one warp per inserted point: beam search over the
//      adjacency snapshot (visit log kept), candidates = visited U current
//      out-row, sort + dedupe, RobustPrune -> staging rows (new_ids/new_len).
//      The snapshot is only read, so every point of a batch sees the same graph
//      (the reference's batch-synchronous guarantee, vamana.py:1-8).
//   2. commit_kernel        -- write the staged rows, count reverse edges per
//      target and register each touched target once.
//   3. sizes / scan / scatter -- CSR of incoming sources per target.
//   4. reverse_kernel       -- one warp per target: merge its row with the
//      incoming sources, sort + dedupe, keep all if <= R else RobustPrune
//      (rows stay (dist,id)-sorted, _kernels.py:378-415).  Candidate order
//      within a group is irrelevant because the merge sorts by (dist, id).
#include <algorithm>
#include <string>

#include <cuda_fp16.h>
#include <cub/cub.cuh>

#include "../../include/peakann_b200.h"
#include "api.cuh"
#include "beam.cuh"
#include "tc_common.cuh"

namespace pk {

int grid_for(long long work, int block);

struct BuildArgs {
    int* ticket = nullptr;  // this launch's item counter (BlockTickets; block-per-item prune kernels)
    SearchParams P;
    DataRef D;
    const int* bids;
    int m;
    int L;
    int H;
    int cap;           // candidate capacity (power of two)
    int vcap;          // visit-log capacity per point
    int S;             // u8 rows staged in shared memory per warp
    double alpha2;
    size_t search_bytes;  // per-warp shared memory, search kernel
    size_t prune_bytes;   // per-warp shared memory, prune kernel
    unsigned* vlog_i;  // [m * vcap]
    double* vlog_d;
    int* vlen;         // [m]
    int* new_ids;      // [m * R]
    int* new_len;      // [m]
    double* new_d;     // [m * R] distances of the out-lists' entries (NaN = unknown), or null
    const double* adjd;  // [n * R] distances of the adjacency rows' entries (NaN = unknown), or null
    unsigned* err;
    long long* stats;  // [4]
    const int* items;  // optional: batch indices to process (overflow of the block prune), count *nitems
    const int* nitems;
};

// phase 1: one warp per inserted point searches the adjacency snapshot and
// logs its visited set (_kernels.py:349-358)
template <int MODE, int QV, bool RING>
__global__ void __launch_bounds__(128, MODE == MODE_SEQ64 ? (QV >= 8 ? 4 : QV >= 4 ? 5 : 8) : 8) build_search_kernel(BuildArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int lane = lane_id();
    BeamSmem sm = A.P.ghash ? carve_beam_gh(smem + (size_t)wib * A.search_bytes,
                                            A.P.ghash + ((size_t)blockIdx.x * wpb + wib) * A.P.ghash_stride, A.L, A.H)
                            : carve_beam(smem + (size_t)wib * A.search_bytes, A.L, A.H);
    if constexpr (RING)
        carve_ring(sm, smem + (size_t)(wib + 1) * A.search_bytes - ring_smem_bytes_dev(A.P.dp, A.P.ring), A.P.dp,
                   A.P.ring);
    unsigned ring_t = 0;
    const MakeAt<MODE, QV, RING> make{A.D};
    long long ev = 0, expansions = 0, un = 0;
    const bool uniq = starts_increasing(A.P);
    for (int t = next_position(A.P.ticket, blockIdx.x * wpb + wib - gridDim.x * wpb, gridDim.x * wpb); t < A.m;
         t = next_position(A.P.ticket, t, gridDim.x * wpb)) {
        const unsigned p = (unsigned)A.bids[t];
        auto dist = make(p);
        WarpBeam<decltype(dist)> wb;
        wb.init(sm, A.L, A.vlog_i + (size_t)t * A.vcap, A.vlog_d + (size_t)t * A.vcap, A.vcap, A.err);
        wb.qid = p;
        wb.rt = ring_t;
        wb.begin_counting(A.P.ubm ? A.P.ubm + ((size_t)blockIdx.x * wpb + wib) * A.P.uwords : nullptr, A.P.uwords);
        {
            PK_PT_BEGIN
            wb.seed(A.P, dist, false, uniq);
            if (A.P.seed_save) wb.save_seed(A.P, p);
            PK_PT_END(6);
        }
        wb.walk(A.P, dist);
        if constexpr (has_screen<decltype(dist)>::value) {
            PK_PT_BEGIN
            if (wb.lazy) wb.finalize_log(A.P, dist);
            PK_PT_END(5);
        }
        un += wb.uniq;
        ev += wb.evals;
        expansions += wb.vl;
        ring_t = wb.rt;
        if (lane == 0) A.vlen[t] = min(wb.vl, A.vcap);
        __syncwarp();
    }
    if (lane == 0 && A.stats) {
        atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 0), (unsigned long long)ev);
        atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 3), (unsigned long long)expansions);
        if (A.P.ubm) atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 4), (unsigned long long)un);
    }
}

// Shared-memory view of the candidate buffers of one warp (host size:
// cand_smem_bytes in api.cuh):
//   kd[cap] f64 | ki[cap] u32 | kp[cap] u16 | alive[cap] u8 | cbuf[32] u32 |
//   qrow[dw] u32 | rows[S][dw + 4] u32 | nrm[S] u32   (the last three: u8 mode)
struct CandSmem {
    double* kd;
    unsigned* ki;
    unsigned short* kp;
    unsigned char* alive;
    unsigned* cbuf;
    unsigned* qrow;
    unsigned* rows;
    unsigned* nrm;
};

__device__ __forceinline__ CandSmem carve_cand(unsigned char* base, int cap, int dw, int S) {
    CandSmem c;
    c.kd = reinterpret_cast<double*>(base);
    c.ki = reinterpret_cast<unsigned*>(base + (size_t)cap * 8);
    c.kp = reinterpret_cast<unsigned short*>(base + (size_t)cap * 12);
    c.alive = base + (size_t)cap * 14;
    c.cbuf = reinterpret_cast<unsigned*>(base + (((size_t)cap * 15 + 3) & ~(size_t)3));
    const size_t q = (((size_t)cap * 15 + 3) & ~(size_t)3) + 128;
    c.qrow = reinterpret_cast<unsigned*>(base + ((q + 15) & ~(size_t)15));
    c.rows = c.qrow + (((size_t)dw + 3) & ~(size_t)3);
    c.nrm = c.rows + (size_t)S * (dw + 4);
    return c;
}

// Stage candidate rows ki[0..c) in input order (slot = position) plus the
// query row, then compute kd[x] = d(query, ki[x]) for x >= from, one lane per
// candidate from shared memory (u8 mode).  Returns the number of staged rows.
__device__ __forceinline__ int stage_and_measure_u8(const DataRef& D, const CandSmem& C, unsigned q, int c, int S,
                                                    int from, long long* ev) {
    const int lane = lane_id();
    const int st = min(c, S);
    for (int w = lane; w < D.dw; w += 32) C.qrow[w] = __ldg(D.X8 + (size_t)q * D.dw + w);
    if (D.dw == 32) {
        stage_u8_rows32(D.X8, C.ki, st, C.rows, C.nrm);
        uint4 qr[8];
        load_row32(C.qrow, qr);
        const unsigned nq = dot32(qr, C.qrow);
        for (int x = from + lane; x < c; x += 32) {
            unsigned dx;
            if (x < st) {
                dx = nq + C.nrm[x] - 2u * dot32(qr, C.rows + (size_t)x * kRs32);
            } else {
                const unsigned* rx = D.X8 + (size_t)C.ki[x] * 32;
                dx = nq + norm32(rx) - 2u * dot32(qr, rx);
            }
            C.kd[x] = (double)dx;
        }
    } else {
        const int rs = D.dw + 1;
        stage_u8_rows(D.X8, D.dw, C.ki, st, C.rows, rs);
        for (int x = from + lane; x < c; x += 32) {
            const unsigned* rx = x < st ? C.rows + (size_t)x * rs : D.X8 + (size_t)C.ki[x] * D.dw;
            C.kd[x] = (double)u8_row_dist(C.qrow, rx, D.dw);
        }
    }
    if (lane == 0) *ev += c - from;
    __syncwarp();
    return st;
}

// sorted, de-duplicated candidates kd/ki/kp[0..c) -> RobustPrune picks in out[]
template <int MODE, int QV>
__device__ __forceinline__ int prune_candidates(const DataRef& D, const CandSmem& C, int c, double alpha2, int R,
                                                int staged, int* out, long long* ev) {
    if (MODE == MODE_EXACT_U8 && D.dw == 32)
        return warp_prune_u8_32(D.X8, C.kd, C.ki, C.kp, c, alpha2, R, C.alive, C.cbuf, out, C.rows, C.nrm, staged,
                                ev);
    if (MODE == MODE_EXACT_U8)
        return warp_prune_u8(D.X8, D.dw, C.kd, C.ki, C.kp, c, alpha2, R, C.alive, C.cbuf, out, C.rows, D.dw + 1,
                             staged, ev);
    if (MODE == MODE_SEQ64 && D.dp <= 128 * QV && D.screen)
        return warp_prune_seq64s<QV>(D.X, D.dp, C.kd, C.ki, c, alpha2, R, C.alive, C.cbuf, out, ev);
    const MakeAt<MODE, QV> make{D};
    return warp_prune(D.X, C.kd, C.ki, c, alpha2, R, C.alive, C.cbuf, out, make, ev);
}

// phase 2: candidates = visited U current out-row (distances recomputed,
// _kernels.py:359-368), canonicalise, RobustPrune -> staged out-list
template <int MODE, int QV>
__global__ void __launch_bounds__(128) build_prune_kernel(BuildArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int lane = lane_id();
    const CandSmem C = carve_cand(smem + (size_t)wib * A.prune_bytes, A.cap, A.D.dw, A.S);
    const MakeAt<MODE, QV> make{A.D};
    long long ev_prune = 0;
    const int R = A.P.R;
    const int total = A.items ? *A.nitems : A.m;
    for (int it = blockIdx.x * wpb + wib; it < total; it += gridDim.x * wpb) {
        const int t = A.items ? A.items[it] : it;
        const unsigned p = (unsigned)A.bids[t];
        const int vl = A.vlen[t];
        const unsigned* vi = A.vlog_i + (size_t)t * A.vcap;
        const double* vd = A.vlog_d + (size_t)t * A.vcap;
        const int nd = __ldg(A.P.deg + p);
        const int* row = A.P.adj + (size_t)p * R;
        int c = min(vl + nd, A.cap);
        if (vl + nd > A.cap && lane == 0) atomicOr(A.err, ERR_CAND_OVERFLOW);
        // candidates in input order: visit log (distances known), then out-row
        for (int x = lane; x < c; x += 32) {
            if (x < vl) {
                C.kd[x] = vd[x];
                C.ki[x] = vi[x];
            } else {
                C.ki[x] = (unsigned)__ldg(row + x - vl);
            }
            C.kp[x] = (unsigned short)x;
        }
        __syncwarp();
        int staged = 0;
        if (MODE == MODE_EXACT_U8) {
            staged = stage_and_measure_u8(A.D, C, p, c, A.S, min(vl, c), &ev_prune);
        } else if (nd > 0) {
            auto dist = make(p);
            for (int e0 = vl; e0 < c; e0 += 32) {
                const int cnt = min(32, c - e0);
                unsigned w = lane < cnt ? C.ki[e0 + lane] : 0u;
                double dd = dist.eval(A.D.X, (int)w, cnt);
                if (lane == 0) ev_prune += cnt;
                if (lane < cnt) C.kd[e0 + lane] = dd;
            }
        }
        const int Pw = next_pow2_dev(c);
        for (int x = c + lane; x < Pw; x += 32) {
            C.kd[x] = __longlong_as_double(0x7ff0000000000000LL);
            C.ki[x] = 0xffffffffu;
            C.kp[x] = 0xffffu;
        }
        __syncwarp();
        warp_sort_pos(C.kd, C.ki, C.kp, Pw);
        c = warp_unique_pos(C.kd, C.ki, C.kp, c, p);
        int* out = A.new_ids + (size_t)t * R;
        int sel = prune_candidates<MODE, QV>(A.D, C, c, A.alpha2, R, staged, out, &ev_prune);
        for (int x = sel + lane; x < R; x += 32) out[x] = -1;
        if (A.new_d)
            for (int x = lane; x < R; x += 32) A.new_d[(size_t)t * R + x] = __longlong_as_double(0x7ff8000000000000LL);
        if (lane == 0) A.new_len[t] = sel;
        __syncwarp();
    }
    if (lane == 0 && A.stats)
        atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 1), (unsigned long long)ev_prune);
}

// write staged rows, count reverse edges, register targets (warp per point)
__global__ void commit_kernel(const int* bids, int m, int R, const int* new_ids, const int* new_len, int* adj,
                              int* deg, int* cnt, int* tslot, int* targets, int* ntargets, const double* new_d,
                              double* adjd) {
    const int lane = lane_id();
    const int wpb = blockDim.x >> 5;
    for (int t = blockIdx.x * wpb + (threadIdx.x >> 5); t < m; t += gridDim.x * wpb) {
        const int p = bids[t];
        const int len = new_len[t];
        for (int x = lane; x < R; x += 32) {
            int u = new_ids[(size_t)t * R + x];
            adj[(size_t)p * R + x] = u;
            if (adjd) adjd[(size_t)p * R + x] = new_d[(size_t)t * R + x];
            if (x < len) {
                if (atomicAdd(cnt + u, 1) == 0) {
                    int s = atomicAdd(ntargets, 1);
                    targets[s] = u;
                    tslot[u] = s;
                }
            }
        }
        if (lane == 0) deg[p] = len;
    }
}

__global__ void sizes_kernel(const int* targets, const int* ntargets, const int* cnt, int* sizes) {
    const int nt = *ntargets;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nt; s += gridDim.x * blockDim.x) sizes[s] = cnt[targets[s]];
}

__global__ void scatter_kernel(const int* bids, int m, int R, const int* new_ids, const int* new_len,
                               const int* tslot, const int* offs, int* fill, int* adds, const double* new_d,
                               double* addd) {
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < (long long)m * R;
         x += (long long)gridDim.x * blockDim.x) {
        int t = (int)(x / R), e = (int)(x % R);
        if (e >= new_len[t]) continue;
        int u = new_ids[x];
        int s = tslot[u];
        int pos = offs[s] + atomicAdd(fill + s, 1);
        adds[pos] = bids[t];
        if (addd) addd[pos] = new_d[x];  // d(p, u) == d(u, p) bit for bit
    }
}

struct RevArgs {
    int* ticket = nullptr;  // this launch's item counter (BlockTickets), zeroed before it
    const float* X;
    int dp;
    DataRef D;
    int S;
    int* adj;
    int* deg;
    int R;
    const int* targets;
    const int* ntargets;
    const int* offs;
    const int* sizes;
    const int* adds;
    double* adist;          // [E] scratch for oversized groups
    unsigned char* aalive;  // [E]
    int* cnt;
    int cap;
    double alpha2;
    size_t warp_bytes;
    long long* stats;
    int capB;       // largest group handled by reverse_big_kernel
    int* biglist;   // groups with cap < candidates <= capB
    int* nbig;
    int rank, world;  // sharded build: this rank re-prunes the targets u % world == rank
    double* adjd;        // [n * R] row-entry distances (NaN = unknown), or null
    const double* addd;  // [E] distances of the batch's new sources to their targets, or null
};

// build context: multi-GPU split (pk_build_vamana_sharded) and the optional
// seeded-beam cache (pk_build_vamana_seeds; single-GPU builds only)
struct Shard {
    int rank = 0, world = 1;
    long long min_shard = 0;
    pk_exchange_fn fn = nullptr;
    void* ctx = nullptr;
    int *xids = nullptr, *xlen = nullptr, *xsend = nullptr, *xrecv = nullptr, *xcnt = nullptr;
    double* seed_bd = nullptr;
    unsigned* seed_bi = nullptr;
    int* seed_bl = nullptr;
};

// rows of the targets this rank re-pruned -> [u, deg, row[R]] records
__global__ void pack_rows_kernel(const int* targets, const int* ntargets, int rank, int world, const int* adj,
                                 const int* deg, int R, int* out, int* npack) {
    const int lane = lane_id();
    const int nt = *ntargets;
    const int wpb = blockDim.x >> 5;
    for (int s = blockIdx.x * wpb + (threadIdx.x >> 5); s < nt; s += gridDim.x * wpb) {
        const int u = targets[s];
        if (u % world != rank) continue;
        int pos = 0;
        if (lane == 0) pos = atomicAdd(npack, 1);
        pos = __shfl_sync(PK_FULL, pos, 0);
        int* rec = out + (size_t)pos * (R + 2);
        if (lane == 0) {
            rec[0] = u;
            rec[1] = deg[u];
        }
        for (int x = lane; x < R; x += 32) rec[2 + x] = adj[(size_t)u * R + x];
    }
}

// apply the other ranks' records (every rank ends with the same graph)
__global__ void unpack_rows_kernel(const int* recv, const int* cnt, int maxc, int world, int rank, int R, int* adj,
                                   int* deg) {
    const int lane = lane_id();
    const int wpb = blockDim.x >> 5;
    const long long tot = (long long)world * maxc;
    for (long long e = blockIdx.x * (long long)wpb + (threadIdx.x >> 5); e < tot; e += (long long)gridDim.x * wpb) {
        const int r = (int)(e / maxc), i = (int)(e % maxc);
        if (r == rank || i >= cnt[r]) continue;
        const int* rec = recv + (size_t)e * (R + 2);
        const int u = rec[0];
        if (lane == 0) deg[u] = rec[1];
        for (int x = lane; x < R; x += 32) adj[(size_t)u * R + x] = rec[2 + x];
    }
}

// Oversized group (more candidates than the shared buffer): RobustPrune by
// repeated selection of the smallest alive key (equal keys = same id, i.e. a
// source already present in the row).  Row entries live in shared memory,
// incoming sources and their distances in global scratch.
template <class MakeDist>
__device__ int prune_by_selection(const RevArgs& A, unsigned u, const MakeDist& make, double* kd, unsigned* ki,
                                  unsigned char* alive_row, unsigned* cbuf, int nd, int off, int size, int* out,
                                  long long* evals) {
    const int lane = lane_id();
    const int tot = nd + size;
    auto du = make(u);
    for (int e0 = 0; e0 < nd; e0 += 32) {
        const int cnt = min(32, nd - e0);
        unsigned w = lane < cnt ? (unsigned)A.adj[(size_t)u * A.R + e0 + lane] : 0u;
        double dd = du.eval(A.X, (int)w, cnt);
        if (lane < cnt) {
            kd[e0 + lane] = dd;
            ki[e0 + lane] = w;
            alive_row[e0 + lane] = w != u;
        }
    }
    for (int e0 = 0; e0 < size; e0 += 32) {
        const int cnt = min(32, size - e0);
        unsigned w = lane < cnt ? (unsigned)A.adds[off + e0 + lane] : 0u;
        double dd = du.eval(A.X, (int)w, cnt);
        if (lane < cnt) {
            A.adist[off + e0 + lane] = dd;
            A.aalive[off + e0 + lane] = w != u;
        }
    }
    *evals += tot;
    __syncwarp();
    auto get = [&](int x, bool& a, double& d, unsigned& i) {
        if (x < nd) { a = alive_row[x]; d = kd[x]; i = ki[x]; }
        else { a = A.aalive[off + x - nd]; d = A.adist[off + x - nd]; i = (unsigned)A.adds[off + x - nd]; }
    };
    auto kill = [&](int x) {
        if (x < nd) alive_row[x] = 0;
        else A.aalive[off + x - nd] = 0;
    };
    int sel = 0;
    while (sel < A.R) {
        double bd = __longlong_as_double(0x7ff0000000000000LL);
        unsigned bi = 0xffffffffu;
        for (int x = lane; x < tot; x += 32) {
            bool a; double d; unsigned i;
            get(x, a, d, i);
            if (a && key_lt(d, i, bd, bi)) { bd = d; bi = i; }
        }
        for (int s = 16; s; s >>= 1) {
            double od = __shfl_xor_sync(PK_FULL, bd, s);
            unsigned oi = __shfl_xor_sync(PK_FULL, bi, s);
            if (key_lt(od, oi, bd, bi)) { bd = od; bi = oi; }
        }
        if (bi == 0xffffffffu) break;
        if (lane == 0) out[sel] = (int)bi;
        ++sel;
        for (int x = lane; x < tot; x += 32) {
            bool a; double d; unsigned i;
            get(x, a, d, i);
            if (a && i == bi) kill(x);
        }
        __syncwarp();
        if (sel >= A.R) break;
        auto dsel = make(bi);
        for (int base = 0; base < tot; base += 32) {
            const int x = base + lane;
            bool a = false; double dx = 0.0; unsigned id = 0;
            if (x < tot) get(x, a, dx, id);
            unsigned b = __ballot_sync(PK_FULL, a);
            const int cnt = __popc(b);
            if (!cnt) continue;
            if (a) cbuf[warp_excl_prefix(b)] = (unsigned)x;
            __syncwarp();
            int sx = lane < cnt ? (int)cbuf[lane] : 0;
            __syncwarp();
            bool a2; double d2 = 0.0; unsigned i2 = 0;
            if (lane < cnt) get(sx, a2, d2, i2);
            double duv = dsel.eval(A.X, (int)i2, cnt);
            *evals += cnt;
            if (lane < cnt && A.alpha2 * duv <= d2) kill(sx);
            __syncwarp();
        }
    }
    return sel;
}

template <int MODE, int QV>
__global__ void __launch_bounds__(128) reverse_kernel(RevArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int lane = lane_id();
    const CandSmem C = carve_cand(smem + (size_t)wib * A.warp_bytes, A.cap, A.D.dw, A.S);
    double* kd = C.kd;
    unsigned* ki = C.ki;
    unsigned* pcbuf = C.cbuf;
    unsigned char* alive = C.alive;
    const MakeAt<MODE, QV> make{A.D};
    const int nt = *A.ntargets;
    long long ev = 0;
    for (int s = blockIdx.x * wpb + wib; s < nt; s += gridDim.x * wpb) {
        const unsigned u = (unsigned)A.targets[s];
        if (A.world > 1 && (int)(u % (unsigned)A.world) != A.rank) {
            // another rank re-prunes this row; only the per-batch counter is reset here
            if (lane == 0) A.cnt[u] = 0;
            continue;
        }
        const int nd = A.deg[u];
        const int off = A.offs[s];
        const int size = A.sizes[s];
        int* row = A.adj + (size_t)u * A.R;
        const int c0 = nd + size;
        int sel;
        if (c0 <= A.cap) {
            for (int x = lane; x < c0; x += 32) {
                ki[x] = x < nd ? (unsigned)row[x] : (unsigned)A.adds[off + x - nd];
                C.kp[x] = (unsigned short)x;
            }
            __syncwarp();
            int staged = 0;
            if (MODE == MODE_EXACT_U8) {
                staged = stage_and_measure_u8(A.D, C, u, c0, A.S, 0, &ev);
            } else {
                auto du = make(u);
                for (int e0 = 0; e0 < c0; e0 += 32) {
                    const int cnt = min(32, c0 - e0);
                    unsigned w = lane < cnt ? ki[e0 + lane] : 0u;
                    double dd = du.eval(A.X, (int)w, cnt);
                    if (lane < cnt) kd[e0 + lane] = dd;
                }
                ev += c0;
            }
            const int Pw = next_pow2_dev(c0);
            for (int x = c0 + lane; x < Pw; x += 32) {
                kd[x] = __longlong_as_double(0x7ff0000000000000LL);
                ki[x] = 0xffffffffu;
                C.kp[x] = 0xffffu;
            }
            __syncwarp();
            warp_sort_pos(kd, ki, C.kp, Pw);
            const int c = warp_unique_pos(kd, ki, C.kp, c0, u);
            if (c <= A.R) {
                for (int x = lane; x < c; x += 32) row[x] = (int)ki[x];
                sel = c;
            } else {
                sel = prune_candidates<MODE, QV>(A.D, C, c, A.alpha2, A.R, staged, row, &ev);
            }
        } else if (c0 <= A.capB) {
            // large group: handled by a whole block in reverse_big_kernel
            if (lane == 0) A.biglist[atomicAdd(A.nbig, 1)] = s;
            __syncwarp();
            continue;
        } else {
            sel = prune_by_selection(A, u, make, kd, ki, alive, pcbuf, nd, off, size, row, &ev);
        }
        __syncwarp();
        for (int x = sel + lane; x < A.R; x += 32) row[x] = -1;
        if (lane == 0) {
            A.deg[u] = sel;
            A.cnt[u] = 0;
        }
        __syncwarp();
    }
    if (lane == 0 && A.stats && ev) atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 2), (unsigned long long)ev);
}

// ---- block-per-item RobustPrune on the integer tensor cores (u8, d = 128) -------------------
// The sequential RobustPrune (_kernels.py:283-315) only ever asks "does pick t
// occlude candidate u": alpha^2 * d(t, u) <= d(p, u).  For the sorted,
// de-duplicated candidates of one item every such bit is computed up front:
// d(t, u) = |t|^2 + |u|^2 - 2 t.u with the dot products of all pairs t < u from
// exact u8 x u8 -> s32 mma.sync tiles (16 x 8 x 32), the occlusion bits packed
// per row; the greedy pass is then bit arithmetic (alive &= ~kill[t]).  The
// picks are identical to the sequential algorithm: the kill decision for (t, u)
// depends only on the pair and on t being picked.
constexpr int BP_CAP = 256;      // candidates per build item (more -> warp path)
constexpr int BP_CAP_MAX = 512;  // reverse groups: third launch with room for 512 (more -> reverse_big_kernel)
constexpr int BP_THREADS = 128;

struct BPSmem {
    unsigned* rows;   // [BP_CAP][32] u8 rows in sorted order, 16-byte chunks XOR-swizzled by (row & 7)
    unsigned* nrm;    // [BP_CAP] |row|^2
    double* kd;       // [BP_CAP] candidate keys (input order, then bitonic-sorted)
    unsigned* ki;
    double* kd2;      // [BP_CAP] de-duplicated, sorted
    unsigned* ki2;
    unsigned* kill;   // [cap][words] occlusion bits: bit u of row t = t occludes u
    int* scal;        // [16] block scalars
    int words;        // bit words per row: 8 (cap <= 256) or cap / 32
};

__host__ __device__ constexpr int bp_words(int cap) { return cap > 256 ? cap / 32 : 8; }

// shared memory of one item with room for `cap` (<= BP_CAP) candidates
__host__ __device__ constexpr size_t bp_smem_bytes(int cap) {
    return (size_t)cap * 32 * 4 + cap * 4 + cap * 8 * 2 + cap * 4 * 2 + (size_t)cap * bp_words(cap) * 4 + 16 * 4 +
           16;
}

__device__ __forceinline__ BPSmem carve_bp(unsigned char* base, int cap) {
    BPSmem S;
    S.rows = reinterpret_cast<unsigned*>(base);
    S.kd = reinterpret_cast<double*>(base + (size_t)cap * 128);
    S.kd2 = S.kd + cap;
    S.nrm = reinterpret_cast<unsigned*>(S.kd2 + cap);
    S.ki = S.nrm + cap;
    S.ki2 = S.ki + cap;
    S.kill = S.ki2 + cap;
    S.words = bp_words(cap);
    S.scal = reinterpret_cast<int*>(S.kill + (size_t)cap * S.words);
    return S;
}

__device__ __forceinline__ int bp_swz(int r, int w) { return r * 32 + (w ^ ((r & 7) << 2)); }

// exact |a - b|^2 of a global u8 row against a register row (dot-product form)
__device__ __forceinline__ unsigned bp_dist_global(const uint4 (&q)[8], unsigned nq, const unsigned* row) {
    uint4 r[8];
    const uint4* v = reinterpret_cast<const uint4*>(row);
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = __ldg(v + i);
    unsigned n0 = 0u, n1 = 0u, d0 = 0u, d1 = 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        n0 = __dp4a(r[i].x, r[i].x, n0);
        n1 = __dp4a(r[i].y, r[i].y, n1);
        n0 = __dp4a(r[i].z, r[i].z, n0);
        n1 = __dp4a(r[i].w, r[i].w, n1);
        d0 = __dp4a(q[i].x, r[i].x, d0);
        d1 = __dp4a(q[i].y, r[i].y, d1);
        d0 = __dp4a(q[i].z, r[i].z, d0);
        d1 = __dp4a(q[i].w, r[i].w, d1);
    }
    return nq + (n0 + n1) - 2u * (d0 + d1);
}

// block bitonic sort of (kd, ki)[0, P) by (dist, id); P a power of two.  One
// compare-exchange per thread and stage (thread -> pair, nobody idles), and a
// block barrier only around the stages that cross a warp's own 64 elements: pair
// p = tid + 128 it lies in elements [64 (p >> 5), 64 (p >> 5) + 64) whenever
// j <= 32, and a warp owns the same pair blocks in every stage, so consecutive
// stages with j <= 32 only need the warp in step (3 block barriers at P = 256
// instead of 36).  Callers enter and leave through a block barrier.
__device__ __forceinline__ void bp_sort(double* kd, unsigned* ki, int P) {
    const int half = P >> 1;
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int p = threadIdx.x; p < half; p += BP_THREADS) {
                const int i = ((p & ~(j - 1)) << 1) | (p & (j - 1));
                const int x = i | j;
                const double a = kd[i], b = kd[x];
                const unsigned ia = ki[i], ib = ki[x];
                if (key_lt(b, ib, a, ia) == ((i & k) == 0)) {
                    kd[i] = b;
                    kd[x] = a;
                    ki[i] = ib;
                    ki[x] = ia;
                }
            }
            const int jn = j > 1 ? (j >> 1) : k;  // the next stage's j (k: first stage of the next k)
            if (j >= 64 || jn >= 64) __syncthreads();
            else __syncwarp();
        }
    __syncthreads();
}

// Reverse groups: kd/ki[0, nd) is the target's current row -- every adjacency
// row is kept (dist, id)-sorted (the build's picks and the re-prunes come out in
// key order) -- and kd/ki[nd, c0) are this batch's few new sources.  Sort the
// sources alone (bitonic over a small power of two), then merge the two sorted
// runs (each element's place = its index + its rank in the other run; equal
// keys are identical entries, row first).  Replaces the full bitonic sort of c0
// keys; kd/ki hold the sorted c0 keys afterwards.
__device__ __forceinline__ void bp_sort_row_plus_adds(const BPSmem& S, int nd, int c0) {
    const int tid = threadIdx.x;
    const int sz = c0 - nd;
    const int P2 = next_pow2_dev(sz < 2 ? 2 : sz);
    for (int x = c0 + tid; x < nd + P2; x += BP_THREADS) {
        S.kd[x] = __longlong_as_double(0x7ff0000000000000LL);
        S.ki[x] = 0xffffffffu;
    }
    __syncthreads();
    if (sz > 1) bp_sort(S.kd + nd, S.ki + nd, P2);
    for (int x = tid; x < c0; x += BP_THREADS) {
        const double d = S.kd[x];
        const unsigned i = S.ki[x];
        int pos;
        if (x < nd) {  // row entry: + number of sources strictly below it
            int lo = 0, hi = sz;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (key_lt(S.kd[nd + mid], S.ki[nd + mid], d, i)) lo = mid + 1;
                else hi = mid;
            }
            pos = x + lo;
        } else {  // source: + number of row entries not above it
            int lo = 0, hi = nd;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (!key_lt(d, i, S.kd[mid], S.ki[mid])) lo = mid + 1;
                else hi = mid;
            }
            pos = x - nd + lo;
        }
        S.kd2[pos] = d;
        S.ki2[pos] = i;
    }
    __syncthreads();
    for (int x = tid; x < c0; x += BP_THREADS) {
        S.kd[x] = S.kd2[x];
        S.ki[x] = S.ki2[x];
    }
    __syncthreads();
}

// drop `self` and repeated (dist, id) entries, keep order -> kd2/ki2; returns the count
__device__ __forceinline__ int bp_unique(const BPSmem& S, int c, unsigned self) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // thread tid owns positions 4 tid .. 4 tid + 3 (c <= 512)
    bool keep[4];
    int mine = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int i = 4 * tid + e;
        keep[e] = false;
        if (i < c) {
            const unsigned id = S.ki[i];
            keep[e] = id != self && !(i > 0 && S.ki[i - 1] == id && S.kd[i - 1] == S.kd[i]);
        }
        mine += keep[e];
    }
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(PK_FULL, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) S.scal[wid] = incl;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < wid; ++w) base += S.scal[w];
    const int total = S.scal[0] + S.scal[1] + S.scal[2] + S.scal[3];
    int o = base + incl - mine;
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if (keep[e]) {
            S.kd2[o] = S.kd[4 * tid + e];
            S.ki2[o] = S.ki[4 * tid + e];
            ++o;
        }
    __syncthreads();
    return total;
}

__device__ __forceinline__ void bp_mma(const unsigned (&a)[4], const unsigned (&b)[2], int (&d)[4]) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ unsigned bp_spread4(unsigned x) {
    return (x & 1u) | ((x & 2u) << 1) | ((x & 4u) << 2) | ((x & 8u) << 3);
}

// RobustPrune of the c sorted unique candidates kd2/ki2 (c > R) -> out[0, sel); returns sel
__device__ int bp_prune(const unsigned* __restrict__ X8, const BPSmem& S, int c, double alpha2, int R, int* out,
                        long long* pairs) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // stage the rows in sorted order (cp.async, 16-byte chunks, swizzled), clear the bits
    for (int e = tid; e < c * 8; e += BP_THREADS) {
        const int x = e >> 3, ch = e & 7;
        const unsigned* src = X8 + (size_t)S.ki2[x] * 32 + ch * 4;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(S.rows + x * 32 + ((ch ^ (x & 7)) << 2));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    for (int e = tid; e < c * S.words; e += BP_THREADS) S.kill[e] = 0u;
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    for (int x = tid; x < c; x += BP_THREADS) {
        unsigned n0 = 0u, n1 = 0u;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint4 v = *reinterpret_cast<const uint4*>(S.rows + x * 32 + ((q ^ (x & 7)) << 2));
            n0 = __dp4a(v.x, v.x, n0);
            n1 = __dp4a(v.y, v.y, n1);
            n0 = __dp4a(v.z, v.z, n0);
            n1 = __dp4a(v.w, v.w, n1);
        }
        S.nrm[x] = n0 + n1;
    }
    __syncthreads();
    // occlusion bits of all pairs t < u: 16-row tiles (snake-assigned to warps) x 8-column tiles
    const int T = (c + 15) >> 4, U = (c + 7) >> 3;
    const int g = lane >> 2, tig = lane & 3;
    for (int i0 = 0; i0 < T; i0 += 4) {
        const int i = ((i0 >> 2) & 1) ? i0 + 3 - wid : i0 + wid;
        if (i >= T) continue;
        const int t0 = 16 * i + g, t1 = t0 + 8;
        const int r0 = min(t0, c - 1), r1 = min(t1, c - 1);
        unsigned a[4][4];
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            a[ks][0] = S.rows[bp_swz(r0, ks * 8 + tig)];
            a[ks][1] = S.rows[bp_swz(r1, ks * 8 + tig)];
            a[ks][2] = S.rows[bp_swz(r0, ks * 8 + 4 + tig)];
            a[ks][3] = S.rows[bp_swz(r1, ks * 8 + 4 + tig)];
        }
        const int n0 = (int)S.nrm[r0], n1 = (int)S.nrm[r1];
        for (int j = 2 * i; j < U; ++j) {
            const int rb = min(8 * j + g, c - 1);
            int d[4] = {0, 0, 0, 0};
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const unsigned b[2] = {S.rows[bp_swz(rb, ks * 8 + tig)], S.rows[bp_swz(rb, ks * 8 + 4 + tig)]};
                bp_mma(a[ks], b, d);
            }
            const int u0 = 8 * j + 2 * tig, u1 = u0 + 1;
            const int m0 = (int)S.nrm[min(u0, c - 1)], m1 = (int)S.nrm[min(u1, c - 1)];
            const double k0 = S.kd2[min(u0, c - 1)], k1 = S.kd2[min(u1, c - 1)];
            const bool v0 = u0 < c, v1 = u1 < c;
            const bool k00 = v0 && u0 > t0 && alpha2 * (double)(n0 + m0 - 2 * d[0]) <= k0;
            const bool k01 = v1 && u1 > t0 && alpha2 * (double)(n0 + m1 - 2 * d[1]) <= k1;
            const bool k10 = v0 && u0 > t1 && alpha2 * (double)(n1 + m0 - 2 * d[2]) <= k0;
            const bool k11 = v1 && u1 > t1 && alpha2 * (double)(n1 + m1 - 2 * d[3]) <= k1;
            const unsigned b00 = __ballot_sync(PK_FULL, k00), b01 = __ballot_sync(PK_FULL, k01);
            const unsigned b10 = __ballot_sync(PK_FULL, k10), b11 = __ballot_sync(PK_FULL, k11);
            if (lane < 16) {
                const int r = lane & 7;
                const unsigned e0 = lane < 8 ? b00 : b10, e1 = lane < 8 ? b01 : b11;
                const unsigned byte = bp_spread4((e0 >> (4 * r)) & 15u) | (bp_spread4((e1 >> (4 * r)) & 15u) << 1);
                const int t = 16 * i + lane;
                if (t < c) reinterpret_cast<unsigned char*>(S.kill)[t * S.words * 4 + j] = (unsigned char)byte;
            }
        }
    }
    __syncthreads();
    // greedy picks (warp 0), 32 candidates (one bit word) at a time: lane j holds
    // candidate 32w + j's occlusion word w, so a pick inside the word is an ffs + a
    // shuffle; the word's picks then clear their bits in later words (OR-reduce)
    if (wid == 0) {
        const int nw = (c + 31) >> 5;
        unsigned acc = 0u;  // lane v: bits of word v occluded by the picks so far
        int sel = 0;
        for (int w = 0; w < nw && sel < R; ++w) {
            const int x = 32 * w + lane;
            const int left = c - 32 * w;
            const unsigned valid = left >= 32 ? 0xffffffffu : (1u << left) - 1u;
            unsigned alive = valid & ~__shfl_sync(PK_FULL, acc, w);
            const unsigned kw = x < c ? S.kill[x * S.words + w] : 0u;
            const int sel0 = sel;
            unsigned picked = 0u;
            while (alive && sel < R) {
                const int j = __ffs(alive) - 1;
                picked |= 1u << j;
                ++sel;
                alive &= ~(1u << j);
                alive &= ~__shfl_sync(PK_FULL, kw, j);
            }
            const bool mine = (picked >> lane) & 1u;
            if (mine) out[sel0 + __popc(picked & ((1u << lane) - 1u))] = (int)S.ki2[x];
            if (sel < R) {
                for (int v = w + 1; v < nw; ++v) {
                    const unsigned r = __reduce_or_sync(PK_FULL, mine ? S.kill[x * S.words + v] : 0u);
                    if (lane == v) acc |= r;
                }
            }
        }
        if (lane == 0) {
            S.scal[8] = sel;
            if (pairs) *pairs += (long long)c * (c - 1) / 2;
        }
    }
    __syncthreads();
    return S.scal[8];
}

// build phase 2 for u8 rows (d = 128): one block per inserted point; items with
// more than BP_CAP candidates are queued for build_prune_kernel
__global__ void __launch_bounds__(BP_THREADS) build_prune_block_kernel(BuildArgs A, int* over, int* nover) {
    extern __shared__ __align__(16) unsigned char smem[];
    const BPSmem S = carve_bp(smem, BP_CAP);
    const int tid = threadIdx.x;
    const int R = A.P.R;
    long long pairs = 0;
    __shared__ int s_tick[2];
    BlockTickets tk{s_tick, 0, 0};
    for (int t = tk.first(A.ticket); t < A.m; __syncthreads(), t = tk.next(A.ticket)) {
        tk.take_next(A.ticket);
        const unsigned p = (unsigned)A.bids[t];
        const int vl = A.vlen[t];
        const int nd = __ldg(A.P.deg + p);
        const int c0 = vl + nd;
        if (c0 > BP_CAP) {
            if (tid == 0) over[atomicAdd(nover, 1)] = t;
            continue;
        }
        const unsigned* vi = A.vlog_i + (size_t)t * A.vcap;
        const double* vd = A.vlog_d + (size_t)t * A.vcap;
        const int* row = A.P.adj + (size_t)p * R;
        uint4 q[8];
        const uint4* qv = reinterpret_cast<const uint4*>(A.D.X8 + (size_t)p * 32);
        unsigned nq0 = 0u, nq1 = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            q[i] = __ldg(qv + i);
            nq0 = __dp4a(q[i].x, q[i].x, nq0);
            nq1 = __dp4a(q[i].y, q[i].y, nq1);
            nq0 = __dp4a(q[i].z, q[i].z, nq0);
            nq1 = __dp4a(q[i].w, q[i].w, nq1);
        }
        const unsigned nq = nq0 + nq1;
        // candidates in input order: visit log (distances known), then the current out-row
        for (int x = tid; x < c0; x += BP_THREADS) {
            if (x < vl) {
                S.kd[x] = vd[x];
                S.ki[x] = vi[x];
            } else {
                const unsigned id = (unsigned)__ldg(row + x - vl);
                S.ki[x] = id;
                S.kd[x] = (double)bp_dist_global(q, nq, A.D.X8 + (size_t)id * 32);
            }
        }
        const int P = next_pow2_dev(c0 < 2 ? 2 : c0);
        for (int x = c0 + tid; x < P; x += BP_THREADS) {
            S.kd[x] = __longlong_as_double(0x7ff0000000000000LL);
            S.ki[x] = 0xffffffffu;
        }
        __syncthreads();
        bp_sort(S.kd, S.ki, P);
        const int c = bp_unique(S, c0, p);
        int* out = A.new_ids + (size_t)t * R;
        // the build always prunes (_kernels.py:370), even c <= R candidates
        int sel = c;
        if (c <= 1) {
            if (tid == 0 && c == 1) out[0] = (int)S.ki2[0];
        } else {
            sel = bp_prune(A.D.X8, S, c, A.alpha2, R, out, &pairs);
        }
        for (int x = sel + tid; x < R; x += BP_THREADS) out[x] = -1;
        if (tid == 0) A.new_len[t] = sel;
        __syncthreads();
    }
    if (tid == 0 && A.stats && pairs)
        atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 1), (unsigned long long)pairs);
}

// reverse-edge re-prune for u8 rows (d = 128): one block per target vertex
// (groups above BP_CAP go to reverse_big_kernel / the selection path as in
// reverse_kernel)
// cap = candidate room of this launch: groups with cap < c0 <= BP_CAP_MAX are
// queued on (mid, nmid) for the next launch (cap 128 -> 256 -> 512, each over
// the previous one's queue; the last launch passes mid = null).
template <int MODE, int QV>
__global__ void __launch_bounds__(BP_THREADS) reverse_block_kernel(RevArgs A, int cap, const int* items,
                                                                   const int* nitems, int* mid, int* nmid) {
    extern __shared__ __align__(16) unsigned char smem[];
    const BPSmem S = carve_bp(smem, cap);
    const int tid = threadIdx.x, wid = tid >> 5;
    const MakeAt<MODE, QV> make{A.D};
    const int nt = items ? *nitems : *A.ntargets;
    long long ev = 0;
    __shared__ int s_tick[2];
    BlockTickets tk{s_tick, 0, 0};
    for (int it = tk.first(A.ticket); it < nt; __syncthreads(), it = tk.next(A.ticket)) {
        tk.take_next(A.ticket);
        const int s = items ? items[it] : it;
        const unsigned u = (unsigned)A.targets[s];
        if (A.world > 1 && (int)(u % (unsigned)A.world) != A.rank) {
            if (tid == 0) A.cnt[u] = 0;
            continue;
        }
        const int nd = A.deg[u];
        const int off = A.offs[s];
        const int size = A.sizes[s];
        int* row = A.adj + (size_t)u * A.R;
        const int c0 = nd + size;
        int sel;
        if (c0 > cap && c0 <= BP_CAP_MAX && mid) {
            if (tid == 0) mid[atomicAdd(nmid, 1)] = s;
            continue;
        }
        if (c0 > BP_CAP_MAX) {
            if (c0 <= A.capB) {
                if (tid == 0) A.biglist[atomicAdd(A.nbig, 1)] = s;
                continue;
            }
            if (wid == 0) {
                sel = prune_by_selection(A, u, make, S.kd, S.ki, reinterpret_cast<unsigned char*>(S.rows), S.nrm, nd,
                                         off, size, row, &ev);
                if (lane_id() == 0) S.scal[9] = sel;
            }
            __syncthreads();
            sel = S.scal[9];
        } else {
            uint4 q[8];
            const uint4* qv = reinterpret_cast<const uint4*>(A.D.X8 + (size_t)u * 32);
            unsigned nq0 = 0u, nq1 = 0u;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                q[i] = __ldg(qv + i);
                nq0 = __dp4a(q[i].x, q[i].x, nq0);
                nq1 = __dp4a(q[i].y, q[i].y, nq1);
                nq0 = __dp4a(q[i].z, q[i].z, nq0);
                nq1 = __dp4a(q[i].w, q[i].w, nq1);
            }
            const unsigned nq = nq0 + nq1;
            for (int x = tid; x < c0; x += BP_THREADS) {
                const unsigned id = x < nd ? (unsigned)row[x] : (unsigned)A.adds[off + x - nd];
                S.ki[x] = id;
                S.kd[x] = (double)bp_dist_global(q, nq, A.D.X8 + (size_t)id * 32);
            }
            if (c0 - nd <= 64 && nd + 64 <= cap) {
                __syncthreads();
                bp_sort_row_plus_adds(S, nd, c0);
            } else {
                const int P = next_pow2_dev(c0 < 2 ? 2 : c0);
                for (int x = c0 + tid; x < P; x += BP_THREADS) {
                    S.kd[x] = __longlong_as_double(0x7ff0000000000000LL);
                    S.ki[x] = 0xffffffffu;
                }
                __syncthreads();
                bp_sort(S.kd, S.ki, P);
            }
            const int c = bp_unique(S, c0, u);
            if (tid == 0) ev += c0;
            if (c <= A.R) {
                for (int x = tid; x < c; x += BP_THREADS) row[x] = (int)S.ki2[x];
                sel = c;
            } else {
                sel = bp_prune(A.D.X8, S, c, A.alpha2, A.R, row, &ev);
            }
        }
        for (int x = sel + tid; x < A.R; x += BP_THREADS) row[x] = -1;
        if (tid == 0) {
            A.deg[u] = sel;
            A.cnt[u] = 0;
        }
        __syncthreads();
    }
    if (tid == 0 && A.stats && ev) atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 2), (unsigned long long)ev);
}

#include "prune_tc.cuh"

// one thread, one full distance between two point ids (exact in every mode)
template <int MODE>
__device__ __forceinline__ double thread_dist(const DataRef& D, unsigned a, unsigned b) {
    if (MODE == MODE_EXACT_U8) return (double)u8_row_dist(D.X8 + (size_t)a * D.dw, D.X8 + (size_t)b * D.dw, D.dw);
    Seq64Member q{D.X + (size_t)a * D.dp, D.dp};
    return q.eval_one(D.X, (int)b);
}

constexpr int kBigThreads = 256;

// Reverse-edge groups with more than A.cap candidates (hub vertices that
// receive hundreds of new in-edges in one batch): one block per group.
// Candidates are sorted by (dist, id) with a block bitonic sort; duplicates
// and the vertex itself are marked dead instead of compacted; the RobustPrune
// picks stay sequential, each kill step runs over all block threads.
template <int MODE, int QV>
__global__ void __launch_bounds__(kBigThreads) reverse_big_kernel(RevArgs A) {
    __shared__ unsigned wbuf[kBigThreads];  // per-warp queues of the fp32 screen
    const bool screen = MODE == MODE_SEQ64 && A.D.dp <= 128 * QV && A.D.screen;
    extern __shared__ __align__(16) unsigned char smem[];
    double* kd = reinterpret_cast<double*>(smem);
    unsigned* ki = reinterpret_cast<unsigned*>(smem + (size_t)A.capB * 8);
    unsigned char* alive = smem + (size_t)A.capB * 12;
    __shared__ int s_t;
    const int tid = threadIdx.x;
    const int nb = *A.nbig;
    long long ev = 0;
    __shared__ int s_tick[2];
    BlockTickets tk{s_tick, 0, 0};
    for (int g = tk.first(A.ticket); g < nb; __syncthreads(), g = tk.next(A.ticket)) {
        tk.take_next(A.ticket);
        const int s = A.biglist[g];
        const unsigned u = (unsigned)A.targets[s];
        const int nd = A.deg[u];
        const int off = A.offs[s];
        const int c0 = nd + A.sizes[s];
        int* row = A.adj + (size_t)u * A.R;
        const int P = next_pow2_dev(c0);
        for (int x = tid; x < P; x += kBigThreads) {
            if (x < c0) {
                const unsigned w = x < nd ? (unsigned)row[x] : (unsigned)A.adds[off + x - nd];
                ki[x] = w;
                kd[x] = thread_dist<MODE>(A.D, u, w);
            } else {
                ki[x] = 0xffffffffu;
                kd[x] = __longlong_as_double(0x7ff0000000000000LL);
            }
        }
        ev += c0;
        __syncthreads();
        for (int k = 2; k <= P; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < P; i += kBigThreads) {
                    const int x = i ^ j;
                    if (x > i) {
                        double a = kd[i], b = kd[x];
                        unsigned ia = ki[i], ib = ki[x];
                        if (key_lt(b, ib, a, ia) == ((i & k) == 0)) {
                            kd[i] = b; kd[x] = a;
                            ki[i] = ib; ki[x] = ia;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int x = tid; x < c0; x += kBigThreads)
            alive[x] = ki[x] != u && !(x > 0 && ki[x - 1] == ki[x] && kd[x - 1] == kd[x]);
        __syncthreads();
        int sel = 0, t = 0;
        while (sel < A.R) {
            if (tid < 32) {
                int nt = -1;
                for (int base = t; base < c0; base += 32) {
                    const int i = base + tid;
                    const unsigned bal = __ballot_sync(PK_FULL, i < c0 && alive[i]);
                    if (bal) { nt = base + __ffs(bal) - 1; break; }
                }
                if (tid == 0) s_t = nt;
            }
            __syncthreads();
            t = s_t;
            if (t < 0) break;
            if (tid == 0) row[sel] = (int)ki[t];  // the row was fully read into ki above
            ++sel;
            if (sel >= A.R) break;
            const unsigned ps = ki[t];
            if (screen) {
                // float data: each warp screens its 32-position chunks of the alive tail
                Fp32Pick<QV> pick;
                pick.load(A.D.X, A.D.dp, ps);
                const int wid = tid >> 5;
                const long long nev = screened_kill_pass<QV>(A.D.X, A.D.dp, ps, pick, kd, ki, alive, wbuf + 32 * wid,
                                                             A.alpha2, t + 1 + 32 * wid, c0, kBigThreads);
                if ((tid & 31) == 0) ev += nev;
            } else {
                for (int x = t + 1 + tid; x < c0; x += kBigThreads) {
                    if (alive[x]) {
                        ++ev;
                        if (A.alpha2 * thread_dist<MODE>(A.D, ps, ki[x]) <= kd[x]) alive[x] = 0;
                    }
                }
            }
            ++t;
            __syncthreads();
        }
        __syncthreads();
        for (int x = sel + tid; x < A.R; x += kBigThreads) row[x] = -1;
        if (A.adjd)
            for (int x = tid; x < A.R; x += kBigThreads) A.adjd[(size_t)u * A.R + x] = __longlong_as_double(0x7ff8000000000000LL);
        if (tid == 0) {
            A.deg[u] = sel;
            A.cnt[u] = 0;
        }
        __syncthreads();
    }
    if (A.stats && ev) atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 2), (unsigned long long)ev);
}

__global__ void robust_prune_api_kernel(const float* X, int dp, unsigned p, const long long* cand_ids,
                                        const double* cand_d, int m, const long long* cur_ids, int dcount,
                                        double alpha2, int R, int cap, long long* out, long long* out_count,
                                        int* scratch_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* kd = reinterpret_cast<double*>(smem);
    unsigned* ki = reinterpret_cast<unsigned*>(smem + (size_t)cap * 8);
    unsigned* pcbuf = reinterpret_cast<unsigned*>(smem + (size_t)cap * 12);
    unsigned char* alive = smem + (size_t)cap * 12 + 128;
    unsigned* ord = reinterpret_cast<unsigned*>(smem + (size_t)cap * 13 + 128);
    const int lane = lane_id();
    const int c0 = m + dcount;
    Seq64Member du{X + (size_t)p * dp, dp};
    // candidates in reference order: given candidates, then current out-list
    for (int x = lane; x < m; x += 32) {
        kd[x] = cand_d[x];
        ki[x] = (unsigned)cand_ids[x];
    }
    for (int e0 = 0; e0 < dcount; e0 += 32) {
        const int cnt = min(32, dcount - e0);
        unsigned w = lane < cnt ? (unsigned)cur_ids[e0 + lane] : 0u;
        double dd = du.eval(X, (int)w, cnt);
        if (lane < cnt) {
            kd[m + e0 + lane] = dd;
            ki[m + e0 + lane] = w;
        }
    }
    __syncwarp();
    // _canon_candidates keeps the FIRST occurrence (in input order) of a
    // duplicated id together with its distance: resolve duplicates before the
    // (dist, id) sort by marking later copies dead.
    for (int x = lane; x < c0; x += 32) {
        bool dupl = ki[x] == p;
        for (int y = 0; y < x && !dupl; ++y) dupl = ki[y] == ki[x];
        ord[x] = dupl ? 1u : 0u;
    }
    __syncwarp();
    for (int x = lane; x < c0; x += 32)
        if (ord[x]) {
            kd[x] = __longlong_as_double(0x7ff0000000000000LL);
            ki[x] = 0xffffffffu;
        }
    const int Pw = next_pow2_dev(c0);
    for (int x = c0 + lane; x < Pw; x += 32) {
        kd[x] = __longlong_as_double(0x7ff0000000000000LL);
        ki[x] = 0xffffffffu;
    }
    __syncwarp();
    warp_sort(kd, ki, Pw);
    int c = 0;
    for (int x = 0; x < c0; ++x)
        if (ki[x] != 0xffffffffu) c = x + 1;
    struct Mk {
        const float* X;
        int dp;
        __device__ Seq64Member operator()(unsigned id) const { return Seq64Member{X + (size_t)id * dp, dp}; }
    } make{X, dp};
    long long ev = 0;
    int sel = warp_prune(X, kd, ki, c, alpha2, R, alive, pcbuf, scratch_out, make, &ev);
    for (int x = lane; x < sel; x += 32) out[x] = scratch_out[x];
    if (lane == 0) *out_count = sel;
}

__global__ void centroid_kernel(const float* X, int n, int dp, double* cen) {
    // one thread per coordinate, sequential over points (the reference order)
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= dp) return;
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc += (double)X[(size_t)j * dp + t];
    cen[t] = acc / (double)n;
}

__global__ void nearest_kernel(const float* X, int n, int dp, const double* cen, double* bd, int* bi) {
    __shared__ double sd[256];
    __shared__ int si[256];
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bid = 0x7fffffff;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        Seq64Vector q{cen, dp};
        double d = q.eval_one(X, j);
        if (d < best || (d == best && j < bid)) { best = d; bid = j; }
    }
    sd[threadIdx.x] = best;
    si[threadIdx.x] = bid;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int x = 1; x < blockDim.x; ++x)
            if (sd[x] < best || (sd[x] == best && si[x] < bid)) { best = sd[x]; bid = si[x]; }
        bd[blockIdx.x] = best;
        bi[blockIdx.x] = bid;
    }
}

__global__ void nearest_final_kernel(const double* bd, const int* bi, int g, long long* out) {
    double best = bd[0];
    int bid = bi[0];
    for (int x = 1; x < g; ++x)
        if (bd[x] < best || (bd[x] == best && bi[x] < bid)) { best = bd[x]; bid = bi[x]; }
    *out = bid;
}

// ---- host driver -----------------------------------------------------------------------------
template <class K>
int config_kernel(K kern, size_t warp_bytes, int want_wpb, int* wpb_out, int* grid_out) {
    int wpb = want_wpb;
    while (wpb > 1 && warp_bytes * wpb > (size_t)max_smem_optin()) wpb >>= 1;
    if (warp_bytes * wpb > (size_t)max_smem_optin()) {
        set_error("per-warp shared memory exceeds the device limit");
        return 2;
    }
    PK_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(warp_bytes * wpb)));
    int per_sm = 0;
    PK_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpb, warp_bytes * wpb));
    *wpb_out = wpb;
    *grid_out = sm_count() * (per_sm < 1 ? 1 : per_sm);
    return 0;
}

// tc_knn.cu: tensor-core screens of all points against the start set
bool tc_supported();
int tc_seed_mask(const float* x, int n, int dp, const int* starts, int s, int take, unsigned* mask, int mw,
                 int* near, cudaStream_t st, const long long* rows_ids = nullptr);
// scan.cu: exact u8 distances of every point to every start on the integer tensor cores
int u8_seed_table(const unsigned* x8, int n, const int* starts, int s, unsigned* tab, cudaStream_t st);

// nearest start of every point from the u8 start-distance table (ties: lowest index)
__global__ void argmin_rows_kernel(const unsigned* __restrict__ tab, int n, int s, int* __restrict__ near) {
    const int lane = lane_id();
    const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = w; r < n; r += nw) {
        const unsigned* row = tab + (size_t)r * s;
        unsigned long long best = ~0ull;
        for (int j = lane; j < s; j += 32) {
            const unsigned long long k = ((unsigned long long)__ldg(row + j) << 32) | (unsigned)j;
            best = k < best ? k : best;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const unsigned long long ob = __shfl_xor_sync(PK_FULL, best, o);
            best = ob < best ? ob : best;
        }
        if (lane == 0) near[r] = (int)(best & 0xffffffffull);
    }
}

// ---- locality order of the batches' points ------------------------------------
// key of position i of the insertion order: (batch of i, nearest start of the
// point); batches are [2^b - 1, 2^(b+1) - 1), so the batch is floor(log2(i + 1))
__global__ void locality_keys_kernel(const int* order, int n, const int* near, int sbits, unsigned* keys, int* vals) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned b = 31u - (unsigned)__clz((unsigned)i + 1u);
        const int p = order[i];
        keys[i] = (b << sbits) | (unsigned)near[p];
        vals[i] = p;
    }
}

// A permutation of `order` that keeps every batch's set of points and sorts
// each batch by nearest start (stable radix sort of the composite keys).
int locality_order(const int* order, int n, const int* near, int s, int** out, cudaStream_t st) {
    int sbits = 1;
    while ((1 << sbits) < s) ++sbits;
    const int end_bit = sbits + 5;  // <= 32 batches
    unsigned *k0 = nullptr, *k1 = nullptr;
    int* v0 = nullptr;
    PK_CHECK(scratch(&k0, (size_t)n, st));
    PK_CHECK(scratch(&k1, (size_t)n, st));
    PK_CHECK(scratch(&v0, (size_t)n, st));
    PK_CHECK(scratch(out, (size_t)n, st));
    {
        ProfScope _ps("locality_keys_kernel", st);
        locality_keys_kernel<<<grid_for(n, 256), 256, 0, st>>>(order, n, near, sbits, k0, v0);
    }
    PK_CHECK_LAUNCH("locality_keys_kernel");
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, k0, k1, v0, *out, n, 0, end_bit, st);
    void* tmp = nullptr;
    PK_CHECK(cudaMallocAsync(&tmp, bytes + 16, st));
    {
        ProfScope _ps("cub_DeviceRadixSort_SortPairs", st);
        PK_CHECK(cub::DeviceRadixSort::SortPairs(tmp, bytes, k0, k1, v0, *out, n, 0, end_bit, st));
    }
    for (void* p : {(void*)k0, (void*)k1, (void*)v0, tmp}) release(p, st);
    return 0;
}

template <int MODE, int QV>
int run_build(const DataRef& D, int n, int R, int L, double alpha, const int* starts, int s, const int* order,
              int* adj, int* deg, long long* stats, int hash_bits, const Shard& SH, cudaStream_t st) {
    const bool u8 = MODE == MODE_EXACT_U8;
    if ((long long)n > (long long)PK_IDMASK) {
        set_error("too many points for the beam kernels (ids are 30-bit)");
        return 2;
    }
    const int H = choose_hash(L, hash_bits, n);
    const int cap = next_pow2(2 * L + 64 + R);
    const int vcap = cap - R;
    // reverse groups: row (<= R) + incoming sources; larger groups take the
    // selection path (prune_by_selection)
    const int capR = next_pow2(std::max(4 * R, 256));
    // staged u8 rows per warp (prune / reverse): more rows = fewer L2 reads in
    // the kill loop, fewer rows = more warps per SM (PK_PRUNE_S / PK_REV_S tune)
    const int S = std::min(cap, env_int("PK_PRUNE_S", 128));
    const int SR = std::min(capR, env_int("PK_REV_S", 128));

    BuildArgs A;
    // row ring of the float searches with lazy keys (beam.cuh carve_ring), behind the beam state
    const bool lazy_screen = MODE == MODE_SEQ64 && D.screen && env_int("PK_LAZY", 1) == 1 && n < (long long)PK_IDMASK;
    int ring = MODE == MODE_SEQ64 && QV >= 4 && env_int("PK_RING_BUILD", 0) == 1 ? ring_slots(D.dp, QV, lazy_screen) : 0;
    if (align16(beam_smem_bytes(L, H)) + align16(ring_smem_bytes(D.dp, ring)) > (size_t)max_smem_optin()) ring = 0;
    // with the ring, the seen table moves to a global slab per warp (carve_beam_gh)
    const bool ghash = ring && env_int("PK_HASH_GLOBAL", 1) == 1;
    A.search_bytes = align16(beam_smem_bytes(L, ghash ? 0 : H)) + align16(ring_smem_bytes(D.dp, ring));
    A.prune_bytes = cand_smem_bytes(cap, D.dw, S, u8);
    auto sk = build_search_kernel<MODE, QV, false>;
    if constexpr (MODE == MODE_SEQ64 && QV >= 4) {
        if (ring) sk = build_search_kernel<MODE, QV, true>;
    }
    auto pkk = build_prune_kernel<MODE, QV>;
    auto rk = reverse_kernel<MODE, QV>;
    int wpb_s, grid_s, wpb_p, grid_p, wpb_r, grid_r, rc;
    if ((rc = config_kernel(sk, A.search_bytes, 4, &wpb_s, &grid_s))) return rc;
    if ((rc = config_kernel(pkk, A.prune_bytes, 2, &wpb_p, &grid_p))) return rc;
    const size_t wbr = cand_smem_bytes(capR, D.dw, SR, u8);
    if ((rc = config_kernel(rk, wbr, 2, &wpb_r, &grid_r))) return rc;
    // u8 rows of d = 128: block-per-item RobustPrune on the integer tensor cores
    const bool blockp = MODE == MODE_EXACT_U8 && D.dw == 32 && env_int("PK_BLOCK_PRUNE", 1) == 1;
    auto bpk = build_prune_block_kernel;
    auto rbk = reverse_block_kernel<MODE, QV>;
    int grid_bp = 0, grid_rb = 0;
    constexpr int kRevCap = 128;  // most reverse groups (row + this batch's sources) fit 128
    if (blockp) {
        const int bytes = (int)bp_smem_bytes(BP_CAP);
        PK_CHECK(cudaFuncSetAttribute(bpk, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        PK_CHECK(cudaFuncSetAttribute(rbk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)bp_smem_bytes(BP_CAP_MAX)));
        int per_sm = 0;
        PK_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bpk, BP_THREADS, bytes));
        grid_bp = sm_count() * std::max(1, per_sm);
        PK_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rbk, BP_THREADS, bp_smem_bytes(kRevCap)));
        grid_rb = sm_count() * std::max(1, per_sm);
    }
    // float data (SEQ64, dp <= 1024): block-per-item RobustPrune on the tensor cores
    const int tcmode = env_int("PK_TC_PRUNE", 1);  // 1: build + reverse, 2: build only, 3: reverse only
    const bool tcp = MODE == MODE_SEQ64 && D.dp <= 128 * QV && QV <= 8 && D.screen && tcmode >= 1 && tcmode <= 3;
    const bool tcb = tcp && tcmode != 3, tcr = tcp && tcmode != 2;
    auto tpk = prune_tc_build_kernel<QV, PT_CAP>;
    auto tpk2 = prune_tc_build_kernel<QV, PT_CAP_BIG>;
    auto trk = prune_tc_reverse_kernel<MODE, QV, PT_CAP>;
    auto trk2 = prune_tc_reverse_kernel<MODE, QV, PT_CAP_BIG>;
    double* nrm64 = nullptr;
    if (tcp) {
        PK_CHECK(cudaFuncSetAttribute(tpk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PT_SMEM));
        PK_CHECK(cudaFuncSetAttribute(tpk2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)pt_smem_bytes(PT_CAP_BIG)));
        PK_CHECK(cudaFuncSetAttribute(trk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PT_SMEM));
        PK_CHECK(cudaFuncSetAttribute(trk2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)pt_smem_bytes(PT_CAP_BIG)));
        PK_CHECK(scratch(&nrm64, (size_t)n, st));
        {
            ProfScope _ps("norms64_kernel", st);
            norms64_kernel<<<sm_count() * 8, 256, 0, st>>>(D.X, n, D.dp, nrm64);
        }
        PK_CHECK_LAUNCH("norms64_kernel");
    }
    // fp16 copy of the rows for the Gram tiles (half the gather bytes, half the K
    // chunks of the tf32 Gram; PK_PRUNE_F16=0: tf32 from the fp32 rows)
    __half* xh = nullptr;
    const int kph = (D.dp + 63) & ~63;
    if (tcp && env_int("PK_PRUNE_F16", 1) == 1) {
        PK_CHECK(scratch(&xh, (size_t)n * kph, st));
        {
            ProfScope _ps("rows_to_half_kernel", st);
            rows_to_half_kernel<<<sm_count() * 16, 256, 0, st>>>(D.X, n, D.dp, kph, xh);
        }
        PK_CHECK_LAUNCH("rows_to_half_kernel");
    }
    // item counters of the block-per-item launches of a batch (BlockTickets), zeroed once per batch:
    // [0] build prune, [1..3] reverse launches, [4] reverse_big_kernel
    int* ptick = nullptr;
    if (env_int("PK_TICKETS", 1) == 1) PK_CHECK(scratch(&ptick, 8, st));
    PTAux aux{nrm64, xh, kph, nullptr};
    const int capB = 8192;
    const size_t big_bytes = (size_t)capB * 13 + 16;
    auto bigk = reverse_big_kernel<MODE, QV>;
    PK_CHECK(cudaFuncSetAttribute(bigk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_bytes));
    const int grid_big = 2 * sm_count();
    int* biglist = nullptr;
    int* nbig = nullptr;

    int maxb = 1;
    while (maxb < n) maxb <<= 1;
    const int mb = std::min(maxb, n);           // largest batch
    const long long E = (long long)mb * R;      // max edges per batch
    const int ub = (int)std::min<long long>(n, E);

    unsigned *vlog_i = nullptr, *err = nullptr;
    double *vlog_d = nullptr, *adist = nullptr;
    int *vlen = nullptr, *new_ids = nullptr, *new_len = nullptr, *cnt = nullptr, *tslot = nullptr;
    int *targets = nullptr, *sizes = nullptr, *offs = nullptr, *fill = nullptr, *adds = nullptr, *ntargets = nullptr;
    unsigned char* aalive = nullptr;
    PK_CHECK(scratch(&vlog_i, (size_t)mb * vcap, st));
    PK_CHECK(scratch(&vlog_d, (size_t)mb * vcap, st));
    PK_CHECK(scratch(&vlen, (size_t)mb, st));
    const bool multi = SH.world > 1;
    // float data on the tensor-core prune path, one GPU: adjacency rows carry the
    // exact distances of their entries (NaN = unknown) so re-prunes need none
    const bool dcache = tcb && tcr && !multi && env_int("PK_ROW_DIST", 1) == 1;
    double *adjd = nullptr, *new_d = nullptr, *addd = nullptr;
    if (dcache) {
        PK_CHECK(scratch(&adjd, (size_t)n * R, st));
        PK_CHECK(scratch(&new_d, (size_t)E, st));
        PK_CHECK(scratch(&addd, (size_t)E, st));
        PK_CHECK(cudaMemsetAsync(adjd, 0xff, sizeof(double) * (size_t)n * R, st));  // all NaN
    }
    if (multi) {
        new_ids = SH.xids;
        new_len = SH.xlen;
    } else {
        PK_CHECK(scratch(&new_ids, (size_t)E, st));
        PK_CHECK(scratch(&new_len, (size_t)mb, st));
    }
    int* npack = nullptr;
    PK_CHECK(scratch(&npack, 1, st));
    int *over = nullptr, *nover = nullptr, *over1 = nullptr;  // over1 / nover[1]: first tensor-core launch's queue
    PK_CHECK(scratch(&over, (size_t)mb, st));
    PK_CHECK(scratch(&over1, (size_t)mb, st));
    PK_CHECK(scratch(&nover, 2, st));
    int *midl = nullptr, *nmid = nullptr, *midl2 = nullptr, *nmid2 = nullptr;
    PK_CHECK(scratch(&midl, (size_t)ub, st));
    PK_CHECK(scratch(&nmid, 1, st));
    PK_CHECK(scratch(&midl2, (size_t)ub, st));
    PK_CHECK(scratch(&nmid2, 1, st));
    PK_CHECK(scratch(&cnt, (size_t)n, st));
    PK_CHECK(scratch(&tslot, (size_t)n, st));
    PK_CHECK(scratch(&targets, (size_t)ub, st));
    PK_CHECK(scratch(&sizes, (size_t)ub + 1, st));
    PK_CHECK(scratch(&offs, (size_t)ub + 1, st));
    PK_CHECK(scratch(&fill, (size_t)ub, st));
    PK_CHECK(scratch(&adds, (size_t)E, st));
    PK_CHECK(scratch(&adist, (size_t)E, st));
    PK_CHECK(scratch(&aalive, (size_t)E, st));
    PK_CHECK(scratch(&ntargets, 1, st));
    PK_CHECK(scratch(&biglist, (size_t)ub, st));
    PK_CHECK(scratch(&nbig, 1, st));
    PK_CHECK(scratch(&err, 1, st));
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, sizes, offs, ub + 1, st);
    PK_CHECK(cudaMallocAsync(&cub_tmp, cub_bytes + 16, st));

    PK_CHECK(cudaMemsetAsync(adj, 0xff, sizeof(int) * (size_t)n * R, st));
    PK_CHECK(cudaMemsetAsync(deg, 0, sizeof(int) * (size_t)n, st));
    PK_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int) * (size_t)n, st));
    PK_CHECK(cudaMemsetAsync(err, 0, sizeof(unsigned), st));

    A.P = SearchParams{D.X, D.dp, adj, R, deg, starts, s};
    A.P.screen = D.screen;
    A.P.prefetch = env_int("PK_PREFETCH", 0) == 1;  // adjacency-row L1 prefetch: measured slower on every configuration
    A.P.prefetch_rows = env_int("PK_PREFETCH_ROWS", 0) == 1 && D.dp >= 512;  // L2 prefetch of candidate rows: a gain before the ticket scheduling, a 2 % loss since
    A.P.lazy = env_int("PK_LAZY", 1) == 1 && n < (long long)PK_IDMASK;
    A.P.ring = ring;
    int* ticket = nullptr;
    if (env_int("PK_TICKETS", 1) == 1) PK_CHECK(scratch(&ticket, 1, st));
    unsigned char* gh = nullptr;
    if (ghash) {
        A.P.ghash_stride = (size_t)H * 2;
        PK_CHECK(scratch(&gh, (size_t)grid_s * wpb_s * A.P.ghash_stride, st));
        A.P.ghash = gh;
    }
    A.P.seed_select = env_int("PK_SEED_SELECT", 1);
    if (SH.seed_bd && SH.seed_bi && SH.seed_bl && SH.world == 1) {
        A.P.seed_bd = SH.seed_bd;
        A.P.seed_bi = SH.seed_bi;
        A.P.seed_bl = SH.seed_bl;
        A.P.seed_save = 1;
    }
    // counting mode (bench.py's untimed pass): exact distinct evaluations -> stats[4]
    unsigned* ubm = nullptr;
    if (stats && env_int("PK_COUNT_UNIQUE", 0) == 1) {
        A.P.uwords = (n + 31) / 32;
        PK_CHECK(scratch(&ubm, (size_t)grid_s * wpb_s * A.P.uwords, st));
        A.P.ubm = ubm;
    }
    // float data, one GPU: the start set pre-screened on the tensor cores; a
    // search fp32-screens only the starts whose bound can reach its take-th
    // (tc_knn.cu tc_seed_mask, beam.cuh seed_select_lazy)
    unsigned* seed_mask = nullptr;
    int* near = nullptr;
    // (replicated on every rank of a sharded build: the mask is per point and the
    // same on every rank, so each rank's searches of its chunk use it unchanged)
    if (MODE == MODE_SEQ64 && D.screen && A.P.lazy && A.P.seed_select && !ubm && L >= 128 && s > L && n >= 4096 &&
        s >= env_int("PK_SEED_TC_MIN", 256) && s <= 8192 && env_int("PK_SEED_TC", 1) == 1 && tc_supported()) {
        const int mw = (s + 31) / 32;
        PK_CHECK(scratch(&seed_mask, (size_t)n * mw, st));
        // (sharded builds: the ranks must agree on the chunks of every batch, and the
        // order below is derived from floating-point screens, so rank 0's order is
        // broadcast -- PK_XCHG_ORDER, below)
        if (env_int("PK_LOCALITY", 1) == 1 && (!multi || R >= 4)) PK_CHECK(scratch(&near, (size_t)n, st));
        if ((rc = tc_seed_mask(D.X, n, D.dp, starts, s, std::min(L, s), seed_mask, mw, near, st))) return rc;
        A.P.seed_mask = seed_mask;
        A.P.seed_mw = mw;
    }
    // Search order inside each batch: a batch's searches and prunes are
    // independent (every search reads the graph as it stood before the batch,
    // the re-prunes sort their candidates), so the points of a batch may run in
    // any order without changing the graph.  Grouped by their nearest start,
    // the warps running at the same time walk the same region of the data and
    // share its rows in L2 instead of each pulling its own from HBM.
    // u8 rows of d = 128: the exact start distances of every point from one
    // integer tensor-core pass (beam.cuh seed_select reads them); the nearest start
    // of every point falls out of the table (the locality key of the u8 builds)
    unsigned* seed_tab = nullptr;
    if (MODE == MODE_EXACT_U8 && D.dw == 32 && D.X8 && A.P.seed_select && !ubm && L >= 128 &&
        (L & (L - 1)) == 0 && s > 32 && (long long)n * s <= (1ll << 31) && env_int("PK_SEED_TAB", 1) == 1) {
        PK_CHECK(scratch(&seed_tab, (size_t)n * s, st));
        if ((rc = u8_seed_table(D.X8, n, starts, s, seed_tab, st))) return rc;
        A.P.seed_tab = seed_tab;
        if (!near && env_int("PK_LOCALITY", 1) == 1 && env_int("PK_LOCALITY_U8", 1) == 1 && n >= (1 << 16) &&
            (!multi || R >= 4)) {
            PK_CHECK(scratch(&near, (size_t)n, st));
            ProfScope _ps("argmin_rows_kernel", st);
            argmin_rows_kernel<<<sm_count() * 8, 256, 0, st>>>(seed_tab, n, s, near);
        }
        PK_CHECK_LAUNCH("argmin_rows_kernel");
    }
    int* lorder = nullptr;
    if (near && n >= (1 << 16) && s <= (1 << 20)) {
        if ((rc = locality_order(order, n, near, s, &lorder, st))) return rc;
        if (multi) {
            // every rank computed the same keys from the same data with the same kernels;
            // rank 0's order is made authoritative anyway (xids holds >= n ints, R >= 4)
            PK_CHECK(cudaMemcpyAsync(SH.xids, lorder, sizeof(int) * (size_t)n, cudaMemcpyDeviceToDevice, st));
            PK_CHECK(cudaStreamSynchronize(st));
            if (SH.fn(SH.ctx, PK_XCHG_ORDER, n, 0) < 0) {
                set_error("search-order broadcast failed");
                return 4;
            }
            PK_CHECK(cudaMemcpyAsync(lorder, SH.xids, sizeof(int) * (size_t)n, cudaMemcpyDeviceToDevice, st));
        }
        order = lorder;
    }
    A.D = D;
    A.L = L;
    A.H = H;
    A.cap = cap;
    A.vcap = vcap;
    A.S = S;
    A.alpha2 = alpha * alpha;
    A.vlog_i = vlog_i;
    A.vlog_d = vlog_d;
    A.vlen = vlen;
    A.new_ids = new_ids;
    A.new_len = new_len;
    A.err = err;
    A.stats = stats;
    A.items = nullptr;
    A.nitems = nullptr;
    A.new_d = new_d;
    A.adjd = adjd;

    RevArgs B;
    B.X = D.X;
    B.dp = D.dp;
    B.D = D;
    B.S = SR;
    B.adj = adj;
    B.deg = deg;
    B.R = R;
    B.targets = targets;
    B.ntargets = ntargets;
    B.offs = offs;
    B.sizes = sizes;
    B.adds = adds;
    B.adist = adist;
    B.aalive = aalive;
    B.cnt = cnt;
    B.cap = capR;
    B.alpha2 = alpha * alpha;
    B.warp_bytes = wbr;
    B.stats = stats;
    B.capB = capB;
    B.biglist = biglist;
    B.nbig = nbig;
    B.rank = 0;
    B.world = 1;
    B.adjd = adjd;
    B.addd = addd;

    for (int lo = 0, batch = 1; lo < n; lo += batch, batch *= 2) {
        const int m = std::min(batch, n - lo);
        // sharded batch: rank r searches + prunes chunk r, then the out-lists are all-gathered
        const bool sharded = multi && m >= SH.min_shard;
        const int chunk = sharded ? (m + SH.world - 1) / SH.world : m;
        const int my_lo = sharded ? std::min(m, SH.rank * chunk) : 0;
        const int my_m = sharded ? std::min(m, my_lo + chunk) - my_lo : m;
        A.bids = order + lo + my_lo;
        A.m = my_m;
        A.new_ids = new_ids + (size_t)my_lo * R;
        A.new_len = new_len + my_lo;
        if (ptick) PK_CHECK(cudaMemsetAsync(ptick, 0, 8 * sizeof(int), st));
        if (my_m > 0) {
            // tickets for the large batches (searches differ in length)
            A.P.ticket = nullptr;
            if (ticket && (long long)my_m > 2ll * grid_s * wpb_s) {
                PK_CHECK(cudaMemsetAsync(ticket, 0, sizeof(int), st));
                A.P.ticket = ticket;
            }
            {
                ProfScope _ps("build_search_kernel", st);
                sk<<<std::min(grid_s, (my_m + wpb_s - 1) / wpb_s), 32 * wpb_s, A.search_bytes * wpb_s, st>>>(A);
            }
            PK_CHECK_LAUNCH("build_search_kernel");
            if (blockp || tcb) {
                PK_CHECK(cudaMemsetAsync(nover, 0, 2 * sizeof(int), st));
                aux.ticket = ptick;
                A.ticket = ptick;
                if (tcb) {
                    {
                        ProfScope _ps("prune_tc_build_kernel", st);
                        tpk<<<std::min(2 * sm_count(), my_m), PT_THREADS, PT_SMEM, st>>>(A, aux, nullptr, nullptr, over1,
                                                                                         nover + 1);
                    }
                    aux.ticket = ptick ? ptick + 5 : nullptr;
                    ProfScope _ps("prune_tc_build_kernel", st);
                    tpk2<<<std::min(sm_count(), my_m), PT_THREADS, pt_smem_bytes(PT_CAP_BIG), st>>>(A, aux, over1, nover + 1,
                                                                                                  over, nover);
                } else {
                    ProfScope _ps("build_prune_block_kernel", st);
                    bpk<<<std::min(grid_bp, my_m), BP_THREADS, bp_smem_bytes(BP_CAP), st>>>(A, over, nover);
                }
                PK_CHECK_LAUNCH("build_prune_block_kernel");
                A.items = over;  // the few items with more than BP_CAP candidates
                A.nitems = nover;
                {
                    ProfScope _ps("build_prune_kernel", st);
                    pkk<<<std::min(grid_p, sm_count()), 32 * wpb_p, A.prune_bytes * wpb_p, st>>>(A);
                }
                A.items = nullptr;
                A.nitems = nullptr;
            } else {
                ProfScope _ps("build_prune_kernel", st);
                pkk<<<std::min(grid_p, (my_m + wpb_p - 1) / wpb_p), 32 * wpb_p, A.prune_bytes * wpb_p, st>>>(A);
            }
            PK_CHECK_LAUNCH("build_prune_kernel");
        }
        if (sharded && SH.fn(SH.ctx, PK_XCHG_OUTLISTS, chunk, 0) < 0) {
            set_error("out-list exchange failed");
            return 4;
        }
        B.rank = sharded ? SH.rank : 0;
        B.world = sharded ? SH.world : 1;
        const int ubb = (int)std::min<long long>(n, (long long)m * R);
        PK_CHECK(cudaMemsetAsync(ntargets, 0, sizeof(int), st));
        PK_CHECK(cudaMemsetAsync(nbig, 0, sizeof(int), st));
        PK_CHECK(cudaMemsetAsync(sizes, 0, sizeof(int) * ((size_t)ubb + 1), st));
        PK_CHECK(cudaMemsetAsync(fill, 0, sizeof(int) * (size_t)ubb, st));
        {
            ProfScope _ps("commit_kernel", st);
            commit_kernel<<<grid_for((long long)m * 32, 256), 256, 0, st>>>(order + lo, m, R, new_ids, new_len, adj, deg,
                                                                             cnt, tslot, targets, ntargets, new_d, adjd);
        }
        PK_CHECK_LAUNCH("commit_kernel");
        {
            ProfScope _ps("sizes_kernel", st);
            sizes_kernel<<<grid_for(ubb, 256), 256, 0, st>>>(targets, ntargets, cnt, sizes);
        }
        PK_CHECK_LAUNCH("sizes_kernel");
        {
            ProfScope _ps("cub_DeviceScan_ExclusiveSum", st);
            PK_CHECK(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, sizes, offs, ubb + 1, st));
        }
        {
            ProfScope _ps("scatter_kernel", st);
            scatter_kernel<<<grid_for((long long)m * R, 256), 256, 0, st>>>(order + lo, m, R, new_ids, new_len, tslot,
                                                                             offs, fill, adds, new_d, addd);
        }
        PK_CHECK_LAUNCH("scatter_kernel");
        if (blockp) {
            PK_CHECK(cudaMemsetAsync(nmid, 0, sizeof(int), st));
            {
                B.ticket = ptick ? ptick + 1 : nullptr;
                ProfScope _ps("reverse_block_kernel", st);
                rbk<<<std::min(grid_rb, ubb), BP_THREADS, bp_smem_bytes(kRevCap), st>>>(B, kRevCap, nullptr, nullptr,
                                                                                       midl, nmid);
            }
            PK_CHECK_LAUNCH("reverse_block_kernel");
            PK_CHECK(cudaMemsetAsync(nmid2, 0, sizeof(int), st));
            {
                B.ticket = ptick ? ptick + 2 : nullptr;
                ProfScope _ps("reverse_block_kernel", st);
                rbk<<<grid_bp, BP_THREADS, bp_smem_bytes(BP_CAP), st>>>(B, BP_CAP, midl, nmid, midl2, nmid2);
            }
            PK_CHECK_LAUNCH("reverse_block_kernel");
            {
                B.ticket = ptick ? ptick + 3 : nullptr;
                ProfScope _ps("reverse_block_kernel", st);
                rbk<<<2 * sm_count(), BP_THREADS, bp_smem_bytes(BP_CAP_MAX), st>>>(B, BP_CAP_MAX, midl2, nmid2,
                                                                                   nullptr, nullptr);
            }
        } else if (tcr) {
            PK_CHECK(cudaMemsetAsync(nmid, 0, sizeof(int), st));
            {
                aux.ticket = ptick ? ptick + 1 : nullptr;
                ProfScope _ps("prune_tc_reverse_kernel", st);
                trk<<<std::min(2 * sm_count(), ubb), PT_THREADS, PT_SMEM, st>>>(B, aux, nullptr, nullptr, midl, nmid);
            }
            PK_CHECK_LAUNCH("prune_tc_reverse_kernel");
            {
                aux.ticket = ptick ? ptick + 2 : nullptr;
                ProfScope _ps("prune_tc_reverse_kernel", st);
                trk2<<<sm_count(), PT_THREADS, pt_smem_bytes(PT_CAP_BIG), st>>>(B, aux, midl, nmid, nullptr, nullptr);
            }
        } else {
            ProfScope _ps("reverse_kernel", st);
            rk<<<std::min(grid_r, (ubb + wpb_r - 1) / wpb_r), 32 * wpb_r, wbr * wpb_r, st>>>(B);
        }
        PK_CHECK_LAUNCH("reverse_kernel");
        {
            B.ticket = ptick ? ptick + 4 : nullptr;
            ProfScope _ps("reverse_big_kernel", st);
            bigk<<<grid_big, kBigThreads, big_bytes, st>>>(B);
        }
        PK_CHECK_LAUNCH("reverse_big_kernel");
        if (sharded) {
            PK_CHECK(cudaMemsetAsync(npack, 0, sizeof(int), st));
            {
                ProfScope _ps("pack_rows_kernel", st);
                pack_rows_kernel<<<grid_for((long long)ubb * 32, 256), 256, 0, st>>>(targets, ntargets, SH.rank, SH.world,
                                                                                    adj, deg, R, SH.xsend, npack);
            }
            PK_CHECK_LAUNCH("pack_rows_kernel");
            int own = 0;
            PK_CHECK(cudaMemcpyAsync(&own, npack, sizeof(int), cudaMemcpyDeviceToHost, st));
            PK_CHECK(cudaStreamSynchronize(st));
            const long long maxc = SH.fn(SH.ctx, PK_XCHG_ROWS, own, 0);
            if (maxc < 0) {
                set_error("row exchange failed");
                return 4;
            }
            if (maxc > 0) {
                ProfScope _ps("unpack_rows_kernel", st);
                unpack_rows_kernel<<<grid_for((long long)SH.world * maxc * 32, 256), 256, 0, st>>>(
                    SH.xrecv, SH.xcnt, (int)maxc, SH.world, SH.rank, R, adj, deg);
            }
            PK_CHECK_LAUNCH("unpack_rows_kernel");
        }
    }
    unsigned herr = 0;
    PK_CHECK(cudaMemcpyAsync(&herr, err, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    if (!multi) {
        release(new_ids, st);
        release(new_len, st);
    }
    for (void* p : {(void*)vlog_i, (void*)vlog_d, (void*)vlen, (void*)cnt, (void*)tslot, (void*)targets, (void*)sizes,
                    (void*)offs, (void*)fill, (void*)adds, (void*)adist, (void*)aalive, (void*)ntargets, (void*)err,
                    (void*)biglist, (void*)nbig, (void*)npack, (void*)over, (void*)over1, (void*)nover, (void*)midl,
                    (void*)nmid, (void*)midl2, (void*)nmid2, (void*)ubm, (void*)nrm64, (void*)xh, (void*)ptick, (void*)adjd, (void*)new_d,
                    (void*)addd, (void*)seed_mask, (void*)seed_tab, (void*)near, (void*)lorder, (void*)gh, (void*)ticket, cub_tmp})
        release(p, st);
    PK_CHECK(cudaStreamSynchronize(st));
    if (herr) {
        set_error(std::string("build capacity exceeded (flags ") + std::to_string(herr) + ")");
        return 3;
    }
    return 0;
}

template <int MODE>
int dispatch_build(const DataRef& D, int n, int R, int L, double alpha, const int* starts, int s, const int* order,
                   int* adj, int* deg, long long* stats, int hash_bits, const Shard& SH, cudaStream_t st) {
    // QV: 128-float (SEQ64 / EXACT32) or 128-byte (u8) chunks per row; SEQ64 rows
    // wider than 1024 floats run without the fp32 screen (QV = 0)
    const int qv = MODE == MODE_EXACT_U8 ? (D.dw + 31) / 32 : (D.dp + 127) / 128;
    if (MODE == MODE_SEQ64 && qv > 8)  // prune_candidates checks dp <= 128 * QV before screening
        return run_build<MODE, 1>(D, n, R, L, alpha, starts, s, order, adj, deg, stats, hash_bits, SH, st);
    if (qv <= 1) return run_build<MODE, 1>(D, n, R, L, alpha, starts, s, order, adj, deg, stats, hash_bits, SH, st);
    if (qv <= 2) return run_build<MODE, 2>(D, n, R, L, alpha, starts, s, order, adj, deg, stats, hash_bits, SH, st);
    if (qv <= 4) return run_build<MODE, 4>(D, n, R, L, alpha, starts, s, order, adj, deg, stats, hash_bits, SH, st);
    if (qv <= 8) return run_build<MODE, 8>(D, n, R, L, alpha, starts, s, order, adj, deg, stats, hash_bits, SH, st);
    set_error("exact integer modes support d <= 1024");
    return 2;
}

}  // namespace pk

using namespace pk;

static int build_entry(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode, int64_t R,
                       int64_t L, double alpha, const int32_t* starts, int64_t s, const int32_t* order,
                       int32_t* adj_out, int32_t* deg_out, int64_t* stats, int hash_bits, const Shard& SH,
                       void* stream) {
    cudaStream_t st = as_stream(stream);
    long long* ls = reinterpret_cast<long long*>(stats);
    DataRef D{x, (int)dp, x8, (int)dw};
    D.screen = env_int("PK_SCREEN", 1) == 1;  // fp32 screen of float-data kill tests (tests compare both)
    if (mode == MODE_EXACT_U8 && !x8) {
        set_error("u8 mode needs the packed rows");
        return 2;
    }
    if (mode == MODE_EXACT_U8)
        return dispatch_build<MODE_EXACT_U8>(D, (int)n, (int)R, (int)L, alpha, starts, (int)s, order, adj_out, deg_out,
                                             ls, hash_bits, SH, st);
    if (mode == MODE_EXACT32)
        return dispatch_build<MODE_EXACT32>(D, (int)n, (int)R, (int)L, alpha, starts, (int)s, order, adj_out, deg_out,
                                            ls, hash_bits, SH, st);
    return dispatch_build<MODE_SEQ64>(D, (int)n, (int)R, (int)L, alpha, starts, (int)s, order, adj_out, deg_out, ls,
                                      hash_bits, SH, st);
}

extern "C" int pk_build_vamana(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                               int64_t R, int64_t L, double alpha, const int32_t* starts, int64_t s,
                               const int32_t* order, int32_t* adj_out, int32_t* deg_out, int64_t* stats,
                               int hash_bits, void* stream) {
    return build_entry(x, n, dp, x8, dw, mode, R, L, alpha, starts, s, order, adj_out, deg_out, stats, hash_bits,
                       Shard{}, stream);
}

extern "C" int pk_build_vamana_seeds(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                                     int64_t R, int64_t L, double alpha, const int32_t* starts, int64_t s,
                                     const int32_t* order, int32_t* adj_out, int32_t* deg_out, int64_t* stats,
                                     int hash_bits, double* seed_bd, uint32_t* seed_bi, int32_t* seed_bl,
                                     void* stream) {
    Shard sh;
    sh.seed_bd = seed_bd;
    sh.seed_bi = reinterpret_cast<unsigned*>(seed_bi);
    sh.seed_bl = reinterpret_cast<int*>(seed_bl);
    return build_entry(x, n, dp, x8, dw, mode, R, L, alpha, starts, s, order, adj_out, deg_out, stats, hash_bits, sh,
                       stream);
}

extern "C" int pk_build_vamana_sharded(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw,
                                       int mode, int64_t R, int64_t L, double alpha, const int32_t* starts, int64_t s,
                                       const int32_t* order, int32_t* adj_out, int32_t* deg_out, int64_t* stats,
                                       int hash_bits, int rank, int world, int64_t min_shard,
                                       pk_exchange_fn exchange, void* ctx, int32_t* xids, int32_t* xlen,
                                       int32_t* xsend, int32_t* xrecv, int32_t* xcnt, void* stream) {
    if (world < 1 || rank < 0 || rank >= world) {
        set_error("invalid rank / world");
        return 2;
    }
    Shard SH;
    SH.rank = rank;
    SH.world = world;
    SH.min_shard = min_shard < 1 ? 1 : min_shard;
    SH.fn = exchange;
    SH.ctx = ctx;
    SH.xids = xids;
    SH.xlen = xlen;
    SH.xsend = xsend;
    SH.xrecv = xrecv;
    SH.xcnt = xcnt;
    if (world > 1 && (!exchange || !xids || !xlen || !xsend || !xrecv || !xcnt)) {
        set_error("sharded build needs the exchange callback and buffers");
        return 2;
    }
    return build_entry(x, n, dp, x8, dw, mode, R, L, alpha, starts, s, order, adj_out, deg_out, stats, hash_bits, SH,
                       stream);
}

extern "C" int pk_robust_prune(const float* x, int64_t n, int64_t dp, int64_t p, const int64_t* cand_ids,
                               const double* cand_sqd, int64_t m, const int64_t* cur_ids, int64_t dcount,
                               double alpha, int64_t R, int64_t* out, int64_t* out_count, void* stream) {
    (void)n;
    cudaStream_t st = as_stream(stream);
    int c0 = (int)(m + dcount);
    int cap = next_pow2(c0 > 32 ? c0 : 32);
    size_t bytes = align16(sort_smem_bytes(cap) + (size_t)cap * 4);
    if (bytes > (size_t)max_smem_optin()) {
        set_error("too many prune candidates for one call");
        return 2;
    }
    int* so = nullptr;
    PK_CHECK(scratch(&so, (size_t)(R > 0 ? R : 1), st));
    PK_CHECK(cudaFuncSetAttribute(robust_prune_api_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    {
        ProfScope _ps("robust_prune_api_kernel", st);
        robust_prune_api_kernel<<<1, 32, bytes, st>>>(x, (int)dp, (unsigned)p, reinterpret_cast<const long long*>(cand_ids),
                                                      cand_sqd, (int)m, reinterpret_cast<const long long*>(cur_ids),
                                                      (int)dcount, alpha * alpha, (int)R, cap,
                                                      reinterpret_cast<long long*>(out),
                                                      reinterpret_cast<long long*>(out_count), so);
    }
    PK_CHECK_LAUNCH("robust_prune_api_kernel");
    release(so, st);
    return 0;
}

extern "C" int pk_nearest_to_centroid(const float* x, int64_t n, int64_t dp, int64_t* out, void* stream) {
    cudaStream_t st = as_stream(stream);
    double* cen = nullptr;
    double* bd = nullptr;
    int* bi = nullptr;
    const int g = 64;
    PK_CHECK(scratch(&cen, (size_t)dp, st));
    PK_CHECK(scratch(&bd, g, st));
    PK_CHECK(scratch(&bi, g, st));
    {
        ProfScope _ps("centroid_kernel", st);
        centroid_kernel<<<(unsigned)((dp + 127) / 128), 128, 0, st>>>(x, (int)n, (int)dp, cen);
    }
    {
        ProfScope _ps("nearest_kernel", st);
        nearest_kernel<<<g, 256, 0, st>>>(x, (int)n, (int)dp, cen, bd, bi);
    }
    {
        ProfScope _ps("nearest_final_kernel", st);
        nearest_final_kernel<<<1, 1, 0, st>>>(bd, bi, g, reinterpret_cast<long long*>(out));
    }
    PK_CHECK_LAUNCH("nearest_to_centroid");
    release(cen, st);
    release(bd, st);
    release(bi, st);
    return 0;
}

// Diagnostics: the build searches' phase timers (see pk_phase_timers).
extern "C" int pk_phase_timers_build(unsigned long long* out8, int reset) {
#ifdef PK_PHASE_TIMERS
    PK_CHECK(cudaDeviceSynchronize());
    PK_CHECK(cudaMemcpyFromSymbol(out8, pk_phase_cycles, sizeof(unsigned long long) * 8));
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        PK_CHECK(cudaMemcpyToSymbol(pk_phase_cycles, z, sizeof z));
    }
#else
    (void)reset;
    for (int i = 0; i < 8; ++i) out8[i] = 0;
#endif
    return 0;
}

// Diagnostics: the tensor-core build prune's phase timers (prune_tc.cuh).
extern "C" int pk_phase_timers_prune(unsigned long long* out8, int reset) {
#ifdef PK_PHASE_TIMERS
    PK_CHECK(cudaDeviceSynchronize());
    PK_CHECK(cudaMemcpyFromSymbol(out8, pk_prune_cycles, sizeof(unsigned long long) * 8));
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        PK_CHECK(cudaMemcpyToSymbol(pk_prune_cycles, z, sizeof z));
    }
#else
    (void)reset;
    for (int i = 0; i < 8; ++i) out8[i] = 0;
#endif
    return 0;
}
