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

#include <cub/cub.cuh>

#include "../../include/peakann_b200.h"
#include "api.cuh"
#include "beam.cuh"

namespace pk {

int grid_for(long long work, int block);

template <int MODE, int QV>
struct BDist;
template <int QV>
struct BDist<PK_MODE_SEQ64, QV> {
    using T = Seq64Member;
    __device__ static T make(const float* X, int dp, unsigned id) { return T{X + (size_t)id * dp, dp}; }
};
template <int QV>
struct BDist<PK_MODE_EXACT32, QV> {
    using T = Exact32<QV>;
    __device__ static T make(const float* X, int dp, unsigned id) {
        T t;
        t.load(X + (size_t)id * dp, dp);
        return t;
    }
};

template <int MODE, int QV>
struct MakeAt {
    const float* X;
    int dp;
    __device__ typename BDist<MODE, QV>::T operator()(unsigned id) const { return BDist<MODE, QV>::make(X, dp, id); }
};

struct BuildArgs {
    SearchParams P;
    const int* bids;
    int m;
    int L;
    int H;
    int cap;           // candidate capacity (power of two)
    int vcap;          // visit-log capacity
    double alpha2;
    size_t warp_bytes;
    unsigned* vlog_i;  // [total_warps * vcap]
    double* vlog_d;
    int* new_ids;      // [m * R]
    int* new_len;      // [m]
    unsigned* err;
    long long* stats;  // [4]
};

template <int MODE, int QV>
__global__ void __launch_bounds__(128) build_batch_kernel(BuildArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int lane = lane_id();
    const int gw = blockIdx.x * wpb + wib;
    unsigned char* mine = smem + (size_t)wib * A.warp_bytes;
    // search view
    BeamSmem sm;
    sm.bd = reinterpret_cast<double*>(mine);
    sm.bi = reinterpret_cast<unsigned*>(mine + (size_t)A.L * 8);
    sm.hash = reinterpret_cast<unsigned*>(mine + (size_t)A.L * 12);
    sm.hmask = (unsigned)A.H - 1u;
    sm.spos = reinterpret_cast<int*>(mine + (size_t)A.L * 12 + (size_t)A.H * 4);
    sm.cbuf = reinterpret_cast<unsigned*>(mine + (size_t)A.L * 12 + (size_t)A.H * 4 + 128);
    // prune view (aliases the search view once the walk is over)
    double* kd = reinterpret_cast<double*>(mine);
    unsigned* ki = reinterpret_cast<unsigned*>(mine + (size_t)A.cap * 8);
    unsigned* pcbuf = reinterpret_cast<unsigned*>(mine + (size_t)A.cap * 12);
    unsigned char* alive = mine + (size_t)A.cap * 12 + 128;

    unsigned* vi = A.vlog_i + (size_t)gw * A.vcap;
    double* vd = A.vlog_d + (size_t)gw * A.vcap;
    const MakeAt<MODE, QV> make{A.P.X, A.P.dp};
    long long ev_search = 0, ev_prune = 0, expansions = 0;
    const int R = A.P.R;
    for (int t = gw; t < A.m; t += gridDim.x * wpb) {
        const unsigned p = (unsigned)A.bids[t];
        auto dist = make(p);
        WarpBeam<decltype(dist)> wb;
        wb.init(sm, A.L, vi, vd, A.vcap, A.err);
        wb.seed(A.P, dist);
        wb.walk(A.P, dist);
        ev_search += wb.evals;
        expansions += wb.vl;
        const int vl = min(wb.vl, A.vcap);
        __syncwarp();
        // candidates: visit log + current out-row (distances recomputed, _kernels.py:359-368)
        for (int x = lane; x < vl; x += 32) {
            kd[x] = vd[x];
            ki[x] = vi[x];
        }
        const int nd = __ldg(A.P.deg + p);
        const int* row = A.P.adj + (size_t)p * R;
        int c = vl;
        for (int e0 = 0; e0 < nd; e0 += 32) {
            const int cnt = min(32, nd - e0);
            unsigned w = lane < cnt ? (unsigned)__ldg(row + e0 + lane) : 0u;
            double dd = dist.eval(A.P.X, (int)w, cnt);
            if (lane == 0) ev_search += cnt;
            if (lane < cnt && c + lane < A.cap) {
                kd[c + lane] = dd;
                ki[c + lane] = w;
            }
            c += cnt;
        }
        if (c > A.cap) {
            if (lane == 0) atomicOr(A.err, ERR_CAND_OVERFLOW);
            c = A.cap;
        }
        const int Pw = next_pow2_dev(c);
        for (int x = c + lane; x < Pw; x += 32) {
            kd[x] = __longlong_as_double(0x7ff0000000000000LL);
            ki[x] = 0xffffffffu;
        }
        __syncwarp();
        warp_sort(kd, ki, Pw);
        c = warp_unique(kd, ki, c, p);
        int* out = A.new_ids + (size_t)t * R;
        int sel = warp_prune(A.P.X, kd, ki, c, A.alpha2, R, alive, pcbuf, out, make, &ev_prune);
        for (int x = sel + lane; x < R; x += 32) out[x] = -1;
        if (lane == 0) A.new_len[t] = sel;
        __syncwarp();
    }
    if (lane == 0 && A.stats) {
        atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 0), (unsigned long long)ev_search);
        atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 1), (unsigned long long)ev_prune);
        atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 3), (unsigned long long)expansions);
    }
}

// write staged rows, count reverse edges, register targets (warp per point)
__global__ void commit_kernel(const int* bids, int m, int R, const int* new_ids, const int* new_len, int* adj,
                              int* deg, int* cnt, int* tslot, int* targets, int* ntargets) {
    const int lane = lane_id();
    const int wpb = blockDim.x >> 5;
    for (int t = blockIdx.x * wpb + (threadIdx.x >> 5); t < m; t += gridDim.x * wpb) {
        const int p = bids[t];
        const int len = new_len[t];
        for (int x = lane; x < R; x += 32) {
            int u = new_ids[(size_t)t * R + x];
            adj[(size_t)p * R + x] = u;
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
                               const int* tslot, const int* offs, int* fill, int* adds) {
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < (long long)m * R;
         x += (long long)gridDim.x * blockDim.x) {
        int t = (int)(x / R), e = (int)(x % R);
        if (e >= new_len[t]) continue;
        int u = new_ids[x];
        int s = tslot[u];
        int pos = offs[s] + atomicAdd(fill + s, 1);
        adds[pos] = bids[t];
    }
}

struct RevArgs {
    const float* X;
    int dp;
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
};

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
    unsigned char* mine = smem + (size_t)wib * A.warp_bytes;
    double* kd = reinterpret_cast<double*>(mine);
    unsigned* ki = reinterpret_cast<unsigned*>(mine + (size_t)A.cap * 8);
    unsigned* pcbuf = reinterpret_cast<unsigned*>(mine + (size_t)A.cap * 12);
    unsigned char* alive = mine + (size_t)A.cap * 12 + 128;
    const MakeAt<MODE, QV> make{A.X, A.dp};
    const int nt = *A.ntargets;
    long long ev = 0;
    for (int s = blockIdx.x * wpb + wib; s < nt; s += gridDim.x * wpb) {
        const unsigned u = (unsigned)A.targets[s];
        const int nd = A.deg[u];
        const int off = A.offs[s];
        const int size = A.sizes[s];
        int* row = A.adj + (size_t)u * A.R;
        const int c0 = nd + size;
        int sel;
        if (c0 <= A.cap) {
            auto du = make(u);
            for (int e0 = 0; e0 < c0; e0 += 32) {
                const int cnt = min(32, c0 - e0);
                const int x = e0 + lane;
                unsigned w = 0u;
                if (lane < cnt) w = x < nd ? (unsigned)row[x] : (unsigned)A.adds[off + x - nd];
                double dd = du.eval(A.X, (int)w, cnt);
                if (lane < cnt) {
                    kd[x] = dd;
                    ki[x] = w;
                }
            }
            ev += c0;
            const int Pw = next_pow2_dev(c0);
            for (int x = c0 + lane; x < Pw; x += 32) {
                kd[x] = __longlong_as_double(0x7ff0000000000000LL);
                ki[x] = 0xffffffffu;
            }
            __syncwarp();
            warp_sort(kd, ki, Pw);
            const int c = warp_unique(kd, ki, c0, u);
            if (c <= A.R) {
                for (int x = lane; x < c; x += 32) row[x] = (int)ki[x];
                sel = c;
            } else {
                sel = warp_prune(A.X, kd, ki, c, A.alpha2, A.R, alive, pcbuf, row, make, &ev);
            }
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

__global__ void starts_bitmap_kernel2(const int* starts, int s, unsigned* bm) {
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < s; x += gridDim.x * blockDim.x)
        atomicOr(bm + (starts[x] >> 5), 1u << (starts[x] & 31));
}

// ---- host driver -----------------------------------------------------------------------------
template <int MODE, int QV>
int run_build(const float* x, int n, int dp, int R, int L, double alpha, const int* starts, int s, const int* order,
              int* adj, int* deg, long long* stats, int hash_bits, cudaStream_t st) {
    const int H = choose_hash(L, hash_bits);
    const int cap = next_pow2(2 * L + 64 + R);
    const int vcap = cap - R;
    const int capR = 1024;
    size_t wb = align16(std::max(beam_smem_bytes(L, H), sort_smem_bytes(cap)));
    int wpb = 4;
    while (wpb > 1 && wb * wpb > (size_t)max_smem_optin()) wpb >>= 1;
    if (wb * wpb > (size_t)max_smem_optin()) {
        set_error("build beam too large for shared memory");
        return 2;
    }
    auto bk = build_batch_kernel<MODE, QV>;
    PK_CHECK(cudaFuncSetAttribute(bk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(wb * wpb)));
    int per_sm = 0;
    PK_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bk, 32 * wpb, wb * wpb));
    if (per_sm < 1) per_sm = 1;
    const int max_grid = sm_count() * per_sm;
    const int total_warps = max_grid * wpb;

    size_t wbr = align16(sort_smem_bytes(capR));
    int wpbr = 4;
    while (wpbr > 1 && wbr * wpbr > (size_t)max_smem_optin()) wpbr >>= 1;
    auto rk = reverse_kernel<MODE, QV>;
    PK_CHECK(cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(wbr * wpbr)));
    int per_sm_r = 0;
    PK_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_r, rk, 32 * wpbr, wbr * wpbr));
    if (per_sm_r < 1) per_sm_r = 1;
    const int grid_r = sm_count() * per_sm_r;

    int maxb = 1;
    while (maxb < n) maxb <<= 1;
    const int mb = std::min(maxb, n);           // largest batch
    const long long E = (long long)mb * R;      // max edges per batch
    const int ub = (int)std::min<long long>(n, E);

    unsigned *vlog_i = nullptr, *bm = nullptr, *err = nullptr;
    double *vlog_d = nullptr, *adist = nullptr;
    int *new_ids = nullptr, *new_len = nullptr, *cnt = nullptr, *tslot = nullptr, *targets = nullptr;
    int *sizes = nullptr, *offs = nullptr, *fill = nullptr, *adds = nullptr, *ntargets = nullptr;
    unsigned char* aalive = nullptr;
    PK_CHECK(scratch(&vlog_i, (size_t)total_warps * vcap, st));
    PK_CHECK(scratch(&vlog_d, (size_t)total_warps * vcap, st));
    PK_CHECK(scratch(&new_ids, (size_t)E, st));
    PK_CHECK(scratch(&new_len, (size_t)mb, st));
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
    PK_CHECK(scratch(&err, 1, st));
    size_t words = (size_t)(n + 31) / 32;
    PK_CHECK(scratch(&bm, words, st));
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, sizes, offs, ub + 1, st);
    PK_CHECK(cudaMallocAsync(&cub_tmp, cub_bytes + 16, st));

    PK_CHECK(cudaMemsetAsync(adj, 0xff, sizeof(int) * (size_t)n * R, st));
    PK_CHECK(cudaMemsetAsync(deg, 0, sizeof(int) * (size_t)n, st));
    PK_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int) * (size_t)n, st));
    PK_CHECK(cudaMemsetAsync(err, 0, sizeof(unsigned), st));
    PK_CHECK(cudaMemsetAsync(bm, 0, words * 4, st));
    {
        ProfScope _ps("starts_bitmap_kernel2", st);
        starts_bitmap_kernel2<<<grid_for(s, 256), 256, 0, st>>>(starts, s, bm);
    }

    BuildArgs A;
    A.P = SearchParams{x, dp, adj, R, deg, starts, s, bm};
    A.L = L;
    A.H = H;
    A.cap = cap;
    A.vcap = vcap;
    A.alpha2 = alpha * alpha;
    A.warp_bytes = wb;
    A.vlog_i = vlog_i;
    A.vlog_d = vlog_d;
    A.new_ids = new_ids;
    A.new_len = new_len;
    A.err = err;
    A.stats = stats;

    RevArgs B;
    B.X = x;
    B.dp = dp;
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

    for (int lo = 0, batch = 1; lo < n; lo += batch, batch *= 2) {
        const int m = std::min(batch, n - lo);
        A.bids = order + lo;
        A.m = m;
        const int g = std::min(max_grid, (m + wpb - 1) / wpb);
        {
            ProfScope _ps("build_batch_kernel", st);
            bk<<<g, 32 * wpb, wb * wpb, st>>>(A);
        }
        PK_CHECK_LAUNCH("build_batch_kernel");
        const int ubb = (int)std::min<long long>(n, (long long)m * R);
        PK_CHECK(cudaMemsetAsync(ntargets, 0, sizeof(int), st));
        PK_CHECK(cudaMemsetAsync(sizes, 0, sizeof(int) * ((size_t)ubb + 1), st));
        PK_CHECK(cudaMemsetAsync(fill, 0, sizeof(int) * (size_t)ubb, st));
        {
            ProfScope _ps("commit_kernel", st);
            commit_kernel<<<grid_for((long long)m * 32, 256), 256, 0, st>>>(order + lo, m, R, new_ids, new_len, adj, deg,
                                                                             cnt, tslot, targets, ntargets);
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
                                                                             offs, fill, adds);
        }
        PK_CHECK_LAUNCH("scatter_kernel");
        const int gr = std::min(grid_r, (ubb + wpbr - 1) / wpbr);
        {
            ProfScope _ps("reverse_kernel", st);
            rk<<<gr, 32 * wpbr, wbr * wpbr, st>>>(B);
        }
        PK_CHECK_LAUNCH("reverse_kernel");
    }
    unsigned herr = 0;
    PK_CHECK(cudaMemcpyAsync(&herr, err, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    for (void* p : {(void*)vlog_i, (void*)vlog_d, (void*)new_ids, (void*)new_len, (void*)cnt, (void*)tslot,
                    (void*)targets, (void*)sizes, (void*)offs, (void*)fill, (void*)adds, (void*)adist,
                    (void*)aalive, (void*)ntargets, (void*)err, (void*)bm, cub_tmp})
        release(p, st);
    PK_CHECK(cudaStreamSynchronize(st));
    if (herr) {
        set_error(std::string("build capacity exceeded (flags ") + std::to_string(herr) + ")");
        return 3;
    }
    return 0;
}

}  // namespace pk

using namespace pk;

extern "C" int pk_build_vamana(const float* x, int64_t n, int64_t dp, int mode, int64_t R, int64_t L, double alpha,
                               const int32_t* starts, int64_t s, const int32_t* order, int32_t* adj_out,
                               int32_t* deg_out, int64_t* stats, int hash_bits, void* stream) {
    cudaStream_t st = as_stream(stream);
    long long* ls = reinterpret_cast<long long*>(stats);
    if (mode == PK_MODE_SEQ64)
        return run_build<PK_MODE_SEQ64, 1>(x, (int)n, (int)dp, (int)R, (int)L, alpha, starts, (int)s, order, adj_out,
                                           deg_out, ls, hash_bits, st);
    int qv = (int)((dp + 127) / 128);
    if (qv <= 1)
        return run_build<PK_MODE_EXACT32, 1>(x, (int)n, (int)dp, (int)R, (int)L, alpha, starts, (int)s, order,
                                             adj_out, deg_out, ls, hash_bits, st);
    if (qv <= 2)
        return run_build<PK_MODE_EXACT32, 2>(x, (int)n, (int)dp, (int)R, (int)L, alpha, starts, (int)s, order,
                                             adj_out, deg_out, ls, hash_bits, st);
    if (qv <= 4)
        return run_build<PK_MODE_EXACT32, 4>(x, (int)n, (int)dp, (int)R, (int)L, alpha, starts, (int)s, order,
                                             adj_out, deg_out, ls, hash_bits, st);
    if (qv <= 8)
        return run_build<PK_MODE_EXACT32, 8>(x, (int)n, (int)dp, (int)R, (int)L, alpha, starts, (int)s, order,
                                             adj_out, deg_out, ls, hash_bits, st);
    set_error("EXACT32 mode supports d <= 1024");
    return 2;
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
