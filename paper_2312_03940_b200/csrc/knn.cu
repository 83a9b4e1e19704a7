// Beam-search kNN, single searches, exact kNN and the dependent-point scan.
#include <algorithm>

#include <cub/cub.cuh>

#include "../../include/peakann_b200.h"
#include "api.cuh"
#include "beam.cuh"

namespace pk {

// ---- beam kNN of member queries (_kernels.py:230-262) --------------------------------
// RING (float data, QV >= 4): candidate rows staged through the per-warp row
// ring (bulk copies into shared memory) instead of registers
template <int MODE, int QV, bool RING>
// (float data: 5 blocks of 96 registers at QV = 8 and 6 blocks of 80 at QV = 4 measured best
// for the member queries -- C5 1.22 -> 1.20 s, C4 0.85 -> 0.73 s; the build searches keep 4 / 5)
__global__ void __launch_bounds__(128, MODE == MODE_SEQ64 ? (QV >= 8 ? 5 : QV >= 4 ? 6 : 8) : 8) beam_knn_kernel(SearchParams P, const long long* __restrict__ qids, int m,
                                                       int L, int kk, int H, size_t warp_bytes,
                                                       long long* __restrict__ out_ids, double* __restrict__ out_d,
                                                       long long* __restrict__ counts, long long* evals_out,
                                                       unsigned char* gbeam, size_t gstride,
                                                       const int* __restrict__ ord) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int lane = lane_id();
    unsigned char* mine = smem + (size_t)wib * warp_bytes;
    BeamSmem sm = gbeam ? carve_beam_spill(mine, gbeam + ((size_t)blockIdx.x * wpb + wib) * gstride, L, H)
                  : P.ghash ? carve_beam_gh(mine, P.ghash + ((size_t)blockIdx.x * wpb + wib) * P.ghash_stride, L, H)
                            : carve_beam(mine, L, H);
    if constexpr (RING) carve_ring(sm, mine + warp_bytes - ring_smem_bytes_dev(P.dp, P.ring), P.dp, P.ring);
    unsigned ring_t = 0;
    long long ev = 0, ex = 0, un = 0;
    const bool uniq = starts_increasing(P);
    for (int t0 = next_position(P.ticket, blockIdx.x * wpb + wib - gridDim.x * wpb, gridDim.x * wpb); t0 < m;
         t0 = next_position(P.ticket, t0, gridDim.x * wpb)) {
        const int t = ord ? __ldg(ord + t0) : t0;  // processing order (locality) != output row order
        const unsigned qi = (unsigned)qids[t];
        auto dist = DistFor<MODE, QV, RING>::make(P.data(), qi);
        WarpBeam<decltype(dist)> wb;
        wb.init(sm, L, nullptr, nullptr, 0, nullptr);
        wb.rt = ring_t;
        wb.begin_counting(P.ubm ? P.ubm + ((size_t)blockIdx.x * wpb + wib) * P.uwords : nullptr, P.uwords);
        {
            PK_PT_BEGIN
            if (P.seed_load) wb.load_seed(P, dist, qi);
            else wb.seed(P, dist, false, uniq);
            PK_PT_END(6);
        }
        if (!P.seed_only) wb.walk(P, dist);
        un += wb.uniq;
        long long* oi = out_ids + (size_t)t * kk;
        double* od = out_d + (size_t)t * kk;
        int got;
        PK_PT_BEGIN
        if constexpr (has_screen<decltype(dist)>::value)
            got = wb.emit(qi, kk, oi, od, [&](unsigned id) { return dist.eval_one(P.X, (int)id); });
        else
            got = wb.emit(qi, kk, oi, od);
        for (int x = got + lane; x < kk; x += 32) {
            oi[x] = -1;
            od[x] = __longlong_as_double(0x7ff0000000000000LL);
        }
        if (lane == 0) counts[t] = got;
        PK_PT_END(5);
        ev += wb.evals;
        ex += wb.vl;
        ring_t = wb.rt;
        __syncwarp();
    }
    if (evals_out && lane == 0 && ev) {
        atomicAdd(reinterpret_cast<unsigned long long*>(evals_out), (unsigned long long)ev);
        atomicAdd(reinterpret_cast<unsigned long long*>(evals_out + 1), (unsigned long long)ex);
        if (P.ubm) atomicAdd(reinterpret_cast<unsigned long long*>(evals_out + 2), (unsigned long long)un);
    }
}

// rows with counts < kk -> list for the exact fallback
__global__ void short_rows_kernel(const long long* counts, int m, int kk, int* list, int* nlist) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x)
        if (counts[t] < kk) list[atomicAdd(nlist, 1)] = t;
}

// ---- single search (beam_search_single, _kernels.py:215-227) ---------------------------
template <class Dist>
__global__ void single_search_kernel(SearchParams P, Dist dist, unsigned self, int L, int k, int H,
                                     long long* top_ids, double* top_d, long long* top_count,
                                     long long* vis_ids, double* vis_d, int vcap, long long* vis_count,
                                     unsigned* vtmp_i, double* vtmp_d, unsigned char* gbeam) {
    extern __shared__ __align__(16) unsigned char smem[];
    BeamSmem sm = gbeam ? carve_beam_spill(smem, gbeam, L, H) : carve_beam(smem, L, H);
    __shared__ unsigned s_err;
    if (threadIdx.x == 0) s_err = 0;
    __syncwarp();
    WarpBeam<Dist> wb;
    wb.init(sm, L, vtmp_i, vtmp_d, vcap, &s_err);
    wb.seed(P, dist, true, false);
    wb.walk(P, dist);
    int got = wb.emit(self, k, top_ids, top_d);
    const int lane = lane_id();
    for (int x = lane; x < min(wb.vl, vcap); x += 32) {
        vis_ids[x] = vtmp_i[x];
        vis_d[x] = vtmp_d[x];
    }
    if (lane == 0) {
        *top_count = got;
        *vis_count = wb.vl;
    }
}

// ---- exact kNN: one block per row --------------------------------------------------------
constexpr int BT = 256;

struct RowQuery {
    const float* qf;   // member row (float), or null
    const double* qd;  // free vector (double), or null
    int self;          // excluded id or -1
};

__device__ __forceinline__ double row_dist(const float* __restrict__ X, int dp, const RowQuery& q, int j) {
    const float* r = X + (size_t)j * dp;
    double acc = 0.0;
    if (q.qf) {
        for (int t = 0; t < dp; t += 4) {
            float4 x = ldg4(r + t), y = ldg4(q.qf + t);
            double a = (double)y.x - (double)x.x; acc = __dadd_rn(acc, __dmul_rn(a, a));
            double b = (double)y.y - (double)x.y; acc = __dadd_rn(acc, __dmul_rn(b, b));
            double c = (double)y.z - (double)x.z; acc = __dadd_rn(acc, __dmul_rn(c, c));
            double e = (double)y.w - (double)x.w; acc = __dadd_rn(acc, __dmul_rn(e, e));
        }
    } else {
        for (int t = 0; t < dp; t += 4) {
            float4 x = ldg4(r + t);
            double a = __ldg(q.qd + t) - (double)x.x; acc = __dadd_rn(acc, __dmul_rn(a, a));
            double b = __ldg(q.qd + t + 1) - (double)x.y; acc = __dadd_rn(acc, __dmul_rn(b, b));
            double c = __ldg(q.qd + t + 2) - (double)x.z; acc = __dadd_rn(acc, __dmul_rn(c, c));
            double e = __ldg(q.qd + t + 3) - (double)x.w; acc = __dadd_rn(acc, __dmul_rn(e, e));
        }
    }
    return acc;
}

// Block-wide exact top-kk of one distance row (the selection of
// _kernels.py:55-83): radix-select the kk-th key, gather keys below it plus
// the smallest ids among equal keys, bitonic-sort the survivors by (dist, id).
__device__ void block_select_row(const double* row, int n, int kk, double* sd, unsigned* si, int P,
                                 long long* out_ids, double* out_d) {
    __shared__ unsigned hist[256];
    __shared__ unsigned long long s_prefix;
    __shared__ int s_want;
    using Scan = cub::BlockScan<int, BT>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int s_base, s_eqseen;
    const int tid = threadIdx.x;
    unsigned long long prefix = 0, mask = 0;
    int want = kk - 1;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int b = tid; b < 256; b += BT) hist[b] = 0;
        __syncthreads();
        for (int j = tid; j < n; j += BT) {
            unsigned long long key = dbits(row[j]);
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid == 0) {
            int acc = 0, b = 0;
            for (; b < 256; ++b) {
                if (acc + (int)hist[b] > want) break;
                acc += hist[b];
            }
            s_want = want - acc;
            s_prefix = prefix | ((unsigned long long)b << shift);
        }
        __syncthreads();
        want = s_want;
        prefix = s_prefix;
        mask |= 255ull << shift;
        __syncthreads();
    }
    const unsigned long long th = prefix;
    const int need_eq = want + 1;  // equal keys admitted, smallest ids first
    if (tid == 0) { s_base = 0; s_eqseen = 0; }
    __syncthreads();
    for (int base = 0; base < n; base += BT) {
        int j = base + tid;
        unsigned long long key = j < n ? dbits(row[j]) : ~0ull;
        int eq = (j < n && key == th) ? 1 : 0;
        int eq_before, eq_total;
        Scan(scan_tmp).ExclusiveSum(eq, eq_before, eq_total);
        __syncthreads();
        int keep = (j < n) && (key < th || (eq && s_eqseen + eq_before < need_eq));
        int pos, tot;
        Scan(scan_tmp).ExclusiveSum(keep, pos, tot);
        if (keep) {
            sd[s_base + pos] = row[j];
            si[s_base + pos] = (unsigned)j;
        }
        __syncthreads();
        if (tid == 0) { s_base += tot; s_eqseen += eq_total; }
        __syncthreads();
    }
    for (int i = kk + tid; i < P; i += BT) {
        sd[i] = __longlong_as_double(0x7ff0000000000000LL);
        si[i] = 0xffffffffu;
    }
    __syncthreads();
    for (int k2 = 2; k2 <= P; k2 <<= 1) {
        for (int j2 = k2 >> 1; j2 > 0; j2 >>= 1) {
            for (int i = tid; i < P; i += BT) {
                int x = i ^ j2;
                if (x > i) {
                    double a = sd[i], b = sd[x];
                    unsigned ia = si[i], ib = si[x];
                    bool asc = (i & k2) == 0;
                    if (key_lt(b, ib, a, ia) == asc) {
                        sd[i] = b; sd[x] = a;
                        si[i] = ib; si[x] = ia;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = tid; i < kk; i += BT) {
        out_ids[i] = si[i];
        out_d[i] = sd[i];
    }
    __syncthreads();
}

// rows: either rowlist (indexes into qids, count in *nrows) or all m rows
__global__ void __launch_bounds__(BT) brute_rows_kernel(const float* __restrict__ X, int n, int dp,
                                                        const long long* __restrict__ qids, const double* qvec,
                                                        const int* rowlist, const int* nrows, int m, int kk,
                                                        double* scratch, double* sbuf_d, unsigned* sbuf_i, int P,
                                                        long long* out_ids, double* out_d) {
    double* row = scratch + (size_t)blockIdx.x * n;
    double* sd = sbuf_d + (size_t)blockIdx.x * P;
    unsigned* si = sbuf_i + (size_t)blockIdx.x * P;
    const int rows = rowlist ? *nrows : m;
    for (int r = blockIdx.x; r < rows; r += gridDim.x) {
        const int t = rowlist ? rowlist[r] : r;
        RowQuery q;
        if (qvec) {
            q.qf = nullptr; q.qd = qvec; q.self = -1;
        } else {
            int i = (int)qids[t];
            q.qf = X + (size_t)i * dp; q.qd = nullptr; q.self = i;
        }
        for (int j = threadIdx.x; j < n; j += BT)
            row[j] = j == q.self ? __longlong_as_double(0x7ff0000000000000LL) : row_dist(X, dp, q, j);
        __syncthreads();
        block_select_row(row, n, kk, sd, si, P, out_ids + (size_t)t * kk, out_d + (size_t)t * kk);
    }
}

// ---- misc small kernels ----------------------------------------------------------------------
__global__ void fill_ids_kernel(long long* ids, double* d, long long count) {
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < count; x += (long long)gridDim.x * blockDim.x) {
        ids[x] = -1;
        d[x] = __longlong_as_double(0x7ff0000000000000LL);
    }
}

__device__ __forceinline__ unsigned ordered_key(float f) {
    unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float from_ordered(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// range[0] = ordered max, range[1] = ordered min over the real coordinates
__global__ void check_exact32_kernel(const float* x, long long total, int dp, int d, int* bad, unsigned* range,
                                     unsigned long long* first_nonfinite) {
    unsigned hi = 0u, lo = 0xffffffffu;
    int b = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int col = (int)(i % dp);
        if (col >= d) continue;
        float v = x[i];
        if (first_nonfinite && !isfinite(v))
            atomicMin(first_nonfinite, (unsigned long long)(i / dp) * (unsigned long long)d + (unsigned long long)col);
        if (v != rintf(v)) b = 1;
        unsigned k = ordered_key(v);
        hi = max(hi, k);
        lo = min(lo, k);
    }
    if (b) atomicOr(bad, 1);
    for (int s = 16; s; s >>= 1) {
        hi = max(hi, __shfl_xor_sync(PK_FULL, hi, s));
        lo = min(lo, __shfl_xor_sync(PK_FULL, lo, s));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(range, hi);
        atomicMin(range + 1, lo);
    }
}

// integer coordinates spanning [lo, hi]: every squared distance and every
// partial sum is an integer <= d * (hi - lo)^2; below 2^24 float32 is exact
__global__ void finish_exact32_kernel(const int* bad, const unsigned* range, int d, int* flag) {
    double span = (double)from_ordered(range[0]) - (double)from_ordered(range[1]);
    double bound = (double)d * span * span;
    // 2: bytes (x - min) hold every coordinate exactly; 1: float32 sums exact.
    // The integer kernels hold a query row in at most 8 slices of 128 floats /
    // 32 packed words, so rows wider than 1024 take the float64 policy.
    *flag = (*bad || d > 1024) ? 0 : span <= 255.0 ? 2 : bound < 16777216.0 ? 1 : 0;
}

__global__ void pack_u8_kernel(const float* x, long long n, int dp, int d, const unsigned* range, int dw,
                               unsigned* out) {
    const float lo = from_ordered(range[1]);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n * dw; i += (long long)gridDim.x * blockDim.x) {
        long long r = i / dw;
        int w = (int)(i % dw);
        unsigned v = 0;
        for (int b = 0; b < 4; ++b) {
            int t = 4 * w + b;
            unsigned byte = t < d ? (unsigned)(x[r * dp + t] - lo) : 0u;
            v |= byte << (8 * b);
        }
        out[i] = v;
    }
}

__global__ void sqrt_kernel(const double* a, long long count, double* out) {
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < count; x += (long long)gridDim.x * blockDim.x)
        out[x] = sqrt(a[x]);
}

__global__ void to_i32_kernel(const long long* a, long long count, int* out) {
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < count; x += (long long)gridDim.x * blockDim.x)
        out[x] = (int)a[x];
}

__global__ void start_bitmap_kernel(const int* starts, int s, unsigned* bm) {
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < s; x += gridDim.x * blockDim.x)
        atomicOr(bm + (starts[x] >> 5), 1u << (starts[x] & 31));
}

int grid_for(long long work, int block) {
    long long g = (work + block - 1) / block;
    long long cap = (long long)sm_count() * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// ---- launch helpers --------------------------------------------------------------------------
int choose_hash(int L, int hash_bits, long long n) {
    int h;
    if (hash_bits <= 0) hash_bits = env_int("PK_HASH_BITS", 0);  // tuning override
    if (hash_bits > 0) {
        h = 1 << hash_bits;
    } else {
        h = next_pow2(16 * L);
        if (h < 512) h = 512;
        if (h > 8192) h = 8192;
    }
    // 16-bit ways hold the quotient id >> log2(h / 4): keep it below 0xffff
    while (((n - 1) >> (__builtin_ctz((unsigned)h) - 2)) >= 0xffff) h <<= 1;
    return h;
}

// keys of the member queries for the locality order: the nearest start (first
// entry of the seeded beam the build saved for the query)
__global__ void seed_near_keys_kernel(const long long* qids, int m, const unsigned* seed_bi, int L, unsigned* keys,
                                      int* vals) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
        keys[t] = seed_bi[(size_t)qids[t] * L] & PK_IDMASK;
        vals[t] = t;
    }
}

// Processing order of a large batch of member queries, grouped by nearest
// start: the warps running at the same time search the same region of the data
// and share its rows in L2 (the results do not depend on the order).
int query_locality_order(const SearchParams& P, const long long* qids, int m, int L, long long n, int** ord,
                         cudaStream_t st) {
    int bits = 1;
    while ((1ll << bits) < n) ++bits;
    unsigned *k0 = nullptr, *k1 = nullptr;
    int* v0 = nullptr;
    PK_CHECK(scratch(&k0, (size_t)m, st));
    PK_CHECK(scratch(&k1, (size_t)m, st));
    PK_CHECK(scratch(&v0, (size_t)m, st));
    PK_CHECK(scratch(ord, (size_t)m, st));
    {
        ProfScope _ps("seed_near_keys_kernel", st);
        seed_near_keys_kernel<<<grid_for(m, 256), 256, 0, st>>>(qids, m, P.seed_bi, L, k0, v0);
    }
    PK_CHECK_LAUNCH("seed_near_keys_kernel");
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, k0, k1, v0, *ord, m, 0, bits, st);
    void* tmp = nullptr;
    PK_CHECK(cudaMallocAsync(&tmp, bytes + 16, st));
    {
        ProfScope _ps("cub_DeviceRadixSort_SortPairs", st);
        PK_CHECK(cub::DeviceRadixSort::SortPairs(tmp, bytes, k0, k1, v0, *ord, m, 0, bits, st));
    }
    for (void* p : {(void*)k0, (void*)k1, (void*)v0, tmp}) release(p, st);
    return 0;
}

// tc_knn.cu
bool tc_supported();
int tc_seed_mask(const float* x, int n, int dp, const int* starts, int s, int take, unsigned* mask, int mw,
                 int* near, cudaStream_t st, const long long* rows_ids);

__global__ void near_keys_kernel(const int* near, int m, unsigned* keys, int* vals) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
        keys[t] = (unsigned)near[t];
        vals[t] = t;
    }
}

// The same order for member queries that have no seeded beams (a graph loaded from
// disk, L != L_build, the ranks of a sharded run): the nearest start of every query
// from one tensor-core screen of the queries against the start rows (the build's
// tc_seed_mask; only its `near` output is used here, an order key, so integer
// data takes the same fp16 screen).  Rows of <= 1,024 coordinates, >= 256 starts.
int near_locality_order(const SearchParams& P, const long long* qids, int m, int** ord, cudaStream_t st) {
    const int mw = (P.s + 31) / 32;
    int* near = nullptr;
    unsigned* mask = nullptr;
    PK_CHECK(scratch(&near, (size_t)m, st));
    PK_CHECK(scratch(&mask, (size_t)m * mw, st));
    int rc = tc_seed_mask(P.X, m, P.dp, P.starts, P.s, 1, mask, mw, near, st, qids);
    release(mask, st);
    if (rc) return rc;
    int bits = 1;
    while ((1 << bits) < P.s) ++bits;
    unsigned *k0 = nullptr, *k1 = nullptr;
    int* v0 = nullptr;
    PK_CHECK(scratch(&k0, (size_t)m, st));
    PK_CHECK(scratch(&k1, (size_t)m, st));
    PK_CHECK(scratch(&v0, (size_t)m, st));
    PK_CHECK(scratch(ord, (size_t)m, st));
    {
        ProfScope _ps("near_keys_kernel", st);
        near_keys_kernel<<<grid_for(m, 256), 256, 0, st>>>(near, m, k0, v0);
    }
    PK_CHECK_LAUNCH("near_keys_kernel");
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, k0, k1, v0, *ord, m, 0, bits, st);
    void* tmp = nullptr;
    PK_CHECK(cudaMallocAsync(&tmp, bytes + 16, st));
    {
        ProfScope _ps("cub_DeviceRadixSort_SortPairs", st);
        PK_CHECK(cub::DeviceRadixSort::SortPairs(tmp, bytes, k0, k1, v0, *ord, m, 0, bits, st));
    }
    for (void* p : {(void*)near, (void*)k0, (void*)k1, (void*)v0, tmp}) release(p, st);
    return 0;
}

template <int MODE, int QV>
int launch_beam_knn(const SearchParams& P, const long long* qids, int m, int L, int kk, int H,
                    long long* out_ids, double* out_d, long long* counts, long long* evals, cudaStream_t st) {
    size_t wb = align16(beam_smem_bytes(L, H));
    // beams past the shared-memory opt-in: the beam goes to a global slab per warp
    const bool spill = wb > (size_t)max_smem_optin();
    const size_t gstride = spill ? spill_slab_bytes(L) : 0;
    if (spill) wb = align16(spill_smem_bytes(H));
    // row ring of the float searches with lazy keys (beam.cuh carve_ring), behind the beam state
    SearchParams Pr = P;
    Pr.ring = MODE == MODE_SEQ64 && QV >= 4 ? ring_slots(P.dp, QV, P.screen && P.lazy) : 0;
    if (spill || wb + align16(ring_smem_bytes(P.dp, Pr.ring)) > (size_t)max_smem_optin()) Pr.ring = 0;
    // with the ring, the seen table moves to a global slab per warp (carve_beam_gh)
    const bool ghash = Pr.ring && env_int("PK_HASH_GLOBAL", 1) == 1;
    if (ghash) wb = align16(beam_smem_bytes(L, 0));
    wb += align16(ring_smem_bytes(P.dp, Pr.ring));
    // warps per block: the most resident warps per SM (wide beams: a block of 2
    // x 64 KB leaves a third warp's worth of the SM's shared memory unused)
    const size_t sm_bytes = (size_t)max_smem_optin() + 1024;  // per-SM capacity (one block's reserve)
    int wpb = 1, best = 0;
    for (int w = 4; w >= 1; w >>= 1) {
        if (wb * w > (size_t)max_smem_optin()) continue;
        const int resident = w * (int)std::min<size_t>(32 / w, sm_bytes / (wb * w + 1024));
        if (resident > best) {
            best = resident;
            wpb = w;
        }
    }
    auto kern = beam_knn_kernel<MODE, QV, false>;
    if constexpr (MODE == MODE_SEQ64 && QV >= 4) {
        if (Pr.ring) kern = beam_knn_kernel<MODE, QV, true>;
    }
    PK_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(wb * wpb)));
    int per_sm = 0;
    PK_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpb, wb * wpb));
    if (per_sm < 1) per_sm = 1;
    long long blocks = ((long long)m + wpb - 1) / wpb;
    long long cap = (long long)sm_count() * per_sm;
    int grid = (int)(blocks < cap ? blocks : cap);
    if (spill) {
        // slabs for at most ~1 GiB of beams (the widest rounds hold few queries)
        const long long max_warps = std::max<long long>(wpb, (1ll << 30) / (long long)gstride);
        grid = (int)std::min<long long>(grid, max_warps / wpb);
    }
    if (grid < 1) grid = 1;
    unsigned char* gbeam = nullptr;
    if (spill) PK_CHECK(scratch(&gbeam, (size_t)grid * wpb * gstride, st));
    unsigned char* gh = nullptr;
    if (ghash) {
        Pr.ghash_stride = (size_t)H * 2;
        PK_CHECK(scratch(&gh, (size_t)grid * wpb * Pr.ghash_stride, st));
        Pr.ghash = gh;
    }
    int* ticket = nullptr;
    if ((long long)m > 2ll * grid * wpb && env_int("PK_TICKETS", 1) == 1) {
        PK_CHECK(scratch(&ticket, 1, st));
        PK_CHECK(cudaMemsetAsync(ticket, 0, sizeof(int), st));
        Pr.ticket = ticket;
    }
    int* ord = nullptr;
    if (P.seed_load && m >= (1 << 16) && env_int("PK_LOCALITY", 1) == 1) {
        const int rc = query_locality_order(P, qids, m, L, P.n_points, &ord, st);
        if (rc) return rc;
    } else if (P.X && P.dp <= 1024 && m >= (1 << 16) && P.s >= 256 && P.s <= 8192 && tc_supported() &&
               env_int("PK_LOCALITY", 1) == 1) {
        const int rc = near_locality_order(P, qids, m, &ord, st);
        if (rc) return rc;
    }
    // counting mode (bench.py's untimed pass): exact number of distinct ids
    // evaluated, added to evals[2] (the caller then passes 3 counters)
    SearchParams Pc = Pr;
    unsigned* ubm = nullptr;
    if (evals && env_int("PK_COUNT_UNIQUE", 0) == 1) {
        Pc.uwords = (int)((P.n_points + 31) / 32);
        PK_CHECK(scratch(&ubm, (size_t)grid * wpb * Pc.uwords, st));
        Pc.ubm = ubm;
    }
    {
        ProfScope _ps("beam_knn_kernel", st);
        kern<<<grid, 32 * wpb, wb * wpb, st>>>(Pc, qids, m, L, kk, H, wb, out_ids, out_d, counts, evals, gbeam,
                                               gstride, ord);
    }
    PK_CHECK_LAUNCH("beam_knn_kernel");
    if (ubm) release(ubm, st);
    if (gbeam) release(gbeam, st);
    if (gh) release(gh, st);
    if (ticket) release(ticket, st);
    if (ord) release(ord, st);
    return 0;
}

template <int MODE>
int dispatch_beam_knn(const SearchParams& P, const long long* qids, int m, int L, int kk, int H,
                      long long* out_ids, double* out_d, long long* counts, long long* evals, cudaStream_t st) {
    int qv = MODE == MODE_EXACT_U8 ? (P.dw + 31) / 32 : (P.dp + 127) / 128;
    if (MODE == MODE_SEQ64 && qv > 8)  // no fp32 screen for rows wider than 1024 floats
        return launch_beam_knn<MODE, 1>(P, qids, m, L, kk, H, out_ids, out_d, counts, evals, st);
    if (qv <= 1) return launch_beam_knn<MODE, 1>(P, qids, m, L, kk, H, out_ids, out_d, counts, evals, st);
    if (qv <= 2) return launch_beam_knn<MODE, 2>(P, qids, m, L, kk, H, out_ids, out_d, counts, evals, st);
    if (qv <= 4) return launch_beam_knn<MODE, 4>(P, qids, m, L, kk, H, out_ids, out_d, counts, evals, st);
    if (qv <= 8) return launch_beam_knn<MODE, 8>(P, qids, m, L, kk, H, out_ids, out_d, counts, evals, st);
    set_error("EXACT32 mode supports d <= 1024");
    return 2;
}

// exact kNN over a row list (or all rows), chunked scratch
int run_brute(const float* x, int n, int dp, const long long* qids, const double* qvec, const int* rowlist,
              const int* nrows, int m, int kk, long long* out_ids, double* out_d, cudaStream_t st) {
    if (kk <= 0 || m <= 0) return 0;
    int P = next_pow2(kk);
    int grid = sm_count();
    // scratch budget: keep the per-block row buffers <= ~2 GiB
    long long per_block = (long long)n * 8 + (long long)P * 12;
    long long maxg = (2ll << 30) / (per_block > 0 ? per_block : 1);
    if (maxg < 1) maxg = 1;
    if (grid > maxg) grid = (int)maxg;
    if (grid > m) grid = m;
    double* scr = nullptr;
    double* sd = nullptr;
    unsigned* si = nullptr;
    PK_CHECK(scratch(&scr, (size_t)grid * n, st));
    PK_CHECK(scratch(&sd, (size_t)grid * P, st));
    PK_CHECK(scratch(&si, (size_t)grid * P, st));
    {
        ProfScope _ps("brute_rows_kernel", st);
        brute_rows_kernel<<<grid, BT, 0, st>>>(x, n, dp, qids, qvec, rowlist, nrows, m, kk, scr, sd, si, P, out_ids, out_d);
    }
    cudaError_t e = cudaGetLastError();
    release(scr, st);
    release(sd, st);
    release(si, st);
    if (e != cudaSuccess) return fail("brute_rows_kernel", e);
    return 0;
}

}  // namespace pk

using namespace pk;

extern "C" int pk_check_exact32(const float* x, int64_t n, int64_t dp, int64_t d, int* out_flag, void* stream) {
    cudaStream_t st = as_stream(stream);
    int* bad = nullptr;
    unsigned* mx = nullptr;
    PK_CHECK(scratch(&bad, 1, st));
    PK_CHECK(scratch(&mx, 2, st));
    PK_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), st));
    PK_CHECK(cudaMemsetAsync(mx, 0, sizeof(unsigned), st));
    PK_CHECK(cudaMemsetAsync(mx + 1, 0xff, sizeof(unsigned), st));
    long long total = n * dp;
    {
        ProfScope _ps("check_exact32_kernel", st);
        check_exact32_kernel<<<grid_for(total, 256), 256, 0, st>>>(x, total, (int)dp, (int)d, bad, mx, nullptr);
    }
    {
        ProfScope _ps("finish_exact32_kernel", st);
        finish_exact32_kernel<<<1, 1, 0, st>>>(bad, mx, (int)d, out_flag);
    }
    PK_CHECK_LAUNCH("check_exact32");
    release(bad, st);
    release(mx, st);
    return 0;
}

__global__ void scan_result_kernel(const int* flag, const unsigned long long* first, long long* out) {
    out[0] = *flag;
    out[1] = *first == ~0ull ? -1ll : (long long)*first;
}

extern "C" int pk_scan_points(const float* x, int64_t n, int64_t dp, int64_t d, int64_t* out, void* stream) {
    cudaStream_t st = as_stream(stream);
    int *bad = nullptr, *flag = nullptr;
    unsigned* mx = nullptr;
    unsigned long long* first = nullptr;
    PK_CHECK(scratch(&bad, 1, st));
    PK_CHECK(scratch(&flag, 1, st));
    PK_CHECK(scratch(&mx, 2, st));
    PK_CHECK(scratch(&first, 1, st));
    PK_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), st));
    PK_CHECK(cudaMemsetAsync(mx, 0, sizeof(unsigned), st));
    PK_CHECK(cudaMemsetAsync(mx + 1, 0xff, sizeof(unsigned), st));
    PK_CHECK(cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), st));
    long long total = n * dp;
    {
        ProfScope _ps("check_exact32_kernel", st);
        check_exact32_kernel<<<grid_for(total, 256), 256, 0, st>>>(x, total, (int)dp, (int)d, bad, mx, first);
    }
    {
        ProfScope _ps("finish_exact32_kernel", st);
        finish_exact32_kernel<<<1, 1, 0, st>>>(bad, mx, (int)d, flag);
        scan_result_kernel<<<1, 1, 0, st>>>(flag, first, reinterpret_cast<long long*>(out));
    }
    PK_CHECK_LAUNCH("scan_points");
    for (void* p : {(void*)bad, (void*)flag, (void*)mx, (void*)first}) release(p, st);
    return 0;
}

extern "C" int pk_pack_u8(const float* x, int64_t n, int64_t dp, int64_t d, uint32_t* out, int64_t dw, void* stream) {
    cudaStream_t st = as_stream(stream);
    int* bad = nullptr;
    unsigned* mx = nullptr;
    PK_CHECK(scratch(&bad, 1, st));
    PK_CHECK(scratch(&mx, 2, st));
    PK_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), st));
    PK_CHECK(cudaMemsetAsync(mx, 0, sizeof(unsigned), st));
    PK_CHECK(cudaMemsetAsync(mx + 1, 0xff, sizeof(unsigned), st));
    long long total = n * dp;
    {
        ProfScope _ps("check_exact32_kernel", st);
        check_exact32_kernel<<<grid_for(total, 256), 256, 0, st>>>(x, total, (int)dp, (int)d, bad, mx, nullptr);
    }
    {
        ProfScope _ps("pack_u8_kernel", st);
        pack_u8_kernel<<<grid_for(n * dw, 256), 256, 0, st>>>(x, n, (int)dp, (int)d, mx, (int)dw, out);
    }
    PK_CHECK_LAUNCH("pack_u8");
    release(bad, st);
    release(mx, st);
    return 0;
}

extern "C" int pk_beam_knn_seeded(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                                  const int32_t* adj, int64_t R, const int32_t* deg, const int32_t* starts, int64_t s,
                                  const int64_t* qids, int64_t m, int64_t L, int64_t k, int64_t* out_ids,
                                  double* out_sqd, int64_t* out_counts, int brute_fallback, int64_t* out_evals,
                                  int hash_bits, const double* seed_bd, const uint32_t* seed_bi, const int32_t* seed_bl,
                                  void* stream);

extern "C" int pk_beam_knn(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                           const int32_t* adj, int64_t R,
                           const int32_t* deg, const int32_t* starts, int64_t s, const int64_t* qids, int64_t m,
                           int64_t L, int64_t k, int64_t* out_ids, double* out_sqd, int64_t* out_counts,
                           int brute_fallback, int64_t* out_evals, int hash_bits, void* stream) {
    return pk_beam_knn_seeded(x, n, dp, x8, dw, mode, adj, R, deg, starts, s, qids, m, L, k, out_ids, out_sqd,
                              out_counts, brute_fallback, out_evals, hash_bits, nullptr, nullptr, nullptr, stream);
}

extern "C" int pk_beam_knn_seeded(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                                  const int32_t* adj, int64_t R, const int32_t* deg, const int32_t* starts, int64_t s,
                                  const int64_t* qids, int64_t m, int64_t L, int64_t k, int64_t* out_ids,
                                  double* out_sqd, int64_t* out_counts, int brute_fallback, int64_t* out_evals,
                                  int hash_bits, const double* seed_bd, const uint32_t* seed_bi, const int32_t* seed_bl,
                                  void* stream) {
    cudaStream_t st = as_stream(stream);
    int64_t kk = k < n - 1 ? k : n - 1;
    if (kk <= 0 || m <= 0) {
        if (m > 0) PK_CHECK(cudaMemsetAsync(out_counts, 0, sizeof(int64_t) * m, st));
        return 0;
    }
    if (L < kk) {
        set_error("beam width L must be >= k");
        return 2;
    }
    if (n > (int64_t)PK_IDMASK) {
        set_error("too many points for the beam kernels (ids are 30-bit)");
        return 2;
    }
    // Start points re-met as neighbours are simply re-evaluated (and dropped
    // by the key-equality check when already in the beam): cheaper than a
    // dependent bitmap load on every neighbour.
    SearchParams P{x, (int)dp, adj, (int)R, deg, starts, (int)s, x8, (int)dw};
    P.screen = env_int("PK_SCREEN", 1) == 1;
    P.n_points = n;
    P.prefetch = env_int("PK_PREFETCH", 0) == 1;  // adjacency-row L1 prefetch: measured slower on every configuration
    P.prefetch_rows = env_int("PK_PREFETCH_ROWS", 0) == 1 && dp >= 512;  // L2 prefetch of candidate rows: a gain before the ticket scheduling, a 2 % loss since
    P.lazy = env_int("PK_LAZY", 1) == 1 && n < (int64_t)PK_IDMASK;
    P.seed_only = env_int("PK_SEED_ONLY", 0);
    P.seed_select = env_int("PK_SEED_SELECT", 1);
    // the counting pass (bench.py) must evaluate the seeds: no cached beams there
    if (seed_bd && seed_bi && seed_bl && !(out_evals && env_int("PK_COUNT_UNIQUE", 0) == 1) &&
        env_int("PK_SEED_CACHE", 1) == 1) {
        P.seed_bd = const_cast<double*>(seed_bd);
        P.seed_bi = const_cast<unsigned*>(reinterpret_cast<const unsigned*>(seed_bi));
        P.seed_bl = const_cast<int*>(seed_bl);
        P.seed_load = 1;
    }
    int H = choose_hash((int)L, hash_bits, n);
    const long long* q = reinterpret_cast<const long long*>(qids);
    long long* oi = reinterpret_cast<long long*>(out_ids);
    long long* oc = reinterpret_cast<long long*>(out_counts);
    long long* ev = reinterpret_cast<long long*>(out_evals);
    if (mode == MODE_EXACT_U8 && !x8) {
        set_error("u8 mode needs the packed rows");
        return 2;
    }
    int rc = mode == MODE_EXACT_U8
                 ? dispatch_beam_knn<MODE_EXACT_U8>(P, q, (int)m, (int)L, (int)kk, H, oi, out_sqd, oc, ev, st)
             : mode == MODE_EXACT32
                 ? dispatch_beam_knn<MODE_EXACT32>(P, q, (int)m, (int)L, (int)kk, H, oi, out_sqd, oc, ev, st)
                 : dispatch_beam_knn<MODE_SEQ64>(P, q, (int)m, (int)L, (int)kk, H, oi, out_sqd, oc, ev, st);
    if (rc) return rc;
    if (brute_fallback) {
        int* list = nullptr;
        int* nl = nullptr;
        PK_CHECK(scratch(&list, (size_t)m, st));
        PK_CHECK(scratch(&nl, 1, st));
        PK_CHECK(cudaMemsetAsync(nl, 0, sizeof(int), st));
        {
            ProfScope _ps("short_rows_kernel", st);
            short_rows_kernel<<<grid_for(m, 256), 256, 0, st>>>(oc, (int)m, (int)kk, list, nl);
        }
        PK_CHECK_LAUNCH("short_rows_kernel");
        // short rows are rare (disconnected or duplicate-heavy regions): read
        // the count so the exact pass and its row scratch run only when needed
        int hshort = 0;
        PK_CHECK(cudaMemcpyAsync(&hshort, nl, sizeof(int), cudaMemcpyDeviceToHost, st));
        PK_CHECK(cudaStreamSynchronize(st));
        if (hshort > 0)
            rc = run_brute(x, (int)n, (int)dp, q, nullptr, list, nl, std::min<int>((int)m, hshort), (int)kk, oi,
                           out_sqd, st);
        release(list, st);
        release(nl, st);
        if (rc) return rc;
    }
    return 0;
}

extern "C" int pk_beam_search_single(const float* x, int64_t n, int64_t dp, const int32_t* adj, int64_t R,
                                     const int32_t* deg, const int32_t* starts, int64_t s, int64_t qid,
                                     const double* qvec, int64_t L, int64_t k, int64_t* top_ids, double* top_sqd,
                                     int64_t* top_count, int64_t* vis_ids, double* vis_sqd, int64_t vcap,
                                     int64_t* vis_count, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (L < k) {
        set_error("beam width L must be >= k");
        return 2;
    }
    SearchParams P{x, (int)dp, adj, (int)R, deg, starts, (int)s};
    int H = choose_hash((int)L, 0, n);
    size_t bytes = align16(beam_smem_bytes((int)L, H));
    unsigned char* gbeam = nullptr;
    if (bytes > (size_t)max_smem_optin()) {  // wide beam: global slab (carve_beam_spill)
        bytes = align16(spill_smem_bytes(H));
        PK_CHECK(scratch(&gbeam, spill_slab_bytes((int)L), st));
    }
    unsigned* vi = nullptr;
    double* vd = nullptr;
    PK_CHECK(scratch(&vi, (size_t)vcap, st));
    PK_CHECK(scratch(&vd, (size_t)vcap, st));
    unsigned self = qid >= 0 ? (unsigned)qid : 0xffffffffu;
    if (qid >= 0) {
        auto kern = single_search_kernel<Seq64Member>;
        PK_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        {
            ProfScope _ps("single_search_kernel", st);
            kern<<<1, 32, bytes, st>>>(P, Seq64Member{x + (size_t)qid * dp, (int)dp}, self, (int)L, (int)k, H,
                                       reinterpret_cast<long long*>(top_ids), top_sqd, reinterpret_cast<long long*>(top_count),
                                       reinterpret_cast<long long*>(vis_ids), vis_sqd, (int)vcap,
                                       reinterpret_cast<long long*>(vis_count), vi, vd, gbeam);
        }
    } else {
        auto kern = single_search_kernel<Seq64Vector>;
        PK_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        {
            ProfScope _ps("single_search_kernel", st);
            kern<<<1, 32, bytes, st>>>(P, Seq64Vector{qvec, (int)dp}, self, (int)L, (int)k, H,
                                       reinterpret_cast<long long*>(top_ids), top_sqd, reinterpret_cast<long long*>(top_count),
                                       reinterpret_cast<long long*>(vis_ids), vis_sqd, (int)vcap,
                                       reinterpret_cast<long long*>(vis_count), vi, vd, gbeam);
        }
    }
    PK_CHECK_LAUNCH("single_search_kernel");
    release(vi, st);
    release(vd, st);
    release(gbeam, st);
    return 0;
}

extern "C" int pk_brute_knn(const float* x, int64_t n, int64_t dp, const int64_t* qids, int64_t m, int64_t k,
                            int64_t* out_ids, double* out_sqd, void* stream) {
    cudaStream_t st = as_stream(stream);
    int64_t kk = k < n - 1 ? k : n - 1;
    if (kk <= 0 || m <= 0) return 0;
    return run_brute(x, (int)n, (int)dp, reinterpret_cast<const long long*>(qids), nullptr, nullptr, nullptr, (int)m,
                     (int)kk, reinterpret_cast<long long*>(out_ids), out_sqd, st);
}

extern "C" int pk_brute_knn_vector(const float* x, int64_t n, int64_t dp, const double* qvec, int64_t k,
                                   int64_t* out_ids, double* out_sqd, void* stream) {
    cudaStream_t st = as_stream(stream);
    int64_t kk = k < n ? k : n;
    if (kk <= 0) return 0;
    return run_brute(x, (int)n, (int)dp, nullptr, qvec, nullptr, nullptr, 1, (int)kk,
                     reinterpret_cast<long long*>(out_ids), out_sqd, st);
}

extern "C" int pk_sqrt(const double* sqd, int64_t count, double* out, void* stream) {
    if (count <= 0) return 0;
    cudaStream_t st = as_stream(stream);
    {
        ProfScope _ps("sqrt_kernel", st);
        sqrt_kernel<<<grid_for(count, 256), 256, 0, st>>>(sqd, count, out);
    }
    PK_CHECK_LAUNCH("sqrt_kernel");
    return 0;
}

// Diagnostics: read (and with reset != 0 clear) the query walks' phase timers;
// all zero unless the library was built with -DPK_PHASE_TIMERS.
extern "C" int pk_phase_timers(unsigned long long* out8, int reset) {
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
