// Exact full scans over all n points for a batch of member queries:
//   * nearest strictly denser point (dp_scan_all, _kernels.py:442-462);
//   * number of points whose (distance, id) key is below a given key -- used
//     to decide whether a query's exact kNN row of width kk would contain its
//     nearest denser point, without building the row (doubling rounds whose
//     beam search came up short, vamana.py:220-225 + dependent.py:80-93).
// Each block holds QT queries in shared memory and streams a chunk of points
// once for all of them; distances are exact in the point set's policy (float64
// in coordinate order, or integer dp4a on u8-packed rows).
#include <algorithm>

#include "../../include/peakann_b200.h"
#include "api.cuh"
#include "common.cuh"

namespace pk {

int grid_for(long long work, int block);

constexpr int kScanThreads = 256;
constexpr int kScanQ = 16;    // queries per block
constexpr int kScanPPT = 4;   // points per thread per block

struct ScanArgs {
    DataRef D;
    int n;
    const long long* rank;     // (n,), SCAN_DENSER
    const long long* qids;     // (m,)
    int m;
    const double* key_d;       // (m,) threshold distances, SCAN_COUNT
    const long long* key_i;    // (m,) threshold ids, SCAN_COUNT
    double* part_d;            // (m, nchunk) partial minima, SCAN_DENSER
    int* part_i;
    long long* count;          // (m,) SCAN_COUNT
};

enum { SCAN_DENSER = 0, SCAN_COUNT = 1, SCAN_DUMP = 2 };

// distances from one point row to the QT staged queries
template <int MODE>
struct QueryTile;

template <>
struct QueryTile<MODE_SEQ64> {
    const float* q;  // smem, QT x dp floats
    int dp;
    __device__ __forceinline__ void dist(const DataRef& D, int j, double* acc) const {
        const float* r = D.X + (size_t)j * dp;
#pragma unroll
        for (int a = 0; a < kScanQ; ++a) acc[a] = 0.0;
        for (int t = 0; t < dp; t += 4) {
            const float4 x = ldg4(r + t);
#pragma unroll
            for (int a = 0; a < kScanQ; ++a) {
                const float* qa = q + a * dp + t;
                double e0 = (double)qa[0] - (double)x.x; acc[a] = __dadd_rn(acc[a], __dmul_rn(e0, e0));
                double e1 = (double)qa[1] - (double)x.y; acc[a] = __dadd_rn(acc[a], __dmul_rn(e1, e1));
                double e2 = (double)qa[2] - (double)x.z; acc[a] = __dadd_rn(acc[a], __dmul_rn(e2, e2));
                double e3 = (double)qa[3] - (double)x.w; acc[a] = __dadd_rn(acc[a], __dmul_rn(e3, e3));
            }
        }
    }
};

// float32 screen of the count scan (SEQ64): per thread, sequential fma over
// the coordinates -- within (dp + 3) 2^-24 relative of the exact sum (all
// terms non-negative), widened to kCountEps below; pairs inside the band get
// the exact float64 value (one_exact)
__device__ __forceinline__ void dist32(const float* q, int dp, const float* __restrict__ X, int j, float* acc) {
    const float* r = X + (size_t)j * dp;
#pragma unroll
    for (int a = 0; a < kScanQ; ++a) acc[a] = 0.f;
    for (int t = 0; t < dp; t += 4) {
        const float4 x = ldg4(r + t);
#pragma unroll
        for (int a = 0; a < kScanQ; ++a) {
            const float4 qa = *reinterpret_cast<const float4*>(q + a * dp + t);
            const float e0 = qa.x - x.x, e1 = qa.y - x.y, e2 = qa.z - x.z, e3 = qa.w - x.w;
            acc[a] = fmaf(e0, e0, acc[a]);
            acc[a] = fmaf(e1, e1, acc[a]);
            acc[a] = fmaf(e2, e2, acc[a]);
            acc[a] = fmaf(e3, e3, acc[a]);
        }
    }
}
__device__ __forceinline__ double one_exact(const float* q, int dp, const float* __restrict__ X, int j) {
    const float* r = X + (size_t)j * dp;
    double acc = 0.0;
    for (int t = 0; t < dp; ++t) {
        const double e = (double)q[t] - (double)__ldg(r + t);
        acc = __dadd_rn(acc, __dmul_rn(e, e));
    }
    return acc;
}

template <>
struct QueryTile<MODE_EXACT_U8> {
    const unsigned* q;  // smem, QT x dw words
    int dw;
    __device__ __forceinline__ void dist(const DataRef& D, int j, double* acc) const {
        const unsigned* r = D.X8 + (size_t)j * dw;
        unsigned s[kScanQ];
#pragma unroll
        for (int a = 0; a < kScanQ; ++a) s[a] = 0u;
        for (int w = 0; w < dw; ++w) {
            const unsigned x = __ldg(r + w);
#pragma unroll
            for (int a = 0; a < kScanQ; ++a) {
                const unsigned v = __vabsdiffu4(q[a * dw + w], x);
                s[a] = __dp4a(v, v, s[a]);
            }
        }
#pragma unroll
        for (int a = 0; a < kScanQ; ++a) acc[a] = (double)s[a];
    }
};

template <int MODE, int OP>
__global__ void __launch_bounds__(kScanThreads) scan_kernel(ScanArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ long long qr[kScanQ];
    __shared__ long long qid[kScanQ];
    __shared__ double kdd[kScanQ];
    __shared__ long long kdi[kScanQ];
    const int q0 = blockIdx.x * kScanQ;
    const int nq = min(kScanQ, A.m - q0);
    const int width = MODE == MODE_EXACT_U8 ? A.D.dw : A.D.dp;
    for (int x = threadIdx.x; x < kScanQ * width; x += kScanThreads) {
        const int a = x / width, t = x % width;
        const long long qi = a < nq ? A.qids[q0 + a] : 0;
        if (MODE == MODE_EXACT_U8)
            reinterpret_cast<unsigned*>(smem)[x] = a < nq ? A.D.X8[(size_t)qi * width + t] : 0u;
        else
            reinterpret_cast<float*>(smem)[x] = a < nq ? A.D.X[(size_t)qi * width + t] : 0.f;
    }
    if (threadIdx.x < kScanQ) {
        const int a = threadIdx.x;
        qid[a] = a < nq ? A.qids[q0 + a] : -1;
        if (OP == SCAN_DENSER) qr[a] = a < nq ? A.rank[A.qids[q0 + a]] : 0x7fffffffffffffffLL;
        if (OP == SCAN_COUNT) {
            kdd[a] = a < nq ? A.key_d[q0 + a] : -1.0;
            kdi[a] = a < nq ? A.key_i[q0 + a] : -1;
        }
    }
    __syncthreads();
    QueryTile<MODE> tile;
    if constexpr (MODE == MODE_EXACT_U8) {
        tile.q = reinterpret_cast<const unsigned*>(smem);
        tile.dw = A.D.dw;
    } else {
        tile.q = reinterpret_cast<const float*>(smem);
        tile.dp = A.D.dp;
    }
    long long rmin = 0x7fffffffffffffffLL;
    if (OP == SCAN_DENSER)
        for (int a = 0; a < kScanQ; ++a) rmin = min(rmin, qr[a]);
    double best[kScanQ];
    int bid[kScanQ];
    int cnt[kScanQ];
#pragma unroll
    for (int a = 0; a < kScanQ; ++a) {
        best[a] = __longlong_as_double(0x7ff0000000000000LL);
        bid[a] = -1;
        cnt[a] = 0;
    }
    const int chunk = kScanThreads * kScanPPT;
    const int j0 = blockIdx.y * chunk;
    if constexpr (OP == SCAN_COUNT && MODE == MODE_EXACT_U8) {
        // register-blocked count scan on packed u8 rows: each thread carries its
        // kScanPPT points through the words together, so every staged query word
        // is read once per kScanPPT points (exact integer distances, any order)
        const int dw = A.D.dw;
        int js[kScanPPT];
        const unsigned* rp[kScanPPT];
        unsigned acc[kScanPPT][kScanQ];
#pragma unroll
        for (int p = 0; p < kScanPPT; ++p) {
            js[p] = j0 + threadIdx.x + p * kScanThreads;
            rp[p] = A.D.X8 + (size_t)min(js[p], A.n - 1) * dw;
#pragma unroll
            for (int a = 0; a < kScanQ; ++a) acc[p][a] = 0u;
        }
        const unsigned* qw = tile.q;
        for (int w = 0; w < dw; ++w) {
            unsigned x[kScanPPT];
#pragma unroll
            for (int p = 0; p < kScanPPT; ++p) x[p] = __ldg(rp[p] + w);
#pragma unroll
            for (int a = 0; a < kScanQ; ++a) {
                const unsigned qa = qw[a * dw + w];
#pragma unroll
                for (int p = 0; p < kScanPPT; ++p) {
                    const unsigned v = __vabsdiffu4(qa, x[p]);
                    acc[p][a] = __dp4a(v, v, acc[p][a]);
                }
            }
        }
#pragma unroll
        for (int p = 0; p < kScanPPT; ++p) {
            if (js[p] >= A.n) continue;
#pragma unroll
            for (int a = 0; a < kScanQ; ++a)
                if (a < nq && (long long)js[p] != qid[a] &&
                    key_lt((double)acc[p][a], (unsigned)js[p], kdd[a], (unsigned)kdi[a]))
                    ++cnt[a];
        }
    }
    for (int jj = threadIdx.x; jj < chunk; jj += kScanThreads) {
        if constexpr (OP == SCAN_COUNT && MODE == MODE_EXACT_U8) break;
        const int j = j0 + jj;
        if (j >= A.n) break;
        long long rj = 0;
        if (OP == SCAN_DENSER) {
            rj = __ldg(A.rank + j);
            if (rj <= rmin) continue;
        }
        if constexpr (OP == SCAN_COUNT && MODE == MODE_SEQ64) {
            float a32[kScanQ];
            dist32(tile.q, tile.dp, A.D.X, j, a32);
            const double eps = (double)(tile.dp + 8) * 1.1920928955078125e-07;
#pragma unroll
            for (int a = 0; a < kScanQ; ++a) {
                if ((long long)j == qid[a] || a >= nq) continue;
                const double v = (double)a32[a], T = kdd[a];
                bool below;
                if (v > 1e-30 && v < 1e30 && T > 1e-30 && v * (1.0 + eps) < T) below = true;
                else if (v > 1e-30 && v < 1e30 && v * (1.0 - eps) > T) below = false;
                else below = key_lt(one_exact(tile.q + a * tile.dp, tile.dp, A.D.X, j), (unsigned)j, T, (unsigned)kdi[a]);
                cnt[a] += below;
            }
            continue;
        }
        double acc[kScanQ];
        tile.dist(A.D, j, acc);
#pragma unroll
        for (int a = 0; a < kScanQ; ++a) {
            if (OP == SCAN_DENSER) {
                if (rj > qr[a] && key_lt(acc[a], (unsigned)j, best[a], (unsigned)bid[a])) {
                    best[a] = acc[a];
                    bid[a] = j;
                }
            } else {
                if ((long long)j != qid[a] && key_lt(acc[a], (unsigned)j, kdd[a], (unsigned)kdi[a])) ++cnt[a];
            }
        }
    }
    const int lane = lane_id(), w = threadIdx.x >> 5;
    if (OP == SCAN_COUNT) {
#pragma unroll
        for (int a = 0; a < kScanQ; ++a) {
            int c = cnt[a];
            for (int s = 16; s; s >>= 1) c += __shfl_xor_sync(PK_FULL, c, s);
            if (lane == 0 && c && a < nq) atomicAdd(reinterpret_cast<unsigned long long*>(A.count + q0 + a),
                                                    (unsigned long long)c);
        }
        return;
    }
    __shared__ double rd[kScanThreads / 32][kScanQ];
    __shared__ int ri[kScanThreads / 32][kScanQ];
#pragma unroll
    for (int a = 0; a < kScanQ; ++a) {
        double d = best[a];
        unsigned i = (unsigned)bid[a];
        for (int s = 16; s; s >>= 1) {
            double od = __shfl_xor_sync(PK_FULL, d, s);
            unsigned oi = __shfl_xor_sync(PK_FULL, i, s);
            if (key_lt(od, oi, d, i)) { d = od; i = oi; }
        }
        if (lane == 0) { rd[w][a] = d; ri[w][a] = (int)i; }
    }
    __syncthreads();
    if (threadIdx.x < nq) {
        const int a = threadIdx.x;
        double d = rd[0][a];
        unsigned i = (unsigned)ri[0][a];
        for (int ww = 1; ww < kScanThreads / 32; ++ww)
            if (key_lt(rd[ww][a], (unsigned)ri[ww][a], d, i)) { d = rd[ww][a]; i = (unsigned)ri[ww][a]; }
        A.part_d[(size_t)(q0 + a) * gridDim.y + blockIdx.y] = d;
        A.part_i[(size_t)(q0 + a) * gridDim.y + blockIdx.y] = (int)i;
    }
}

__global__ void scan_reduce_kernel(const double* part_d, const int* part_i, int m, int nchunk, long long* out_id,
                                   double* out_d) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    double d = __longlong_as_double(0x7ff0000000000000LL);
    unsigned i = 0xffffffffu;
    for (int c = 0; c < nchunk; ++c) {
        const double od = part_d[(size_t)t * nchunk + c];
        const unsigned oi = (unsigned)part_i[(size_t)t * nchunk + c];
        if (key_lt(od, oi, d, i)) { d = od; i = oi; }
    }
    out_id[t] = i == 0xffffffffu ? -1 : (long long)i;
    out_d[t] = d;
}

// rows resolved by the full scan: lam/delta scattered, the rest kept
__global__ void short_resolve_kernel(const long long* qids, int m, const long long* sid, const double* ssq,
                                     const long long* cnt, long long kk, long long* lam, double* delta,
                                     unsigned char* unres) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const bool ok = sid[t] >= 0 && cnt[t] < kk;
    if (ok) {
        lam[qids[t]] = sid[t];
        delta[qids[t]] = sqrt(ssq[t]);
    }
    unres[t] = !ok;
}

template <int MODE, int OP>
int launch_scan(ScanArgs A, cudaStream_t st, int* nchunk_out) {
    const int nchunk = (A.n + kScanThreads * kScanPPT - 1) / (kScanThreads * kScanPPT);
    const int width = MODE == MODE_EXACT_U8 ? A.D.dw : A.D.dp;
    const size_t sm = (size_t)kScanQ * width * 4;
    auto kern = scan_kernel<MODE, OP>;
    if (sm > 48 * 1024) PK_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dim3 grid((unsigned)((A.m + kScanQ - 1) / kScanQ), (unsigned)nchunk);
    {
        ProfScope _ps(OP == SCAN_DENSER ? "scan_denser_kernel" : "scan_count_kernel", st);
        kern<<<grid, kScanThreads, sm, st>>>(A);
    }
    PK_CHECK_LAUNCH("scan_kernel");
    *nchunk_out = nchunk;
    return 0;
}

template <int OP>
int dispatch_scan(int mode, ScanArgs A, cudaStream_t st, int* nchunk) {
    // EXACT32 data is integer-valued: the float64 path computes the same values
    if (mode == MODE_EXACT_U8) return launch_scan<MODE_EXACT_U8, OP>(A, st, nchunk);
    return launch_scan<MODE_SEQ64, OP>(A, st, nchunk);
}

extern int compact_flagged(const long long* in, const unsigned char* flags, long long n, long long* out,
                           long long* count, cudaStream_t st);

}  // namespace pk

using namespace pk;

int dp_scan_u8_tc(const uint32_t* x8, int64_t n, const int64_t* rank, const int64_t* qids, int64_t m, int64_t* out_id,
                  double* out_sqd, cudaStream_t st);

extern "C" int pk_dp_scan(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                          const int64_t* rank, const int64_t* qids, int64_t m, int64_t* out_id, double* out_sqd,
                          void* stream) {
    cudaStream_t st = as_stream(stream);
    if (m <= 0) return 0;
    if (mode == MODE_EXACT_U8 && !x8) {
        set_error("u8 mode needs the packed rows");
        return 2;
    }
    if (mode == MODE_EXACT_U8 && dw == 32 && n < (1ll << 30) && env_int("PK_U8_TC_SCAN", 1) == 1)
        return dp_scan_u8_tc(x8, n, rank, qids, m, out_id, out_sqd, as_stream(stream));
    ScanArgs A{};
    A.D = DataRef{x, (int)dp, x8, (int)dw};
    A.n = (int)n;
    A.rank = reinterpret_cast<const long long*>(rank);
    A.qids = reinterpret_cast<const long long*>(qids);
    A.m = (int)m;
    const int nchunk = (int)((n + kScanThreads * kScanPPT - 1) / (kScanThreads * kScanPPT));
    PK_CHECK(scratch(&A.part_d, (size_t)m * nchunk, st));
    PK_CHECK(scratch(&A.part_i, (size_t)m * nchunk, st));
    int nc = 0;
    int rc = dispatch_scan<SCAN_DENSER>(mode, A, st, &nc);
    if (rc) return rc;
    {
        ProfScope _ps("scan_reduce_kernel", st);
        scan_reduce_kernel<<<(unsigned)((m + 127) / 128), 128, 0, st>>>(A.part_d, A.part_i, (int)m, nc,
                                                                      reinterpret_cast<long long*>(out_id), out_sqd);
    }
    PK_CHECK_LAUNCH("scan_reduce_kernel");
    release(A.part_d, st);
    release(A.part_i, st);
    return 0;
}

// ---- u8 rows of d = 128 (32 words): count scan on the integer tensor cores ----------------
// Exact u8 x u8 -> s32 mma.sync tiles (m16n8k32): a block holds 64 queries (4
// warps x 16 rows, A fragments in registers) and streams 64-point tiles of the
// packed rows through shared memory (cp.async, double-buffered, 16-byte chunks
// XOR-swizzled by row); every accumulator becomes the exact integer distance
// |q|^2 + |x|^2 - 2 q.x and is compared with the row's key.
constexpr int CU_Q = 64, CU_P = 64;

__device__ __forceinline__ int cu_swz(int r, int w) { return r * 32 + (w ^ ((r & 7) << 2)); }

__device__ __forceinline__ void cu_mma(const unsigned (&a)[4], unsigned b0, unsigned b1, int (&d)[4]) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cu_stage(const unsigned* __restrict__ X8, int n, int p0, unsigned* dst) {
    for (int e = threadIdx.x; e < CU_P * 8; e += 128) {
        const int r = e >> 3, ch = e & 7;
        const int j = min(p0 + r, n - 1);
        const unsigned d = (unsigned)__cvta_generic_to_shared(dst + r * 32 + ((ch ^ (r & 7)) << 2));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(X8 + (size_t)j * 32 + ch * 4)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// OP = SCAN_COUNT: count[q] += #{j != q : (d, j) < key}; OP = SCAN_DENSER:
// best[q] = min over j with rank[j] > rank[q] of the packed key (d << 32 | j)
// (exact integer distances < 2^32, ids < 2^30: the u64 order is the (d, id) order).
// OP = SCAN_DUMP: dump[q * n + j] = d(Q8 row q, X8 row j) for every column (qids
// null: query q is row q of Q8).  Query rows come from Q8, columns from X8.
template <int OP>
__global__ void __launch_bounds__(128) u8_tc_scan_kernel(const unsigned* __restrict__ Q8,
                                                        const unsigned* __restrict__ X8, int n,
                                                        const long long* __restrict__ qids, int m,
                                                        const double* __restrict__ key_d,
                                                        const long long* __restrict__ key_i,
                                                        const long long* __restrict__ rank, int tiles_per_block,
                                                        long long* __restrict__ count,
                                                        unsigned long long* __restrict__ best,
                                                        unsigned* __restrict__ dump) {
    __shared__ __align__(16) unsigned qs[CU_Q * 32];
    __shared__ __align__(16) unsigned ps[2][CU_P * 32];
    __shared__ unsigned pn[2][CU_P];
    __shared__ long long pr[2][CU_P];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int q0 = blockIdx.x * CU_Q;
    for (int e = tid; e < CU_Q * 8; e += 128) {
        const int r = e >> 3, ch = e & 7;
        const long long qi = qids ? qids[min(q0 + r, m - 1)] : (long long)min(q0 + r, m - 1);
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(Q8 + (size_t)qi * 32 + ch * 4));
        *reinterpret_cast<uint4*>(qs + r * 32 + ((ch ^ (r & 7)) << 2)) = v;
    }
    const int t0 = blockIdx.y * tiles_per_block;
    const int ntile = (n + CU_P - 1) / CU_P;
    const int t1 = min(ntile, t0 + tiles_per_block);
    if (t0 < t1) cu_stage(X8, n, t0 * CU_P, ps[0]);
    __syncthreads();
    // this warp's 16 query rows: A fragments, norms, keys
    const int ra = warp * 16 + g, rb = ra + 8;
    unsigned a[4][4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
        a[ks][0] = qs[cu_swz(ra, ks * 8 + tig)];
        a[ks][1] = qs[cu_swz(rb, ks * 8 + tig)];
        a[ks][2] = qs[cu_swz(ra, ks * 8 + 4 + tig)];
        a[ks][3] = qs[cu_swz(rb, ks * 8 + 4 + tig)];
    }
    unsigned na = 0u, nb = 0u;
    for (int w = 0; w < 32; ++w) {
        const unsigned x = qs[cu_swz(ra, w)], y = qs[cu_swz(rb, w)];
        na = __dp4a(x, x, na);
        nb = __dp4a(y, y, nb);
    }
    const bool va = q0 + ra < m, vb = q0 + rb < m;
    const long long sa = (va && qids) ? qids[q0 + ra] : -1, sb = (vb && qids) ? qids[q0 + rb] : -1;
    double ka = -1.0, kb = -1.0;
    unsigned ia = 0u, ib = 0u;
    long long rka = 0x7fffffffffffffffLL, rkb = 0x7fffffffffffffffLL;
    if constexpr (OP == SCAN_COUNT) {
        ka = va ? key_d[q0 + ra] : -1.0;
        kb = vb ? key_d[q0 + rb] : -1.0;
        ia = va ? (unsigned)key_i[q0 + ra] : 0u;
        ib = vb ? (unsigned)key_i[q0 + rb] : 0u;
    } else if constexpr (OP == SCAN_DENSER) {
        if (va) rka = rank[sa];
        if (vb) rkb = rank[sb];
    }
    int ca = 0, cb = 0;
    unsigned long long ba = ~0ull, bb = ~0ull;
    for (int t = t0; t < t1; ++t) {
        const int buf = (t - t0) & 1;
        if (t + 1 < t1) cu_stage(X8, n, (t + 1) * CU_P, ps[buf ^ 1]);
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncthreads();
        const unsigned* P = ps[buf];
        if (tid < CU_P) {
            unsigned s0 = 0u;
            for (int w = 0; w < 32; ++w) {
                const unsigned x = P[cu_swz(tid, w)];
                s0 = __dp4a(x, x, s0);
            }
            pn[buf][tid] = s0;
            if constexpr (OP == SCAN_DENSER) {
                const int j = t * CU_P + tid;
                pr[buf][tid] = j < n ? rank[j] : -1;
            }
        }
        __syncthreads();
        const int pbase = t * CU_P;
#pragma unroll
        for (int nt = 0; nt < CU_P / 8; ++nt) {
            int d[4] = {0, 0, 0, 0};
            const int col = nt * 8 + g;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                cu_mma(a[ks], P[cu_swz(col, ks * 8 + tig)], P[cu_swz(col, ks * 8 + 4 + tig)], d);
            const int c0 = nt * 8 + 2 * tig;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = pbase + c0 + h;
                if (j >= n) continue;
                const unsigned pj = pn[buf][c0 + h];
                const unsigned ua = na + pj - 2u * (unsigned)d[h], ub = nb + pj - 2u * (unsigned)d[2 + h];
                if constexpr (OP == SCAN_DUMP) {
                    if (va) dump[(size_t)(q0 + ra) * n + j] = ua;
                    if (vb) dump[(size_t)(q0 + rb) * n + j] = ub;
                } else if constexpr (OP == SCAN_COUNT) {
                    if (va && (long long)j != sa && key_lt((double)ua, (unsigned)j, ka, ia)) ++ca;
                    if (vb && (long long)j != sb && key_lt((double)ub, (unsigned)j, kb, ib)) ++cb;
                } else {
                    const long long rj = pr[buf][c0 + h];
                    const unsigned long long pa = ((unsigned long long)ua << 32) | (unsigned)j;
                    const unsigned long long pb = ((unsigned long long)ub << 32) | (unsigned)j;
                    if (rj > rka && pa < ba) ba = pa;
                    if (rj > rkb && pb < bb) bb = pb;
                }
            }
        }
        __syncthreads();
    }
    if constexpr (OP == SCAN_COUNT) {
        ca += __shfl_xor_sync(PK_FULL, ca, 1);
        ca += __shfl_xor_sync(PK_FULL, ca, 2);
        cb += __shfl_xor_sync(PK_FULL, cb, 1);
        cb += __shfl_xor_sync(PK_FULL, cb, 2);
        if (tig == 0) {
            if (va && ca) atomicAdd(reinterpret_cast<unsigned long long*>(count + q0 + ra), (unsigned long long)ca);
            if (vb && cb) atomicAdd(reinterpret_cast<unsigned long long*>(count + q0 + rb), (unsigned long long)cb);
        }
    } else if constexpr (OP == SCAN_DENSER) {
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            ba = min(ba, __shfl_xor_sync(PK_FULL, ba, o));
            bb = min(bb, __shfl_xor_sync(PK_FULL, bb, o));
        }
        if (tig == 0) {
            if (va && ba != ~0ull) atomicMin(best + q0 + ra, ba);
            if (vb && bb != ~0ull) atomicMin(best + q0 + rb, bb);
        }
    }
}

__global__ void u8_tc_best_kernel(const unsigned long long* best, int m, long long* out_id, double* out_d) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const unsigned long long b = best[t];
    out_id[t] = b == ~0ull ? -1 : (long long)(b & 0xffffffffull);
    out_d[t] = b == ~0ull ? __longlong_as_double(0x7ff0000000000000LL) : (double)(unsigned)(b >> 32);
}

// grid: one block per 64 queries x point splits (~32 blocks per SM overall)
template <int OP>
int launch_u8_tc_scan(const unsigned* x8, int64_t n, const int64_t* qids, int64_t m, const double* key_d,
                      const int64_t* key_i, const int64_t* rank, long long* count, unsigned long long* best,
                      cudaStream_t st, const unsigned* q8 = nullptr, unsigned* dump = nullptr) {
    const int qt = (int)((m + CU_Q - 1) / CU_Q);
    const int ntile = (int)((n + CU_P - 1) / CU_P);
    int splits = std::max(1, std::min(ntile, (sm_count() * 32 + qt - 1) / qt));
    const int per = (ntile + splits - 1) / splits;
    splits = (ntile + per - 1) / per;
    ProfScope _ps(OP == SCAN_COUNT ? "count_u8_tc_kernel" : OP == SCAN_DUMP ? "seed_u8_tc_kernel" : "denser_u8_tc_kernel",
                  st);
    u8_tc_scan_kernel<OP><<<dim3(qt, splits), 128, 0, st>>>(
        q8 ? q8 : x8, x8, (int)n, reinterpret_cast<const long long*>(qids), (int)m, key_d, reinterpret_cast<const long long*>(key_i),
        reinterpret_cast<const long long*>(rank), per, count, best, dump);
    PK_CHECK_LAUNCH("u8_tc_scan_kernel");
    return 0;
}

__global__ void gather_rows8_kernel(const unsigned* x8, const int* starts, int s, unsigned* out) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < s * 32; t += gridDim.x * blockDim.x)
        out[t] = x8[(size_t)starts[t >> 5] * 32 + (t & 31)];
}

namespace pk {
// Exact squared distances of every u8 row (d = 128) to every start:
// tab[i * s + j] = |x_i - x_starts[j]|^2, from one integer tensor-core pass over
// the gathered start rows (build.cu: the build's seeding reads them).
int u8_seed_table(const unsigned* x8, int n, const int* starts, int s, unsigned* tab, cudaStream_t st) {
    unsigned* rows = nullptr;
    PK_CHECK(scratch(&rows, (size_t)s * 32, st));
    gather_rows8_kernel<<<(s * 32 + 255) / 256, 256, 0, st>>>(x8, starts, s, rows);
    PK_CHECK_LAUNCH("gather_rows8_kernel");
    const int rc = launch_u8_tc_scan<SCAN_DUMP>(rows, s, nullptr, n, nullptr, nullptr, nullptr, nullptr, nullptr, st,
                                                x8, tab);
    release(rows, st);
    return rc;
}
}  // namespace pk

int dp_scan_u8_tc(const uint32_t* x8, int64_t n, const int64_t* rank, const int64_t* qids, int64_t m, int64_t* out_id,
                  double* out_sqd, cudaStream_t st) {
    unsigned long long* best = nullptr;
    PK_CHECK(scratch(&best, (size_t)m, st));
    PK_CHECK(cudaMemsetAsync(best, 0xff, sizeof(unsigned long long) * (size_t)m, st));
    int rc = launch_u8_tc_scan<SCAN_DENSER>(x8, n, qids, m, nullptr, nullptr, rank, nullptr, best, st);
    if (rc) return rc;
    {
        ProfScope _ps("u8_tc_best_kernel", st);
        u8_tc_best_kernel<<<(unsigned)((m + 127) / 128), 128, 0, st>>>(best, (int)m, reinterpret_cast<long long*>(out_id),
                                                                    out_sqd);
    }
    PK_CHECK_LAUNCH("u8_tc_best_kernel");
    release(best, st);
    return 0;
}

extern "C" int pk_count_below(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                              const int64_t* qids, int64_t m, const double* key_d, const int64_t* key_i,
                              int64_t* out_count, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (m <= 0) return 0;
    ScanArgs A{};
    A.D = DataRef{x, (int)dp, x8, (int)dw};
    A.n = (int)n;
    A.qids = reinterpret_cast<const long long*>(qids);
    A.m = (int)m;
    A.key_d = key_d;
    A.key_i = reinterpret_cast<const long long*>(key_i);
    A.count = reinterpret_cast<long long*>(out_count);
    PK_CHECK(cudaMemsetAsync(out_count, 0, sizeof(int64_t) * (size_t)m, st));
    if (mode == MODE_EXACT_U8 && dw == 32 && x8 && env_int("PK_U8_TC_SCAN", 1) == 1)
        return launch_u8_tc_scan<SCAN_COUNT>(x8, n, qids, m, key_d, key_i, nullptr,
                                             reinterpret_cast<long long*>(out_count), nullptr, st);
    int nc = 0;
    return dispatch_scan<SCAN_COUNT>(mode, A, st, &nc);
}

namespace pk {
int tc_count_decide(const float* x, int n, int dp, const long long* qids, int m, const double* key_d,
                    const long long* key_i, long long kk, long long* cnt,
                    int (*exact_count)(const long long*, int, const double*, const long long*, long long*, void*),
                    void* ctx, cudaStream_t st);
bool tc_supported();
}  // namespace pk

namespace {
struct CountCtx {
    const float* x;
    int64_t n, dp;
    const uint32_t* x8;
    int64_t dw;
    int mode;
    void* stream;
};
int exact_count_cb(const long long* q, int m, const double* kd, const long long* ki, long long* out, void* ctx) {
    const CountCtx& C = *static_cast<const CountCtx*>(ctx);
    return pk_count_below(C.x, C.n, C.dp, C.x8, C.dw, C.mode, reinterpret_cast<const int64_t*>(q), m, kd,
                          reinterpret_cast<const int64_t*>(ki), reinterpret_cast<int64_t*>(out), C.stream);
}
}  // namespace

extern "C" int pk_resolve_short_scanned(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw,
                                        int mode, const int64_t* qids, int64_t m, int64_t kk, const int64_t* dp_id,
                                        const double* dp_sqd, int64_t* lam, double* delta, int64_t* unresolved,
                                        int64_t* n_unresolved, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (m <= 0) {
        PK_CHECK(cudaMemsetAsync(n_unresolved, 0, sizeof(int64_t), st));
        return 0;
    }
    long long* cnt = nullptr;
    unsigned char* fl = nullptr;
    PK_CHECK(scratch(&cnt, (size_t)m, st));
    PK_CHECK(scratch(&fl, (size_t)m, st));
    int rc;
    // float data: the decision count < kk from tensor-core bounds, exact counts
    // only for the rows they leave open
    if (mode == MODE_SEQ64 && x && m >= env_int("PK_TC_COUNT_MIN", 64) && n >= 4096 && env_int("PK_TC_COUNT", 1) == 1 &&
        tc_supported()) {
        CountCtx C{x, n, dp, x8, dw, mode, stream};
        rc = tc_count_decide(x, (int)n, (int)dp, reinterpret_cast<const long long*>(qids), (int)m, dp_sqd,
                             reinterpret_cast<const long long*>(dp_id), kk, cnt, exact_count_cb, &C, st);
    } else {
        rc = pk_count_below(x, n, dp, x8, dw, mode, qids, m, dp_sqd, dp_id, reinterpret_cast<int64_t*>(cnt), stream);
    }
    if (rc) return rc;
    {
        ProfScope _ps("short_resolve_kernel", st);
        short_resolve_kernel<<<(unsigned)((m + 127) / 128), 128, 0, st>>>(
            reinterpret_cast<const long long*>(qids), (int)m, reinterpret_cast<const long long*>(dp_id), dp_sqd, cnt,
            kk, reinterpret_cast<long long*>(lam), delta, fl);
    }
    PK_CHECK_LAUNCH("short_resolve_kernel");
    rc = compact_flagged(reinterpret_cast<const long long*>(qids), fl, m, reinterpret_cast<long long*>(unresolved),
                         reinterpret_cast<long long*>(n_unresolved), st);
    for (void* p : {(void*)cnt, (void*)fl}) release(p, st);
    return rc;
}

extern "C" int pk_resolve_short(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                                const int64_t* rank, const int64_t* qids, int64_t m, int64_t kk, int64_t* lam,
                                double* delta, int64_t* unresolved, int64_t* n_unresolved, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (m <= 0) {
        PK_CHECK(cudaMemsetAsync(n_unresolved, 0, sizeof(int64_t), st));
        return 0;
    }
    int64_t* sid = nullptr;
    double* ssq = nullptr;
    PK_CHECK(scratch(&sid, (size_t)m, st));
    PK_CHECK(scratch(&ssq, (size_t)m, st));
    int rc = pk_dp_scan(x, n, dp, x8, dw, mode, rank, qids, m, sid, ssq, stream);
    if (rc) return rc;
    rc = pk_resolve_short_scanned(x, n, dp, x8, dw, mode, qids, m, kk, sid, ssq, lam, delta, unresolved, n_unresolved,
                                  stream);
    release(sid, st);
    release(ssq, st);
    return rc;
}
