// Exact kNN on the tensor cores (the reference's brute_knn_batch,
// _kernels.py:86-104, for BruteForceIndex / the exact pipeline mode).
//
// 1. Screening: a tcgen05 GEMM of fp16 queries x fp16 points (K-major, TMA
//    tiles with 128-byte swizzle, fp32 accumulators in TMEM) with a fused
//    epilogue that turns every accumulator into ||q||^2 + ||p||^2 - 2 q.p and
//    keeps, per query row, the K' = 64 smallest screened distances (self
//    excluded).  Warp-specialised, one CTA per 128-query block (optionally a
//    slice of the points): warp 0 issues TMA, warp 1 issues tcgen05.mma (one
//    elected lane) into a double-buffered TMEM accumulator (2 x 256 columns),
//    warps 2-5 drain TMEM (tcgen05.ld) while the next tile accumulates.
// 2. Rescoring: one warp per query recomputes the K' candidates with the
//    reference's float64 sequential distance, sorts by (dist, id) and emits the
//    first kk -- the same keys the reference selects among.  A per-row
//    certificate checks that every screened-out point lies beyond the exact
//    kk-th distance given the fp16 error bound; rows that fail are counted and
//    reported (and recomputed exactly by the caller when requested).
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "../../include/peakann_b200.h"
#include "api.cuh"
#include "common.cuh"
#include "tc_common.cuh"

namespace pk {

int grid_for(long long work, int block);

constexpr int TC_BM = 128;          // queries per tile (UMMA M)
constexpr int TC_BN = 256;          // points per tile (UMMA N)
constexpr int TC_BK = 64;           // fp16 elements per stage (128-byte rows)
constexpr int TC_STAGES = 4;
constexpr int TC_KP = 64;           // screened candidates kept per row (K'), two halves
constexpr int TC_KPH = TC_KP / 2;   // one max-heap per (row, column half of the tile)
constexpr int TC_EPI = 8;           // epilogue warps: 2 per TMEM lane group (column halves)
constexpr int TC_THREADS = 64 + 32 * TC_EPI;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2;
constexpr int TC_B_BYTES = (TC_BN / 2) * TC_BK * 2;  // each CTA of the pair holds half the point tile
constexpr int TC_STAGE_BYTES = TC_A_BYTES + TC_B_BYTES;
constexpr int TC_LIST_BYTES = TC_KP * TC_BM * 8;
constexpr int TC_CH = 16;           // accumulator columns per tcgen05.ld in the epilogue
constexpr size_t TC_SMEM =
    1024 + (size_t)TC_STAGES * TC_STAGE_BYTES + TC_LIST_BYTES + 256 + 2 * TC_BN * 4 + TC_CH * 32 * TC_EPI * 4 +
    2 * TC_BN * 4;

struct TcArgs {
    const float* qn;       // (m,) ||q||^2 of the fp16-rounded-from rows (fp32 originals)
    const float* pn;       // (n,)
    const long long* qids; // (m,) member ids (self exclusion), may be null
    int m, n, kblocks;     // kblocks = Kp / 64
    int tiles_per_split;   // point tiles handled by one CTA
    int dbg;
    int nsplit;
    int* out_id;           // (m, nsplit, K') screened ids (-1 = empty)
    float* out_d;          // (m, nsplit, K') screened distances
    const int* prank;      // (n,) density rank: only points with prank > qrank[row] are kept
    const int* qrank;      // (m,) (both null: plain kNN)
    float* dump = nullptr;  // non-null: write every screened distance, dump[row * dump_ld + col] (no heaps)
    long long dump_ld = 0;
    // count mode (cnt_key non-null, no heaps): per row, the points j != self, j !=
    // cnt_kid[row] certainly below cnt_key[row] (hi < key) -> cnt_lo, possibly
    // below (lo <= key or non-finite screen) -> cnt_hi; bounds as in tc_seed_mask
    const double* cnt_key = nullptr;
    const long long* cnt_kid = nullptr;
    unsigned* cnt_lo = nullptr;
    unsigned* cnt_hi = nullptr;
    const float* pmax2 = nullptr;  // max ||p||^2 (device scalar)
    float cnt_eps = 0.f, cnt_abs = 0.f;
};

// ---- screening kernel ------------------------------------------------------------------
// CTA pair (cluster of 2 along x): CTA r owns query rows (2*pair + r)*128.. and loads
// point rows t*256 + r*128.. of every tile; the leader issues M=256 x N=256 MMAs that
// read both CTAs' smem and write each CTA's 128 rows into its own TMEM.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1) tc_screen_kernel(const __grid_constant__ CUtensorMap map_q,
                                                                  const __grid_constant__ CUtensorMap map_p, TcArgs A) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // offset from the shared array itself (not an integer round trip) so every
    // access below compiles to LDS/STS instead of generic loads/stores
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* stage_base = smem;
    float* lst_d = reinterpret_cast<float*>(smem + (size_t)TC_STAGES * TC_STAGE_BYTES);
    int* lst_i = reinterpret_cast<int*>(lst_d + TC_KP * TC_BM);
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(lst_i + TC_KP * TC_BM);
    unsigned long long* full = bars;
    unsigned long long* empty = bars + TC_STAGES;
    unsigned long long* tfull = bars + 2 * TC_STAGES;
    unsigned long long* tempty = bars + 2 * TC_STAGES + 2;
    unsigned* tmem_slot = reinterpret_cast<unsigned*>(bars + 2 * TC_STAGES + 4);
    float* pn_s = reinterpret_cast<float*>(bars + 2 * TC_STAGES + 8);  // [2][TC_BN]
    float* stg = pn_s + 2 * TC_BN;  // [TC_CH][32 * TC_EPI] chunk distances per epilogue thread
    int* rk_s = reinterpret_cast<int*>(stg + TC_CH * 32 * TC_EPI);  // [2][TC_BN] point ranks (dp scan)

    const int warp = threadIdx.x >> 5;
    const int lane = lane_id();
    const int qblock = blockIdx.x;
    const int split = blockIdx.y;
    const int ntiles_total = (A.n + TC_BN - 1) / TC_BN;
    const int t0 = split * A.tiles_per_split;
    const int t1 = min(ntiles_total, t0 + A.tiles_per_split);

    const unsigned rank = cluster_rank();
    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 2 * TC_EPI);  // one arrival per epilogue warp of both CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const unsigned tmem = *tmem_slot;
    const unsigned full_lead = mapa_shared(smem_u32(full), 0);
    const unsigned tempty_lead = mapa_shared(smem_u32(tempty), 0);

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            unsigned phase = 0;
            for (int t = t0; t < t1; ++t) {
                for (int kb = 0; kb < A.kblocks; ++kb) {
                    mbar_wait(empty + stage, phase ^ 1);
                    unsigned char* sa = stage_base + (size_t)stage * TC_STAGE_BYTES;
                    if (rank == 0) mbar_expect_tx(full + stage, 2 * TC_STAGE_BYTES);
                    const unsigned fb = full_lead + 8u * (unsigned)stage;
                    tma_load_2d_pair(&map_q, sa, fb, kb * TC_BK, qblock * TC_BM);
                    tma_load_2d_pair(&map_p, sa + TC_A_BYTES, fb, kb * TC_BK, t * TC_BN + (int)rank * (TC_BN / 2));
                    if (++stage == TC_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1 && rank == 0) {
        // instruction descriptor: F32 accumulate, F16 x F16, both K-major, N = 256, M = 256 (pair)
        const unsigned idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((unsigned)(TC_BN >> 3) << 17) |
                               ((unsigned)((2 * TC_BM) >> 4) << 24);
        int stage = 0;
        unsigned phase = 0;
        int acc = 0;
        unsigned aphase = 0;
        for (int t = t0; t < t1; ++t) {
            mbar_wait(tempty + acc, aphase ^ 1);
            tc_fence_after();
            const unsigned tmem_d = tmem + (unsigned)(acc * TC_BN);
            for (int kb = 0; kb < A.kblocks; ++kb) {
                mbar_wait(full + stage, phase);
                tc_fence_after();
                if (lane == 0) {
                    unsigned char* sa = stage_base + (size_t)stage * TC_STAGE_BYTES;
                    const unsigned long long da = umma_desc_sw128(sa);
                    const unsigned long long db = umma_desc_sw128(sa + TC_A_BYTES);
#pragma unroll
                    for (int k = 0; k < TC_BK / 16; ++k)  // 16 fp16 = 32 bytes per UMMA_K step
                        if (!(A.dbg & 2)) tc_mma_f16_pair(tmem_d, da + (unsigned long long)(2 * k), db + (unsigned long long)(2 * k),
                                        idesc, (kb | k) != 0);
                    tc_commit_pair(empty + stage);
                }
                __syncwarp();
                if (++stage == TC_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (lane == 0) tc_commit_pair(tfull + acc);
            __syncwarp();
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
    } else if (warp >= 2) {
        // epilogue: thread owns TMEM lane (query row) 32 * (warp % 4) + lane and
        // one column half of every tile (warps 2-5: columns 0-127, 6-9: 128-255)
        const int ew = warp & 3;
        const int half = (warp - 2) >> 2;
        const int et = (warp - 2) * 32 + lane;  // epilogue thread 0..255
        const int row = ew * 32 + lane;
        const int tid = row;  // list column
        float* hd = lst_d + (size_t)half * TC_KPH * TC_BM;  // this half's heap, [TC_KPH][TC_BM]
        int* hi = lst_i + (size_t)half * TC_KPH * TC_BM;
        const int q = qblock * TC_BM + row;
        const bool live = q < A.m;
        const long long self = (live && A.qids) ? A.qids[q] : -1;
        const float qn = live ? A.qn[q] : 0.f;
        const int myrank = (A.prank && live) ? A.qrank[q] : 0;
        for (int k = 0; k < TC_KPH; ++k) {
            hd[k * TC_BM + tid] = __int_as_float(0x7f800000);
            hi[k * TC_BM + tid] = -1;
        }
        float thr = __int_as_float(0x7f800000);
        int acc = 0;
        unsigned aphase = 0;
        // count mode state
        double ckey = 0.0;
        long long ckid = -1;
        float cerr = 0.f;
        unsigned c_lo = 0u, c_hi = 0u;
        if (A.cnt_key && live) {
            ckey = A.cnt_key[q];
            ckid = A.cnt_kid[q];
            const float p2 = *A.pmax2;
            cerr = A.cnt_eps * sqrtf(qn) * sqrtf(p2) + A.cnt_abs * (sqrtf(qn) + sqrtf(p2)) + 1e-6f * (qn + p2);
        }
        constexpr int kChunks = TC_BN / TC_CH / 2;  // chunks per column half
        for (int t = t0; t < t1; ++t) {
            // this tile's point norms, staged once for the 256 epilogue threads
            for (int x = et; x < TC_BN; x += 32 * TC_EPI) {
                const int col = t * TC_BN + x;
                pn_s[acc * TC_BN + x] = col < A.n ? __ldg(A.pn + col) : 0.f;
                if (A.prank) rk_s[acc * TC_BN + x] = col < A.n ? __ldg(A.prank + col) : -1;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(32 * TC_EPI) : "memory");
            mbar_wait(tfull + acc, aphase);
            tc_fence_after();
            const unsigned taddr = tmem + ((unsigned)(ew * 32) << 16) + (unsigned)(acc * TC_BN);
            for (int cc = 0; cc < kChunks; ++cc) {
                const int ch = half * kChunks + cc;
                unsigned v[TC_CH];
                __syncwarp();
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                    "[%16];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15])
                    : "r"(taddr + (unsigned)(ch * TC_CH)));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (A.dbg & 1) continue;  // warp-uniform (profiling aid)
                const int cbase = t * TC_BN + ch * TC_CH;
                const float* pnt = pn_s + acc * TC_BN + ch * TC_CH;
                // distances of the chunk, bit mask of the ones below this half's K'-th
                float pv[TC_CH];
#pragma unroll
                for (int j = 0; j < TC_CH; j += 4) {
                    const float4 t4 = *reinterpret_cast<const float4*>(pnt + j);
                    pv[j] = t4.x;
                    pv[j + 1] = t4.y;
                    pv[j + 2] = t4.z;
                    pv[j + 3] = t4.w;
                }
                unsigned mask = 0;
#pragma unroll
                for (int j = 0; j < TC_CH; ++j) {
                    const float dd = qn + pv[j] - 2.f * __uint_as_float(v[j]);
                    v[j] = __float_as_uint(dd);
                    mask |= (dd < thr ? 1u : 0u) << j;
                }
                if (A.cnt_key) {  // count mode
                    if (live) {
#pragma unroll
                        for (int j = 0; j < TC_CH; ++j) {
                            const long long col = cbase + j;
                            if (col < A.n && col != self && col != ckid) {
                                const float dd = __uint_as_float(v[j]);
                                const float mg = cerr + 1e-5f * fabsf(dd);
                                const bool fin = isfinite(dd + mg);
                                c_lo += (fin && (double)(dd + mg) < ckey) ? 1u : 0u;
                                c_hi += (!fin || !((double)(dd - mg) > ckey)) ? 1u : 0u;
                            }
                        }
                    }
                    continue;
                }
                if (A.dump) {  // dump mode: every column of the row, self included
                    if (live) {
                        float* o = A.dump + (size_t)q * A.dump_ld + cbase;
#pragma unroll
                        for (int j = 0; j < TC_CH; ++j)
                            if (cbase + j < A.n) o[j] = __uint_as_float(v[j]);
                    }
                    continue;
                }
                if (A.prank) {  // nearest-denser search: only strictly denser points compete
                    const int* rk = rk_s + acc * TC_BN + ch * TC_CH;
#pragma unroll
                    for (int j = 0; j < TC_CH; ++j)
                        if (rk[j] <= myrank) mask &= ~(1u << j);
                }
                if (!live) mask = 0;
                if (__any_sync(PK_FULL, mask != 0)) {
#pragma unroll
                    for (int j = 0; j < TC_CH; ++j) stg[j * 32 * TC_EPI + et] = __uint_as_float(v[j]);
                }
                if (cbase + TC_CH > A.n) mask &= A.n > cbase ? (1u << (A.n - cbase)) - 1u : 0u;
                if (self >= cbase && self < cbase + TC_CH) mask &= ~(1u << (int)(self - cbase));
                // every lane walks its own pending candidates: the warp runs max-popcount
                // iterations instead of one per column
                while (mask) {
                    const int j = __ffs(mask) - 1;
                    mask &= mask - 1u;
                    const float dd = stg[j * 32 * TC_EPI + et];
                    if (!(dd < thr)) continue;
                    // binary max-heap: replace the root, sift down
                    int i = 0;
                    for (;;) {
                        const int l = 2 * i + 1;
                        if (l >= TC_KPH) break;
                        const int r = l + 1;
                        const float dl = hd[l * TC_BM + tid];
                        const float dr = r < TC_KPH ? hd[r * TC_BM + tid] : -1.f;
                        const int cidx = dr > dl ? r : l;
                        const float dc = dr > dl ? dr : dl;
                        if (dc <= dd) break;
                        hd[i * TC_BM + tid] = dc;
                        hi[i * TC_BM + tid] = hi[cidx * TC_BM + tid];
                        i = cidx;
                    }
                    hd[i * TC_BM + tid] = dd;
                    hi[i * TC_BM + tid] = cbase + j;
                    thr = hd[tid];
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_lead + 8u * (unsigned)acc);
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
        if (A.cnt_key && live) {
            atomicAdd(A.cnt_lo + q, c_lo);
            atomicAdd(A.cnt_hi + q, c_hi);
        }
        if (live && !A.dump && !A.cnt_key) {
            const size_t base = ((size_t)q * A.nsplit + split) * TC_KP + (size_t)half * TC_KPH;
            for (int k = 0; k < TC_KPH; ++k) {
                A.out_id[base + k] = hi[k * TC_BM + tid];
                A.out_d[base + k] = hd[k * TC_BM + tid];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ---- operand preparation -------------------------------------------------------------------
// fp16 rows (K padded to a multiple of 64 with zeros) and fp32 squared norms
__global__ void tc_prep_kernel(const float* __restrict__ X, int dp, const long long* rows, int m, int kp,
                               __half* out, float* nrm) {
    // one warp per row (a block per row spent its time launching: 31 ms for the
    // 1.28 M rows of C5 where the copy needs ~1.5 ms of HBM time)
    const int lane = threadIdx.x & 31;
    const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = w; r < m; r += nw) {
        const long long src = rows ? rows[r] : r;
        const float* x = X + (size_t)src * dp;
        __half2* o = reinterpret_cast<__half2*>(out + (size_t)r * kp);
        double acc = 0.0;
        // dp is a multiple of 4 (16-byte rows), kp a multiple of 64
        for (int t = lane * 4; t < kp; t += 128) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (t < dp) v = *reinterpret_cast<const float4*>(x + t);
            o[t >> 1] = __halves2half2(__float2half_rn(v.x), __float2half_rn(v.y));
            o[(t >> 1) + 1] = __halves2half2(__float2half_rn(v.z), __float2half_rn(v.w));
            acc += (double)v.x * (double)v.x + (double)v.y * (double)v.y + (double)v.z * (double)v.z +
                   (double)v.w * (double)v.w;
        }
        for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(PK_FULL, acc, s);
        if (lane == 0) nrm[r] = (float)acc;
    }
}

// (dist, id) bitonic sort of P (power of two) entries in shared memory by one warp
__device__ __forceinline__ void warp_bitonic(double* kd, unsigned* ki, int P, int lane) {
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < P; i += 32) {
                const int x = i ^ j;
                if (x > i) {
                    const double a = kd[i], b = kd[x];
                    const unsigned ia = ki[i], ib = ki[x];
                    if (key_lt(b, ib, a, ia) == ((i & k) == 0)) {
                        kd[i] = b;
                        kd[x] = a;
                        ki[i] = ib;
                        ki[x] = ia;
                    }
                }
            }
            __syncwarp();
        }
}

// ---- exact rescoring ---------------------------------------------------------------------
// one warp per query: float64 sequential distances of the screened candidates,
// (dist, id) sort, first kk out; certificate: every screened-out point has
// screened distance >= the split's worst kept value, true >= screened - eps.
__global__ void tc_rescore_kernel(const float* __restrict__ X, int dp, const long long* __restrict__ qids, int m,
                                  int nsplit, const int* cand_i, const float* cand_d, int kk, float eps_scale,
                                  const float* qn, float pmax, long long* out_ids, double* out_d,
                                  unsigned long long* uncertified, unsigned char* row_flag, int P) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int lane = lane_id();
    double* kd = reinterpret_cast<double*>(smem) + (size_t)wib * P;
    unsigned* ki = reinterpret_cast<unsigned*>(reinterpret_cast<double*>(smem) + (size_t)wpb * P) + (size_t)wib * P;
    for (int t = blockIdx.x * wpb + wib; t < m; t += gridDim.x * wpb) {
        const long long qi = qids[t];
        const int c = nsplit * TC_KP;
        Seq64Member dq{X + (size_t)qi * dp, dp};
        const double eps = (double)eps_scale * sqrt((double)qn[t]) * (double)pmax;
        // 1. order the candidates by screened distance
        for (int x = lane; x < P; x += 32) {
            const int id = x < c ? cand_i[(size_t)t * c + x] : -1;
            kd[x] = id >= 0 ? (double)cand_d[(size_t)t * c + x] : __longlong_as_double(0x7ff0000000000000LL);
            ki[x] = id >= 0 ? (unsigned)id : 0xffffffffu;
        }
        __syncwarp();
        warp_bitonic(kd, ki, P, lane);
        // 2. exact distances only where the screened value allows a place in the top kk:
        //    true kk-th <= s_kk + eps and true >= screened - eps
        const double bound = kd[kk - 1] + 2.0 * eps;
        __syncwarp();
        for (int x = lane; x < P; x += 32) {
            if (ki[x] != 0xffffffffu && kd[x] <= bound) {
                kd[x] = dq.eval_one(X, (int)ki[x]);
            } else {
                kd[x] = __longlong_as_double(0x7ff0000000000000LL);
                ki[x] = 0xffffffffu;
            }
        }
        __syncwarp();
        warp_bitonic(kd, ki, P, lane);
        for (int x = lane; x < kk; x += 32) {
            out_ids[(size_t)t * kk + x] = ki[x] == 0xffffffffu ? -1 : (long long)ki[x];
            out_d[(size_t)t * kk + x] = kd[x];
        }
        // certificate
        const double tk = kd[kk - 1];
        bool ok = true;
        // one heap per (split, column half): each full heap bounds what it screened out
        for (int s = lane; s < 2 * nsplit; s += 32) {
            float worst = -1.f;
            bool full = true;
            for (int k = 0; k < TC_KPH; ++k) {
                const size_t o = (size_t)t * c + (size_t)s * TC_KPH + k;
                if (cand_i[o] < 0) full = false;
                worst = fmaxf(worst, cand_d[o]);
            }
            if (full && !((double)worst - eps > tk)) ok = false;
        }
        ok = __all_sync(PK_FULL, ok);
        if (lane == 0) {
            if (row_flag) row_flag[t] = ok ? 0 : 1;
            if (!ok && uncertified) atomicAdd(uncertified, 1ull);
        }
        __syncwarp();
    }
}

// ---- host -----------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    return fn;
}

static int make_map(CUtensorMap* map, const __half* base, int rows, int kp, int box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return 2;
    }
    cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kp * 2};
    cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)base, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed");
        return 2;
    }
    return 0;
}

__global__ void tc_max_kernel(const float* v, int n, float* out) {
    float mx = 0.f;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) mx = fmaxf(mx, v[i]);
    for (int s = 16; s; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(PK_FULL, mx, s));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(mx));
}

bool tc_supported() {
    int dev = 0, major = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    return major == 10;
}

}  // namespace pk

using namespace pk;

// shared host driver: exact kNN (prank == null) or nearest strictly denser
// point (prank / qrank, kk = 1) through tensor-core screening + rescoring
static int tc_knn_core(const float* x, int64_t n, int64_t dp, const int64_t* qids, int64_t m, int64_t kk,
                       const int* prank, const int* qrank, int64_t* out_ids, double* out_sqd, uint8_t* row_flags,
                       uint64_t* uncertified, cudaStream_t st) {
    if (kk <= 0 || m <= 0) return 0;
    if (kk > TC_KP / 2) {
        set_error("tensor-core kNN keeps k <= 32");
        return 2;
    }
    if (!tc_supported()) {
        set_error("tensor-core kNN needs an sm_100 device");
        return 2;
    }
    const int kp = (int)((dp + TC_BK - 1) / TC_BK * TC_BK);
    __half *qh = nullptr, *ph = nullptr;
    float *qn = nullptr, *pn = nullptr, *pmax = nullptr;
    long long* iota = nullptr;
    PK_CHECK(scratch(&qh, (size_t)m * kp, st));
    PK_CHECK(scratch(&ph, (size_t)n * kp, st));
    PK_CHECK(scratch(&qn, (size_t)m, st));
    PK_CHECK(scratch(&pn, (size_t)n, st));
    PK_CHECK(scratch(&pmax, 1, st));
    {
        ProfScope _ps("tc_prep_kernel", st);
        tc_prep_kernel<<<(unsigned)std::min<long long>(((long long)(m) + 7) / 8, 148ll * 32), 256, 0, st>>>(x, (int)dp, reinterpret_cast<const long long*>(qids), (int)m, kp,
                                                    qh, qn);
        tc_prep_kernel<<<(unsigned)std::min<long long>(((long long)(n) + 7) / 8, 148ll * 32), 256, 0, st>>>(x, (int)dp, nullptr, (int)n, kp, ph, pn);
    }
    PK_CHECK(cudaMemsetAsync(pmax, 0, sizeof(float), st));
    {
        ProfScope _ps("tc_max_kernel", st);
        tc_max_kernel<<<grid_for(n, 256), 256, 0, st>>>(pn, (int)n, pmax);
    }
    PK_CHECK_LAUNCH("tc_prep");
    CUtensorMap mq, mp;
    int rc = make_map(&mq, qh, (int)m, kp, TC_BM);
    if (rc) return rc;
    rc = make_map(&mp, ph, (int)n, kp, TC_BN / 2);
    if (rc) return rc;
    const int qblocks = (int)((m + 2 * TC_BM - 1) / (2 * TC_BM)) * 2;  // whole CTA pairs
    const int ntiles = (int)((n + TC_BN - 1) / TC_BN);
    // column splits fill the GPU for small query counts; at most 16 so the rescoring
    // list (nsplit * K' per row) stays within one warp's shared memory budget
    int nsplit = std::max(1, std::min(std::min(ntiles, 16), (2 * sm_count() + qblocks - 1) / qblocks));
    const int per = (ntiles + nsplit - 1) / nsplit;
    nsplit = (ntiles + per - 1) / per;
    TcArgs A;
    A.qn = qn;
    A.pn = pn;
    A.qids = reinterpret_cast<const long long*>(qids);
    A.m = (int)m;
    A.n = (int)n;
    A.kblocks = kp / TC_BK;
    A.tiles_per_split = per;
    A.nsplit = nsplit;
    A.dbg = getenv("PK_TC_DEBUG") ? atoi(getenv("PK_TC_DEBUG")) : 0;
    A.prank = prank;
    A.qrank = qrank;
    PK_CHECK(scratch(&A.out_id, (size_t)m * nsplit * TC_KP, st));
    PK_CHECK(scratch(&A.out_d, (size_t)m * nsplit * TC_KP, st));
    PK_CHECK(cudaFuncSetAttribute(tc_screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM));
    {
        ProfScope _ps("tc_screen_kernel", st);
        tc_screen_kernel<<<dim3((unsigned)qblocks, (unsigned)nsplit), TC_THREADS, TC_SMEM, st>>>(mq, mp, A);
    }
    PK_CHECK_LAUNCH("tc_screen_kernel");
    // rescoring
    float hmax = 0.f;
    PK_CHECK(cudaMemcpyAsync(&hmax, pmax, sizeof(float), cudaMemcpyDeviceToHost, st));
    PK_CHECK(cudaStreamSynchronize(st));
    const int P = next_pow2(nsplit * TC_KP);
    const int wpb = 4;
    const size_t rs_smem = (size_t)wpb * P * 12;
    if (rs_smem > 48 * 1024)
        PK_CHECK(cudaFuncSetAttribute(tc_rescore_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs_smem));
    // |q.p error| <= (2 * 2^-11 + d * 2^-24) |q| |p| for fp16 operands with fp32 accumulation
    const float eps_scale = 2.f * (2.f * ldexpf(1.f, -11) + (float)kp * ldexpf(1.f, -24));
    {
        ProfScope _ps("tc_rescore_kernel", st);
        tc_rescore_kernel<<<(unsigned)std::min<long long>((m + wpb - 1) / wpb, 65535), 32 * wpb, rs_smem, st>>>(
            x, (int)dp, reinterpret_cast<const long long*>(qids), (int)m, nsplit, A.out_id, A.out_d, (int)kk,
            eps_scale, qn, sqrtf(hmax), reinterpret_cast<long long*>(out_ids), out_sqd,
            reinterpret_cast<unsigned long long*>(uncertified), row_flags, P);
    }
    PK_CHECK_LAUNCH("tc_rescore_kernel");
    for (void* p : {(void*)qh, (void*)ph, (void*)qn, (void*)pn, (void*)pmax, (void*)A.out_id, (void*)A.out_d})
        release(p, st);
    (void)iota;
    return 0;
}

__global__ void widen_ids_kernel(const int* in, int m, long long* out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m) out[t] = in[t];
}

namespace pk {
// One warp per row of a screened chunk: hi = v + e, lo = v - e bound the exact
// squared distance (e: the fp16-operand / fp32-accumulation bound of the
// screen, the fp16 subnormal term, fp32 rounding of the norms, and a 1e-5
// relative margin); T = the take-th smallest hi; bit j of the row's mask is set
// unless lo_j > T (such a start is certainly outside the take nearest).  A
// non-finite screen (fp16 overflow) keeps its start a candidate with hi = +inf.
__global__ void seed_mask_kernel(const float* __restrict__ dump, long long ld, int rows, int s, int take,
                                 const float* __restrict__ qn, const float* __restrict__ smax2, float eps, float eabs,
                                 unsigned* __restrict__ mask, int mw, int* __restrict__ near) {
    extern __shared__ unsigned seed_sh[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int spad = (s + 31) & ~31;
    unsigned* hi = seed_sh + (size_t)w * (spad + 256);
    unsigned* bins = hi + spad;
    const float sm2 = *smax2;
    for (int r = blockIdx.x * wpb + w; r < rows; r += gridDim.x * wpb) {
        const float* drow = dump + (size_t)r * ld;
        const float q2 = qn[r];
        const float e = eps * sqrtf(q2) * sqrtf(sm2) + eabs * (sqrtf(q2) + sqrtf(sm2)) + 1e-6f * (q2 + sm2);
        float best = __int_as_float(0x7f800000);
        int bj = 0;
        for (int x = lane; x < s; x += 32) {
            const float v = drow[x];
            const float h = v + e + 1e-5f * fabsf(v);
            hi[x] = isfinite(h) ? __float_as_uint(fmaxf(h, 0.f)) : 0x7f800000u;
            if (v < best) {
                best = v;
                bj = x;
            }
        }
        if (near) {
            // screened nearest start (a locality key for the search order, not a result)
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const float ob = __shfl_xor_sync(PK_FULL, best, o);
                const int oj = __shfl_xor_sync(PK_FULL, bj, o);
                if (ob < best || (ob == best && oj < bj)) {
                    best = ob;
                    bj = oj;
                }
            }
            if (lane == 0) near[r] = bj;
        }
        __syncwarp();
        int need = 0;
        const float T = __uint_as_float(warp_radix_kth(hi, s, take, bins, need));
        for (int b = 0; b < s; b += 32) {
            bool keep = false;
            if (b + lane < s) {
                const float v = drow[b + lane];
                keep = !(v - e - 1e-5f * fabsf(v) > T) || !isfinite(v);
            }
            const unsigned m = __ballot_sync(PK_FULL, keep);
            if (lane == 0) mask[(size_t)r * mw + (b >> 5)] = m;
        }
        __syncwarp();
    }
}

// Tensor-core pre-screen of a build's start set: mask[i * mw + j / 32] bit j
// set iff start j may be among the take nearest starts of point i (exact float64
// squared distances).  The points are screened against the starts in chunks of
// rows on the tcgen05 kernel (fp16 operands, fp32 TMEM accumulation, every
// distance dumped), each chunk reduced to its bits by seed_mask_kernel.  Used by
// beam.cuh seed_select_lazy to skip the fp32 screens of far starts.
// `rows` (optional): the screened points are x[rows[0 .. n)] instead of x[0 .. n)
// (mask and near are indexed by position either way).
int tc_seed_mask(const float* x, int n, int dp, const int* starts, int s, int take, unsigned* mask, int mw,
                 int* near, cudaStream_t st, const long long* rows_ids) {
    if (!tc_supported()) {
        set_error("tensor-core screens need an sm_100 device");
        return 2;
    }
    const int kp = (dp + TC_BK - 1) / TC_BK * TC_BK;
    const long long ld = (s + 3) / 4 * 4;
    // equal chunks of <= 256 MB of screens (none much smaller than the others)
    const long long cmax = env_int("PK_SEED_CHUNK", 0) >= 2 * TC_BM ? env_int("PK_SEED_CHUNK", 0)
                                                                      : std::max<long long>(2 * TC_BM, (256ll << 20) / (ld * 4));
    const long long nchunk = (n + cmax - 1) / cmax;
    const int chunk = (int)((n + nchunk - 1) / nchunk);
    __half *qh = nullptr, *ph = nullptr;
    float *pn = nullptr, *qn = nullptr, *smax2 = nullptr, *dump = nullptr;
    long long* sid = nullptr;
    PK_CHECK(scratch(&qh, (size_t)chunk * kp, st));
    PK_CHECK(scratch(&ph, (size_t)s * kp, st));
    PK_CHECK(scratch(&pn, (size_t)s, st));
    PK_CHECK(scratch(&qn, (size_t)chunk, st));
    PK_CHECK(scratch(&smax2, 1, st));
    PK_CHECK(scratch(&sid, (size_t)s, st));
    PK_CHECK(scratch(&dump, (size_t)chunk * ld, st));
    widen_ids_kernel<<<(s + 255) / 256, 256, 0, st>>>(starts, s, sid);
    {
        ProfScope _ps("tc_prep_kernel", st);
        tc_prep_kernel<<<(unsigned)std::min<long long>(((long long)(s) + 7) / 8, 148ll * 32), 256, 0, st>>>(x, dp, sid, s, kp, ph, pn);
    }
    PK_CHECK(cudaMemsetAsync(smax2, 0, sizeof(float), st));
    {
        ProfScope _ps("tc_max_kernel", st);
        tc_max_kernel<<<grid_for(s, 256), 256, 0, st>>>(pn, s, smax2);
    }
    PK_CHECK_LAUNCH("tc_seed_prep");
    CUtensorMap mq, mp;
    int rc = make_map(&mp, ph, s, kp, TC_BN / 2);
    if (rc) return rc;
    PK_CHECK(cudaFuncSetAttribute(tc_screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM));
    // |screen - d| <= eps |x| |start|_max for normal fp16 operands (both roundings,
    // kp fp32 accumulations, factor 2 of the cross term); subnormal fp16 operands
    // add <= 2^-24 sqrt(kp) (|x| + |start|_max), taken twice
    const float eps = 2.f * (2.f * ldexpf(1.f, -11) + (float)kp * ldexpf(1.f, -24));
    const float eabs = 2.f * sqrtf((float)kp) * ldexpf(1.f, -24);
    constexpr int kMaskWarps = 8;
    const size_t msmem = (size_t)kMaskWarps * (((s + 31) & ~31) + 256) * sizeof(unsigned);
    PK_CHECK(cudaFuncSetAttribute(seed_mask_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem));
    int per_sm = 0;
    PK_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, seed_mask_kernel, kMaskWarps * 32, msmem));
    for (int r0 = 0; r0 < n; r0 += chunk) {
        const int rows = std::min(chunk, n - r0);
        {
            ProfScope _ps("tc_prep_kernel", st);
            tc_prep_kernel<<<(unsigned)std::min<long long>(((long long)(rows) + 7) / 8, 148ll * 32), 256, 0, st>>>(rows_ids ? x : x + (size_t)r0 * dp, dp, rows_ids ? rows_ids + r0 : nullptr, rows, kp, qh, qn);
        }
        if ((rc = make_map(&mq, qh, rows, kp, TC_BM))) return rc;
        TcArgs A;
        A.qn = qn;
        A.pn = pn;
        A.qids = nullptr;
        A.m = rows;
        A.n = s;
        A.kblocks = kp / TC_BK;
        A.tiles_per_split = (s + TC_BN - 1) / TC_BN;
        A.nsplit = 1;
        A.dbg = 0;
        A.prank = nullptr;
        A.qrank = nullptr;
        A.out_id = nullptr;
        A.out_d = nullptr;
        A.dump = dump;
        A.dump_ld = ld;
        {
            ProfScope _ps("tc_seed_screen_kernel", st);
            const int qblocks = (rows + 2 * TC_BM - 1) / (2 * TC_BM) * 2;
            tc_screen_kernel<<<dim3((unsigned)qblocks, 1u), TC_THREADS, TC_SMEM, st>>>(mq, mp, A);
        }
        PK_CHECK_LAUNCH("tc_seed_screen_kernel");
        {
            ProfScope _ps("seed_mask_kernel", st);
            const int grid = std::min(sm_count() * std::max(1, per_sm), (rows + kMaskWarps - 1) / kMaskWarps);
            seed_mask_kernel<<<grid, kMaskWarps * 32, msmem, st>>>(dump, ld, rows, s, take, qn, smax2, eps, eabs,
                                                                   mask + (size_t)r0 * mw, mw,
                                                                   near ? near + r0 : nullptr);
        }
        PK_CHECK_LAUNCH("seed_mask_kernel");
    }
    for (void* p : {(void*)qh, (void*)ph, (void*)pn, (void*)qn, (void*)smax2, (void*)sid, (void*)dump}) release(p, st);
    return 0;
}

long long tc_count_stats[2] = {0, 0};  // rows screened / rows sent to the exact count

// Per row: the decision count < kk from the tensor-core bounds where they settle
// it (cnt = the bound), else the row is flagged for the exact count.
__global__ void count_decide_kernel(const unsigned* lo, const unsigned* hi, int m, long long kk, long long* cnt,
                                    unsigned char* flag) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const bool below = (long long)hi[t] < kk, above = (long long)lo[t] >= kk;
    cnt[t] = below ? (long long)hi[t] : (long long)lo[t];
    flag[t] = !(below || above);
}

__global__ void iota64_kernel(long long* out, int m) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m) out[t] = t;
}

__global__ void gather_rows_kernel(const long long* rows, const long long* nrows, const long long* qids,
                                   const double* key_d, const long long* key_i, long long* sq, double* sd,
                                   long long* si) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= *nrows) return;
    const long long r = rows[t];
    sq[t] = qids[r];
    sd[t] = key_d[r];
    si[t] = key_i[r];
}

__global__ void scatter_counts_kernel(const long long* rows, const long long* nrows, const long long* sc,
                                      long long* cnt) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t < *nrows) cnt[rows[t]] = sc[t];
}

int compact_flagged(const long long* in, const unsigned char* flags, long long n, long long* out, long long* count,
                    cudaStream_t st);

// count[r] such that (count[r] < kk) == (#{j != qids[r] : (d(q, j), j) < (key_d[r],
// key_i[r])} < kk), the count itself exact whenever the tensor-core bounds leave
// the decision open: member rows screened against all points on tcgen05 (fp16
// operands, fp32 accumulators, counting epilogue), undecided rows counted by
// `exact_count(rows, m', keys...)` (the scan kernels).  Used by the doubling
// rounds' short-row resolution (scan.cu pk_resolve_short_scanned) on float data.
int tc_count_decide(const float* x, int n, int dp, const long long* qids, int m, const double* key_d,
                    const long long* key_i, long long kk, long long* cnt,
                    int (*exact_count)(const long long*, int, const double*, const long long*, long long*, void*),
                    void* ctx, cudaStream_t st) {
    if (!tc_supported()) {
        set_error("tensor-core screens need an sm_100 device");
        return 2;
    }
    const int kp = (dp + TC_BK - 1) / TC_BK * TC_BK;
    __half *qh = nullptr, *ph = nullptr;
    float *qn = nullptr, *pn = nullptr, *pmax2 = nullptr;
    unsigned *lo = nullptr, *hi = nullptr;
    PK_CHECK(scratch(&qh, (size_t)m * kp, st));
    PK_CHECK(scratch(&ph, (size_t)n * kp, st));
    PK_CHECK(scratch(&qn, (size_t)m, st));
    PK_CHECK(scratch(&pn, (size_t)n, st));
    PK_CHECK(scratch(&pmax2, 1, st));
    PK_CHECK(scratch(&lo, (size_t)m, st));
    PK_CHECK(scratch(&hi, (size_t)m, st));
    {
        ProfScope _ps("tc_prep_kernel", st);
        tc_prep_kernel<<<(unsigned)std::min<long long>(((long long)(m) + 7) / 8, 148ll * 32), 256, 0, st>>>(x, dp, qids, m, kp, qh, qn);
        tc_prep_kernel<<<(unsigned)std::min<long long>(((long long)(n) + 7) / 8, 148ll * 32), 256, 0, st>>>(x, dp, nullptr, n, kp, ph, pn);
    }
    PK_CHECK(cudaMemsetAsync(pmax2, 0, sizeof(float), st));
    PK_CHECK(cudaMemsetAsync(lo, 0, sizeof(unsigned) * (size_t)m, st));
    PK_CHECK(cudaMemsetAsync(hi, 0, sizeof(unsigned) * (size_t)m, st));
    {
        ProfScope _ps("tc_max_kernel", st);
        tc_max_kernel<<<grid_for(n, 256), 256, 0, st>>>(pn, n, pmax2);
    }
    PK_CHECK_LAUNCH("tc_count_prep");
    CUtensorMap mq, mp;
    int rc = make_map(&mq, qh, m, kp, TC_BM);
    if (rc) return rc;
    if ((rc = make_map(&mp, ph, n, kp, TC_BN / 2))) return rc;
    const int qblocks = (m + 2 * TC_BM - 1) / (2 * TC_BM) * 2;
    const int ntiles = (n + TC_BN - 1) / TC_BN;
    int nsplit = std::max(1, std::min(ntiles, (2 * sm_count() + qblocks - 1) / qblocks));
    const int per = (ntiles + nsplit - 1) / nsplit;
    nsplit = (ntiles + per - 1) / per;
    TcArgs A;
    A.qn = qn;
    A.pn = pn;
    A.qids = qids;
    A.m = m;
    A.n = n;
    A.kblocks = kp / TC_BK;
    A.tiles_per_split = per;
    A.nsplit = nsplit;
    A.dbg = 0;
    A.prank = nullptr;
    A.qrank = nullptr;
    A.out_id = nullptr;
    A.out_d = nullptr;
    A.cnt_key = key_d;
    A.cnt_kid = key_i;
    A.cnt_lo = lo;
    A.cnt_hi = hi;
    A.pmax2 = pmax2;
    A.cnt_eps = 2.f * (2.f * ldexpf(1.f, -11) + (float)kp * ldexpf(1.f, -24));
    A.cnt_abs = 2.f * sqrtf((float)kp) * ldexpf(1.f, -24);
    PK_CHECK(cudaFuncSetAttribute(tc_screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM));
    {
        ProfScope _ps("tc_count_screen_kernel", st);
        tc_screen_kernel<<<dim3((unsigned)qblocks, (unsigned)nsplit), TC_THREADS, TC_SMEM, st>>>(mq, mp, A);
    }
    PK_CHECK_LAUNCH("tc_count_screen_kernel");
    for (void* p : {(void*)qh, (void*)ph, (void*)qn, (void*)pn, (void*)pmax2}) release(p, st);
    unsigned char* flag = nullptr;
    long long *rows = nullptr, *nrows = nullptr, *iota = nullptr;
    PK_CHECK(scratch(&flag, (size_t)m, st));
    PK_CHECK(scratch(&rows, (size_t)m, st));
    PK_CHECK(scratch(&nrows, 1, st));
    PK_CHECK(scratch(&iota, (size_t)m, st));
    count_decide_kernel<<<(m + 255) / 256, 256, 0, st>>>(lo, hi, m, kk, cnt, flag);
    iota64_kernel<<<(m + 255) / 256, 256, 0, st>>>(iota, m);
    PK_CHECK_LAUNCH("count_decide_kernel");
    if ((rc = compact_flagged(iota, flag, m, rows, nrows, st))) return rc;
    long long nb = 0;
    PK_CHECK(cudaMemcpyAsync(&nb, nrows, sizeof(long long), cudaMemcpyDeviceToHost, st));
    PK_CHECK(cudaStreamSynchronize(st));
    if (nb > 0) {
        long long *sq = nullptr, *si = nullptr, *sc = nullptr;
        double* sd = nullptr;
        PK_CHECK(scratch(&sq, (size_t)nb, st));
        PK_CHECK(scratch(&si, (size_t)nb, st));
        PK_CHECK(scratch(&sd, (size_t)nb, st));
        PK_CHECK(scratch(&sc, (size_t)nb, st));
        gather_rows_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(rows, nrows, qids, key_d, key_i, sq, sd, si);
        PK_CHECK_LAUNCH("gather_rows_kernel");
        if ((rc = exact_count(sq, (int)nb, sd, si, sc, ctx))) return rc;
        scatter_counts_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(rows, nrows, sc, cnt);
        PK_CHECK_LAUNCH("scatter_counts_kernel");
        for (void* p : {(void*)sq, (void*)si, (void*)sd, (void*)sc}) release(p, st);
    }
    tc_count_stats[0] += m;
    tc_count_stats[1] += nb;
    for (void* p : {(void*)lo, (void*)hi, (void*)flag, (void*)rows, (void*)nrows, (void*)iota}) release(p, st);
    return 0;
}
}  // namespace pk

extern "C" int pk_brute_knn_tc(const float* x, int64_t n, int64_t dp, const int64_t* qids, int64_t m, int64_t k,
                               int64_t* out_ids, double* out_sqd, uint8_t* row_flags, uint64_t* uncertified,
                               void* stream) {
    const int64_t kk = k < n - 1 ? k : n - 1;
    return tc_knn_core(x, n, dp, qids, m, kk, nullptr, nullptr, out_ids, out_sqd, row_flags, uncertified,
                       as_stream(stream));
}

__global__ void rank32_kernel(const long long* rank, long long n, const long long* qids, long long m, int* prank,
                              int* qrank) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n + m; i += (long long)gridDim.x * blockDim.x) {
        if (i < n) prank[i] = (int)rank[i];
        else qrank[i - n] = (int)rank[qids[i - n]];
    }
}

extern "C" int pk_dp_scan_tc(const float* x, int64_t n, int64_t dp, const int64_t* rank, const int64_t* qids, int64_t m,
                             int64_t* out_id, double* out_sqd, uint8_t* row_flags, uint64_t* uncertified, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (m <= 0) return 0;
    if (n >= (1ll << 31)) {
        set_error("tensor-core dp scan needs n < 2^31");
        return 2;
    }
    int *prank = nullptr, *qrank = nullptr;
    PK_CHECK(scratch(&prank, (size_t)n, st));
    PK_CHECK(scratch(&qrank, (size_t)m, st));
    {
        ProfScope _ps("rank32_kernel", st);
        rank32_kernel<<<grid_for(n + m, 256), 256, 0, st>>>(reinterpret_cast<const long long*>(rank), n,
                                                            reinterpret_cast<const long long*>(qids), m, prank, qrank);
    }
    PK_CHECK_LAUNCH("rank32_kernel");
    const int rc = tc_knn_core(x, n, dp, qids, m, 1, prank, qrank, out_id, out_sqd, row_flags, uncertified, st);
    release(prank, st);
    release(qrank, st);
    return rc;
}

extern "C" int pk_tc_count_stats(int64_t* out2, int reset) {
    out2[0] = tc_count_stats[0];
    out2[1] = tc_count_stats[1];
    if (reset) tc_count_stats[0] = tc_count_stats[1] = 0;
    return 0;
}
