// RobustPrune for float data on the tensor cores (SEQ64 mode, dp <= 1024).
//
// The sequential RobustPrune (_kernels.py:283-315) only ever asks "does pick
// t occlude candidate u": alpha^2 * d(t, u) <= d(p, u), with d(t, u) the
// reference's sequential float64 distance.  For the <= 256 sorted, unique
// candidates of one item the kernel decides every pair t < u up front:
//
//  * the Gram matrix G = C C^T of the candidate rows is one tcgen05 GEMM
//    (kind::tf32, fp32 accumulators in TMEM): the rows stream through shared
//    memory in 32-float K chunks (cp.async gathers into the 128-byte-swizzled
//    K-major layout, 4 stages), tile 0 = rows 0-127 x columns 0-255 (TMEM
//    columns 0-255), tile 1 = rows 128-255 x columns 128-255 (columns 256-383);
//  * the epilogue (thread = TMEM lane = candidate row) forms
//    d~ = |t|^2 + |u|^2 - 2 G~ (float64 norms precomputed once per build) and a
//    rigorous bound E = 2 eg |t||u| + 1e-12 (|t|^2 + |u|^2) with
//    eg = 2^-9 + (dp + 8) 2^-23 (tf32 inputs keep >= 10 mantissa bits; fp32
//    accumulation), then sets the occlusion bit where alpha^2 (d~ + E) <= d(p,u)
//    and an "uncertain" bit where neither that nor alpha^2 (d~ - E) > d(p,u)
//    holds;
//  * the greedy picks (warp 0) are bit arithmetic; an uncertain pair (t, u)
//    whose t is picked while u is alive is decided exactly (fp32 screen with its
//    guard band, the reference's float64 sequential value where that cannot
//    call it) -- the picks are identical to the sequential algorithm.
//
// Each candidate row is read once per item (instead of once per pick), which
// is what bounded the warp-per-item kill passes (HBM re-reads).
//
// Textually included by build.cu inside namespace pk, after the definitions it
// uses (BuildArgs, RevArgs, BPSmem, bp_sort, bp_unique, prune_by_selection).
#pragma once

constexpr int PT_CAP = 256;
constexpr int PT_THREADS = 128;
constexpr int PT_STAGES = 4;
constexpr int PT_STAGE_BYTES = PT_CAP * 128;  // 256 rows x 32 fp32
constexpr size_t PT_SMEM = 1024 + (size_t)PT_STAGES * PT_STAGE_BYTES  // K-chunk stages
                           + (size_t)PT_CAP * 8 * 4                    // kd, kd2, nrm, sq (f64)
                           + (size_t)PT_CAP * 4 * 2                    // ki, ki2
                           + (size_t)PT_CAP * 8 * 4 * 2                // kill, unc bit rows
                           + 256;                                      // barriers, scalars

struct PTSmem {
    unsigned char* stage;  // [PT_STAGES][PT_CAP][128 B], 1024-aligned
    double* nrm;           // [PT_CAP] |x|^2 of the sorted candidates
    double* sq;            // [PT_CAP] |x|
    unsigned* kill;        // [PT_CAP][8]
    unsigned* unc;         // [PT_CAP][8]
    unsigned long long* bar;  // [PT_STAGES] MMAs of the stage's chunk done
    unsigned* tmem_slot;
    BPSmem S;              // kd, ki, kd2, ki2, scal (bp_sort / bp_unique)
};

__device__ __forceinline__ PTSmem carve_pt(unsigned char* raw) {
    PTSmem P;
    unsigned char* base = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    P.stage = base;
    unsigned char* q = base + (size_t)PT_STAGES * PT_STAGE_BYTES;
    P.S.kd = reinterpret_cast<double*>(q);
    P.S.kd2 = P.S.kd + PT_CAP;
    P.nrm = P.S.kd2 + PT_CAP;
    P.sq = P.nrm + PT_CAP;
    P.S.ki = reinterpret_cast<unsigned*>(P.sq + PT_CAP);
    P.S.ki2 = P.S.ki + PT_CAP;
    P.kill = P.S.ki2 + PT_CAP;
    P.unc = P.kill + PT_CAP * 8;
    P.bar = reinterpret_cast<unsigned long long*>(P.unc + PT_CAP * 8);
    P.tmem_slot = reinterpret_cast<unsigned*>(P.bar + PT_STAGES + 1);
    P.S.scal = reinterpret_cast<int*>(P.tmem_slot + 2);
    P.S.rows = nullptr;
    P.S.nrm = nullptr;
    P.S.kill = nullptr;
    return P;
}

__device__ __forceinline__ void tc_mma_tf32(unsigned tmem_d, unsigned long long da, unsigned long long db,
                                            unsigned idesc, unsigned accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld16(unsigned taddr, float (&v)[16]) {
    unsigned r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// per-CTA pipeline state (identical in every thread)
struct PTPipe {
    unsigned tmem;
    unsigned phase;  // bit s: parity of the next completion of bar[s]
};

// float64 |x|^2 of every point (warp per row), for the Gram epilogue
__global__ void norms64_kernel(const float* __restrict__ X, long long n, int dp, double* __restrict__ out) {
    const int lane = lane_id();
    const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = w; r < n; r += nw) {
        const float4* row = reinterpret_cast<const float4*>(X + (size_t)r * dp);
        double acc = 0.0;
        for (int f = lane; f < (dp >> 2); f += 32) {
            const float4 v = __ldg(row + f);
            acc = fma((double)v.x, (double)v.x, acc);
            acc = fma((double)v.y, (double)v.y, acc);
            acc = fma((double)v.z, (double)v.z, acc);
            acc = fma((double)v.w, (double)v.w, acc);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(PK_FULL, acc, o);
        if (lane == 0) out[r] = acc;
    }
}

// Copy K chunk kc (floats 32 kc .. 32 kc + 31) of the c sorted candidates into
// stage buffer `st`: row r at r * 128 bytes, 16-byte piece j at (j ^ (r & 7)).
__device__ __forceinline__ void pt_stage_chunk(const float* __restrict__ X, int dp, const unsigned* ki2, int c, int kc,
                                               unsigned char* st) {
    for (int e = threadIdx.x; e < c * 8; e += PT_THREADS) {
        const int r = e >> 3, j = e & 7;
        const int col = kc * 32 + j * 4;
        unsigned char* dst = st + r * 128 + ((j ^ (r & 7)) << 4);
        if (col < dp) {
            const float* src = X + (size_t)ki2[r] * dp + col;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
        } else {
            *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// Gram matrix of the c (<= 256) sorted candidates into TMEM (tile 0 at column
// 0, tile 1 at column 256), then the occlusion / uncertain bit rows.
template <int QV>
__device__ void pt_gram_bits(const float* __restrict__ X, int dp, const PTSmem& P, PTPipe& pp, int c, double alpha2) {
    const int tid = threadIdx.x;
    const int nk = (dp + 31) >> 5;
    const int n0 = min(256, (c + 15) & ~15);
    const bool two = c > 128;
    const int n1 = two ? ((c - 128 + 15) & ~15) : 0;
    const unsigned id0 = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(n0 >> 3) << 17) | ((128u >> 4) << 24);
    const unsigned id1 = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(n1 >> 3) << 17) | ((128u >> 4) << 24);
    // prologue: chunks 0 .. PT_STAGES - 2
    for (int k = 0; k < PT_STAGES - 1; ++k) {
        if (k < nk) pt_stage_chunk(X, dp, P.S.ki2, c, k, P.stage + (size_t)k * PT_STAGE_BYTES);
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    for (int kc = 0; kc < nk; ++kc) {
        // refill the stage the MMAs of chunk kc - 1 read (wait for them first)
        const int kn = kc + PT_STAGES - 1;
        const int sn = kn % PT_STAGES;
        if (kc >= 1) {
            mbar_wait(P.bar + sn, (pp.phase >> sn) & 1u);
            pp.phase ^= 1u << sn;
        }
        if (kn < nk) pt_stage_chunk(X, dp, P.S.ki2, c, kn, P.stage + (size_t)sn * PT_STAGE_BYTES);
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group %0;\n" ::"n"(PT_STAGES - 1) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const int s = kc % PT_STAGES;
            unsigned char* sb = P.stage + (size_t)s * PT_STAGE_BYTES;
            const unsigned long long d0 = umma_desc_sw128(sb);
            const unsigned long long d1 = umma_desc_sw128(sb + 128 * 128);
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 8 tf32 = 32 bytes per UMMA_K step
                tc_mma_tf32(pp.tmem, d0 + 2ull * k, d0 + 2ull * k, id0, (kc | k) != 0);
                if (two) tc_mma_tf32(pp.tmem + 256u, d1 + 2ull * k, d1 + 2ull * k, id1, (kc | k) != 0);
            }
            tc_commit(P.bar + s);
        }
    }
    // the last chunk's commit tracks every MMA of the item
    {
        const int s = (nk - 1) % PT_STAGES;
        mbar_wait(P.bar + s, (pp.phase >> s) & 1u);
        pp.phase ^= 1u << s;
    }
    tc_fence_after();

    // epilogue: thread tid = TMEM lane; tile 0 row t = tid, tile 1 row t = 128 + tid
    const int warp = tid >> 5;
    const double eg = 0.001953125 + (double)(dp + 8) * 1.1920928955078125e-07;
    for (int tile = 0; tile < (two ? 2 : 1); ++tile) {
        const int t = tile * 128 + tid;
        const int cbase = tile * 128;                  // first candidate column of the tile
        const int ncol = tile ? n1 : n0;
        const unsigned tbase = pp.tmem + ((unsigned)(warp * 32) << 16) + (tile ? 256u : 0u);
        const bool live = t < c;
        const double nt = live ? P.nrm[t] : 0.0, st = live ? P.sq[t] : 0.0;
        // columns below this warp's first row hold only pairs u <= t: skip whole words
        const int w0 = (cbase + 32 * warp - cbase) >> 5;  // word offset inside the tile
        for (int wd = w0; wd * 32 < ncol; ++wd) {
            unsigned kb = 0u, ub = 0u;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = wd * 32 + h * 16;
                if (col >= ncol) break;
                float g[16];
                tmem_ld16(tbase + (unsigned)col, g);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int u = cbase + col + i;
                    if (live && u > t && u < c) {
                        const double dt = nt + P.nrm[u] - 2.0 * (double)g[i];
                        const double E = 2.0 * eg * st * P.sq[u] + 1e-12 * (nt + P.nrm[u]);
                        const double K = P.S.kd2[u];
                        const double hi = alpha2 * (dt + E) * (1.0 + 1e-12);
                        const double lo = alpha2 * (dt - E) * (1.0 - 1e-12);
                        const unsigned bit = 1u << (h * 16 + i);
                        if (hi <= K) kb |= bit;
                        else if (!(lo > K)) ub |= bit;
                    }
                }
            }
            if (live) {
                const int word = (cbase >> 5) + wd;
                P.kill[t * 8 + word] = kb;
                P.unc[t * 8 + word] = ub;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
}

// Greedy picks over the bit rows (warp 0); uncertain pairs of a picked t are
// decided exactly.  Returns sel (picks written to out[0, sel)).
template <int QV>
__device__ int pt_greedy(const float* __restrict__ X, int dp, const PTSmem& P, int c, double alpha2, int R, int* out,
                         long long* exact_pairs) {
    const int lane = lane_id();
    const int nw = (c + 31) >> 5;
    // lane l < nw holds alive word l
    unsigned alive = 0u;
    if (lane < nw) alive = (c - 32 * lane >= 32) ? 0xffffffffu : ((1u << (c - 32 * lane)) - 1u);
    int sel = 0;
    long long nex = 0;
    while (sel < R) {
        const unsigned nz = __ballot_sync(PK_FULL, alive != 0u);
        if (!nz) break;
        const int wl = __ffs(nz) - 1;
        const int t = 32 * wl + __ffs(__shfl_sync(PK_FULL, alive, wl)) - 1;
        if (lane == wl) alive &= ~(1u << (t & 31));
        const unsigned tid_t = P.S.ki2[t];
        if (lane == 0) out[sel] = (int)tid_t;
        ++sel;
        if (sel >= R) break;
        unsigned kill = lane < nw ? P.kill[t * 8 + lane] : 0u;
        unsigned unc = lane < nw ? (P.unc[t * 8 + lane] & alive) : 0u;
        if (__any_sync(PK_FULL, unc != 0u)) {
            Fp32Pick<QV> pick;
            pick.load(X, dp, tid_t);
            const Seq64Member dx{X + (size_t)tid_t * dp, dp};
            for (int w = 0; w < nw; ++w) {
                unsigned b = __shfl_sync(PK_FULL, unc, w);
                unsigned kw = 0u;
                while (b) {
                    const int j = __ffs(b) - 1;
                    b &= b - 1;
                    const int u = 32 * w + j;
                    const unsigned uid = P.S.ki2[u];
                    const float s = Fp32Pick<QV>::reduce(pick.partial(X, dp, uid));
                    int v = screen_le(alpha2, s, P.S.kd2[u]);
                    if (v == 2) {
                        double duv = 0.0;
                        if (lane == 0) duv = dx.eval_one(X, (int)uid);
                        duv = __shfl_sync(PK_FULL, duv, 0);
                        v = alpha2 * duv <= P.S.kd2[u] ? 1 : 0;
                    }
                    if (v == 1) kw |= 1u << j;
                    ++nex;
                }
                if (lane == w) kill |= kw;
            }
        }
        alive &= ~kill;
    }
    if (lane == 0 && exact_pairs) *exact_pairs += nex;
    return sel;
}

// one item: sorted unique candidates in P.S.kd2/ki2 (c > R) -> picks
template <int QV>
__device__ int pt_prune(const float* __restrict__ X, int dp, const double* __restrict__ nrm64, const PTSmem& P,
                        PTPipe& pp, int c, double alpha2, int R, int* out, long long* exact_pairs) {
    for (int x = threadIdx.x; x < c; x += PT_THREADS) {
        const double v = nrm64[P.S.ki2[x]];
        P.nrm[x] = v;
        P.sq[x] = sqrt(v);
    }
    __syncthreads();
    pt_gram_bits<QV>(X, dp, P, pp, c, alpha2);
    if ((threadIdx.x >> 5) == 0) {
        const int sel = pt_greedy<QV>(X, dp, P, c, alpha2, R, out, exact_pairs);
        if (lane_id() == 0) P.S.scal[8] = sel;
    }
    __syncthreads();
    return P.S.scal[8];
}

__device__ __forceinline__ void pt_setup(const PTSmem& P, PTPipe& pp) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < PT_STAGES; ++s) mbar_init(P.bar + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(P.tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pp.tmem = *P.tmem_slot;
    pp.phase = 0u;
}

__device__ __forceinline__ void pt_teardown(const PTSmem& P, const PTPipe& pp) {
    tc_fence_before();
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(pp.tmem), "r"(512));
    }
}

// build phase 2 for float data: one block per inserted point (items with more
// than PT_CAP candidates are queued for build_prune_kernel)
template <int QV>
__global__ void __launch_bounds__(PT_THREADS, 1) prune_tc_build_kernel(BuildArgs A, const double* __restrict__ nrm64,
                                                                      int* over, int* nover) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const PTSmem P = carve_pt(smem_raw);
    PTPipe pp;
    pt_setup(P, pp);
    const int tid = threadIdx.x;
    const int R = A.P.R;
    const int dp = A.D.dp;
    const float* X = A.D.X;
    long long pairs = 0, exact_pairs = 0;
    for (int t = blockIdx.x; t < A.m; t += gridDim.x) {
        const unsigned p = (unsigned)A.bids[t];
        const int vl = A.vlen[t];
        const int nd = __ldg(A.P.deg + p);
        const int c0 = vl + nd;
        if (c0 > PT_CAP) {
            if (tid == 0) over[atomicAdd(nover, 1)] = t;
            continue;
        }
        const unsigned* vi = A.vlog_i + (size_t)t * A.vcap;
        const double* vd = A.vlog_d + (size_t)t * A.vcap;
        const int* row = A.P.adj + (size_t)p * R;
        const Seq64Member dq{X + (size_t)p * dp, dp};
        for (int x = tid; x < c0; x += PT_THREADS) {
            if (x < vl) {
                P.S.kd[x] = vd[x];
                P.S.ki[x] = vi[x];
            } else {
                const unsigned id = (unsigned)__ldg(row + x - vl);
                P.S.ki[x] = id;
                P.S.kd[x] = dq.eval_one(X, (int)id);
            }
        }
        const int Pw = next_pow2_dev(c0 < 2 ? 2 : c0);
        for (int x = c0 + tid; x < Pw; x += PT_THREADS) {
            P.S.kd[x] = __longlong_as_double(0x7ff0000000000000LL);
            P.S.ki[x] = 0xffffffffu;
        }
        __syncthreads();
        bp_sort(P.S.kd, P.S.ki, Pw);
        const int c = bp_unique(P.S, c0, p);
        int* out = A.new_ids + (size_t)t * R;
        // the build always prunes (_kernels.py:370), even c <= R candidates
        int sel = c;
        if (c <= 1) {
            if (tid == 0 && c == 1) out[0] = (int)P.S.ki2[0];
        } else {
            sel = pt_prune<QV>(X, dp, nrm64, P, pp, c, A.alpha2, R, out, &exact_pairs);
            if (tid == 0) pairs += (long long)c * (c - 1) / 2;
        }
        for (int x = sel + tid; x < R; x += PT_THREADS) out[x] = -1;
        if (tid == 0) A.new_len[t] = sel;
        __syncthreads();
    }
    if (tid == 0 && A.stats && pairs)
        atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 1), (unsigned long long)(pairs + exact_pairs));
    pt_teardown(P, pp);
}

// reverse-edge re-prune for float data: one block per target vertex with at most
// PT_CAP candidates (larger groups: reverse_big_kernel / the selection path)
template <int MODE, int QV>
__global__ void __launch_bounds__(PT_THREADS, 1) prune_tc_reverse_kernel(RevArgs A, const double* __restrict__ nrm64) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const PTSmem P = carve_pt(smem_raw);
    PTPipe pp;
    pt_setup(P, pp);
    const int tid = threadIdx.x, wid = tid >> 5;
    const MakeAt<MODE, QV> make{A.D};
    const int dp = A.dp;
    const float* X = A.X;
    const int nt = *A.ntargets;
    long long ev = 0;
    for (int s = blockIdx.x; s < nt; s += gridDim.x) {
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
        if (c0 > PT_CAP) {
            if (c0 <= A.capB) {
                if (tid == 0) A.biglist[atomicAdd(A.nbig, 1)] = s;
                continue;
            }
            if (wid == 0) {
                sel = prune_by_selection(A, u, make, P.S.kd, P.S.ki, reinterpret_cast<unsigned char*>(P.kill),
                                         P.unc, nd, off, size, row, &ev);
                if (lane_id() == 0) P.S.scal[9] = sel;
            }
            __syncthreads();
            sel = P.S.scal[9];
        } else {
            const Seq64Member du{X + (size_t)u * dp, dp};
            for (int x = tid; x < c0; x += PT_THREADS) {
                const unsigned id = x < nd ? (unsigned)row[x] : (unsigned)A.adds[off + x - nd];
                P.S.ki[x] = id;
                P.S.kd[x] = du.eval_one(X, (int)id);
            }
            const int Pw = next_pow2_dev(c0 < 2 ? 2 : c0);
            for (int x = c0 + tid; x < Pw; x += PT_THREADS) {
                P.S.kd[x] = __longlong_as_double(0x7ff0000000000000LL);
                P.S.ki[x] = 0xffffffffu;
            }
            __syncthreads();
            bp_sort(P.S.kd, P.S.ki, Pw);
            const int c = bp_unique(P.S, c0, u);
            if (tid == 0) ev += c0;
            if (c <= A.R) {
                for (int x = tid; x < c; x += PT_THREADS) row[x] = (int)P.S.ki2[x];
                sel = c;
            } else {
                long long ex = 0;
                sel = pt_prune<QV>(X, dp, nrm64, P, pp, c, A.alpha2, A.R, row, &ex);
                if (tid == 0) ev += ex;
            }
        }
        for (int x = sel + tid; x < A.R; x += PT_THREADS) row[x] = -1;
        if (tid == 0) {
            A.deg[u] = sel;
            A.cnt[u] = 0;
        }
        __syncthreads();
    }
    if (tid == 0 && A.stats && ev) atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 2), (unsigned long long)ev);
    pt_teardown(P, pp);
}

