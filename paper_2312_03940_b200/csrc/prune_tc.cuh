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
//    K-major layout, 2 stages), pass 0 = rows 0-127 x columns 0-255, pass 1 =
//    rows 128-255 x columns 128-255, each into the CTA's 256 TMEM columns (two
//    CTAs per SM, so one item's staging overlaps the other's sort / greedy);
//  * the epilogue (thread = TMEM lane = candidate row) forms
//    d~ = |t|^2 + |u|^2 - 2 G~ (float64 norms precomputed once per build) and a
//    rigorous bound E = 2 (eg |t||u| + ea (|t| + |u| + 1)) + 1e-12 (|t|^2 + |u|^2)
//    with eg = 2^-9 + (dp + 8) 2^-23 (tf32 inputs keep >= 10 mantissa bits;
//    fp32 accumulation) and ea = (dp + 8) 2^-126 (subnormals flushed to zero);
//    a non-finite accumulator (overflow) is always "uncertain"; then sets the
//    occlusion bit where alpha^2 (d~ + E) <= d(p,u)
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

// Phase timers of the tensor-core prune (diagnostics build only, -DPK_PHASE_TIMERS):
// clock64 cycles of thread 0 per phase summed over blocks into pk_prune_cycles[]
// -- 0 candidates + sort + unique, 1 norms / row pointers, 2 Gram staging + MMAs,
// 3 epilogue (bit rows), 4 greedy picks, 5 output; [6] = exact pair decisions,
// [7] = items.  Read by pk_phase_timers_prune.
#ifdef PK_PHASE_TIMERS
static __device__ unsigned long long pk_prune_cycles[8];
#define PT_T0 pp.t0 = clock64();
#define PT_TICK(ph)                                                                                        \
    do {                                                                                                   \
        if (threadIdx.x == 0 && pp.t0 >= 0) {                                                              \
            const long long _n = clock64();                                                                \
            atomicAdd(&pk_prune_cycles[ph], (unsigned long long)(_n - pp.t0));                             \
            pp.t0 = _n;                                                                                   \
        }                                                                                                  \
    } while (0)
#define PT_COUNT(slot, v)                                                               \
    do {                                                                                \
        if (threadIdx.x == 0 && pp.t0 >= 0) atomicAdd(&pk_prune_cycles[slot], (unsigned long long)(v)); \
    } while (0)
#else
#define PT_T0
#define PT_TICK(ph) do { } while (0)
#define PT_COUNT(slot, v) do { } while (0)
#endif

constexpr int PT_CAP = 512;   // candidates per item, two-CTA-per-SM kernels (bit rows in 128-row blocks)
constexpr int PT_CAP_BIG = 1024;  // reverse groups of 513..1024 candidates: one CTA per SM
constexpr int PT_THREADS = 128;
constexpr int PT_STAGES = 2;  // two CTAs per SM (TMEM 2 x 256 columns, smem 2 x ~100 KB)
constexpr int PT_STAGE_BYTES = 256 * 128;  // 256 row slots x 32 fp32
// shared memory of a kernel with room for `cap` candidates
__host__ __device__ constexpr size_t pt_smem_bytes(int cap) {
    return 1024 + (size_t)PT_STAGES * PT_STAGE_BYTES  // K-chunk stages
           + (size_t)cap * 8 * 4                      // kd, kd2, nrm, sq (f64)
           + (size_t)cap * 4 * 2                      // ki, ki2
           + (size_t)128 * (cap / 32) * 4 * 2         // kill, unc bit rows (one 128-row block)
           + (size_t)cap * 8                          // row pointers
           + 256;                                     // barriers, scalars
}
constexpr size_t PT_SMEM = pt_smem_bytes(PT_CAP);

struct PTSmem {
    unsigned char* stage;  // [PT_STAGES][256][128 B], 1024-aligned
    double* nrm;           // [PT_CAP] |x|^2 of the sorted candidates
    double* sq;            // [PT_CAP] |x|
    unsigned* kill;        // [128][words] bit rows of the current 128-candidate block
    unsigned* unc;         // [128][words]
    int words;             // bit words per row (cap / 32)
    unsigned long long* rowp;  // [PT_CAP] global address of each sorted candidate row
    // fp32 operands of the epilogue's first-pass decision (pt_gram_pass), in the
    // space of S.ki / S.kd, which are dead between pt_unique and the next item:
    float* su32;               // [cap] |u| rounded up
    float2* ab32;              // [cap] (A_u rounded down, B_u rounded up); NaN = out of the fp32 range
    unsigned long long* bar;  // [PT_STAGES] MMAs of the stage's chunk done
    unsigned* tmem_slot;
    BPSmem S;              // kd, ki, kd2, ki2, scal (bp_sort / bp_unique)
};

template <int CAP>
__device__ __forceinline__ PTSmem carve_pt(unsigned char* raw) {
    constexpr int PT_SORT = CAP, PT_WORDS = CAP / 32;
    PTSmem P;
    P.words = PT_WORDS;
    unsigned char* base = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    P.stage = base;
    unsigned char* q = base + (size_t)PT_STAGES * PT_STAGE_BYTES;
    P.S.kd = reinterpret_cast<double*>(q);
    P.S.kd2 = P.S.kd + PT_SORT;
    P.nrm = P.S.kd2 + PT_SORT;
    P.sq = P.nrm + CAP;
    P.S.ki = reinterpret_cast<unsigned*>(P.sq + CAP);
    P.S.ki2 = P.S.ki + PT_SORT;
    P.kill = P.S.ki2 + PT_SORT;
    P.unc = P.kill + 128 * PT_WORDS;
    P.rowp = reinterpret_cast<unsigned long long*>(P.unc + 128 * PT_WORDS);
    P.bar = P.rowp + CAP;
    P.tmem_slot = reinterpret_cast<unsigned*>(P.bar + PT_STAGES + 1);
    P.S.scal = reinterpret_cast<int*>(P.tmem_slot + 2);
    P.S.rows = nullptr;
    P.S.nrm = nullptr;
    P.S.kill = nullptr;
    P.su32 = reinterpret_cast<float*>(P.S.ki);
    P.ab32 = reinterpret_cast<float2*>(P.S.kd);
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
    long long t0;    // phase timers (diagnostics build): start of the current phase
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

// Per-build inputs of the tensor-core prune: float64 |x|^2 of every point and,
// for the fp16 Gram (PK_PRUNE_F16, default), an fp16 copy of the rows padded to
// kp = a multiple of 64 coordinates.  xh == nullptr: tf32 Gram from the fp32 rows.
struct PTAux {
    const double* nrm64;
    const __half* xh;
    int kp;
    int* ticket;  // this launch's item counter (zeroed before it): items are handed out one at a time
};

using PTTickets = BlockTickets;

// fp16 copy of every row (round to nearest), K padded with zeros to kp
__global__ void rows_to_half_kernel(const float* __restrict__ X, long long n, int dp, int kp, __half* __restrict__ out) {
    const long long total = n * (long long)(kp >> 1);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / (kp >> 1);
        const int t = (int)(i - r * (kp >> 1)) * 2;
        const float a = t < dp ? __ldg(X + (size_t)r * dp + t) : 0.f;
        const float b = t + 1 < dp ? __ldg(X + (size_t)r * dp + t + 1) : 0.f;
        reinterpret_cast<__half2*>(out)[i] = __halves2half2(__float2half_rn(a), __float2half_rn(b));
    }
}

// Copy K chunk kc (floats 32 kc .. 32 kc + 31) of the pass's rows into stage
// buffer `st` (slot x at x * 128 bytes, 16-byte piece j at (j ^ (x & 7))):
// A rows r0 .. r0 + na - 1 at slots 0 .., and, when the B block is separate
// (b0 != r0), B rows b0 .. b0 + nb - 1 at slots 128 ..
// Per-thread staging plan of one Gram pass: thread tid always copies 16-byte
// piece j = tid & 7 of slots x = (tid >> 3) + 16 i (i < 16): the source row
// pointer (already offset by the piece) and the swizzled destination offset
// are computed once per pass, so a K chunk costs one add + one cp.async per
// piece.  Slot x holds A row r0 + x (x < na) and, when the B block is separate
// (b0 != r0), B row b0 + x - 128 at x >= 128; with b0 == r0 slot x is row r0 + x.
struct PTStagePlan {
    const float* src[16];
    unsigned dst[16];
    unsigned live;  // bit i: slot (tid >> 3) + 16 i is copied
    int j;
};

__device__ __forceinline__ void pt_stage_plan(const unsigned long long* rowp, int r0, int na, int b0, int nb,
                                              PTStagePlan& pl) {
    const int tid = threadIdx.x;
    pl.j = tid & 7;
    pl.live = 0u;
    const int tot = (b0 == r0) ? nb : 128 + nb;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int x = (tid >> 3) + 16 * i;
        int r = -1;
        if (x < tot) {
            if (b0 == r0) r = r0 + x;
            else if (x < 128) r = x < na ? r0 + x : -1;
            else r = b0 + x - 128;
        }
        pl.src[i] = r >= 0 ? reinterpret_cast<const float*>(rowp[r]) + pl.j * 4 : nullptr;
        pl.dst[i] = (unsigned)(x * 128 + ((pl.j ^ (x & 7)) << 4));
        if (r >= 0) pl.live |= 1u << i;
    }
}

// Copy K chunk kc (floats 32 kc .. 32 kc + 31) of the planned slots into stage
// buffer `st` (row slot x at x * 128 bytes, 16-byte piece j at (j ^ (x & 7))).
// (rowbytes = the row's length in bytes: dp * 4 for fp32 rows, kp * 2 for the
// fp16 copy, whose chunk of 128 bytes holds 64 coordinates)
__device__ __forceinline__ void pt_stage_chunk(int rowbytes, const PTStagePlan& pl, int kc, unsigned char* st) {
    const bool in = kc * 128 + pl.j * 16 < rowbytes;
    const unsigned sbase = smem_u32(st);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        if (!((pl.live >> i) & 1u)) continue;
        if (in) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + pl.dst[i]), "l"(pl.src[i] + kc * 32)
                         : "memory");
        } else {
            *reinterpret_cast<float4*>(st + pl.dst[i]) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// One Gram pass: rows r0 .. r0 + 127 (A) x columns b0 .. b0 + nb - 1 (B) of the
// sorted candidates into TMEM columns 0 .. N - 1 (nb <= 256 when b0 == r0, else
// <= 128), then the occlusion / uncertain bit words of rows r0 + tid for those
// columns (pairs u > t only).
template <int QV>
__device__ void pt_gram_pass(const float* __restrict__ X, int dp, const PTSmem& P, PTPipe& pp, int c, int r0, int b0,
                             int nb, double alpha2, int rowbytes, bool f16) {
    const int tid = threadIdx.x;
    const int nk = (rowbytes + 127) >> 7;
    const int na = min(128, c - r0);
    const int ncol = (nb + 15) & ~15;
    // fp32 accumulators; operands tf32 (format 2) or f16 (format 0), K-major
    const unsigned fmt = f16 ? 0u : 2u;
    const unsigned idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((unsigned)(ncol >> 3) << 17) | ((128u >> 4) << 24);
    PTStagePlan pl;
    pt_stage_plan(P.rowp, r0, na, b0, nb, pl);
    const unsigned boff = (b0 == r0) ? 0u : 128u * 128u;  // B operand offset inside a stage
    // prologue: chunks 0 .. PT_STAGES - 2
    for (int k = 0; k < PT_STAGES - 1; ++k) {
        if (k < nk) pt_stage_chunk(rowbytes, pl, k, P.stage + (size_t)k * PT_STAGE_BYTES);
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
        if (kn < nk) pt_stage_chunk(rowbytes, pl, kn, P.stage + (size_t)sn * PT_STAGE_BYTES);
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group %0;\n" ::"n"(PT_STAGES - 1) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const int s = kc % PT_STAGES;
            unsigned char* sb = P.stage + (size_t)s * PT_STAGE_BYTES;
            const unsigned long long da = umma_desc_sw128(sb);
            const unsigned long long db = umma_desc_sw128(sb + boff);
            if (f16) {
#pragma unroll
                for (int k = 0; k < 4; ++k)  // 16 f16 = 32 bytes per UMMA_K step
                    tc_mma_f16(pp.tmem, da + 2ull * k, db + 2ull * k, idesc, (kc | k) != 0);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)  // 8 tf32 = 32 bytes per UMMA_K step
                    tc_mma_tf32(pp.tmem, da + 2ull * k, db + 2ull * k, idesc, (kc | k) != 0);
            }
            tc_commit(P.bar + s);
        }
    }
    // the last chunk's commit tracks every MMA of the pass
    {
        const int s = (nk - 1) % PT_STAGES;
        mbar_wait(P.bar + s, (pp.phase >> s) & 1u);
        pp.phase ^= 1u << s;
    }
    tc_fence_after();
    PT_TICK(2);

    // epilogue: thread tid = TMEM lane, candidate row t = r0 + tid
    const int warp = tid >> 5;
    // relative bound of the tf32 Gram (inputs keep >= 10 mantissa bits, fp32
    // accumulation) and an absolute term for subnormal inputs / partial sums
    // flushed to zero: <= (dp + 8) 2^-126 (|t| + |u| + 1)
    // fp16 operands (round to nearest, 11 significant bits; below 2^-14 the
    // spacing is 2^-24): |x^ - x| <= 2^-11 |x| + 2^-25 per coordinate, so
    // |G^ - G| <= 2^-10 (1 + 2^-10) |t||u| + 2^-25 sqrt(dp) (|t| + |u|) (1 + 2^-10),
    // plus the same fp32 accumulation term; a coordinate past the fp16 range makes
    // the accumulator non-finite (decided exactly below)
    const double eg = f16 ? 0.0009775171065493646 + (double)(dp + 8) * 1.1932570e-07
                          : 0.001953125 + (double)(dp + 8) * 1.1920928955078125e-07;
    const double eabs = f16 ? 5.9604644775390625e-08 * sqrt((double)dp) : (double)(dp + 8) * 1.1754943508222875e-38;
    const int t = r0 + tid;
    const unsigned tbase = pp.tmem + ((unsigned)(warp * 32) << 16);
    const bool live = t < c;
    const double nt = live ? P.nrm[t] : 0.0, st = live ? P.sq[t] : 0.0;
    // First-pass decision in fp32 (the float64 form below costs ~17 FP64 operations
    // per pair, and FP64 issue is what bounded this epilogue).  With E = c1 |u| + c0
    // + 1e-12 |u|^2, c1 = 2 eg |t| + 2 eabs, c0 = 2 eabs (|t| + 1) + 1e-12 |t|^2:
    //   alpha^2 (d~ + E) <= K  <=>  (|t|^2 + c0) - 2 G~ + c1 |u| <= A_u = K / alpha^2 - |u|^2 (1 + 1e-12)
    //   alpha^2 (d~ - E) >  K  <=>  (|t|^2 - c0) - 2 G~ - c1 |u| >  B_u = K / alpha^2 - |u|^2 (1 - 1e-12)
    // Per-row and per-candidate terms are rounded outwards (pt_prune: su32, ab32),
    // and `tol` covers the fp32 roundings of each side, so a pair the fp32 test
    // calls is called the same way by exact arithmetic; every other pair (and any
    // operand outside the fp32 range: NaN) is "uncertain" -- the fp32 slack widens
    // the uncertain band (2 E ~ 2^-9 |t||u|) by ~1e-6 of it.
    const double c1d = 2.0 * eg * st + 2.0 * eabs;
    const double c0d = 2.0 * eabs * (st + 1.0) + 1e-12 * nt;
    float Pt = __double2float_ru(nt + c0d), Mt = __double2float_rd(nt - c0d);
    const float c1f = __double2float_ru(c1d);
    if (!(Pt < 1e30f) || !(c1f < 1e30f)) Pt = Mt = __int_as_float(0x7fc00000);
    // in the diagonal block, columns below this warp's first row hold only pairs u <= t
    for (int wd = (b0 == r0) ? warp : 0; wd * 32 < ncol; ++wd) {
        unsigned kb = 0u, ub = 0u;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int col = wd * 32 + h * 16;
            if (col >= ncol) break;
            float g[16];
            tmem_ld16(tbase + (unsigned)col, g);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int u = b0 + col + i;
                if (live && u > t && u < c) {
                    const unsigned bit = 1u << (h * 16 + i);
                    if (!isfinite(g[i])) {  // fp32 accumulator overflow (huge coordinates): decide exactly
                        ub |= bit;
                        continue;
                    }
                    const float y = c1f * P.su32[u];
                    const float2 ab = P.ab32[u];
                    const float tol = fmaf(4e-7f, Pt + 2.f * fabsf(g[i]) + y, 1e-30f);
                    if (fmaf(-2.f, g[i], Pt) + y + tol <= ab.x) kb |= bit;
                    else if (!(fmaf(-2.f, g[i], Mt) - y - tol > ab.y)) ub |= bit;
                }
            }
        }
        if (live) {
            const int word = (b0 >> 5) + wd;
            P.kill[tid * P.words + word] = kb;
            P.unc[tid * P.words + word] = ub;
        }
    }
    tc_fence_before();
    __syncthreads();
    PT_TICK(3);
}

// Bit rows of candidates r0 .. r0 + 127 against every later candidate: the
// diagonal block (columns r0 .. r0 + 255) then 128-column blocks up to c.
template <int QV>
__device__ void pt_gram_rows(const float* __restrict__ X, int dp, const PTSmem& P, PTPipe& pp, int c, int r0,
                             double alpha2, int rowbytes, bool f16) {
    pt_gram_pass<QV>(X, dp, P, pp, c, r0, r0, min(256, c - r0), alpha2, rowbytes, f16);
    for (int b0 = r0 + 256; b0 < c; b0 += 128)
        pt_gram_pass<QV>(X, dp, P, pp, c, r0, b0, min(128, c - b0), alpha2, rowbytes, f16);
}

// Greedy picks (warp 0) among the candidates of the current row block
// [r0, r0 + 128) whose bit rows are in P.kill / P.unc; uncertain pairs of a
// picked t are decided exactly.  `alive` (lane l: word l), `sel` persist across
// blocks.  Returns true when the picks are complete (sel == R or no candidate
// is left), false when the next alive candidate lies beyond this block.
template <int QV>
__device__ bool pt_greedy_block(const float* __restrict__ X, int dp, const PTSmem& P, int c, int r0, double alpha2,
                                int R, int* out, double* out_d, unsigned& alive, int& sel, long long& nex) {
    const int lane = lane_id();
    const int nw = (c + 31) >> 5;
    // the alive word the next pick comes from is also held warp-uniform (wl, aw),
    // updated from a broadcast read of the pick's kill word: the serial chain per
    // pick is ffs -> one shared-memory read -> and, without a ballot + shuffle
    int wl = 0;
    unsigned aw = 0u;
    while (sel < R) {
        if (aw == 0u) {
            const unsigned nz = __ballot_sync(PK_FULL, alive != 0u);
            if (!nz) return true;
            wl = __ffs(nz) - 1;
            aw = __shfl_sync(PK_FULL, alive, wl);
        }
        const int t = 32 * wl + __ffs(aw) - 1;
        if (t >= r0 + 128) return false;
        aw &= aw - 1u;
        if (lane == wl) alive = aw;
        const unsigned tid_t = P.S.ki2[t];
        if (lane == 0) {
            out[sel] = (int)tid_t;
            if (out_d) out_d[sel] = P.S.kd2[t];
        }
        ++sel;
        if (sel >= R) return true;
        const int row = (t - r0) * P.words;
        unsigned kill = lane < nw ? P.kill[row + lane] : 0u;
        unsigned kill_wl = P.kill[row + wl];
        unsigned unc = lane < nw ? (P.unc[row + lane] & alive) : 0u;
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
                if (w == wl) kill_wl |= kw;
            }
        }
        alive &= ~kill;
        aw &= ~kill_wl;
    }
    return true;
}

// drop `self` and repeated (dist, id) entries of the sorted kd/ki[0, c) (c <=
// CAP), keep order -> kd2/ki2; returns the count (block-wide)
template <int CAP>
__device__ __forceinline__ int pt_unique(const BPSmem& S, int c, unsigned self) {
    constexpr int E = CAP / PT_THREADS;  // positions per thread
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    bool keep[E];
    int mine = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = E * tid + e;
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
    for (int e = 0; e < E; ++e)
        if (keep[e]) {
            S.kd2[o] = S.kd[E * tid + e];
            S.ki2[o] = S.ki[E * tid + e];
            ++o;
        }
    __syncthreads();
    return total;
}

// one item: sorted unique candidates in P.S.kd2/ki2 (c <= PT_CAP) -> picks.
// Bit rows are computed one 128-candidate block at a time, only as far as the
// greedy needs them (R picks usually come from the first block).
template <int QV>
__device__ int pt_prune(const float* __restrict__ X, int dp, const PTAux& aux, const PTSmem& P,
                        PTPipe& pp, int c, double alpha2, int R, int* out, double* out_d, long long* exact_pairs) {
    const bool f16 = aux.xh != nullptr;
    const int rowbytes = f16 ? aux.kp * 2 : dp * 4;
    for (int x = threadIdx.x; x < c; x += PT_THREADS) {
        const unsigned id = P.S.ki2[x];
        const double v = aux.nrm64[id];
        P.nrm[x] = v;
        P.sq[x] = sqrt(v);
        P.rowp[x] = f16 ? reinterpret_cast<unsigned long long>(aux.xh + (size_t)id * aux.kp)
                        : reinterpret_cast<unsigned long long>(X + (size_t)id * dp);
        // fp32 operands of the epilogue's first-pass decision (see pt_gram_pass)
        const double Kq = P.S.kd2[x] / alpha2;
        const double slack = 1e-14 * (Kq + v);
        const double Au = Kq - v * (1.0 + 1e-12) - slack, Bu = Kq - v * (1.0 - 1e-12) + slack;
        float af = __double2float_rd(Au), bf = __double2float_ru(Bu);
        const float sf = __double2float_ru(P.sq[x]);
        if (!(fabsf(af) < 1e30f) || !(fabsf(bf) < 1e30f) || !(sf < 1e30f)) af = bf = __int_as_float(0x7fc00000);
        P.su32[x] = sf;
        P.ab32[x] = make_float2(af, bf);
    }
    __syncthreads();
    PT_TICK(1);
    const int lane = lane_id();
    const int nw = (c + 31) >> 5;
    unsigned alive = 0u;  // warp 0: lane l holds alive word l
    if (lane < nw) alive = (c - 32 * lane >= 32) ? 0xffffffffu : ((1u << (c - 32 * lane)) - 1u);
    int sel = 0;
    long long nex = 0;
    for (int r0 = 0; r0 < c; r0 += 128) {
        pt_gram_rows<QV>(X, dp, P, pp, c, r0, alpha2, rowbytes, f16);
        if ((threadIdx.x >> 5) == 0) {
            const bool done = pt_greedy_block<QV>(X, dp, P, c, r0, alpha2, R, out, out_d, alive, sel, nex);
            if (lane == 0) {
                P.S.scal[8] = sel;
                P.S.scal[9] = done;
            }
        }
        __syncthreads();
        PT_TICK(4);
        if (P.S.scal[9]) break;
    }
    PT_COUNT(6, nex);
    PT_COUNT(7, 1);
    if (threadIdx.x == 0 && exact_pairs) *exact_pairs += nex;
    const int r = P.S.scal[8];
    __syncthreads();
    return r;
}

__device__ __forceinline__ void pt_setup(const PTSmem& P, PTPipe& pp) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < PT_STAGES; ++s) mbar_init(P.bar + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(P.tmem_slot)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pp.tmem = *P.tmem_slot;
    pp.phase = 0u;
    pp.t0 = -1;  // phase timers: only the kernels that start them (PT_T0) are timed
}

__device__ __forceinline__ void pt_teardown(const PTSmem& P, const PTPipe& pp) {
    tc_fence_before();
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(pp.tmem), "r"(256));
    }
}

// build phase 2 for float data: one block per inserted point (items with more
// than PT_CAP candidates are queued for build_prune_kernel)
// CAP = PT_CAP (two CTAs per SM) over the whole batch, then CAP = PT_CAP_BIG (one
// CTA per SM) over the items the first launch queued on (over, nover); what
// that one queues goes to build_prune_kernel (a warp per item: 20 ms for a
// 600-candidate item, which a launch then waits for)
template <int QV, int CAP>
__global__ void __launch_bounds__(PT_THREADS, CAP == PT_CAP ? 2 : 1)
    prune_tc_build_kernel(BuildArgs A, const PTAux aux, const int* items, const int* nitems, int* over, int* nover) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const PTSmem P = carve_pt<CAP>(smem_raw);
    PTPipe pp;
    pt_setup(P, pp);
    const int tid = threadIdx.x;
    const int R = A.P.R;
    const int dp = A.D.dp;
    const float* X = A.D.X;
    long long pairs = 0, exact_pairs = 0;
    __shared__ int s_tick[2];
    PTTickets tk{s_tick, 0, 0};
    const int total = items ? *nitems : A.m;
    for (int it = tk.first(aux.ticket); it < total; __syncthreads(), it = tk.next(aux.ticket)) {
        PT_T0
        tk.take_next(aux.ticket);
        const int t = items ? items[it] : it;
        const unsigned p = (unsigned)A.bids[t];
        const int vl = A.vlen[t];
        const int nd = __ldg(A.P.deg + p);
        const int c0 = vl + nd;
        if (c0 > CAP) {
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
                const double cd = A.adjd ? A.adjd[(size_t)p * R + x - vl] : 0.0;
                P.S.kd[x] = (A.adjd && !isnan(cd)) ? cd : dq.eval_one(X, (int)id);
            }
        }
        const int Pw = next_pow2_dev(c0 < 2 ? 2 : c0);
        for (int x = c0 + tid; x < Pw; x += PT_THREADS) {
            P.S.kd[x] = __longlong_as_double(0x7ff0000000000000LL);
            P.S.ki[x] = 0xffffffffu;
        }
        __syncthreads();
        bp_sort(P.S.kd, P.S.ki, Pw);
        const int c = pt_unique<CAP>(P.S, c0, p);
        PT_TICK(0);
        if (c > CAP) {  // more unique candidates than one Gram holds: warp path
            if (tid == 0) over[atomicAdd(nover, 1)] = t;
            __syncthreads();
            continue;
        }
        int* out = A.new_ids + (size_t)t * R;
        double* out_d = A.new_d ? A.new_d + (size_t)t * R : nullptr;
        // the build always prunes (_kernels.py:370), even c <= R candidates
        int sel = c;
        if (c <= 1) {
            if (tid == 0 && c == 1) {
                out[0] = (int)P.S.ki2[0];
                if (out_d) out_d[0] = P.S.kd2[0];
            }
        } else {
            sel = pt_prune<QV>(X, dp, aux, P, pp, c, A.alpha2, R, out, out_d, &exact_pairs);
            if (tid == 0) pairs += (long long)c * (c - 1) / 2;
        }
        for (int x = sel + tid; x < R; x += PT_THREADS) {
            out[x] = -1;
            if (out_d) out_d[x] = __longlong_as_double(0x7ff8000000000000LL);
        }
        if (tid == 0) A.new_len[t] = sel;
        __syncthreads();
        PT_TICK(5);
    }
    if (tid == 0 && A.stats && pairs)
        atomicAdd(reinterpret_cast<unsigned long long*>(A.stats + 1), (unsigned long long)(pairs + exact_pairs));
    pt_teardown(P, pp);
}

// reverse-edge re-prune for float data: one block per target vertex with at most
// PT_CAP candidates (larger groups: reverse_big_kernel / the selection path)
// CAP = PT_CAP (two CTAs per SM) over every target: groups of PT_CAP + 1 ..
// PT_CAP_BIG candidates are queued on (mid, nmid) for the CAP = PT_CAP_BIG
// launch (one CTA per SM) over items = mid.
template <int MODE, int QV, int CAP>
__global__ void __launch_bounds__(PT_THREADS, CAP == PT_CAP ? 2 : 1)
    prune_tc_reverse_kernel(RevArgs A, const PTAux aux, const int* items, const int* nitems, int* mid, int* nmid) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const PTSmem P = carve_pt<CAP>(smem_raw);
    PTPipe pp;
    pt_setup(P, pp);
    const int tid = threadIdx.x, wid = tid >> 5;
    const MakeAt<MODE, QV> make{A.D};
    const int dp = A.dp;
    const float* X = A.X;
    const int nt = items ? *nitems : *A.ntargets;
    long long ev = 0;
    __shared__ int s_tick[2];
    PTTickets tk{s_tick, 0, 0};
    for (int it = tk.first(aux.ticket); it < nt; __syncthreads(), it = tk.next(aux.ticket)) {
        tk.take_next(aux.ticket);
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
        if (c0 > CAP && mid && c0 <= PT_CAP_BIG) {
            if (tid == 0) mid[atomicAdd(nmid, 1)] = s;
            continue;
        }
        if (c0 > CAP) {
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
            if (A.adjd)
                for (int x = tid; x < A.R; x += PT_THREADS) A.adjd[(size_t)u * A.R + x] = __longlong_as_double(0x7ff8000000000000LL);
        } else {
            const Seq64Member du{X + (size_t)u * dp, dp};
            for (int x = tid; x < c0; x += PT_THREADS) {
                const unsigned id = x < nd ? (unsigned)row[x] : (unsigned)A.adds[off + x - nd];
                P.S.ki[x] = id;
                double cd = 0.0;
                bool known = false;
                if (A.adjd) {  // row entries and new sources carry their exact distances (NaN = unknown)
                    cd = x < nd ? A.adjd[(size_t)u * A.R + x] : A.addd[off + x - nd];
                    known = !isnan(cd);
                }
                P.S.kd[x] = known ? cd : du.eval_one(X, (int)id);
            }
            const int Pw = next_pow2_dev(c0 < 2 ? 2 : c0);
            for (int x = c0 + tid; x < Pw; x += PT_THREADS) {
                P.S.kd[x] = __longlong_as_double(0x7ff0000000000000LL);
                P.S.ki[x] = 0xffffffffu;
            }
            __syncthreads();
            bp_sort(P.S.kd, P.S.ki, Pw);
            const int c = pt_unique<CAP>(P.S, c0, u);
            if (tid == 0) ev += c0;
            double* rowd = A.adjd ? A.adjd + (size_t)u * A.R : nullptr;
            if (c <= A.R) {
                for (int x = tid; x < c; x += PT_THREADS) {
                    row[x] = (int)P.S.ki2[x];
                    if (rowd) rowd[x] = P.S.kd2[x];
                }
                sel = c;
            } else {
                long long ex = 0;
                sel = pt_prune<QV>(X, dp, aux, P, pp, c, A.alpha2, A.R, row, rowd, &ex);
                if (tid == 0) ev += ex;
            }
            if (rowd)
                for (int x = sel + tid; x < A.R; x += PT_THREADS) rowd[x] = __longlong_as_double(0x7ff8000000000000LL);
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

