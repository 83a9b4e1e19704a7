/*
 * peakann_b200 -- C ABI of the B200-native density-peaks hot path.
 *
 * The reference package's de-facto FFI for this path is its numba kernel
 * module, /root/reference/pkg/src/peakann/_kernels.py: free functions over
 * plain arrays (float32 points, int32 adjacency, int64 ids, float64 squared
 * distances).  Each entry point below replaces one of those functions (or
 * one numpy stage of the Python layer) and names the reference interface it
 * stands in for.  All pointers are DEVICE pointers (caller-owned; nothing is
 * retained after return) unless marked "host"; every call is enqueued on the
 * given cudaStream_t (passed as void*) and returns 0 on success or a nonzero
 * code, with a message from pk_last_error().
 *
 * Point layout: row-major float32 (n, dp) with dp = d rounded up to a
 * multiple of 4 and zero padding (adds exactly +0.0 to squared distances).
 * `mode` selects the distance policy: PK_MODE_SEQ64 (per-lane sequential
 * float64 in index order -- bit-identical to _kernels.py:21-38 for any data),
 * PK_MODE_EXACT32 (warp-split float32, legal only when pk_check_exact32
 * proved every partial sum is an exactly representable integer) or
 * PK_MODE_EXACT_U8 (integer data spanning <= 255 packed as bytes in x8 by
 * pk_pack_u8, rows of dw words; exact integer dp4a arithmetic).  x8 may be
 * null in the other modes.
 */
#ifndef PEAKANN_B200_H
#define PEAKANN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PK_MODE_SEQ64 0
#define PK_MODE_EXACT32 1
#define PK_MODE_EXACT_U8 2

#define PK_DENSITY_KTH 0
#define PK_DENSITY_KTH_NORMALIZED 1
#define PK_DENSITY_EXP_SUM 2
#define PK_DENSITY_SUM_EXP 3
#define PK_DENSITY_SUM 4

int pk_version(void);
const char* pk_last_error(void);
/* number of SMs / opt-in shared memory per block of the current device (host out) */
int pk_device_info(int* sm_count, int* smem_optin);

/* Launch accounting (no reference counterpart; used by bench.py): every
 * kernel launch is counted per kernel name; with pk_prof_enable(1) each launch
 * is also bracketed by CUDA events on its stream.  pk_prof_collect writes
 * "name count total_ms\n" lines into buf (host) and returns the full length;
 * reset != 0 clears the counters. */
void pk_prof_enable(int on);
/* Restrict event timing to the comma-separated kernel names ("" = all);
 * launch counting is unaffected. */
void pk_prof_only(const char* names);
int pk_prof_collect(char* buf, int len, int reset);

/* Distance-policy classification into *out_flag (device int): 2 when every
 * coordinate is an integer and max - min <= 255 (PK_MODE_EXACT_U8 is exact),
 * 1 when integer with d * (max - min)^2 < 2^24 (PK_MODE_EXACT32 is exact),
 * else 0 (PK_MODE_SEQ64).  Replaces: nothing (the reference always uses the
 * float64 loop of _kernels.py:21-38; the exact modes reproduce its values). */
int pk_check_exact32(const float* x, int64_t n, int64_t dp, int64_t d, int* out_flag, void* stream);

/* Pack integer coordinates as bytes (x - min), 4 per uint32 word, rows of dw
 * = ceil(d/4) words (zero padded).  Only valid when pk_check_exact32 gave 2. */
int pk_pack_u8(const float* x, int64_t n, int64_t dp, int64_t d, uint32_t* out, int64_t dw, void* stream);

/* Beam-search kNN of member queries.  Replaces _kernels.beam_knn_batch
 * (_kernels.py:230-262); with brute_fallback=1 also the short-row exact
 * recompute of VamanaIndex.knn_batch (vamana.py:220-225).
 * out_ids (m,kk) int64 (-1 pad), out_sqd (m,kk) float64 (+inf pad),
 * out_counts (m,) int64 (counts BEFORE the fallback), kk = min(k, n-1).
 * out_evals (device int64[2], may be null) accumulates distance evaluations
 * and expansions (adjacency rows read).
 * hash_bits: log2 of the per-query seen-table size (0 = automatic). */
int pk_beam_knn(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                const int32_t* adj, int64_t R,
                const int32_t* deg, const int32_t* starts, int64_t s, const int64_t* qids, int64_t m,
                int64_t L, int64_t k, int64_t* out_ids, double* out_sqd, int64_t* out_counts,
                int brute_fallback, int64_t* out_evals, int hash_bits, void* stream);

/* pk_beam_knn starting each member query from its beam saved by
 * pk_build_vamana_seeds (L must equal the build's L, same start list). */
int pk_beam_knn_seeded(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                       const int32_t* adj, int64_t R, const int32_t* deg, const int32_t* starts, int64_t s,
                       const int64_t* qids, int64_t m, int64_t L, int64_t k, int64_t* out_ids, double* out_sqd,
                       int64_t* out_counts, int brute_fallback, int64_t* out_evals, int hash_bits,
                       const double* seed_bd, const uint32_t* seed_bi, const int32_t* seed_bl, void* stream);

/* One search from an explicit start list for a member query (qid >= 0) or a
 * float64 query vector (qid < 0, qvec = dp doubles, zero padded).  Replaces
 * _kernels.beam_search_single (_kernels.py:215-227) as used by beam_search /
 * find_knn_with_fallback (vamana.py:62-84, 175-197): writes the first k
 * entries of sorted(visited U beam) without qid into top_ids/top_sqd (k
 * slots), their count into *top_count, and the visit log (expansion order)
 * into vis_ids/vis_sqd (capacity vcap; *vis_count may exceed vcap on overflow).
 * Counts are device int64. */
int pk_beam_search_single(const float* x, int64_t n, int64_t dp, const int32_t* adj, int64_t R,
                          const int32_t* deg, const int32_t* starts, int64_t s, int64_t qid,
                          const double* qvec, int64_t L, int64_t k, int64_t* top_ids, double* top_sqd,
                          int64_t* top_count, int64_t* vis_ids, double* vis_sqd, int64_t vcap,
                          int64_t* vis_count, void* stream);

/* Exact kNN of member queries with (dist,id) order, self excluded.
 * Replaces _kernels.brute_knn_batch (_kernels.py:86-104). kk = min(k, n-1). */
int pk_brute_knn(const float* x, int64_t n, int64_t dp, const int64_t* qids, int64_t m, int64_t k,
                 int64_t* out_ids, double* out_sqd, void* stream);

/* Same contract as pk_brute_knn (kk <= 32), on the tensor cores: a tcgen05
 * fp16 GEMM screens the K' = 64 nearest candidates of every query (fused
 * distance + top-K' epilogue), then each row is rescored with the float64
 * sequential distance and sorted by (dist, id).  row_flags (device u8, m)
 * marks rows whose error-bound certificate failed (the caller recomputes them
 * with pk_brute_knn); *uncertified (device u64) counts them. */
int pk_brute_knn_tc(const float* x, int64_t n, int64_t dp, const int64_t* qids, int64_t m, int64_t k,
                    int64_t* out_ids, double* out_sqd, uint8_t* row_flags, uint64_t* uncertified, void* stream);

/* Exact kNN of one float64 vector, no exclusion, kk = min(k, n).
 * Replaces _kernels.brute_knn_vector (_kernels.py:107-118). */
int pk_brute_knn_vector(const float* x, int64_t n, int64_t dp, const double* qvec, int64_t k,
                        int64_t* out_ids, double* out_sqd, void* stream);

/* Whole Vamana build: batches of 1, 2, 4, ... over `order`, each a fused
 * beam-search + RobustPrune (_kernels.build_batch, _kernels.py:338-375), the
 * out-list commit and the reverse-edge re-prune (_kernels.apply_reverse_edges,
 * _kernels.py:378-415, grouped as in vamana.py:157-167).  Replaces the batch
 * loop of build_vamana (vamana.py:141-169).  adj_out (n,R) int32 (-1 pad),
 * deg_out (n,) int32.  starts/order are int32 device arrays (sampled on the
 * host from the reference's PCG64 stream, vamana.py:132-143).
 * stats (device int64[4], may be null): search evals, prune evals,
 * reverse evals, expansions. */
int pk_build_vamana(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                    int64_t R, int64_t L, double alpha,
                    const int32_t* starts, int64_t s, const int32_t* order, int32_t* adj_out,
                    int32_t* deg_out, int64_t* stats, int hash_bits, void* stream);

/* pk_build_vamana that also saves, per inserted point p, the beam its search
 * starts from (after seeding with the start list): seed_bd / seed_bi are
 * [n][L] (the beam's key slots and id words), seed_bl [n] the lengths.  A later
 * pk_beam_knn_seeded of member queries with the same L and start list starts
 * from these beams instead of seeding again (same inputs, same seeded beam). */
int pk_build_vamana_seeds(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode, int64_t R,
                          int64_t L, double alpha, const int32_t* starts, int64_t s, const int32_t* order,
                          int32_t* adj_out, int32_t* deg_out, int64_t* stats, int hash_bits, double* seed_bd,
                          uint32_t* seed_bi, int32_t* seed_bl, void* stream);

/* Sharded build: one process per GPU, every rank holds the full point set
 * and ends with the full graph (identical on every rank and to
 * pk_build_vamana).  A batch of m >= min_shard points is split into world
 * contiguous chunks of c = ceil(m / world); rank r searches and prunes chunk r
 * into xids[(r*c + t) * R ...] / xlen[r*c + t], then calls
 *     exchange(ctx, PK_XCHG_OUTLISTS, c, 0)
 * which must all-gather xids[0, world*c*R) and xlen[0, world*c) in place.
 * Reverse-edge re-prunes run on the targets u with u % world == rank; their
 * rows are packed as [u, deg, row[R]] (R + 2 int32) into xsend and
 *     maxc = exchange(ctx, PK_XCHG_ROWS, own_count, 0)
 * must all-gather the counts into xcnt[world] (device int32) and
 * xsend[0, maxc*(R+2)) into xrecv[0, world*maxc*(R+2)), returning maxc (< 0 =
 * error).  Buffers: xids >= (B + world) * R, xlen >= B + world with B the
 * largest batch (<= n), xsend >= U * (R+2), xrecv >= world * U * (R+2) with
 * U = min(n, B * R).  Smaller batches run replicated (no exchange).
 * Replaces the batch loop of vamana.py:146-169 with the multi-GPU split
 * SURVEY.md section 8(e) step 6 describes. */
typedef int64_t (*pk_exchange_fn)(void* ctx, int kind, int64_t a, int64_t b);
#define PK_XCHG_OUTLISTS 0
#define PK_XCHG_ROWS 1
/* exchange(ctx, PK_XCHG_ORDER, n, 0): broadcast xids[0, n) from rank 0 (the
 * search order inside the batches, float builds with the start pre-screen:
 * every rank derives it from the same data, rank 0's copy is authoritative) */
#define PK_XCHG_ORDER 2
int pk_build_vamana_sharded(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                            int64_t R, int64_t L, double alpha,
                            const int32_t* starts, int64_t s, const int32_t* order, int32_t* adj_out,
                            int32_t* deg_out, int64_t* stats, int hash_bits, int rank, int world,
                            int64_t min_shard, pk_exchange_fn exchange, void* ctx, int32_t* xids,
                            int32_t* xlen, int32_t* xsend, int32_t* xrecv, int32_t* xcnt, void* stream);

/* Host helper (no device work): numpy's Generator.permutation(n) on a PCG64
 * stream given as state = {state_hi, state_lo, inc_hi, inc_lo} plus the
 * buffered 32-bit half (has_uint32, uinteger), written as int32 into `out`
 * (the build's insertion order, vamana.py:141-143).  state_out (optional):
 * {state_hi, state_lo, has_uint32, uinteger} after the draws. */
int pk_pcg64_permutation(const uint64_t* state, int has_uint32, uint32_t uinteger, int64_t n, int32_t* out,
                         uint64_t* state_out);

/* Host helper (no device work): parse the vertex records of a PECG graph file
 * (everything after the 16-byte header and the start ids: per vertex a u32
 * degree followed by that many u32 neighbour ids; vamana.py:243-267 replaces
 * its per-vertex Python loop) into adj (n, R) int32 padded with -1 and
 * deg (n,) int32.  Returns 0, or 3 = truncated at vertex info[0], 4 = vertex
 * info[0] has degree info[1] > R, 5 = info[0] trailing bytes. */
int pk_parse_pecg(const uint32_t* words, int64_t nwords, int64_t n, int64_t R, int32_t* adj, int32_t* deg,
                  int64_t* info);

/* Diagnostics: the beam walk's per-phase clock64 cycle sums (expand, row
 * prefetch, fp32 screens, resolve, merge, emit, seeding); zeros unless the
 * library was compiled with -DPK_PHASE_TIMERS (tools/variant.sh). */
int pk_phase_timers(unsigned long long* out8, int reset);
int pk_phase_timers_build(unsigned long long* out8, int reset);
/* the tensor-core build prune: candidates + sort, norms, Gram, epilogue, greedy,
 * output; [6] exact pair decisions, [7] items */
int pk_phase_timers_prune(unsigned long long* out8, int reset);

/* Host helper: index of the first non-finite value of x[0, count) in
 * row-major order (-1 if none) -> *first_bad; all host threads scan.  The
 * PointSet finiteness check (core.py:17-54). */
int pk_find_nonfinite(const float* x, int64_t count, int64_t* first_bad);

/* One pass over a freshly uploaded point set: out[0] = the pk_check_exact32
 * flag (0 / 1 / 2), out[1] = flat index (row * d + column) of the first
 * non-finite coordinate, -1 if none (device int64[2]).  The PointSet
 * validation of core.py:17-54 fused with the distance-policy check. */
int pk_scan_points(const float* x, int64_t n, int64_t dp, int64_t d, int64_t* out, void* stream);

/* Nearest strictly denser point of each query (rank[p] > rank[q], order
 * (dist, id)) through the tensor-core screen of pk_brute_knn_tc restricted to
 * denser points, float64 rescoring and the same error-bound certificate.
 * Replaces _kernels.dp_scan_all (_kernels.py:442-462) for batches; rows the
 * certificate rejects are flagged (row_flags, *uncertified) and must be
 * recomputed with pk_dp_scan.  out_id (m,) int64 (-1 = none), out_sqd (m,)
 * float64. */
int pk_dp_scan_tc(const float* x, int64_t n, int64_t dp, const int64_t* rank, const int64_t* qids, int64_t m,
                  int64_t* out_id, double* out_sqd, uint8_t* row_flags, uint64_t* uncertified, void* stream);

/* RobustPrune of vertex p over explicit candidates (ids, squared distances)
 * merged with its current out-list cur_ids (distances recomputed).  Replaces
 * _kernels.robust_prune_standalone (_kernels.py:318-335).  out (R,) int64,
 * *out_count device int64. */
int pk_robust_prune(const float* x, int64_t n, int64_t dp, int64_t p, const int64_t* cand_ids,
                    const double* cand_sqd, int64_t m, const int64_t* cur_ids, int64_t dcount,
                    double alpha, int64_t R, int64_t* out, int64_t* out_count, void* stream);

/* Replaces _kernels.nearest_to_centroid (_kernels.py:418-435). *out device int64. */
int pk_nearest_to_centroid(const float* x, int64_t n, int64_t dp, int64_t* out, void* stream);

/* sqrt of squared distances, elementwise (index.py:131-139, vamana.py:226). */
int pk_sqrt(const double* sqd, int64_t count, double* out, void* stream);

/* Densities from (n,k) neighbour distances (true distances, not squared) and
 * ids.  Replaces density.compute_densities (density.py:92-113) including
 * numpy's pairwise row summation order. */
int pk_densities(int kind, const int64_t* ids, const double* dists, int64_t n, int64_t k, double* rho,
                 void* stream);

/* kth_normalized from a given base density vector: rho*k / sum(base[ids])
 * (density.density_kth_normalized, density.py:48-55, 69-73). */
int pk_normalize_rho(const double* base, const int64_t* ids, int64_t n, int64_t k, double* out, void* stream);

/* pk_normalize_rho for the rows of points row0 .. row0 + m - 1 only (one rank's
 * chunk of the kNN rows; base covers all n points): out[i] = base[row0 + i] * k
 * / sum_j base[ids[i][j]] in numpy's summation order (density.py:48-55). */
int pk_normalize_rho_rows(const double* base, const int64_t* ids, int64_t row0, int64_t m, int64_t k, double* out,
                          void* stream);

/* rank[i] in 1..n, higher = denser, ties by smaller id; *nan_flag (device
 * int) set when rho has a NaN.  Replaces density.rank_order (density.py:116-129). */
int pk_rank_order(const double* rho, int64_t n, int64_t* rank, int* nan_flag, void* stream);

/* First strictly denser entry of each (dist,id)-sorted row.  Replaces
 * dependent._resolve_from_lists (dependent.py:80-93): fills lam/delta for
 * resolved rows, appends unresolved qids (ascending order preserved) to
 * unresolved, count in *n_unresolved (device int64).  `skip` (>= 0) is a
 * qid dropped from the unresolved list (the global density peak,
 * dependent.py:112). */
int pk_resolve_lists(const int64_t* rank, const int64_t* qids, int64_t m, const int64_t* ids,
                     const double* dists, int64_t k, int64_t* lam, double* delta, int64_t* unresolved,
                     int64_t* n_unresolved, int64_t skip, const int64_t* counts, int64_t* short_out,
                     int64_t* n_short, void* stream);
/* (counts, short_out, n_short may be null; with counts, rows whose beam
 * search found fewer than k entries are not resolved from their partial
 * list but appended to short_out for pk_resolve_short.) */

/* Closest strictly denser point over all n for each query.  Replaces
 * _kernels.dp_scan_all (_kernels.py:442-462).  out_id (m,) int64,
 * out_sqd (m,) float64. */
int pk_dp_scan(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
               const int64_t* rank, const int64_t* qids, int64_t m, int64_t* out_id, double* out_sqd,
               void* stream);

/* out_count[t] = #{ j != qids[t] : (d(qids[t], j), j) < (key_d[t], key_i[t]) },
 * i.e. the position the key would take in the query's exact kNN row. */
int pk_count_below(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                   const int64_t* qids, int64_t m, const double* key_d, const int64_t* key_i,
                   int64_t* out_count, void* stream);

/* Doubling-round rows whose beam search came up short.  The reference
 * replaces them with exact kNN rows of width kk (vamana.py:220-225) and takes
 * the first strictly denser entry (dependent.py:80-93); that entry is the
 * nearest denser point p* iff fewer than kk keys precede p*'s key.  So: one
 * dp scan + one count scan, no row.  Resolved rows fill lam/delta, the others
 * are appended (input order) to unresolved, count in *n_unresolved. */
int pk_resolve_short(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                     const int64_t* rank, const int64_t* qids, int64_t m, int64_t kk, int64_t* lam,
                     double* delta, int64_t* unresolved, int64_t* n_unresolved, void* stream);
/* pk_resolve_short with the dp scan already done (dp_id / dp_sqd = the exact
 * nearest denser point of each row, e.g. from pk_dp_scan_tc): the count scan
 * and the resolution only. */
int pk_resolve_short_scanned(const float* x, int64_t n, int64_t dp, const uint32_t* x8, int64_t dw, int mode,
                             const int64_t* qids, int64_t m, int64_t kk, const int64_t* dp_id, const double* dp_sqd,
                             int64_t* lam, double* delta, int64_t* unresolved, int64_t* n_unresolved, void* stream);
/* Counters of the tensor-core count decision used by pk_resolve_short_scanned on
 * float data: out2[0] = rows screened, out2[1] = rows the bounds left open (sent
 * to the exact count scan); reset != 0 zeroes them.  Diagnostics only. */
int pk_tc_count_stats(int64_t* out2, int reset);

/* Scatter: lam[qids[i]] = src_id[i], delta[qids[i]] = sqrt(src_sqd[i])
 * (dependent.py:125-127). */
int pk_scatter_dependents(const int64_t* qids, int64_t m, const int64_t* src_id, const double* src_sqd,
                          int64_t* lam, double* delta, void* stream);

/* index of the maximum rank (dependent.py:108: argmax(rank)); *out device int64 */
int pk_argmax_rank(const int64_t* rank, int64_t n, int64_t* out, void* stream);

/* Policies (cluster.py:134-180).  flags are device uint8 (n,).
 *   noise:      flag[i] = rho[i] < rho_min
 *   threshold:  flag[i] = !noise[i] && delta[i] >= delta_min
 *   product:    the n_c non-noise ids with the largest delta*rho, ties by
 *               larger delta then smaller id (lexsort, cluster.py:145-172);
 *               requires n_c < number of non-noise points
 *   local:      flag[i] = !noise[i] && rank[i] > max rank over its kNN row
 *   orphans:    flag[i] |= lam[i] < 0 && !noise[i]   (cluster.py:248-253) */
int pk_flag_noise(const double* rho, int64_t n, double rho_min, uint8_t* noise, int64_t* n_noise, void* stream);
int pk_centers_threshold(const double* delta, const uint8_t* noise, int64_t n, double delta_min,
                         uint8_t* center, void* stream);
int pk_centers_product(const double* rho, const double* delta, const uint8_t* noise, int64_t n, int64_t n_c,
                       uint8_t* center, void* stream);
int pk_centers_local(const int64_t* rank, const int64_t* nbr_ids, int64_t k, const uint8_t* noise, int64_t n,
                     uint8_t* center, void* stream);
int pk_promote_orphans(const int64_t* lam, const uint8_t* noise, int64_t n, uint8_t* center, void* stream);

/* Union-find assignment by pointer jumping on parent[i] = skip[i] ? i : lam[i]
 * (dependency edges point strictly up in density rank, so each component is a
 * tree rooted at its center / noise point).  Replaces assign_clusters +
 * UnionFind (cluster.py:183-220, unionfind.py:16-41).  center/noise are
 * device uint8 flags; labels (n,) int64.  status (device int64[2]):
 * status[0] = 0 ok, 1 = a non-skip point with lam < 0 (status[1] = smallest
 * such id), 3 = a component without center/noise (status[1] = smallest id). */
int pk_assign_clusters(const int64_t* lam, const uint8_t* center, const uint8_t* noise, int64_t n,
                       int64_t* labels, int64_t* status, void* stream);

/* ids of set flags in ascending order: out (capacity n), *count device int64 */
int pk_flags_to_ids(const uint8_t* flags, int64_t n, int64_t* out, int64_t* count, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PEAKANN_B200_H */
