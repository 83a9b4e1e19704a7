/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the peakann-b200 parity tests.
 *
 * A plain-C restatement of the reference's numba kernels
 * (/root/reference/pkg/src/peakann/_kernels.py) plus the host-side batch loop
 * of build_vamana (vamana.py:106-172).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library;
 * the product path (paper_2312_03940_b200/) never links or calls it.
 *
 * Faithfulness notes (what the parity tests depend on):
 *  - distances: float32 coordinates, float64 accumulation in index order
 *    t = 0..d-1 (_kernels.py:21-38);
 *  - every ordering is (squared distance, id) (_kernels.py:8-9);
 *  - the beam search keeps the reference's data structures: a per-query
 *    zeroed visited/inbeam byte map of size n, O(L) sorted inserts, and
 *    re-evaluation of evicted nodes (_kernels.py:125-185, 244-249), so the
 *    timed CPU baseline does the same work the reference does;
 *  - parallel loops are OpenMP "for" over independent queries / targets and
 *    write disjoint outputs, so results do not depend on the thread count.
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py -> tests/golden/*.npz; tests/test_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t i64;
typedef int32_t i32;

/* ---- distances (_kernels.py:21-38) ----------------------------------- */

static inline double sq_to_vec(const float *data, i64 d, i64 j, const double *q) {
    const float *x = data + j * d;
    double acc = 0.0;
    for (i64 t = 0; t < d; ++t) {
        double df = q[t] - (double)x[t];
        acc += df * df;
    }
    return acc;
}

double or_point_sqdist(const float *data, i64 d, i64 i, i64 j) {
    const float *a = data + i * d, *b = data + j * d;
    double acc = 0.0;
    for (i64 t = 0; t < d; ++t) {
        double df = (double)a[t] - (double)b[t];
        acc += df * df;
    }
    return acc;
}

static void row_as_f64(const float *data, i64 d, i64 i, double *q) {
    for (i64 t = 0; t < d; ++t) q[t] = (double)data[i * d + t];
}

/* ---- key helpers ------------------------------------------------------ */

static inline int key_less(double da, i64 ia, double db, i64 ib) {
    return da < db || (da == db && ia < ib);
}

/* stable merge sort of (d, id) pairs by d only (numpy argsort kind=mergesort) */
static void stable_sort_by_d(double *dd, i64 *ids, i64 m, double *td, i64 *ti) {
    for (i64 w = 1; w < m; w *= 2) {
        for (i64 lo = 0; lo < m; lo += 2 * w) {
            i64 mid = lo + w < m ? lo + w : m, hi = lo + 2 * w < m ? lo + 2 * w : m;
            i64 a = lo, b = mid, o = lo;
            while (a < mid && b < hi) {
                if (dd[b] < dd[a]) { td[o] = dd[b]; ti[o++] = ids[b++]; }
                else { td[o] = dd[a]; ti[o++] = ids[a++]; }
            }
            while (a < mid) { td[o] = dd[a]; ti[o++] = ids[a++]; }
            while (b < hi) { td[o] = dd[b]; ti[o++] = ids[b++]; }
        }
        memcpy(dd, td, (size_t)m * sizeof(double));
        memcpy(ids, ti, (size_t)m * sizeof(i64));
    }
}

/* stable merge sort of (id, d) pairs by id only */
static void stable_sort_by_id(i64 *ids, double *dd, i64 m, i64 *ti, double *td) {
    for (i64 w = 1; w < m; w *= 2) {
        for (i64 lo = 0; lo < m; lo += 2 * w) {
            i64 mid = lo + w < m ? lo + w : m, hi = lo + 2 * w < m ? lo + 2 * w : m;
            i64 a = lo, b = mid, o = lo;
            while (a < mid && b < hi) {
                if (ids[b] < ids[a]) { ti[o] = ids[b]; td[o++] = dd[b++]; }
                else { ti[o] = ids[a]; td[o++] = dd[a++]; }
            }
            while (a < mid) { ti[o] = ids[a]; td[o++] = dd[a++]; }
            while (b < hi) { ti[o] = ids[b]; td[o++] = dd[b++]; }
        }
        memcpy(dd, td, (size_t)m * sizeof(double));
        memcpy(ids, ti, (size_t)m * sizeof(i64));
    }
}

/* k-th smallest (0-based) of a copy of row (quickselect; value only) */
static double kth_value(double *tmp, i64 n, i64 kth) {
    i64 lo = 0, hi = n - 1;
    while (lo < hi) {
        double piv = tmp[lo + (hi - lo) / 2];
        i64 i = lo, j = hi;
        while (i <= j) {
            while (tmp[i] < piv) ++i;
            while (tmp[j] > piv) --j;
            if (i <= j) { double t = tmp[i]; tmp[i] = tmp[j]; tmp[j] = t; ++i; --j; }
        }
        if (kth <= j) hi = j;
        else if (kth >= i) lo = i;
        else return tmp[kth];
    }
    return tmp[kth];
}

/* top-kk of a distance row with (dist, id) order (_kernels.py:55-83) */
static void select_k(const double *row, i64 n, i64 kk, i64 *out_ids, double *out_d, double *scratch) {
    memcpy(scratch, row, (size_t)n * sizeof(double));
    double th = kth_value(scratch, n, kk - 1);
    i64 c = 0;
    for (i64 j = 0; j < n; ++j)
        if (row[j] < th) { out_ids[c] = j; out_d[c++] = row[j]; }
    for (i64 j = 0; j < n && c < kk; ++j)
        if (row[j] == th) { out_ids[c] = j; out_d[c++] = row[j]; }
    double *td = scratch;
    i64 *ti = (i64 *)malloc((size_t)kk * sizeof(i64));
    stable_sort_by_d(out_d, out_ids, kk, td, ti);
    free(ti);
}

/* ---- exact kNN (_kernels.py:86-118) ----------------------------------- */

void or_brute_knn_batch(const float *data, i64 n, i64 d, const i64 *qids, i64 m, i64 k,
                        i64 *out_ids, double *out_d) {
    i64 kk = k < n - 1 ? k : n - 1;
    for (i64 t = 0; t < m * (kk > 0 ? kk : 0); ++t) { out_ids[t] = -1; out_d[t] = INFINITY; }
    if (kk <= 0) return;
#pragma omp parallel
    {
        double *row = (double *)malloc((size_t)n * sizeof(double));
        double *scr = (double *)malloc((size_t)n * sizeof(double));
        double *q = (double *)malloc((size_t)d * sizeof(double));
#pragma omp for schedule(dynamic, 4)
        for (i64 t = 0; t < m; ++t) {
            i64 i = qids[t];
            row_as_f64(data, d, i, q);
            for (i64 j = 0; j < n; ++j) row[j] = sq_to_vec(data, d, j, q);
            row[i] = INFINITY;
            select_k(row, n, kk, out_ids + t * kk, out_d + t * kk, scr);
        }
        free(row); free(scr); free(q);
    }
}

void or_brute_knn_vector(const float *data, i64 n, i64 d, const double *q, i64 k,
                         i64 *out_ids, double *out_d) {
    i64 kk = k < n ? k : n;
    double *row = (double *)malloc((size_t)n * sizeof(double));
    double *scr = (double *)malloc((size_t)n * sizeof(double));
    for (i64 j = 0; j < n; ++j) row[j] = sq_to_vec(data, d, j, q);
    select_k(row, n, kk, out_ids, out_d, scr);
    free(row); free(scr);
}

/* ---- greedy beam search (_kernels.py:125-212) -------------------------- */

typedef struct {
    i64 *bi; double *bd;     /* beam, (dist,id)-sorted, capacity L   */
    i64 *vi; double *vd;     /* visit log, capacity n                */
    uint8_t *visited, *inbeam;
    double *q;
    i64 evals;               /* distance evaluations performed        */
} beam_ws;

static i64 beam_put(beam_ws *w, i64 bl, i64 L, i64 id, double dist) {
    i64 pos = bl;
    for (i64 t = 0; t < bl; ++t)
        if (key_less(dist, id, w->bd[t], w->bi[t])) { pos = t; break; }
    if (bl < L) {
        for (i64 t = bl; t > pos; --t) { w->bi[t] = w->bi[t - 1]; w->bd[t] = w->bd[t - 1]; }
        w->bi[pos] = id; w->bd[pos] = dist; w->inbeam[id] = 1;
        return bl + 1;
    }
    if (pos >= L) return bl;
    w->inbeam[w->bi[L - 1]] = 0;
    for (i64 t = L - 1; t > pos; --t) { w->bi[t] = w->bi[t - 1]; w->bd[t] = w->bd[t - 1]; }
    w->bi[pos] = id; w->bd[pos] = dist; w->inbeam[id] = 1;
    return bl;
}

/* returns beam length; *vl = number of expansions */
static i64 beam_walk(const float *data, i64 d, const i32 *adj, i64 R, const i32 *deg,
                     const i64 *starts, i64 s, i64 L, beam_ws *w, i64 *vl_out) {
    i64 bl = 0;
    for (i64 a = 0; a < s; ++a) {
        i64 st = starts[a];
        if (w->inbeam[st]) continue;
        w->evals++;
        bl = beam_put(w, bl, L, st, sq_to_vec(data, d, st, w->q));
    }
    i64 vl = 0;
    for (;;) {
        i64 pos = -1;
        for (i64 t = 0; t < bl; ++t)
            if (!w->visited[w->bi[t]]) { pos = t; break; }
        if (pos < 0) break;
        i64 p = w->bi[pos];
        w->visited[p] = 1;
        w->vi[vl] = p; w->vd[vl] = w->bd[pos]; ++vl;
        for (i64 e = 0; e < deg[p]; ++e) {
            i64 nb = adj[p * R + e];
            if (w->inbeam[nb]) continue;
            w->evals++;
            bl = beam_put(w, bl, L, nb, sq_to_vec(data, d, nb, w->q));
        }
    }
    *vl_out = vl;
    return bl;
}

/* visited U unvisited-beam, (dist,id)-sorted; returns count */
static i64 gather_candidates(beam_ws *w, i64 bl, i64 vl, i64 *ci, double *cd, i64 *ti, double *td) {
    i64 c = 0;
    for (i64 t = 0; t < vl; ++t) { ci[c] = w->vi[t]; cd[c++] = w->vd[t]; }
    for (i64 t = 0; t < bl; ++t)
        if (!w->visited[w->bi[t]]) { ci[c] = w->bi[t]; cd[c++] = w->bd[t]; }
    stable_sort_by_id(ci, cd, c, ti, td);
    stable_sort_by_d(cd, ci, c, td, ti);
    return c;
}

static int ws_alloc(beam_ws *w, i64 n, i64 d, i64 L) {
    w->bi = (i64 *)malloc((size_t)L * sizeof(i64));
    w->bd = (double *)malloc((size_t)L * sizeof(double));
    w->vi = (i64 *)malloc((size_t)n * sizeof(i64));
    w->vd = (double *)malloc((size_t)n * sizeof(double));
    w->visited = (uint8_t *)calloc((size_t)n, 1);
    w->inbeam = (uint8_t *)calloc((size_t)n, 1);
    w->q = (double *)malloc((size_t)d * sizeof(double));
    w->evals = 0;
    return w->bi && w->bd && w->vi && w->vd && w->visited && w->inbeam && w->q;
}

static void ws_free(beam_ws *w) {
    free(w->bi); free(w->bd); free(w->vi); free(w->vd); free(w->visited); free(w->inbeam); free(w->q);
}

/* one search for an arbitrary float64 query (beam_search_single, _kernels.py:215-227).
 * cand buffers need n entries, vis buffers n entries. Returns candidate count;
 * *vl = visit count. */
i64 or_beam_search_single(const float *data, i64 n, i64 d, const i32 *adj, i64 R, const i32 *deg,
                          const i64 *starts, i64 s, const double *q, i64 L,
                          i64 *cand_ids, double *cand_d, i64 *vis_ids, double *vis_d, i64 *vl_out) {
    beam_ws w;
    ws_alloc(&w, n, d, L);
    memcpy(w.q, q, (size_t)d * sizeof(double));
    i64 vl;
    i64 bl = beam_walk(data, d, adj, R, deg, starts, s, L, &w, &vl);
    i64 *ti = (i64 *)malloc((size_t)(n + 1) * sizeof(i64));
    double *td = (double *)malloc((size_t)(n + 1) * sizeof(double));
    i64 c = gather_candidates(&w, bl, vl, cand_ids, cand_d, ti, td);
    memcpy(vis_ids, w.vi, (size_t)vl * sizeof(i64));
    memcpy(vis_d, w.vd, (size_t)vl * sizeof(double));
    *vl_out = vl;
    free(ti); free(td); ws_free(&w);
    return c;
}

/* beam_knn_batch (_kernels.py:230-262); evals_out (optional) counts distance evaluations */
void or_beam_knn_batch(const float *data, i64 n, i64 d, const i32 *adj, i64 R, const i32 *deg,
                       const i64 *starts, i64 s, const i64 *qids, i64 m, i64 L, i64 k,
                       i64 *out_ids, double *out_d, i64 *counts, i64 *evals_out) {
    i64 kk = k < n - 1 ? k : n - 1;
    for (i64 t = 0; t < m * (kk > 0 ? kk : 0); ++t) { out_ids[t] = -1; out_d[t] = INFINITY; }
    for (i64 t = 0; t < m; ++t) counts[t] = 0;
    if (kk <= 0) return;
    i64 total_evals = 0;
#pragma omp parallel reduction(+ : total_evals)
    {
#pragma omp for schedule(dynamic, 16)
        for (i64 t = 0; t < m; ++t) {
            /* per-query allocation and zeroing, as the reference does */
            beam_ws w;
            ws_alloc(&w, n, d, L);
            i64 i = qids[t];
            row_as_f64(data, d, i, w.q);
            i64 vl;
            i64 bl = beam_walk(data, d, adj, R, deg, starts, s, L, &w, &vl);
            i64 cap = vl + bl;
            i64 *ci = (i64 *)malloc((size_t)cap * sizeof(i64) + 8);
            double *cd = (double *)malloc((size_t)cap * sizeof(double) + 8);
            i64 *ti = (i64 *)malloc((size_t)cap * sizeof(i64) + 8);
            double *td = (double *)malloc((size_t)cap * sizeof(double) + 8);
            i64 c = gather_candidates(&w, bl, vl, ci, cd, ti, td);
            i64 got = 0;
            for (i64 x = 0; x < c && got < kk; ++x) {
                if (ci[x] == i) continue;
                out_ids[t * kk + got] = ci[x];
                out_d[t * kk + got] = cd[x];
                ++got;
            }
            counts[t] = got;
            total_evals += w.evals;
            free(ci); free(cd); free(ti); free(td);
            ws_free(&w);
        }
    }
    if (evals_out) *evals_out = total_evals;
}

/* ---- robust prune and graph build (_kernels.py:269-415) ---------------- */

/* drop p and duplicate ids (first occurrence in id order wins), sort (dist,id) */
static i64 canonicalise(i64 *ids, double *dd, i64 m, i64 p, i64 *ti, double *td) {
    stable_sort_by_id(ids, dd, m, ti, td);
    i64 c = 0, prev = -1;
    for (i64 t = 0; t < m; ++t) {
        i64 v = ids[t];
        if (v == prev || v == p) continue;
        ids[c] = v; dd[c++] = dd[t];
        prev = v;
    }
    stable_sort_by_d(dd, ids, c, td, ti);
    return c;
}

static i64 prune_sorted(const float *data, i64 d, const i64 *ids, const double *dd, i64 c,
                        double alpha2, i64 R, i64 *out, uint8_t *alive, double *pq) {
    memset(alive, 1, (size_t)c);
    i64 sel = 0;
    for (i64 t = 0; t < c; ++t) {
        if (!alive[t]) continue;
        i64 ps = ids[t];
        out[sel++] = ps;
        if (sel >= R) break;
        row_as_f64(data, d, ps, pq);
        for (i64 u = t + 1; u < c; ++u) {
            if (!alive[u]) continue;
            if (alpha2 * sq_to_vec(data, d, ids[u], pq) <= dd[u]) alive[u] = 0;
        }
    }
    return sel;
}

/* robust_prune_standalone (_kernels.py:318-335); returns selected count */
i64 or_robust_prune(const float *data, i64 n, i64 d, i64 p, const i64 *cand_ids, const double *cand_d,
                    i64 m, const i64 *cur_ids, i64 dcount, double alpha, i64 R, i64 *out) {
    (void)n;
    i64 tot = m + dcount;
    i64 *ids = (i64 *)malloc((size_t)tot * sizeof(i64) + 8);
    double *dd = (double *)malloc((size_t)tot * sizeof(double) + 8);
    i64 *ti = (i64 *)malloc((size_t)tot * sizeof(i64) + 8);
    double *td = (double *)malloc((size_t)tot * sizeof(double) + 8);
    uint8_t *alive = (uint8_t *)malloc((size_t)tot + 8);
    double *q = (double *)malloc((size_t)d * sizeof(double));
    row_as_f64(data, d, p, q);
    for (i64 t = 0; t < m; ++t) { ids[t] = cand_ids[t]; dd[t] = cand_d[t]; }
    for (i64 t = 0; t < dcount; ++t) { ids[m + t] = cur_ids[t]; dd[m + t] = sq_to_vec(data, d, cur_ids[t], q); }
    i64 c = canonicalise(ids, dd, tot, p, ti, td);
    i64 sel = prune_sorted(data, d, ids, dd, c, alpha * alpha, R, out, alive, q);
    free(ids); free(dd); free(ti); free(td); free(alive); free(q);
    return sel;
}

/* build_batch (_kernels.py:338-375): new_ids (m,R) int32 (-1 padded), new_len (m,) */
static void build_batch(const float *data, i64 n, i64 d, const i32 *adj, const i32 *deg,
                        const i64 *starts, i64 s, const i64 *bids, i64 m, i64 L, double alpha2, i64 R,
                        i32 *new_ids, i64 *new_len) {
#pragma omp parallel for schedule(dynamic, 4)
    for (i64 t = 0; t < m; ++t) {
        beam_ws w;
        ws_alloc(&w, n, d, L);
        i64 p = bids[t];
        row_as_f64(data, d, p, w.q);
        i64 vl;
        beam_walk(data, d, adj, R, deg, starts, s, L, &w, &vl);
        i64 dc = deg[p], tot = vl + dc;
        i64 *ids = (i64 *)malloc((size_t)tot * sizeof(i64) + 8);
        double *dd = (double *)malloc((size_t)tot * sizeof(double) + 8);
        i64 *ti = (i64 *)malloc((size_t)tot * sizeof(i64) + 8);
        double *td = (double *)malloc((size_t)tot * sizeof(double) + 8);
        uint8_t *alive = (uint8_t *)malloc((size_t)tot + 8);
        i64 *out = (i64 *)malloc((size_t)R * sizeof(i64));
        double *pq = (double *)malloc((size_t)d * sizeof(double));
        for (i64 x = 0; x < vl; ++x) { ids[x] = w.vi[x]; dd[x] = w.vd[x]; }
        for (i64 x = 0; x < dc; ++x) {
            i64 nb = adj[p * R + x];
            ids[vl + x] = nb;
            dd[vl + x] = sq_to_vec(data, d, nb, w.q);
        }
        i64 c = canonicalise(ids, dd, tot, p, ti, td);
        i64 sel = prune_sorted(data, d, ids, dd, c, alpha2, R, out, alive, pq);
        for (i64 x = 0; x < R; ++x) new_ids[t * R + x] = x < sel ? (i32)out[x] : -1;
        new_len[t] = sel;
        free(ids); free(dd); free(ti); free(td); free(alive); free(out); free(pq);
        ws_free(&w);
    }
}

/* apply_reverse_edges (_kernels.py:378-415) over CSR groups */
static void reverse_edges(const float *data, i64 d, i32 *adj, i32 *deg, const i64 *targets, i64 nt,
                          const i64 *offsets, const i64 *adds, double alpha2, i64 R) {
#pragma omp parallel for schedule(dynamic, 8)
    for (i64 t = 0; t < nt; ++t) {
        i64 u = targets[t];
        i64 dc = deg[u], extra = offsets[t + 1] - offsets[t], tot = dc + extra;
        i64 *ids = (i64 *)malloc((size_t)tot * sizeof(i64) + 8);
        double *dd = (double *)malloc((size_t)tot * sizeof(double) + 8);
        i64 *ti = (i64 *)malloc((size_t)tot * sizeof(i64) + 8);
        double *td = (double *)malloc((size_t)tot * sizeof(double) + 8);
        uint8_t *alive = (uint8_t *)malloc((size_t)tot + 8);
        i64 *out = (i64 *)malloc((size_t)R * sizeof(i64));
        double *q = (double *)malloc((size_t)d * sizeof(double));
        row_as_f64(data, d, u, q);
        i64 c = 0;
        for (i64 x = 0; x < dc; ++x) { ids[c] = adj[u * R + x]; dd[c] = sq_to_vec(data, d, ids[c], q); ++c; }
        for (i64 x = offsets[t]; x < offsets[t + 1]; ++x) { ids[c] = adds[x]; dd[c] = sq_to_vec(data, d, ids[c], q); ++c; }
        c = canonicalise(ids, dd, tot, u, ti, td);
        i64 sel;
        if (c <= R) {
            sel = c;
            for (i64 x = 0; x < sel; ++x) adj[u * R + x] = (i32)ids[x];
        } else {
            sel = prune_sorted(data, d, ids, dd, c, alpha2, R, out, alive, q);
            for (i64 x = 0; x < sel; ++x) adj[u * R + x] = (i32)out[x];
        }
        for (i64 x = sel; x < R; ++x) adj[u * R + x] = -1;
        deg[u] = (i32)sel;
        free(ids); free(dd); free(ti); free(td); free(alive); free(out); free(q);
    }
}

/* pairs (target, source) sorted by target, stable on source position */
typedef struct { i64 u, p, pos; } edge_t;
static int edge_cmp(const void *a, const void *b) {
    const edge_t *x = (const edge_t *)a, *y = (const edge_t *)b;
    if (x->u != y->u) return x->u < y->u ? -1 : 1;
    return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

/* build_vamana batch loop (vamana.py:141-169). starts / order come from the
 * caller (numpy PCG64 stream, vamana.py:132-143). adj (n,R) int32 and deg (n,)
 * are outputs. */
void or_build_vamana(const float *data, i64 n, i64 d, i64 R, i64 L, double alpha,
                     const i64 *starts, i64 s, const i64 *order, i32 *adj, i32 *deg) {
    double alpha2 = alpha * alpha;
    for (i64 x = 0; x < n * R; ++x) adj[x] = -1;
    for (i64 x = 0; x < n; ++x) deg[x] = 0;
    i64 maxb = 1;
    while (maxb < n) maxb *= 2;
    i32 *new_ids = (i32 *)malloc((size_t)(maxb < n ? maxb : n) * R * sizeof(i32) + 8);
    i64 *new_len = (i64 *)malloc((size_t)(maxb < n ? maxb : n) * sizeof(i64) + 8);
    edge_t *edges = (edge_t *)malloc((size_t)(maxb < n ? maxb : n) * R * sizeof(edge_t) + 8);
    i64 *targets = (i64 *)malloc((size_t)(maxb < n ? maxb : n) * R * sizeof(i64) + 8);
    i64 *offsets = (i64 *)malloc(((size_t)(maxb < n ? maxb : n) * R + 1) * sizeof(i64) + 8);
    i64 *adds = (i64 *)malloc((size_t)(maxb < n ? maxb : n) * R * sizeof(i64) + 8);
    i64 lo = 0, batch = 1;
    while (lo < n) {
        i64 hi = lo + batch < n ? lo + batch : n, m = hi - lo;
        const i64 *bids = order + lo;
        build_batch(data, n, d, adj, deg, starts, s, bids, m, L, alpha2, R, new_ids, new_len);
        i64 ne = 0;
        for (i64 t = 0; t < m; ++t) {
            i64 p = bids[t];
            for (i64 x = 0; x < R; ++x) adj[p * R + x] = new_ids[t * R + x];
            deg[p] = (i32)new_len[t];
            for (i64 x = 0; x < new_len[t]; ++x) {
                edges[ne].u = new_ids[t * R + x]; edges[ne].p = p; edges[ne].pos = ne; ++ne;
            }
        }
        if (ne > 0) {
            qsort(edges, (size_t)ne, sizeof(edge_t), edge_cmp);
            i64 nt = 0;
            for (i64 x = 0; x < ne; ++x) {
                if (x == 0 || edges[x].u != edges[x - 1].u) { targets[nt] = edges[x].u; offsets[nt++] = x; }
                adds[x] = edges[x].p;
            }
            offsets[nt] = ne;
            reverse_edges(data, d, adj, deg, targets, nt, offsets, adds, alpha2, R);
        }
        lo = hi;
        batch *= 2;
    }
    free(new_ids); free(new_len); free(edges); free(targets); free(offsets); free(adds);
}

/* ---- misc ---------------------------------------------------------------- */

i64 or_nearest_to_centroid(const float *data, i64 n, i64 d) {
    double *cen = (double *)calloc((size_t)d, sizeof(double));
    for (i64 j = 0; j < n; ++j)
        for (i64 t = 0; t < d; ++t) cen[t] += (double)data[j * d + t];
    for (i64 t = 0; t < d; ++t) cen[t] /= (double)n;
    double best = INFINITY;
    i64 bid = -1;
    for (i64 j = 0; j < n; ++j) {
        double dj = sq_to_vec(data, d, j, cen);
        if (dj < best) { best = dj; bid = j; }
    }
    free(cen);
    return bid;
}

/* dp_scan_all (_kernels.py:442-462) */
void or_dp_scan_all(const float *data, i64 n, i64 d, const i64 *rank, const i64 *qids, i64 m,
                    i64 *out_id, double *out_d) {
#pragma omp parallel
    {
        double *q = (double *)malloc((size_t)d * sizeof(double));
#pragma omp for schedule(dynamic, 1)
        for (i64 t = 0; t < m; ++t) {
            i64 i = qids[t];
            row_as_f64(data, d, i, q);
            i64 ri = rank[i];
            double best = INFINITY;
            i64 bid = -1;
            for (i64 j = 0; j < n; ++j) {
                if (rank[j] > ri) {
                    double dj = sq_to_vec(data, d, j, q);
                    if (dj < best || (dj == best && j < bid)) { best = dj; bid = j; }
                }
            }
            out_id[t] = bid;
            out_d[t] = best;
        }
        free(q);
    }
}

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void or_set_num_threads(int t) {
#ifdef _OPENMP
    omp_set_num_threads(t);
#else
    (void)t;
#endif
}
