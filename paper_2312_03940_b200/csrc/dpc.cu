// Densities, rank order, dependent-point bookkeeping, center/noise policies and
// the union-find assignment (density.py, dependent.py, cluster.py, unionfind.py).
#include <cub/cub.cuh>

#include <algorithm>
#include <string>

#include "../../include/peakann_b200.h"
#include "api.cuh"
#include "common.cuh"

namespace pk {

int grid_for(long long work, int block);

// numpy's pairwise summation for a contiguous float64 run (the inner loop of
// `arr.sum(axis=1)`): sequential below 8 items, 8 interleaved accumulators up
// to 128, recursive halving (rounded to a multiple of 8) above.
__device__ double np_pairwise_sum(const double* a, int n) {
    // explicit stack instead of recursion
    int lo_stack[32], n_stack[32];
    double acc_stack[32];
    int side[32];
    int sp = 0;
    int lo = 0, len = n;
    double result = 0.0;
    for (;;) {
        if (len <= 128) {
            double res;
            if (len < 8) {
                res = 0.0;
                for (int i = 0; i < len; ++i) res += a[lo + i];
            } else {
                double r[8];
                for (int j = 0; j < 8; ++j) r[j] = a[lo + j];
                int i = 8;
                for (; i < len - (len % 8); i += 8)
                    for (int j = 0; j < 8; ++j) r[j] += a[lo + i + j];
                res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
                for (; i < len; ++i) res += a[lo + i];
            }
            // unwind: combine with finished left halves
            while (sp > 0 && side[sp - 1] == 1) {
                --sp;
                res = acc_stack[sp] + res;
            }
            if (sp == 0) {
                result = res;
                break;
            }
            // finished a left half: store it, continue with the right half
            side[sp - 1] = 1;
            acc_stack[sp - 1] = res;
            int plo = lo_stack[sp - 1], pn = n_stack[sp - 1];
            int n2 = pn / 2;
            n2 -= n2 % 8;
            lo = plo + n2;
            len = pn - n2;
            continue;
        }
        // split: push frame, descend into the left half
        lo_stack[sp] = lo;
        n_stack[sp] = len;
        side[sp] = 0;
        ++sp;
        int n2 = len / 2;
        n2 -= n2 % 8;
        len = n2;
    }
    return result;
}

__global__ void density_rows_kernel(int kind, const double* dists, long long n, int k, double* rho, double* tmp) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double* row = dists + i * k;
        double* t = tmp + i * k;
        double v;
        if (kind == PK_DENSITY_KTH || kind == PK_DENSITY_KTH_NORMALIZED) {
            v = 1.0 / row[k - 1];
        } else if (kind == PK_DENSITY_EXP_SUM) {
            for (int j = 0; j < k; ++j) t[j] = row[j] * row[j];
            v = exp(-np_pairwise_sum(t, k) / (double)k);
        } else if (kind == PK_DENSITY_SUM_EXP) {
            for (int j = 0; j < k; ++j) t[j] = exp(-(row[j] * row[j]));
            v = np_pairwise_sum(t, k) / (double)k;
        } else {
            v = -np_pairwise_sum(row, k);
        }
        rho[i] = v;
    }
}

// rho * k / sum(rho[neighbours]) with inf for zero / nan (density.py:48-55)
// (rows i of this call are points row0 + i: a rank's own chunk of the kNN rows)
__global__ void normalize_kernel(const double* base, const long long* ids, long long n, int k, double* out,
                                 double* tmp, long long row0) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double* t = tmp + i * k;
        for (int j = 0; j < k; ++j) t[j] = base[ids[i * k + j]];
        double den = np_pairwise_sum(t, k);
        double v = base[row0 + i] * (double)k / den;
        if (den == 0.0 || isnan(v)) v = __longlong_as_double(0x7ff0000000000000LL);
        out[i] = v;
    }
}

// descending-order radix key for rho: bigger rho -> smaller key; -0.0 == +0.0
__global__ void rank_keys_kernel(const double* rho, long long n, unsigned long long* keys, long long* vals, int* nan_flag) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double r = rho[i];
        if (isnan(r)) atomicOr(nan_flag, 1);
        if (r == 0.0) r = 0.0;
        unsigned long long b = (unsigned long long)__double_as_longlong(r);
        // ascending order key of r, then complemented for descending
        unsigned long long asc = (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
        keys[i] = ~asc;
        vals[i] = i;
    }
}

__global__ void rank_scatter_kernel(const long long* order, long long n, long long* rank) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
        rank[order[j]] = n - j;
}

// first denser entry per row; unresolved flagged (dependent.py:80-93)
__global__ void resolve_kernel(const long long* rank, const long long* qids, long long m, const long long* ids,
                               const double* dists, int k, long long* lam, double* delta, unsigned char* unres,
                               long long skip, const long long* counts, unsigned char* shortf) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x) {
        long long q = qids[t];
        if (counts) {
            // a row the beam search could not fill: resolved by pk_resolve_short
            const bool sh = counts[t] < k;
            shortf[t] = sh;
            if (sh) {
                unres[t] = 0;
                continue;
            }
        }
        long long rq = rank[q];
        int hit = -1;
        for (int j = 0; j < k; ++j) {
            long long id = ids[t * k + j];
            if (id >= 0 && rank[id] > rq) { hit = j; break; }
        }
        if (hit >= 0) {
            lam[q] = ids[t * k + hit];
            delta[q] = dists[t * k + hit];
            unres[t] = 0;
        } else {
            unres[t] = q != skip;
        }
    }
}

__global__ void scatter_dep_kernel(const long long* qids, long long m, const long long* sid, const double* ssq,
                                   long long* lam, double* delta) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x) {
        lam[qids[t]] = sid[t];
        delta[qids[t]] = sqrt(ssq[t]);
    }
}

__global__ void noise_kernel(const double* rho, long long n, double rho_min, unsigned char* noise) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        noise[i] = rho[i] < rho_min;
}

__global__ void threshold_kernel(const double* delta, const unsigned char* noise, long long n, double dmin,
                                 unsigned char* center) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        center[i] = !noise[i] && delta[i] >= dmin;
}

__device__ __forceinline__ unsigned long long desc_key(double v) {
    if (v == 0.0) v = 0.0;
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    unsigned long long asc = (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
    return ~asc;
}

// products for non-noise points (cluster.py:145-152); noise gets a key after everything
__global__ void product_keys_kernel(const double* rho, const double* delta, const unsigned char* noise, long long n,
                                    unsigned long long* kprod, unsigned long long* kdelta, long long* vals) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double dl = delta[i], r = rho[i];
        double pr = dl * r;
        if (isinf(dl)) pr = __longlong_as_double(0x7ff0000000000000LL);
        if (isnan(pr)) pr = dl == 0.0 ? 0.0 : __longlong_as_double(0x7ff0000000000000LL);
        kprod[i] = noise[i] ? ~0ull : desc_key(pr);
        kdelta[i] = desc_key(dl);
        vals[i] = i;
    }
}

__global__ void gather_keys_kernel(const unsigned long long* k, const long long* order, long long n,
                                   unsigned long long* out) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
        out[j] = k[order[j]];
}

__global__ void mark_first_kernel(const long long* order, long long nc, unsigned char* center) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < nc; j += (long long)gridDim.x * blockDim.x)
        center[order[j]] = 1;
}

__global__ void local_kernel(const long long* rank, const long long* nbr, int k, const unsigned char* noise,
                             long long n, unsigned char* center) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        long long best = rank[nbr[i * k]];
        for (int j = 1; j < k; ++j) best = max(best, rank[nbr[i * k + j]]);
        center[i] = !noise[i] && rank[i] > best;
    }
}

__global__ void orphan_kernel(const long long* lam, const unsigned char* noise, long long n, unsigned char* center) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (lam[i] < 0 && !noise[i]) center[i] = 1;
}

// pointer jumping: parent = skip ? self : lam
__global__ void parent_init_kernel(const long long* lam, const unsigned char* center, const unsigned char* noise,
                                   long long n, long long* par, long long* status) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        bool skip = center[i] || noise[i];
        long long l = lam[i];
        if (!skip && (l < 0 || l >= n)) {
            atomicMin(reinterpret_cast<unsigned long long*>(status + 1), (unsigned long long)i);
            atomicMax(reinterpret_cast<unsigned long long*>(status), 1ull);
            l = i;
        }
        par[i] = skip ? i : l;
    }
}

__global__ void jump_kernel(const long long* par, long long n, long long* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = par[par[i]];
}

__global__ void label_kernel(const long long* root, const unsigned char* center, const unsigned char* noise,
                             long long n, long long* labels, long long* status) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        long long r = root[i];
        if (center[r] || noise[r]) {
            labels[i] = r;
        } else {
            labels[i] = -1;
            atomicMin(reinterpret_cast<unsigned long long*>(status + 2), (unsigned long long)i);
        }
    }
}

__global__ void status_final_kernel(long long* status) {
    // status[0]: 0 ok, 1 missing dependent (status[1] id), 3 orphan component (status[1] id)
    if (status[0] == 0 && status[2] != 0x7fffffffffffffffLL) {
        status[0] = 3;
        status[1] = status[2];
    }
}

__global__ void flags_u8_to_int(const unsigned char* f, long long n, int* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = f[i];
}

__global__ void argmax_rank_kernel(const long long* rank, long long n, long long* out) {
    // rank is a permutation of 1..n: the argmax is where rank == n
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (rank[i] == n) *out = i;
}

int sort_pairs_u64(const unsigned long long* kin, unsigned long long* kout, const long long* vin, long long* vout,
                   long long n, cudaStream_t st) {
    size_t bytes = 0;
    PK_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, 0, 64, st));
    void* tmp = nullptr;
    PK_CHECK(cudaMallocAsync(&tmp, bytes + 16, st));
    {
        ProfScope _ps("cub_DeviceRadixSort_SortPairs", st);
        PK_CHECK(cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, (int)n, 0, 64, st));
    }
    release(tmp, st);
    return 0;
}

// out[j] = in[i] for the flagged i, in order; *count = number flagged
int compact_flagged(const long long* in, const unsigned char* flags, long long n, long long* out, long long* count,
                    cudaStream_t st) {
    size_t bytes = 0;
    PK_CHECK(cub::DeviceSelect::Flagged(nullptr, bytes, in, flags, out, count, (int)n, st));
    void* tmp = nullptr;
    PK_CHECK(cudaMallocAsync(&tmp, bytes + 16, st));
    {
        ProfScope _ps("cub_DeviceSelect_Flagged", st);
        PK_CHECK(cub::DeviceSelect::Flagged(tmp, bytes, in, flags, out, count, (int)n, st));
    }
    release(tmp, st);
    return 0;
}

__global__ void iota_kernel(long long* a, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        a[i] = i;
}

}  // namespace pk

using namespace pk;

extern "C" int pk_densities(int kind, const int64_t* ids, const double* dists, int64_t n, int64_t k, double* rho,
                            void* stream) {
    cudaStream_t st = as_stream(stream);
    if (n <= 0) return 0;
    if (kind < 0 || kind > 4 || k < 1) {
        set_error("bad density kind or k");
        return 2;
    }
    double* tmp = nullptr;
    PK_CHECK(scratch(&tmp, (size_t)n * k, st));
    int g = grid_for(n, 128);
    if (kind == PK_DENSITY_KTH_NORMALIZED) {
        double* base = nullptr;
        PK_CHECK(scratch(&base, (size_t)n, st));
        {
            ProfScope _ps("density_rows_kernel", st);
            density_rows_kernel<<<g, 128, 0, st>>>(PK_DENSITY_KTH, dists, n, (int)k, base, tmp);
        }
        {
            ProfScope _ps("normalize_kernel", st);
            normalize_kernel<<<g, 128, 0, st>>>(base, reinterpret_cast<const long long*>(ids), n, (int)k, rho, tmp, 0);
        }
        release(base, st);
    } else {
        {
            ProfScope _ps("density_rows_kernel", st);
            density_rows_kernel<<<g, 128, 0, st>>>(kind, dists, n, (int)k, rho, tmp);
        }
    }
    PK_CHECK_LAUNCH("density kernels");
    release(tmp, st);
    return 0;
}

extern "C" int pk_normalize_rho_rows(const double* base, const int64_t* ids, int64_t row0, int64_t m, int64_t k,
                                     double* out, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (m <= 0) return 0;
    double* tmp = nullptr;
    PK_CHECK(scratch(&tmp, (size_t)m * k, st));
    {
        ProfScope _ps("normalize_kernel", st);
        normalize_kernel<<<grid_for(m, 128), 128, 0, st>>>(base, reinterpret_cast<const long long*>(ids), m, (int)k, out,
                                                          tmp, row0);
    }
    PK_CHECK_LAUNCH("normalize_kernel");
    release(tmp, st);
    return 0;
}

extern "C" int pk_normalize_rho(const double* base, const int64_t* ids, int64_t n, int64_t k, double* out,
                                void* stream) {
    return pk_normalize_rho_rows(base, ids, 0, n, k, out, stream);
}

extern "C" int pk_rank_order(const double* rho, int64_t n, int64_t* rank, int* nan_flag, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (n <= 0) return 0;
    unsigned long long *k0 = nullptr, *k1 = nullptr;
    long long *v0 = nullptr, *v1 = nullptr;
    PK_CHECK(scratch(&k0, (size_t)n, st));
    PK_CHECK(scratch(&k1, (size_t)n, st));
    PK_CHECK(scratch(&v0, (size_t)n, st));
    PK_CHECK(scratch(&v1, (size_t)n, st));
    PK_CHECK(cudaMemsetAsync(nan_flag, 0, sizeof(int), st));
    int g = grid_for(n, 256);
    {
        ProfScope _ps("rank_keys_kernel", st);
        rank_keys_kernel<<<g, 256, 0, st>>>(rho, n, k0, v0, nan_flag);
    }
    PK_CHECK_LAUNCH("rank_keys_kernel");
    // stable LSD radix sort: equal densities keep ascending ids (lexsort, density.py:126)
    int rc = sort_pairs_u64(k0, k1, v0, v1, n, st);
    if (rc) return rc;
    {
        ProfScope _ps("rank_scatter_kernel", st);
        rank_scatter_kernel<<<g, 256, 0, st>>>(v1, n, reinterpret_cast<long long*>(rank));
    }
    PK_CHECK_LAUNCH("rank_scatter_kernel");
    for (void* p : {(void*)k0, (void*)k1, (void*)v0, (void*)v1}) release(p, st);
    return 0;
}

extern "C" int pk_resolve_lists(const int64_t* rank, const int64_t* qids, int64_t m, const int64_t* ids,
                                const double* dists, int64_t k, int64_t* lam, double* delta, int64_t* unresolved,
                                int64_t* n_unresolved, int64_t skip, const int64_t* counts, int64_t* short_out,
                                int64_t* n_short, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (m <= 0) {
        PK_CHECK(cudaMemsetAsync(n_unresolved, 0, sizeof(int64_t), st));
        if (n_short) PK_CHECK(cudaMemsetAsync(n_short, 0, sizeof(int64_t), st));
        return 0;
    }
    if (counts && (!short_out || !n_short)) {
        set_error("pk_resolve_lists: counts given without a short-row output");
        return 2;
    }
    unsigned char* fl = nullptr;
    unsigned char* sf = nullptr;
    PK_CHECK(scratch(&fl, (size_t)m, st));
    if (counts) PK_CHECK(scratch(&sf, (size_t)m, st));
    if (k == 0) {
        PK_CHECK(cudaMemsetAsync(fl, 1, (size_t)m, st));
        if (sf) PK_CHECK(cudaMemsetAsync(sf, 0, (size_t)m, st));
    } else {
        {
            ProfScope _ps("resolve_kernel", st);
            resolve_kernel<<<grid_for(m, 256), 256, 0, st>>>(
                reinterpret_cast<const long long*>(rank), reinterpret_cast<const long long*>(qids), m,
                reinterpret_cast<const long long*>(ids), dists, (int)k, reinterpret_cast<long long*>(lam), delta, fl, skip,
                reinterpret_cast<const long long*>(counts), sf);
        }
        PK_CHECK_LAUNCH("resolve_kernel");
    }
    // unresolved (and short) qids, input order preserved
    int rc = compact_flagged(reinterpret_cast<const long long*>(qids), fl, m, reinterpret_cast<long long*>(unresolved),
                             reinterpret_cast<long long*>(n_unresolved), st);
    if (!rc && sf)
        rc = compact_flagged(reinterpret_cast<const long long*>(qids), sf, m, reinterpret_cast<long long*>(short_out),
                             reinterpret_cast<long long*>(n_short), st);
    release(fl, st);
    if (sf) release(sf, st);
    return rc;
}

extern "C" int pk_scatter_dependents(const int64_t* qids, int64_t m, const int64_t* src_id, const double* src_sqd,
                                     int64_t* lam, double* delta, void* stream) {
    if (m <= 0) return 0;
    cudaStream_t st = as_stream(stream);
    {
        ProfScope _ps("scatter_dep_kernel", st);
        scatter_dep_kernel<<<grid_for(m, 256), 256, 0, st>>>(reinterpret_cast<const long long*>(qids), m,
                                                            reinterpret_cast<const long long*>(src_id), src_sqd,
                                                            reinterpret_cast<long long*>(lam), delta);
    }
    PK_CHECK_LAUNCH("scatter_dep_kernel");
    return 0;
}

extern "C" int pk_argmax_rank(const int64_t* rank, int64_t n, int64_t* out, void* stream) {
    if (n <= 0) return 0;
    cudaStream_t st = as_stream(stream);
    {
        ProfScope _ps("argmax_rank_kernel", st);
        argmax_rank_kernel<<<grid_for(n, 256), 256, 0, st>>>(reinterpret_cast<const long long*>(rank), n,
                                                            reinterpret_cast<long long*>(out));
    }
    PK_CHECK_LAUNCH("argmax_rank_kernel");
    return 0;
}

extern "C" int pk_flag_noise(const double* rho, int64_t n, double rho_min, uint8_t* noise, int64_t* n_noise,
                             void* stream) {
    if (n <= 0) return 0;
    cudaStream_t st = as_stream(stream);
    {
        ProfScope _ps("noise_kernel", st);
        noise_kernel<<<grid_for(n, 256), 256, 0, st>>>(rho, n, rho_min, noise);
    }
    PK_CHECK_LAUNCH("noise_kernel");
    if (n_noise) {
        size_t bytes = 0;
        PK_CHECK(cub::DeviceReduce::Sum(nullptr, bytes, noise, reinterpret_cast<long long*>(n_noise), (int)n, st));
        void* tmp = nullptr;
        PK_CHECK(cudaMallocAsync(&tmp, bytes + 16, st));
        {
            ProfScope _ps("cub_DeviceReduce_Sum", st);
            PK_CHECK(cub::DeviceReduce::Sum(tmp, bytes, noise, reinterpret_cast<long long*>(n_noise), (int)n, st));
        }
        release(tmp, st);
    }
    return 0;
}

extern "C" int pk_centers_threshold(const double* delta, const uint8_t* noise, int64_t n, double delta_min,
                                    uint8_t* center, void* stream) {
    if (n <= 0) return 0;
    cudaStream_t st = as_stream(stream);
    {
        ProfScope _ps("threshold_kernel", st);
        threshold_kernel<<<grid_for(n, 256), 256, 0, st>>>(delta, noise, n, delta_min, center);
    }
    PK_CHECK_LAUNCH("threshold_kernel");
    return 0;
}

extern "C" int pk_centers_product(const double* rho, const double* delta, const uint8_t* noise, int64_t n,
                                  int64_t n_c, uint8_t* center, void* stream) {
    if (n <= 0) return 0;
    cudaStream_t st = as_stream(stream);
    unsigned long long *kp = nullptr, *kdl = nullptr, *ka = nullptr, *kb = nullptr;
    long long *v0 = nullptr, *v1 = nullptr;
    PK_CHECK(scratch(&kp, (size_t)n, st));
    PK_CHECK(scratch(&kdl, (size_t)n, st));
    PK_CHECK(scratch(&ka, (size_t)n, st));
    PK_CHECK(scratch(&kb, (size_t)n, st));
    PK_CHECK(scratch(&v0, (size_t)n, st));
    PK_CHECK(scratch(&v1, (size_t)n, st));
    int g = grid_for(n, 256);
    {
        ProfScope _ps("product_keys_kernel", st);
        product_keys_kernel<<<g, 256, 0, st>>>(rho, delta, noise, n, kp, kdl, v0);
    }
    PK_CHECK_LAUNCH("product_keys_kernel");
    // lexsort((id, -delta, -prod)): stable sort by -delta, then stable sort by -prod
    int rc = sort_pairs_u64(kdl, ka, v0, v1, n, st);
    if (rc) return rc;
    {
        ProfScope _ps("gather_keys_kernel", st);
        gather_keys_kernel<<<g, 256, 0, st>>>(kp, v1, n, ka);
    }
    rc = sort_pairs_u64(ka, kb, v1, v0, n, st);
    if (rc) return rc;
    PK_CHECK(cudaMemsetAsync(center, 0, (size_t)n, st));
    {
        ProfScope _ps("mark_first_kernel", st);
        mark_first_kernel<<<grid_for(n_c, 256), 256, 0, st>>>(v0, n_c, center);
    }
    PK_CHECK_LAUNCH("mark_first_kernel");
    for (void* p : {(void*)kp, (void*)kdl, (void*)ka, (void*)kb, (void*)v0, (void*)v1}) release(p, st);
    return 0;
}

extern "C" int pk_centers_local(const int64_t* rank, const int64_t* nbr_ids, int64_t k, const uint8_t* noise,
                                int64_t n, uint8_t* center, void* stream) {
    if (n <= 0) return 0;
    cudaStream_t st = as_stream(stream);
    {
        ProfScope _ps("local_kernel", st);
        local_kernel<<<grid_for(n, 256), 256, 0, st>>>(reinterpret_cast<const long long*>(rank),
                                                      reinterpret_cast<const long long*>(nbr_ids), (int)k, noise, n, center);
    }
    PK_CHECK_LAUNCH("local_kernel");
    return 0;
}

extern "C" int pk_promote_orphans(const int64_t* lam, const uint8_t* noise, int64_t n, uint8_t* center, void* stream) {
    if (n <= 0) return 0;
    cudaStream_t st = as_stream(stream);
    {
        ProfScope _ps("orphan_kernel", st);
        orphan_kernel<<<grid_for(n, 256), 256, 0, st>>>(reinterpret_cast<const long long*>(lam), noise, n, center);
    }
    PK_CHECK_LAUNCH("orphan_kernel");
    return 0;
}

extern "C" int pk_assign_clusters(const int64_t* lam, const uint8_t* center, const uint8_t* noise, int64_t n,
                                  int64_t* labels, int64_t* status, void* stream) {
    if (n <= 0) return 0;
    cudaStream_t st = as_stream(stream);
    long long *a = nullptr, *b = nullptr;
    PK_CHECK(scratch(&a, (size_t)n, st));
    PK_CHECK(scratch(&b, (size_t)n, st));
    long long init[3] = {0, 0x7fffffffffffffffLL, 0x7fffffffffffffffLL};
    PK_CHECK(cudaMemcpyAsync(status, init, sizeof(init), cudaMemcpyHostToDevice, st));
    int g = grid_for(n, 256);
    long long* s = reinterpret_cast<long long*>(status);
    {
        ProfScope _ps("parent_init_kernel", st);
        parent_init_kernel<<<g, 256, 0, st>>>(reinterpret_cast<const long long*>(lam), center, noise, n, a, s);
    }
    // ceil(log2 n) + 1 rounds of pointer jumping reach every root of a forest
    int rounds = 1;
    while ((1ll << rounds) < n) ++rounds;
    for (int r = 0; r <= rounds; ++r) {
        {
            ProfScope _ps("jump_kernel", st);
            jump_kernel<<<g, 256, 0, st>>>(a, n, b);
        }
        std::swap(a, b);
    }
    {
        ProfScope _ps("label_kernel", st);
        label_kernel<<<g, 256, 0, st>>>(a, center, noise, n, reinterpret_cast<long long*>(labels), s);
    }
    {
        ProfScope _ps("status_final_kernel", st);
        status_final_kernel<<<1, 1, 0, st>>>(s);
    }
    PK_CHECK_LAUNCH("assign kernels");
    // the memcpy source is a host stack array: make sure it was consumed
    PK_CHECK(cudaStreamSynchronize(st));
    release(a, st);
    release(b, st);
    return 0;
}

extern "C" int pk_flags_to_ids(const uint8_t* flags, int64_t n, int64_t* out, int64_t* count, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (n <= 0) {
        PK_CHECK(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
        return 0;
    }
    long long* iota = nullptr;
    PK_CHECK(scratch(&iota, (size_t)n, st));
    {
        ProfScope _ps("iota_kernel", st);
        iota_kernel<<<grid_for(n, 256), 256, 0, st>>>(iota, n);
    }
    int rc = compact_flagged(iota, flags, n, reinterpret_cast<long long*>(out), reinterpret_cast<long long*>(count), st);
    release(iota, st);
    return rc;
}
