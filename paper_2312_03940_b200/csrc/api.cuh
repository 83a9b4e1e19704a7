// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>

namespace pk {

void set_error(const std::string& msg);
int fail(const char* where, cudaError_t e);

#define PK_CHECK(call)                                   \
    do {                                                 \
        cudaError_t _e = (call);                         \
        if (_e != cudaSuccess) return ::pk::fail(#call, _e); \
    } while (0)

#define PK_CHECK_LAUNCH(where)                                   \
    do {                                                         \
        cudaError_t _e = cudaGetLastError();                     \
        if (_e != cudaSuccess) return ::pk::fail(where, _e);     \
    } while (0)

int sm_count();
int max_smem_optin();

inline int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// stream-ordered scratch allocation (cudaMallocAsync pool)
template <class T>
cudaError_t scratch(T** p, size_t count, cudaStream_t st) {
    return cudaMallocAsync(reinterpret_cast<void**>(p), count * sizeof(T) + 16, st);
}
inline void release(void* p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

// per-warp shared memory sizes
inline size_t beam_smem_bytes(int L, int H) {
    return (((((size_t)L * 12 + 7) & ~(size_t)7) + (size_t)H * 2 + 15) & ~(size_t)15) + 128 + 4 * 64;
}
// spilled beam (carve_beam_spill): shared memory for the seen table and scratch,
// a global slab of spill_slab_bytes(L) per warp for the beam itself
inline size_t spill_smem_bytes(int H) { return (((size_t)H * 2 + 15) & ~(size_t)15) + 128 + 4 * 64; }
inline size_t spill_slab_bytes(int L) { return ((size_t)L * 12 + 15) & ~(size_t)15; }
// row ring behind the beam state (carve_ring): slots x dp floats + one mbarrier per slot
inline size_t ring_smem_bytes(int dp, int slots) { return slots ? (size_t)slots * dp * 4 + (size_t)slots * 8 : 0; }
// slots of the row ring for a float search with lazy keys (PK_RING = 2 or 4; default
// 0 = rows through registers, which is faster since the searches are handed out by
// tickets -- profiles/r2_ring_ab.md): rows of >= 1 KB that the fp32 screen covers
inline int ring_slots(int dp, int qv, bool lazy_screen);
inline size_t sort_smem_bytes(int cap) {
    return (size_t)cap * 13 + 128;
}
inline size_t align16(size_t b) { return (b + 15) & ~(size_t)15; }
// candidate buffers of the prune kernels (layout: carve_cand in build.cu)
inline size_t cand_smem_bytes(int cap, int dw, int S, bool u8) {
    size_t keys = align16(((((size_t)cap * 15 + 3) & ~(size_t)3) + 128));
    if (!u8) return keys;
    return align16(keys + (((size_t)dw + 3) & ~(size_t)3) * 4 + (size_t)S * (dw + 4) * 4 + (size_t)S * 4);
}

int choose_hash(int L, int hash_bits, long long n);

// integer tuning knob from the environment (default when unset / invalid)
inline int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    if (!v || !*v) return dflt;
    char* end = nullptr;
    const long x = std::strtol(v, &end, 10);
    return (end && *end == 0 && x >= 0) ? (int)x : dflt;  // "0" switches a default-on knob off
}

inline int ring_slots(int dp, int qv, bool lazy_screen) {
    if (!lazy_screen || dp < 256 || dp > 128 * qv) return 0;
    int s = env_int("PK_RING", 0);
    if (s <= 0) return 0;
    if (s > 8) s = 8;
    while (s & (s - 1)) s &= s - 1;  // power of two
    return s;
}

// ---- launch accounting -------------------------------------------------------
// Every kernel launch site opens a ProfScope: launches are always counted per
// kernel name; with pk_prof_enable(1) a CUDA event pair brackets the launch on
// its stream so the host can read per-kernel device time (bench.py roofline).
struct ProfScope {
    const char* name;
    cudaStream_t st;
    int slot;
    ProfScope(const char* n, cudaStream_t s);
    ~ProfScope();
};

}  // namespace pk
